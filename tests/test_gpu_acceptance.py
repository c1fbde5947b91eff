"""Acceptance-style checks in the spirit of the reference's criteria C2-C8
(pkg/tests/test_acceptance.py), run through the GPU path."""

import math
from fractions import Fraction

import numpy as np
import pytest
import torch

import paper_1905_13746_b200 as gnb
from paper_1905_13746_b200 import dense
from paper_1905_13746_b200.model import Label

pytestmark = pytest.mark.gpu


def _rec(sid, label, size, ops):
    return gnb.SampleRecord(sid, label, size, gnb.OpcodeHistogram.from_counts(ops))


def test_c2_posterior_matches_exact_rational_bayes():
    """200 micro-instances: GPU scores -> normalized posterior vs exact Fractions."""
    rng = np.random.default_rng(77)
    pool = ("a", "b", "c", "d")
    worst = 0.0
    for case in range(200):
        feats = tuple(sorted(rng.choice(pool, size=int(rng.integers(1, 5)), replace=False)))
        alpha = int(rng.integers(1, 3))
        cm = {o: int(rng.integers(0, 6)) for o in feats}
        cb = {o: int(rng.integers(0, 6)) for o in feats}
        n_m, n_b = int(rng.integers(1, 4)), int(rng.integers(1, 4))
        samples = [_rec(f"m{i}", Label.MALWARE, 1, {**({o: c for o, c in cm.items() if c}
                                                     if i == 0 else {}), "zz": 1})
                   for i in range(n_m)]
        samples += [_rec(f"b{i}", Label.BENIGN, 1, {**({o: c for o, c in cb.items() if c}
                                                    if i == 0 else {}), "zz": 1})
                    for i in range(n_b)]
        model = gnb.train_group(samples, gnb.FeatureSet(feats, 4), float(alpha))
        hist = {o: int(rng.integers(0, 4)) for o in feats + ("noise",)}
        h = gnb.OpcodeHistogram.from_counts(hist)
        joint = {}
        for lab, n_c, counts in ((Label.MALWARE, n_m, cm), (Label.BENIGN, n_b, cb)):
            tot = sum(counts.values())
            pr = Fraction(n_c, n_m + n_b)
            for o in feats:
                pr *= Fraction(counts[o] + alpha, tot + alpha * len(feats)) ** h.get(o, 0)
            joint[lab] = pr
        want = joint[Label.MALWARE] / (joint[Label.MALWARE] + joint[Label.BENIGN])
        got = gnb.normalized_posterior(gnb.log_posterior(model, h))[Label.MALWARE]
        worst = max(worst, abs(got - float(want)))
    assert worst < 1e-9


def test_c3_feature_selection_double_loop_oracle():
    rng = np.random.default_rng(33)
    pool = ["add", "call", "jmp", "lea", "mov", "pop", "push", "ret", "sub", "xor"]
    for case in range(40):
        vocab = list(rng.choice(pool, size=int(rng.integers(2, 11)), replace=False))
        samples = []
        for i in range(12):
            ops = {op: int(rng.integers(1, 40)) for op in
                   rng.choice(vocab, size=int(rng.integers(1, len(vocab) + 1)), replace=False)}
            samples.append(_rec(f"c{case}-{i}", Label.MALWARE if i % 2 == 0 else Label.BENIGN,
                                100 + i, ops))
        tot = {Label.MALWARE: 0, Label.BENIGN: 0}
        cnt = {Label.MALWARE: {}, Label.BENIGN: {}}
        for s in samples:
            for op, n in s.histogram.entries.items():
                cnt[s.label][op] = cnt[s.label].get(op, 0) + n
                tot[s.label] += n
        score = {op: abs(cnt[Label.MALWARE].get(op, 0) / tot[Label.MALWARE]
                         - cnt[Label.BENIGN].get(op, 0) / tot[Label.BENIGN])
                 for op in set(cnt[Label.MALWARE]) | set(cnt[Label.BENIGN])}
        k = int(rng.integers(1, 12))
        want = tuple(op for op, _ in sorted(score.items(), key=lambda kv: (-kv[1], kv[0]))[:k])
        cfg = gnb.GroupingConfig(min_per_class=1)
        bundle = gnb.train_bundle(gnb.partition_by_group(samples, cfg)[0], k, created_at="t")
        assert bundle.models[0].features.opcodes == want


def test_c4_sequential_and_parallel_identical_with_errors():
    rng = np.random.default_rng(404)
    samples = []
    for g in range(3):
        for i in range(14):
            lab = Label.MALWARE if i % 2 else Label.BENIGN
            ops = {f"op{int(j)}": int(rng.integers(1, 9)) for j in rng.choice(12, 5, replace=False)}
            samples.append(_rec(f"s{g}-{i}", lab, g * 5120 + i, ops))
    bundle = gnb.train_bundle(gnb.partition_by_group(samples, gnb.GroupingConfig())[0], 6,
                              created_at="t")
    work = list(samples) * 3
    work[7] = _rec("big", Label.UNKNOWN, 512000 + 5, {"op1": 1})
    seq = gnb.classify_sequential(bundle, gnb.Workload(tuple(work), lanes=1), warmup=False)
    for lanes in (1, 2, 4, 8):
        par = gnb.classify_parallel(bundle, gnb.Workload(tuple(work), lanes=lanes), warmup=False)
        assert par.predictions == seq.predictions and par.errors == seq.errors
    assert seq.errors == ((7, "size_bytes 512005 outside [0, 512000)"),)


def test_c7_exclusion_and_fallback():
    short = {5, 8, 61}
    samples = []
    for g in range(100):
        for i in range(5 if g in short else 6):
            samples.append(_rec(f"m{g}-{i}", Label.MALWARE, g * 5120 + i, {"evil": 3 + i % 2, "mov": 1}))
        for i in range(6):
            samples.append(_rec(f"b{g}-{i}", Label.BENIGN, g * 5120 + i, {"mov": 3, "add": 1 + i % 2}))
    corpus = gnb.partition_by_group(samples, gnb.GroupingConfig())[0]
    assert gnb.trainable_groups(corpus, corpus.config) == set(range(100)) - short
    bundle = gnb.train_bundle(corpus, 3, created_at="t")
    assert bundle.trained_ids == tuple(sorted(set(range(100)) - short))
    probes = tuple(_rec(f"p{g}", Label.UNKNOWN, g * 5120 + 100, {"mov": 2, "evil": 1})
                   for g in sorted(short))
    run = gnb.classify_sequential(bundle, gnb.Workload(probes, lanes=1), warmup=False)
    assert [p.effective_group for p in run.predictions] == [6, 9, 62]


@pytest.mark.parametrize("divergence,lo,hi", [(1.0, 1.0, 1.0), (0.0, 0.45, 0.55)])
def test_c8_learnability(divergence, lo, hi):
    """Disjoint class vocabularies are fully learnable; identical ones are not."""
    n, V = 60_000, 40
    x, size, lab = dense.generate(n, V, divergence=divergence, seed=11, group_rows=[n])
    tr, te = slice(0, 40_000), slice(40_000, n)
    st = dense.fit_stats(x[tr], size[tr], lab[tr], n_classes=2, group_size_bytes=5120,
                         max_size_bytes=5120)
    fin = dense.fin_train(st.sums.cpu().numpy(), st.counts.cpu().numpy(), k=20, alpha=1.0,
                          min_per_class=6)
    F = int(fin.n_features[0])
    t = dense.DeviceTables.build(fin.log_prior[:1], fin.log_lik[:1, :, :F], np.zeros(1, np.int32),
                                 group_size_bytes=5120, max_size_bytes=5120)
    feats = torch.from_numpy(fin.features[0, :F].astype(np.int64)).cuda()
    pred, _ = dense.predict(x[te][:, feats].contiguous(), size[te].contiguous(), t)
    acc = float((pred == lab[te]).float().mean())
    assert lo <= acc <= hi
