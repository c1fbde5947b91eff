"""The GPU drop-in on the reference's OWN objects (groupnb from baseline/_ref):
train_bundle / train_bundles / train_group / classify_parallel answer in groupnb
types and equal the reference's own results bit for bit -- bundle JSON
byte-identical, Tp predictions == the reference's Tc (classify_sequential) --
on one device and sharded over several (here: shards on the visible GPUs,
round-robin)."""

import numpy as np
import pytest
import torch

from refpkg import groupnb

gn = groupnb()
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(gn is None, reason="baseline/_ref not installed")]

from paper_1905_13746_b200 import api  # noqa: E402


def _corpus(seed, groups=6, per=25, vocab=80, div=0.4):
    spec = gn.SyntheticSpec(group_count=groups, samples_per_group_per_class=per,
                            vocabulary_size=vocab, divergence=div, seed=seed)
    corpus = gn.generate_synthetic(spec)
    train, _ = gn.partition_by_group(corpus, gn.GroupingConfig())
    return corpus, train


def _devices(n):
    return [i % torch.cuda.device_count() for i in range(n)]


@pytest.mark.parametrize("seed,k,ndev", [(0, 10, 1), (1, 40, 1), (2, 200, 2), (3, 7, 3)])
def test_train_bundle_equals_reference(seed, k, ndev):
    corpus, train = _corpus(seed)
    ref = gn.train_bundle(train, k=k, alpha=0.5 + seed, created_at="t")
    got = api.train_bundle(train, k, 0.5 + seed, created_at="t", devices=_devices(ndev))
    assert type(got) is gn.ModelBundle
    assert gn.bundle_to_json(got) == gn.bundle_to_json(ref)
    assert got.trained_ids == ref.trained_ids


@pytest.mark.parametrize("seed,ndev", [(0, 1), (1, 2), (4, 4)])
def test_classify_parallel_equals_reference_tc(seed, ndev):
    corpus, train = _corpus(seed)
    bundle = gn.train_bundle(train, k=30, created_at="t")
    rng = np.random.default_rng(seed)
    samples = [corpus[i] for i in rng.integers(0, len(corpus), size=2000)]
    for j in (3, 999, 1500):
        samples[j] = gn.SampleRecord(f"big{j}", gn.Label.UNKNOWN, 512000 + j,
                                     gn.OpcodeHistogram.from_counts({"op01": 1}))
    work = gn.Workload(tuple(samples), lanes=4)
    tc = gn.classify_sequential(bundle, work)
    tp = api.classify_parallel(bundle, work, devices=_devices(ndev))
    assert type(tp) is gn.TimedRun
    assert tp.predictions == tc.predictions and tp.errors == tc.errors
    assert all(type(p) is gn.Prediction for p in tp.predictions if p is not None)


def test_train_bundles_equals_reference():
    corpus, train = _corpus(7)
    ks = (20, 40, 80)
    ref = gn.train_bundles(train, ks, created_at="t")
    got = api.train_bundles(train, ks, created_at="t")
    assert sorted(got) == sorted(ref)
    for k in ks:
        assert gn.bundle_to_json(got[k]) == gn.bundle_to_json(ref[k])


def test_train_group_equals_reference():
    corpus, train = _corpus(8)
    for g in sorted(train.groups)[:3]:
        table = gn.score_opcodes(train.groups[g], group=g)
        for k in (1, 5, 50):
            feats = gn.select_top_k(table, k)
            ref = gn.train_group(train.groups[g], feats, 1.0, group=g)
            got = api.train_group(train.groups[g], feats, 1.0, group=g)
            assert type(got) is gn.GroupModel and got == ref
    f = gn.FeatureSet(("op01", "op01", "op02"), 3)            # duplicates: reference totals
    assert api.train_group(train.groups[0], f, 1.0) == gn.train_group(train.groups[0], f, 1.0)


def _err(fn):
    try:
        fn()
    except Exception as e:  # noqa: BLE001
        return type(e), str(e)
    return None


def test_errors_are_the_references():
    mk = lambda sid, lab, size, ops: gn.SampleRecord(  # noqa: E731
        sid, lab, size, gn.OpcodeHistogram.from_counts(ops))
    M, B, U = gn.Label.MALWARE, gn.Label.BENIGN, gn.Label.UNKNOWN
    cases = []
    # unlabeled sample inside a trainable group
    s = [mk(f"m{i}", M, 10, {"a": 2}) for i in range(6)] + [mk(f"b{i}", B, 10, {"b": 1})
                                                           for i in range(6)]
    cases.append(s + [mk("u", U, 11, {"a": 1})])
    # all histograms empty: no opcode occurrences to score
    cases.append([mk(f"m{i}", M, 10, {}) for i in range(6)] + [mk(f"b{i}", B, 10, {})
                                                              for i in range(6)])
    # benign side empty
    cases.append([mk(f"m{i}", M, 10, {"a": 1}) for i in range(6)] + [mk(f"b{i}", B, 10, {})
                                                                    for i in range(6)])
    # nothing trainable at all (only UNKNOWN): an empty bundle, no error
    cases.append([mk(f"u{i}", U, 10, {"a": 1}) for i in range(20)])
    for samples in cases:
        train, _ = gn.partition_by_group(samples, gn.GroupingConfig())
        for k, alpha in ((3, 1.0), (0, 1.0), (3, -1.0)):
            want = _err(lambda: gn.train_bundle(train, k, alpha, created_at="t"))
            got = _err(lambda: api.train_bundle(train, k, alpha, created_at="t"))
            assert got == want
            if want is None:
                assert gn.bundle_to_json(api.train_bundle(train, k, alpha, created_at="t")) == \
                    gn.bundle_to_json(gn.train_bundle(train, k, alpha, created_at="t"))
    only_m = [mk("m", M, 10, {"a": 1})]
    for feats, alpha in ((gn.FeatureSet(("a",), 1), 1.0), (gn.FeatureSet((), 1), 1.0),
                         (gn.FeatureSet(("a",), 1), 0)):
        assert _err(lambda: api.train_group(only_m, feats, alpha)) == \
            _err(lambda: gn.train_group(only_m, feats, alpha))
    empty = gn.build_bundle([], gn.GroupingConfig(), gn.BundleMeta(3, 1.0, 0, "t"))
    with pytest.raises(gn.errors.EmptyBundleError):
        api.classify_parallel(empty, gn.Workload((), lanes=1))


def test_hand_built_corpus_groups_by_key():
    """A GroupedCorpus whose dict keys disagree with the sizes trains by key, as
    the reference does (engine.py:170-172)."""
    corpus, train = _corpus(9, groups=3)
    moved = gn.GroupedCorpus(train.config, {g + 10: v for g, v in train.groups.items()})
    assert gn.bundle_to_json(api.train_bundle(moved, 9, created_at="t")) == \
        gn.bundle_to_json(gn.train_bundle(moved, 9, created_at="t"))
    bad = gn.GroupedCorpus(train.config, {150: train.groups[0]})
    assert _err(lambda: api.train_bundle(bad, 9, created_at="t")) == \
        _err(lambda: gn.train_bundle(bad, 9, created_at="t"))
