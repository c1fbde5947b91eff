"""Object-level drop-in (train_bundle / classify_*) vs the reference's golden outputs."""

import json

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_1905_13746_b200 as gnb  # noqa: E402
from paper_1905_13746_b200.model import Label  # noqa: E402

_CODE = {0: Label.BENIGN, 1: Label.MALWARE, -1: Label.UNKNOWN}


def _samples(z, which):
    vocab = z["vocab"].tolist()
    x = z[f"{which}_x"]
    size = z[f"{which}_size"]
    labels = z["train_label"] if which == "train" else np.full(len(size), -1)
    out = []
    for i in range(len(size)):
        nz = np.nonzero(x[i])[0]
        hist = gnb.OpcodeHistogram.from_counts({vocab[j]: int(x[i, j]) for j in nz})
        out.append(gnb.SampleRecord(f"{which}{i}", _CODE[int(labels[i])], int(size[i]), hist))
    return out


def _config(z):
    return gnb.GroupingConfig(int(z["group_size_bytes"]), int(z["max_size_bytes"]),
                              int(z["min_per_class"]))


def test_train_bundle_and_classify_match_reference(golden):
    name, z = golden
    cfg = _config(z)
    train, rejected = gnb.partition_by_group(_samples(z, "train"), cfg)
    assert not rejected
    bundle = gnb.train_bundle(train, k=int(z["k"]), alpha=float(z["alpha"]), created_at="golden")
    doc = json.loads(str(z["bundle_json"]))
    assert list(bundle.trained_ids) == [m["group"] for m in doc["models"]]
    for m in doc["models"]:
        got = bundle.models[m["group"]]
        assert list(got.features.opcodes) == m["features"]
        for c in (Label.MALWARE, Label.BENIGN):
            assert got.log_prior[c] == m["log_prior"][c.value]
            assert [got.log_likelihood[c][op] for op in m["features"]] == \
                [m["log_likelihood"][c.value][op] for op in m["features"]]
            assert got.train_counts[c] == m["train_counts"][c.value]
    test = _samples(z, "test")
    run = gnb.classify_parallel(bundle, gnb.Workload(tuple(test), lanes=4))
    for i, p in enumerate(run.predictions):
        want = int(z["pred_label"][i])
        if want < 0:
            assert p is None
            continue
        assert p.label is _CODE[want]
        assert p.log_posterior[Label.BENIGN] == z["pred_lp"][i, 0]
        assert p.log_posterior[Label.MALWARE] == z["pred_lp"][i, 1]
        assert p.effective_group == int(z["pred_group"][i])
    assert [i for i, _ in run.errors] == z["err_index"].tolist()
    assert [m for _, m in run.errors] == z["err_msg"].tolist()
    assert run.elapsed_ns > 0


def test_single_sample_entry_points():
    # pkg/tests/test_classifier.py:21-41, 116-121 worked example
    import math
    s = [gnb.SampleRecord("m", Label.MALWARE, 10, gnb.OpcodeHistogram.from_counts({"a": 2})),
         gnb.SampleRecord("b", Label.BENIGN, 11, gnb.OpcodeHistogram.from_counts({"b": 2}))]
    model = gnb.train_group(s, gnb.FeatureSet(("a", "b"), 2), 1.0, group=3)
    assert model.log_likelihood[Label.MALWARE]["a"] == math.log(3 / 4)
    assert model.log_likelihood[Label.BENIGN]["a"] == math.log(1 / 4)
    pred = gnb.predict(model, gnb.OpcodeHistogram.from_counts({"a": 1}))
    assert pred.label is Label.MALWARE and pred.effective_group == 3
    assert pred.log_posterior[Label.MALWARE] == math.log(1 / 2) + math.log(3 / 4)
    empty = gnb.log_posterior(model, gnb.OpcodeHistogram.from_counts({}))
    assert empty[Label.MALWARE] == model.log_prior[Label.MALWARE]


def test_errors_match_reference_contract():
    cfg = gnb.GroupingConfig()
    meta = gnb.BundleMeta(k=3, alpha=1.0, seed=0, created_at="t")
    empty = gnb.build_bundle([], cfg, meta)
    with pytest.raises(gnb.EmptyBundleError):
        gnb.classify_parallel(empty, gnb.Workload((), lanes=1))
    only_m = [gnb.SampleRecord("m", Label.MALWARE, 10, gnb.OpcodeHistogram.from_counts({"a": 1}))]
    with pytest.raises(gnb.InsufficientClassError):
        gnb.train_group(only_m, gnb.FeatureSet(("a",), 1), 1.0)
    with pytest.raises(gnb.InvalidConfigError):
        gnb.train_group(only_m, gnb.FeatureSet((), 1), 1.0)
    with pytest.raises(gnb.InvalidConfigError):
        gnb.Workload((), lanes=0)


def _jsonl(z, which):
    vocab = z["vocab"].tolist()
    x = z[f"{which}_x"]
    size = z[f"{which}_size"]
    labels = z["train_label"] if which == "train" else np.full(len(size), -1)
    out = []
    for i in range(len(size)):
        d = {"id": f"{which}{i}", "size_bytes": int(size[i]),
             "opcodes": {vocab[j]: int(x[i, j]) for j in np.nonzero(x[i])[0]}}
        if labels[i] >= 0:
            d["label"] = "malware" if labels[i] == 1 else "benign"
        if int(size[i]) >= 0:
            out.append(json.dumps(d))
        else:   # negative sizes are not valid JSONL records; keep them as oversize rows
            d["size_bytes"] = 10**9
            out.append(json.dumps(d))
    return "\n".join(out)


def test_dense_corpus_pipeline_matches_reference(golden):
    """JSONL -> C++ ingest -> device fit / gather / predict == reference outputs."""
    from paper_1905_13746_b200 import ingest
    from paper_1905_13746_b200.api import classify_corpus, train_bundle_corpus
    name, z = golden
    cfg = _config(z)
    train = ingest.read_corpus(_jsonl(z, "train"))
    bundle = train_bundle_corpus(train, cfg, int(z["k"]), float(z["alpha"]), created_at="g")
    doc = json.loads(str(z["bundle_json"]))
    assert list(bundle.trained_ids) == [m["group"] for m in doc["models"]]
    for m in doc["models"]:
        got = bundle.models[m["group"]]
        assert list(got.features.opcodes) == m["features"]
        for c in (Label.MALWARE, Label.BENIGN):
            assert [got.log_likelihood[c][op] for op in m["features"]] == \
                [m["log_likelihood"][c.value][op] for op in m["features"]]
    test = ingest.read_corpus(_jsonl(z, "test"), allow_unlabeled=True)
    lab, lp, eff, errors, elapsed = classify_corpus(bundle, test)
    want = z["pred_label"].astype(int)
    assert lab.tolist() == want.tolist()
    ok = want >= 0
    assert lp[ok].tobytes() == z["pred_lp"][ok].tobytes()
    assert eff[ok].tolist() == z["pred_group"][ok].tolist()
    assert [i for i, _ in errors] == np.nonzero(~ok)[0].tolist()


def test_jsonl_to_jsonl_matches_reference_bytes():
    """JSONL in -> device fit + classify -> JSONL out, byte-identical to the reference's
    train_bundle / classify_sequential / write_predictions (tests/golden/writer.npz)."""
    from conftest import load_golden
    from paper_1905_13746_b200 import ingest
    from paper_1905_13746_b200.api import classify_corpus, train_bundle_corpus
    w = load_golden("writer")
    cfg = gnb.GroupingConfig()
    bundle = train_bundle_corpus(ingest.read_corpus(str(w["train_text"])), cfg, int(w["k"]),
                                 1.0, created_at="golden")
    test = ingest.read_corpus(str(w["text_in"]), allow_unlabeled=True)
    lab, lp, eff, errors, _ = classify_corpus(bundle, test)
    assert test.predictions_jsonl(lab, lp, eff, cfg.max_size_bytes) == str(w["out"])
