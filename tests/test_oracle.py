"""Pin the CPU oracle to the reference: golden vectors made by the reference itself.

Fixtures: tests/golden/*.npz from tests/golden/make_golden.py, which runs the
reference's train_bundle (engine.py:157) and classify_sequential
(engine.py:209).  Everything here is bit-exact (==, not approx).
"""

import json

import numpy as np
import pytest

from oracle import oracle as O


def _golden_models(z):
    """Parse the reference's bundle JSON into {group: (features, prior[b,m], ll[b|m, F], counts)}."""
    doc = json.loads(str(z["bundle_json"]))
    vocab = {op: i for i, op in enumerate(z["vocab"].tolist())}
    out = {}
    for m in doc["models"]:
        feats = np.array([vocab[op] for op in m["features"]])
        prior = np.array([m["log_prior"]["benign"], m["log_prior"]["malware"]])
        ll = np.array([[m["log_likelihood"][c][op] for op in m["features"]]
                       for c in ("benign", "malware")])
        counts = np.array([m["train_counts"]["benign"], m["train_counts"]["malware"]])
        out[m["group"]] = (feats, prior, ll, counts)
    return doc, out


def _fit(z):
    return O.train_bundle_dense(
        z["train_x"], z["train_size"], z["train_label"], len(z["vocab"]),
        width=int(z["group_size_bytes"]), limit=int(z["max_size_bytes"]),
        min_per_class=int(z["min_per_class"]), k=int(z["k"]), alpha=float(z["alpha"]))


def test_fit_matches_reference_bundle(golden):
    name, z = golden
    doc, ref = _golden_models(z)
    got = _fit(z)
    assert sorted(got) == sorted(ref)
    for g, (feats, prior, ll, counts) in ref.items():
        t = got[g]
        assert t.features.tolist() == feats.tolist(), (name, g)
        assert t.log_prior.tobytes() == prior.tobytes(), (name, g)
        assert t.log_lik.tobytes() == ll.tobytes(), (name, g)
        assert t.train_counts.tolist() == counts.tolist()


def test_predict_matches_reference_predictions(golden):
    name, z = golden
    _, ref = _golden_models(z)
    models = _fit(z)
    width, limit = int(z["group_size_bytes"]), int(z["max_size_bytes"])
    F = max(len(t.features) for t in models.values())
    ids, route, prior, ll = O.pack_models(models, limit // width, F)
    xg = O.gather_rows(z["test_x"].astype(np.int64), z["test_size"], models,
                       width=width, limit=limit, n_features=F)
    label, lp = O.predict_dense(xg, z["test_size"], route, prior, ll, width=width, limit=limit)
    assert label.tolist() == z["pred_label"].astype(np.int32).tolist()
    ok = label >= 0
    assert lp[ok].tobytes() == z["pred_lp"][ok].tobytes()
    g = O.group_of(z["test_size"], width, limit)
    eff = np.where(ok, np.array(ids)[route[np.maximum(g, 0)]], -1)
    assert eff.tolist() == z["pred_group"].tolist()
    msgs = [O.oversize_message(int(z["test_size"][i]), limit) for i in np.nonzero(~ok)[0]]
    assert msgs == z["err_msg"].tolist()
    assert np.nonzero(~ok)[0].tolist() == z["err_index"].tolist()


@pytest.mark.parametrize("query,expected", [(2, 2), (3, 4), (6, 4), (0, 1), (1, 1)])
def test_route_known_answers(query, expected):
    # pkg/tests/test_engine.py:117-121
    assert O.route_table([1, 2, 4], 100)[query] == expected


def test_route_linear_scan():
    # pkg/tests/test_engine.py:123-133
    rng = np.random.default_rng(47)
    for _ in range(30):
        ids = sorted(int(g) for g in rng.choice(100, size=int(rng.integers(1, 8)), replace=False))
        table = O.route_table(ids, 100)
        for g in range(100):
            higher = [i for i in ids if i >= g]
            assert table[g] == (min(higher) if higher else max(ids))


def test_fit_stats_sums_and_squares():
    rng = np.random.default_rng(3)
    x = rng.integers(0, 50, size=(500, 7))
    size = rng.integers(-100, 30000, size=500)
    label = rng.integers(-1, 4, size=500)
    S, Q, n, bad, oor = O.fit_stats(x, size, label, 3, 5120, 25600)
    g = O.group_of(size, 5120, 25600)
    for gg in range(5):
        for c in range(3):
            m = (g == gg) & (label == c)
            assert (S[gg, c] == x[m].sum(0)).all()
            assert (Q[gg, c] == (x[m] ** 2).sum(0)).all()
            assert n[gg, c] == m.sum()
    assert oor == int((g < 0).sum())
    assert bad == int(((g >= 0) & ((label < 0) | (label >= 3))).sum())


def test_worked_example_train_and_score():
    # pkg/tests/test_classifier.py:21-41, 116-121: malware {a:2}, benign {b:2}, features (a, b)
    S_g = np.array([[0, 2], [2, 0]])            # [benign, malware] x [a, b]
    t = O.train_tables(S_g, np.array([1, 1]), np.array([0, 1]), 1.0, 3)
    import math
    assert t.log_lik[1].tolist() == [math.log(3 / 4), math.log(1 / 4)]
    assert t.log_lik[0].tolist() == [math.log(1 / 4), math.log(3 / 4)]
    label, lp = O.predict_dense(np.array([[1, 0]]), np.array([10]), np.zeros(100, np.int32),
                                t.log_prior[None], t.log_lik[None], width=5120, limit=512000)
    assert label.tolist() == [1]
    assert lp[0, 1] == math.log(0.5) + 1 * math.log(3 / 4)


def test_tie_goes_to_benign():
    # pkg/tests/test_classifier.py:162-170
    S_g = np.array([[1, 1], [1, 1]])
    t = O.train_tables(S_g, np.array([1, 1]), np.array([0, 1]), 1.0, 0)
    label, lp = O.predict_dense(np.array([[4, 0]]), np.array([10]), np.zeros(100, np.int32),
                                t.log_prior[None], t.log_lik[None], width=5120, limit=512000)
    assert lp[0, 0] == lp[0, 1] and label.tolist() == [0]
