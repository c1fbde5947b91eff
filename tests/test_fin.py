"""FIN (host C++ in libgnb.so) against the reference's golden bundles -- CPU only.

The sums fed to FIN here come from the oracle's exact integer fit; the GPU
fit is checked against the same oracle in test_gpu_fit.py.
"""

import json

import numpy as np
import pytest

from oracle import oracle as O
from paper_1905_13746_b200 import dense


def _ref_models(z):
    doc = json.loads(str(z["bundle_json"]))
    vocab = {op: i for i, op in enumerate(z["vocab"].tolist())}
    return {m["group"]: m for m in doc["models"]}, vocab


def test_fin_train_bit_exact(golden):
    name, z = golden
    width, limit = int(z["group_size_bytes"]), int(z["max_size_bytes"])
    S, _, n, _, _ = O.fit_stats(z["train_x"], z["train_size"], z["train_label"], 2, width, limit)
    k = int(z["k"])
    fin = dense.fin_train(S.astype(np.float64), n.astype(np.float64), k=k,
                          alpha=float(z["alpha"]), min_per_class=int(z["min_per_class"]))
    ref, vocab = _ref_models(z)
    assert sorted(np.nonzero(fin.state == 1)[0].tolist()) == sorted(ref)
    for g, m in ref.items():
        F = int(fin.n_features[g])
        assert [int(v) for v in fin.features[g, :F]] == [vocab[op] for op in m["features"]]
        assert fin.log_prior[g, 0] == m["log_prior"]["benign"]
        assert fin.log_prior[g, 1] == m["log_prior"]["malware"]
        for c, cname in ((0, "benign"), (1, "malware")):
            want = np.array([m["log_likelihood"][cname][op] for op in m["features"]])
            assert fin.log_lik[g, c, :F].tobytes() == want.tobytes()


def test_fin_insufficient_states():
    S = np.zeros((3, 2, 4))
    S[0, 0] = [1, 2, 0, 0]          # malware total 0 -> -1
    S[1, 1] = [0, 0, 3, 1]          # benign total 0 -> -2
    S[2, 0] = [1, 0, 0, 0]
    S[2, 1] = [0, 1, 0, 0]
    n = np.array([[6, 6], [6, 6], [6, 5]], dtype=np.float64)
    fin = dense.fin_train(S, n, k=2, alpha=1.0, min_per_class=6)
    assert fin.state.tolist() == [-1, -2, 0]


def test_fin_tables_multiclass_matches_oracle():
    rng = np.random.default_rng(5)
    S = rng.integers(0, 1000, size=(16, 40)).astype(np.float64)
    n = rng.integers(1, 50, size=16).astype(np.float64)
    feats = rng.choice(40, size=12, replace=False)
    prior, ll = dense.fin_tables(S, n, feats, 0.5)
    t = O.train_tables(S.astype(np.int64), n.astype(np.int64), feats, 0.5, 0)
    assert prior.tobytes() == t.log_prior.tobytes()
    assert ll.tobytes() == t.log_lik.tobytes()


@pytest.mark.parametrize("k", [1, 3, 100])
def test_fin_random_vs_oracle(k):
    rng = np.random.default_rng(k)
    for _ in range(20):
        V = int(rng.integers(1, 30))
        S = rng.integers(0, 5, size=(2, 2, V)) * rng.integers(0, 2, size=(2, 2, V))
        n = rng.integers(0, 9, size=(2, 2))
        fin = dense.fin_train(S.astype(float), n.astype(float), k=k, alpha=1.0, min_per_class=2)
        for g in range(2):
            if (n[g] < 2).any():
                assert fin.state[g] == 0
                continue
            try:
                feats, _ = O.select_features(S[g], k, g)
            except O.OracleError:
                assert fin.state[g] in (-1, -2)
                continue
            t = O.train_tables(S[g], n[g], feats, 1.0, g)
            F = len(feats)
            assert fin.state[g] == 1
            assert fin.features[g, :F].tolist() == feats.tolist()
            assert fin.log_prior[g].tobytes() == t.log_prior.tobytes()
            assert fin.log_lik[g, :, :F].tobytes() == t.log_lik.tobytes()
