"""The C oracle (CPU baseline) equals the numpy oracle (pinned to the reference) bit-for-bit."""

import numpy as np
import pytest

from oracle import oracle as O


@pytest.mark.parametrize("threads", [1, 4])
@pytest.mark.parametrize("C", [2, 5])
def test_c_predict_matches_numpy(threads, C):
    rng = np.random.default_rng(C * 10 + threads)
    S, F, G = 3, 37, 6
    prior = np.log(rng.dirichlet(np.ones(C), size=S))
    ll = np.log(rng.dirichlet(np.ones(F), size=(S, C)))
    route = rng.integers(0, S, size=G).astype(np.int32)
    x = rng.poisson(2.0, size=(2001, F))
    size = rng.integers(-5, G * 10 + 5, size=2001)
    lab, lp = O.c_predict(x, size, route, prior, ll, width=10, limit=G * 10, threads=threads)
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=10, limit=G * 10)
    assert lab.tolist() == want.tolist()
    assert lp.tobytes() == wlp.tobytes()


def test_c_fit_matches_numpy():
    rng = np.random.default_rng(2)
    x = rng.poisson(3.0, size=(3000, 21))
    size = rng.integers(-5, 50, size=3000)
    label = rng.integers(-1, 4, size=3000)
    a = O.c_fit_stats(x, size, label, 3, 10, 40)
    b = O.fit_stats(x, size, label, 3, 10, 40)
    for u, v in zip(a, b):
        assert np.array_equal(np.asarray(u), np.asarray(v))


def test_c_predict_golden(golden):
    name, z = golden
    width, limit = int(z["group_size_bytes"]), int(z["max_size_bytes"])
    models = O.train_bundle_dense(z["train_x"], z["train_size"], z["train_label"],
                                  len(z["vocab"]), width=width, limit=limit,
                                  min_per_class=int(z["min_per_class"]), k=int(z["k"]),
                                  alpha=float(z["alpha"]))
    F = max(len(t.features) for t in models.values())
    ids, route, prior, ll = O.pack_models(models, limit // width, F)
    xg = O.gather_rows(z["test_x"].astype(np.int64), z["test_size"], models,
                       width=width, limit=limit, n_features=F)
    size = np.clip(z["test_size"], -1, 2**31 - 1)
    lab, lp = O.c_predict(xg, size, route, prior, ll, width=width, limit=limit, threads=3)
    assert lab.tolist() == z["pred_label"].astype(np.int32).tolist()
    ok = lab >= 0
    assert lp[ok].tobytes() == z["pred_lp"][ok].tobytes()


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16])
def test_c_predict_narrow_storage(dtype):
    rng = np.random.default_rng(4)
    prior = np.log(rng.dirichlet(np.ones(2), size=2))
    ll = np.log(rng.dirichlet(np.ones(30), size=(2, 2)))
    route = np.array([0, 1, 1], np.int32)
    x = rng.integers(0, np.iinfo(dtype).max, size=(999, 30))
    size = rng.integers(-2, 31, size=999)
    a = O.c_predict(x.astype(dtype), size, route, prior, ll, width=10, limit=30, threads=3)
    b = O.predict_dense(x, size, route, prior, ll, width=10, limit=30)
    assert a[0].tolist() == b[0].tolist()
    assert a[1].tobytes() == b[1].tobytes()
