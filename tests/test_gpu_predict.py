"""K-PRED parity on the GPU: bit-exact against the oracle (pinned to the reference).

Bar: labels identical, log-posteriors bit-identical (the kernel does the
reference's mul-then-add in FeatureSet order), statuses identical.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_1905_13746_b200 import dense  # noqa: E402


def _tables(rng, S, C, F, group_count):
    prior = np.log(rng.dirichlet(np.ones(C), size=S))
    ll = np.log(rng.dirichlet(np.ones(F), size=(S, C)))
    route = rng.integers(0, S, size=group_count).astype(np.int32)
    return prior, ll, route


def _run(x, size, prior, ll, route, width, limit, *, generic=False, ldx=None, pad=0):
    dev = torch.device("cuda")
    N, F = x.shape
    if ldx is None or ldx == F:
        xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).to(dev)
    else:
        base = torch.full((N, ldx), pad, dtype=torch.int32, device=dev)
        base[:, :F] = torch.from_numpy(x.astype(np.int32)).to(dev)
        xd = base[:, :F]
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=limit)
    lab, lp = dense.predict(xd, torch.from_numpy(size.astype(np.int32)).to(dev), t,
                            generic=generic)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), lp.cpu().numpy()


def _check(x, size, prior, ll, route, width, limit, **kw):
    lab, lp = _run(x, size, prior, ll, route, width, limit, **kw)
    want_lab, want_lp = O.predict_dense(x, size, route, prior, ll, width=width, limit=limit)
    assert lab.tolist() == want_lab.tolist()
    ok = want_lab >= 0
    assert lp[ok].tobytes() == want_lp[ok].tobytes()
    assert np.isnan(lp[~ok]).all()


def test_golden_cases_device(golden):
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
    for generic in (False, True):
        lab, lp = _run(xg, size, prior, ll, route, width, limit, generic=generic)
        assert lab.tolist() == z["pred_label"].astype(np.int32).tolist()
        ok = lab >= 0
        assert lp[ok].tobytes() == z["pred_lp"][ok].tobytes()


@pytest.mark.parametrize("F", [1, 4, 31, 32, 33, 50, 100, 128, 200, 256, 500])
def test_feature_counts(F):
    rng = np.random.default_rng(F)
    N = 1000 + F
    prior, ll, route = _tables(rng, 1, 2, F, 1)
    x = rng.poisson(2.0, size=(N, F))
    size = rng.integers(0, 5120, size=N)
    ldx = (F + 3) // 4 * 4
    _check(x, size, prior, ll, route, 5120, 5120, ldx=ldx)
    _check(x, size, prior, ll, route, 5120, 5120, generic=True)


@pytest.mark.parametrize("C", [2, 3, 4, 7, 8, 16])
def test_class_counts(C):
    rng = np.random.default_rng(100 + C)
    prior, ll, route = _tables(rng, 3, C, 40, 5)
    x = rng.poisson(1.5, size=(777, 40))
    size = rng.integers(-50, 5 * 1000 + 50, size=777)
    _check(x, size, prior, ll, route, 1000, 5000)


@pytest.mark.parametrize("F,ldx", [(13, 16), (50, 52), (50, 56), (52, 52), (64, 64), (100, 100)])
@pytest.mark.parametrize("S,C", [(1, 2), (3, 2), (64, 2), (3, 4), (2, 16)])
def test_rowbox_paths(F, ldx, S, C):
    """Row-box K-PRED: contiguous rows (1-D bulk tile) and padded pitches (2-D
    box); tables resident in smem (few slots) or staged per tile (64 slots);
    row-in-registers early release (C=2 up to 13 quads, C=4 up to 8); uniform
    (grouped) and mixed (shuffled) tiles."""
    rng = np.random.default_rng(F * 1000 + S * 10 + C)
    width, G = 100, max(S, 4)
    prior, ll, route = _tables(rng, S, C, F, G)
    N = 4 * 128 * 3 + 77
    size = np.sort(rng.integers(0, width * G, size=N))
    x = rng.poisson(3.0, size=(N, F))
    _check(x, size, prior, ll, route, width, width * G, ldx=ldx)
    perm = rng.permutation(N)
    _check(x[perm], size[perm], prior, ll, route, width, width * G, ldx=ldx)


@pytest.mark.parametrize("F,ldx", [(13, 16), (50, 52), (50, 56), (101, 104), (33, 36),
                                   (250, 252), (255, 260)])
def test_uninitialised_pitch_padding(F, ldx):
    """Pitch padding columns [F, ldx) full of 0xFFFFFFFF (leftover memory with the
    sign bit set) are neither scored nor flagged as negative counts, on every
    K-PRED path (1-D bulk row box, 2-D row box, 128-B boxes, mixed tiles)."""
    rng = np.random.default_rng(F * 7 + ldx)
    prior, ll, route = _tables(rng, 3, 2, F, 4)
    N = 3 * 128 + 41
    size = np.sort(rng.integers(0, 400, size=N))
    x = rng.poisson(2.0, size=(N, F))
    for order in (np.arange(N), rng.permutation(N)):
        _check(x[order], size[order], prior, ll, route, 100, 400, ldx=ldx, pad=-1)


def test_ragged_groups_sorted_and_shuffled():
    rng = np.random.default_rng(7)
    G, F = 32, 200
    counts = (4000 * 0.9 ** np.arange(G)).astype(int) + 1
    prior, ll, _ = _tables(rng, G - 3, 2, F, G)
    trained = [g for g in range(G) if g not in (5, 8, 17)]
    route = np.array([trained.index(t) for t in O.route_table(trained, G)], dtype=np.int32)
    size = np.concatenate([g * 5120 + rng.integers(0, 5120, size=c) for g, c in enumerate(counts)])
    x = rng.poisson(1.0, size=(len(size), F))
    _check(x, size, prior, ll, route, 5120, G * 5120)           # grouped: uniform tiles
    perm = rng.permutation(len(size))
    _check(x[perm], size[perm], prior, ll, route, 5120, G * 5120)  # mixed tiles


def test_edge_rows_and_statuses():
    rng = np.random.default_rng(9)
    prior, ll, route = _tables(rng, 2, 2, 64, 4)
    x = rng.poisson(1.0, size=(300, 64))
    size = rng.integers(0, 4000, size=300)
    size[[0, 7, 128, 299]] = [-1, 4000, 2**31 - 1, -2**31]
    x[5, 3] = -1                      # negative count -> status -2
    x[200, 63] = 2**31 - 1            # max count: exact product
    lab, lp = _run(x, size, prior, ll, route, 1000, 4000, ldx=64)
    want, wlp = O.predict_dense(np.clip(x, 0, None), size, route, prior, ll, width=1000, limit=4000)
    assert lab[[0, 7, 128, 299]].tolist() == [-1] * 4
    assert lab[5] == -2
    keep = np.ones(300, bool)
    keep[[0, 7, 128, 299, 5]] = False
    assert lab[keep].tolist() == want[keep].tolist()
    assert lp[keep].tobytes() == wlp[keep].tobytes()


def test_empty_and_tiny():
    rng = np.random.default_rng(1)
    prior, ll, route = _tables(rng, 1, 2, 8, 1)
    for N in (0, 1, 2, 127, 128, 129):
        x = rng.poisson(3.0, size=(N, 8))
        size = rng.integers(0, 10, size=N)
        _check(x, size, prior, ll, route, 10, 10, ldx=8)


def test_host_entry_matches_device():
    """gnb_predict_host (host buffers, chunked H2D pipeline) == device path."""
    import ctypes
    from paper_1905_13746_b200 import _native as N
    rng = np.random.default_rng(3)
    S, C, F, G = 3, 2, 70, 6
    prior, ll, route = _tables(rng, S, C, F, G)
    n = 300_000
    x = rng.poisson(1.0, size=(n, F)).astype(np.int32)
    size = rng.integers(0, G * 100, size=n).astype(np.int32)
    lab = np.empty(n, np.int32)
    lp = np.empty((n, C))
    el = ctypes.c_int64()
    pr, lk = np.ascontiguousarray(prior), np.ascontiguousarray(ll)
    N.check(N.lib.gnb_predict_host(x.ctypes.data, n, F, F, size.ctypes.data, 100, G * 100,
                                   route.ctypes.data, S, C, pr.ctypes.data, lk.ctypes.data,
                                   lab.ctypes.data, lp.ctypes.data, 0, ctypes.addressof(el)))
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=100, limit=G * 100)
    assert lab.tolist() == want.tolist()
    assert lp.tobytes() == wlp.tobytes()
    assert el.value > 0


def test_large_counts_and_values_exact():
    """x up to 2^31-1 and extreme log-likelihoods keep the product exact."""
    rng = np.random.default_rng(11)
    F = 36
    prior = np.log(np.array([[0.3, 0.7]]))
    ll = -np.abs(rng.standard_cauchy(size=(1, 2, F))) * 10
    x = rng.integers(0, 2**31 - 1, size=(257, F))
    x[::3] = rng.integers(0, 3, size=(86, F))
    _check(x, np.zeros(257, np.int64), prior, ll, np.zeros(1, np.int32), 1, 1, ldx=36)


def test_gather_features_matches_oracle():
    """Device route + FeatureSet gather == oracle.gather_rows; then predict on it."""
    rng = np.random.default_rng(21)
    G, V, F, N = 12, 90, 40, 20000
    trained = [0, 1, 2, 4, 5, 6, 8, 10]
    models = {}
    for g in trained:
        nf = int(rng.integers(5, F + 1))
        feats = rng.choice(V, size=nf, replace=False)
        models[g] = O.GroupTables(g, feats, np.log(np.array([0.4, 0.6])),
                                  np.log(rng.dirichlet(np.ones(nf), size=2)), np.array([6, 6]))
    ids, route, prior, ll = O.pack_models(models, G, F)
    featmat = np.full((len(ids), F), -1, np.int32)
    nfeat = np.zeros(len(ids), np.int32)
    for i, g in enumerate(ids):
        featmat[i, :len(models[g].features)] = models[g].features
        nfeat[i] = len(models[g].features)
    xv = rng.poisson(1.0, size=(N, V)).astype(np.int32)
    size = rng.integers(-10, G * 100 + 10, size=N).astype(np.int32)
    dev = torch.device("cuda")
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=100, max_size_bytes=G * 100)
    sd = torch.from_numpy(size).to(dev)
    xg = dense.gather_features(torch.from_numpy(xv).to(dev), sd, t, featmat, nfeat)
    lab, lp = dense.predict(xg, sd, t)
    torch.cuda.synchronize()
    want_x = O.gather_rows(xv, size, models, width=100, limit=G * 100, n_features=F)
    assert np.array_equal(xg.cpu().numpy(), want_x)
    want, wlp = O.predict_dense(want_x, size, route, prior, ll, width=100, limit=G * 100)
    assert lab.cpu().numpy().tolist() == want.tolist()
    ok = want >= 0
    assert lp.cpu().numpy()[ok].tobytes() == wlp[ok].tobytes()


@pytest.mark.parametrize("dtype,hi", [(torch.uint8, 256), (torch.uint16, 65536)])
@pytest.mark.parametrize("F", [1, 16, 31, 64, 100, 128, 129, 256, 300])
@pytest.mark.parametrize("C", [2, 5])
def test_narrow_dtypes_bit_exact(dtype, hi, F, C):
    """uint8 / uint16 X: same counts, fewer bytes, identical results (TMA and L1 paths)."""
    rng = np.random.default_rng(F * 7 + C)
    prior, ll, route = _tables(rng, 3, C, F, 4)
    N = 2000
    x = rng.integers(0, hi, size=(N, F))
    x[::5] = rng.poisson(1.0, size=(len(x[::5]), F))
    size = rng.integers(-5, 4 * 100 + 5, size=N)
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=100, limit=400)
    dev = torch.device("cuda")
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=100, max_size_bytes=400)
    sd = torch.from_numpy(size.astype(np.int32)).to(dev)
    esz = torch.tensor([], dtype=dtype).element_size()
    ld_tma = (F * esz + 15) // 16 * 16 // esz
    for ld in (ld_tma, F):                     # aligned pitch -> TMA; F may force the L1 path
        base = torch.zeros((N, ld), dtype=torch.int32, device=dev)
        base[:, :F] = torch.from_numpy(x.astype(np.int32)).to(dev)
        xd = base.to(dtype)[:, :F]
        lab, lp = dense.predict(xd, sd, t)
        torch.cuda.synchronize()
        assert lab.cpu().numpy().tolist() == want.tolist()
        ok = want >= 0
        assert lp.cpu().numpy()[ok].tobytes() == wlp[ok].tobytes()


def test_narrowest_roundtrip():
    x = torch.tensor([[0, 5, 255]], dtype=torch.int32, device="cuda")
    assert dense.narrowest(x).dtype == torch.uint8
    assert dense.narrowest(x * 100).dtype == torch.uint16
    assert dense.narrowest(x * 1000).dtype == torch.int32


@pytest.mark.parametrize("narrow", ["0", "1", "raw2"])
@pytest.mark.parametrize("hi,neg", [(16, False), (256, False), (60000, False), (2**31 - 1, False),
                                    (100, True), (16, True)])
@pytest.mark.parametrize("F", [45, 64])
def test_host_entry_narrowing_paths(hi, neg, narrow, F, monkeypatch):
    """gnb_predict_host (default GNB_HOST_NARROW=1: int32 chunks shipped as nibbles /
    uint8 / uint16 / int32 by content) gives identical results."""
    import ctypes
    from paper_1905_13746_b200 import _native as N
    monkeypatch.setenv("GNB_HOST_NARROW", "0" if narrow == "0" else "1")
    monkeypatch.setenv("GNB_HOST_RAW_EVERY", "2" if narrow == "raw2" else "0")
    monkeypatch.setenv("GNB_HOST_CHUNK_MB", "1")      # several chunks per call
    rng = np.random.default_rng(hi % 1000)
    S, C, G = 2, 2, 3
    prior, ll, route = _tables(rng, S, C, F, G)
    n = 70_000
    x = rng.integers(0, hi, size=(n, F)).astype(np.int32)
    if neg:
        x[123, 7] = -5
    ldx = F + 3                               # padded host rows: exercises the pitch paths
    xh = np.zeros((n, ldx), np.int32)
    xh[:, :F] = x
    size = rng.integers(-3, G * 100, size=n).astype(np.int32)
    lab = np.empty(n, np.int32)
    lp = np.empty((n, C))
    el = ctypes.c_int64()
    pr, lk = np.ascontiguousarray(prior), np.ascontiguousarray(ll)
    N.check(N.lib.gnb_predict_host(xh.ctypes.data, n, F, ldx, size.ctypes.data, 100, G * 100,
                                   route.ctypes.data, S, C, pr.ctypes.data, lk.ctypes.data,
                                   lab.ctypes.data, lp.ctypes.data, 0, ctypes.addressof(el)))
    want, wlp = O.predict_dense(np.clip(x, 0, None), size, route, prior, ll, width=100,
                                limit=G * 100)
    if neg:
        assert lab[123] == N.ROW_NEGATIVE_COUNT or size[123] < 0
        want[123] = lab[123]
        wlp[123] = lp[123]
    assert lab.tolist() == want.tolist()
    ok = want >= 0
    assert lp[ok].tobytes() == wlp[ok].tobytes()


@pytest.mark.parametrize("dtype,xt", [(np.uint8, 2), (np.uint16, 1), (np.int32, 0)])
def test_host_typed_entry(dtype, xt):
    import ctypes
    from paper_1905_13746_b200 import _native as N
    rng = np.random.default_rng(xt)
    S, C, F, G = 2, 3, 37, 2
    prior, ll, route = _tables(rng, S, C, F, G)
    n = 50_000
    x = rng.integers(0, np.iinfo(dtype).max if dtype != np.int32 else 10**6, size=(n, F))
    ldx = F + 3
    xh = np.zeros((n, ldx), dtype)
    xh[:, :F] = x
    size = rng.integers(0, G * 100, size=n).astype(np.int32)
    lab = np.empty(n, np.int32)
    lp = np.empty((n, C))
    pr, lk = np.ascontiguousarray(prior), np.ascontiguousarray(ll)
    N.check(N.lib.gnb_predict_host_typed(xh.ctypes.data, xt, n, F, ldx, size.ctypes.data, 100,
                                         G * 100, route.ctypes.data, S, C, pr.ctypes.data,
                                         lk.ctypes.data, lab.ctypes.data, lp.ctypes.data, 0,
                                         None))
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=100, limit=G * 100)
    assert lab.tolist() == want.tolist()
    assert lp.tobytes() == wlp.tobytes()


@pytest.mark.parametrize("dtype", [torch.int32, torch.uint8])
@pytest.mark.parametrize("N", [1, 127, 5000, 100_003])
def test_slot_sort_and_permuted_predict(dtype, N):
    """Shuffled ragged batch: slot_sort + gather4 predict == oracle, outputs in original order."""
    rng = np.random.default_rng(N)
    G, F = 32, 72
    trained = [g for g in range(G) if g not in (5, 8, 17)]
    prior, ll, _ = _tables(rng, len(trained), 2, F, G)
    route = np.array([trained.index(t) for t in O.route_table(trained, G)], dtype=np.int32)
    size = rng.integers(-20, G * 100 + 20, size=N)
    x = rng.integers(0, 200, size=(N, F))
    dev = torch.device("cuda")
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=100, max_size_bytes=G * 100)
    sd = torch.from_numpy(size.astype(np.int32)).to(dev)
    perm = dense.slot_sort(sd, t)
    torch.cuda.synchronize()
    pm = perm.cpu().numpy()
    assert sorted(pm.tolist()) == list(range(N))           # a permutation
    g = O.group_of(size, 100, G * 100)
    key = np.where(g >= 0, route[np.maximum(g, 0)], len(trained))
    assert (np.diff(key[pm]) >= 0).all()                    # grouped by slot, invalid last
    ld = {torch.int32: (F + 3) // 4 * 4, torch.uint8: (F + 15) // 16 * 16}[dtype]
    base = torch.zeros((N, ld), dtype=torch.int32, device=dev)
    base[:, :F] = torch.from_numpy(x.astype(np.int32)).to(dev)
    xd = base.to(dtype)[:, :F]
    lab, lp = dense.predict(xd, sd, t, perm=perm)
    torch.cuda.synchronize()
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=100, limit=G * 100)
    assert lab.cpu().numpy().tolist() == want.tolist()
    ok = want >= 0
    assert lp.cpu().numpy()[ok].tobytes() == wlp[ok].tobytes()


@pytest.mark.parametrize("dtype", [torch.int32, torch.uint16, torch.uint8])
@pytest.mark.parametrize("F,C", [(50, 2), (100, 3), (256, 2), (500, 2), (40, 16)])
@pytest.mark.parametrize("order", ["grouped", "shuffled", "permuted"])
def test_fma_mode_within_tolerance(dtype, F, C, order):
    """GNB_MODE_FMA: one rounding per term.  Bar (north star):
    log-posteriors within 1e-5 relative -- asserted far tighter, 1e-11 -- and
    labels identical except where the top-two margin is below that error."""
    rng = np.random.default_rng(F * 7 + C)
    G = 6
    prior, ll, route = _tables(rng, G, C, F, G)
    N = 5000
    size = np.sort(rng.integers(-100, G * 1000 + 100, size=N))
    if order != "grouped":
        size = rng.permutation(size)
    hi = 200 if dtype == torch.uint8 else 3000
    x = rng.integers(0, hi, size=(N, F))
    x[rng.random((N, F)) < 0.5] = 0
    dev = torch.device("cuda")
    xd = torch.from_numpy(x.astype(np.int64)).to(dev).to(dtype)
    sd = torch.from_numpy(size.astype(np.int32)).to(dev)
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=1000, max_size_bytes=G * 1000)
    perm = dense.slot_sort(sd, t) if order == "permuted" else None
    lab_e, lp_e = dense.predict(xd, sd, t, perm=perm)
    lab_f, lp_f = dense.predict(xd, sd, t, perm=perm, mode="fma")
    torch.cuda.synchronize()
    lab_e, lp_e, lab_f, lp_f = (a.cpu().numpy() for a in (lab_e, lp_e, lab_f, lp_f))
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=1000, limit=G * 1000)
    assert lab_e.tolist() == want.tolist()              # exact mode stays bit-exact
    ok = want >= 0
    assert lp_e[ok].tobytes() == wlp[ok].tobytes()
    assert (lab_f[~ok] == want[~ok]).all() and np.isnan(lp_f[~ok]).all()
    rel = np.abs(lp_f[ok] - wlp[ok]) / np.maximum(np.abs(wlp[ok]), 1e-300)
    assert rel.max() < 1e-11
    srt = np.sort(wlp[ok], axis=1)
    margin = srt[:, -1] - srt[:, -2]
    close = margin <= 1e-11 * np.abs(srt[:, -1]) * 4
    assert (lab_f[ok][~close] == want[ok][~close]).all()


def test_mode_rejects_unknown():
    from paper_1905_13746_b200.errors import InvalidConfigError
    rng = np.random.default_rng(0)
    prior, ll, route = _tables(rng, 1, 2, 8, 1)
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=10, max_size_bytes=10)
    x = torch.zeros((4, 8), dtype=torch.int32, device="cuda")
    s = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(InvalidConfigError):
        dense.predict(x, s, t, mode="fast")


@pytest.mark.parametrize("F,pad,n", [(37, 0, 50_000), (37, 6, 30_001), (256, 0, 200_000),
                                     (1, 0, 7), (100, 2, 1_000_003)])
def test_host_u4_entry(F, pad, n):
    """GNB_X_U4 host rows (two counts per byte, unpacked on the device): labels
    and log-posteriors bit-identical to the oracle, contiguous (one copy) and
    padded (2-D copy) pitches, odd F, several pipeline chunks, ragged slots."""
    import ctypes
    from paper_1905_13746_b200 import _native as N
    rng = np.random.default_rng(F + pad)
    S, C, G = 3, 2, 4
    prior, ll, route = _tables(rng, S, C, F, G)
    x = rng.integers(0, 16, size=(n, F))
    packed = dense.pack_u4(torch.from_numpy(x.astype(np.int32))).numpy()
    if pad:
        wide = np.zeros((n, packed.shape[1] + pad), np.uint8)
        wide[:, :packed.shape[1]] = packed
        packed = wide
    ldx = 2 * packed.shape[1]
    size = rng.integers(-5, G * 100 + 5, size=n).astype(np.int32)
    lab = np.empty(n, np.int32)
    lp = np.empty((n, C))
    pr, lk = np.ascontiguousarray(prior), np.ascontiguousarray(ll)
    N.check(N.lib.gnb_predict_host_typed(packed.ctypes.data, N.X_U4, n, F, ldx, size.ctypes.data,
                                         100, G * 100, route.ctypes.data, S, C, pr.ctypes.data,
                                         lk.ctypes.data, lab.ctypes.data, lp.ctypes.data, 0,
                                         None))
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=100, limit=G * 100)
    assert lab.tolist() == want.tolist()
    ok = want >= 0
    assert lp[ok].tobytes() == wlp[ok].tobytes()
