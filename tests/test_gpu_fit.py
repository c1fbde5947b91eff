"""K-FIT parity on the GPU: exact integer statistics vs the oracle."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_1905_13746_b200 import dense  # noqa: E402


def _fit(x, size, label, C, width, limit, ldx=None, sumsq=True):
    dev = torch.device("cuda")
    N, V = x.shape
    ld = ldx or (V + 3) // 4 * 4
    base = torch.zeros((N, ld), dtype=torch.int32, device=dev)
    base[:, :V] = torch.from_numpy(x.astype(np.int32)).to(dev)
    st = dense.fit_stats(base[:, :V], torch.from_numpy(size.astype(np.int32)).to(dev),
                         torch.from_numpy(label.astype(np.int32)).to(dev), n_classes=C,
                         group_size_bytes=width, max_size_bytes=limit, sumsq=sumsq)
    torch.cuda.synchronize()
    return st


def _check(x, size, label, C, width, limit, **kw):
    st = _fit(x, size, label, C, width, limit, **kw)
    S, Q, n, bad, oor = O.fit_stats(x, size, label, C, width, limit)
    assert np.array_equal(st.sums.cpu().numpy(), S.astype(np.float64))
    if st.sumsq is not None:
        assert np.array_equal(st.sumsq.cpu().numpy(), Q.astype(np.float64))
    assert np.array_equal(st.counts.cpu().numpy(), n.astype(np.float64))
    assert st.status.cpu().tolist() == [bad, oor]


def test_golden_training_sets(golden):
    _, z = golden
    _check(z["train_x"], z["train_size"], z["train_label"], 2,
           int(z["group_size_bytes"]), int(z["max_size_bytes"]))


@pytest.mark.parametrize("V", [1, 5, 32, 33, 64, 100, 128, 256, 1000])
def test_vocab_sizes(V):
    rng = np.random.default_rng(V)
    N = 3000
    x = rng.poisson(2.0, size=(N, V))
    size = rng.integers(0, 5120, size=N)
    label = rng.integers(0, 2, size=N)
    _check(x, size, label, 2, 5120, 5120)


@pytest.mark.parametrize("C", [2, 3, 16])
def test_classes_groups_and_bad_rows(C):
    rng = np.random.default_rng(C)
    N, V, G = 5000, 128, 7
    x = rng.poisson(1.0, size=(N, V))
    size = rng.integers(-100, G * 1000 + 100, size=N)
    label = rng.integers(-1, C + 1, size=N)
    _check(x, size, label, C, 1000, G * 1000)


def test_many_keys_spill_to_global():
    """G*C*V larger than shared memory: keys beyond the smem cap use global atomics."""
    rng = np.random.default_rng(4)
    N, V, G = 20000, 256, 100
    x = rng.poisson(0.5, size=(N, V))
    size = rng.integers(0, 512000, size=N)
    label = rng.integers(0, 2, size=N)
    _check(x, size, label, 2, 5120, 512000)


def test_large_values_exact():
    rng = np.random.default_rng(8)
    x = rng.integers(0, 2**20, size=(4096, 40))
    _check(x, np.zeros(4096, np.int64), rng.integers(0, 2, size=4096), 2, 1, 1)


def test_accumulate_over_chunks_equals_one_pass():
    rng = np.random.default_rng(12)
    N, V = 10000, 96
    x = rng.poisson(1.0, size=(N, V)).astype(np.int32)
    size = rng.integers(0, 3000, size=N).astype(np.int32)
    label = rng.integers(0, 2, size=N).astype(np.int32)
    dev = torch.device("cuda")
    xd, sd, ld = (torch.from_numpy(a).to(dev) for a in (x, size, label))
    whole = dense.fit_stats(xd, sd, ld, n_classes=2, group_size_bytes=1000, max_size_bytes=3000)
    acc = None
    for lo in range(0, N, 3333):
        acc = dense.fit_stats(xd[lo:lo + 3333], sd[lo:lo + 3333], ld[lo:lo + 3333], n_classes=2,
                              group_size_bytes=1000, max_size_bytes=3000, out=acc,
                              accumulate=acc is not None)
    torch.cuda.synchronize()
    assert torch.equal(whole.sums, acc.sums) and torch.equal(whole.counts, acc.counts)
    assert torch.equal(whole.sumsq, acc.sumsq)


@pytest.mark.parametrize("dtype,hi", [(torch.uint8, 256), (torch.uint16, 65536)])
@pytest.mark.parametrize("V", [1, 33, 64, 100, 128, 129, 256, 300])
@pytest.mark.parametrize("C", [2, 16])
def test_narrow_storage_fit(dtype, hi, V, C):
    """uint8 / uint16 X: identical statistics to the int32 oracle."""
    rng = np.random.default_rng(V * 3 + C)
    N, G = 4000, 3
    x = rng.integers(0, hi, size=(N, V))
    size = rng.integers(-10, G * 100 + 10, size=N)
    label = rng.integers(-1, C + 1, size=N)
    dev = torch.device("cuda")
    esz = torch.tensor([], dtype=dtype).element_size()
    ld = (V * esz + 15) // 16 * 16 // esz
    base = torch.zeros((N, ld), dtype=torch.int32, device=dev)
    base[:, :V] = torch.from_numpy(x.astype(np.int32)).to(dev)
    xd = base.to(dtype)[:, :V]
    st = dense.fit_stats(xd, torch.from_numpy(size.astype(np.int32)).to(dev),
                         torch.from_numpy(label.astype(np.int32)).to(dev), n_classes=C,
                         group_size_bytes=100, max_size_bytes=G * 100)
    torch.cuda.synchronize()
    S, Q, n, bad, oor = O.fit_stats(x, size, label, C, 100, G * 100)
    assert np.array_equal(st.sums.cpu().numpy(), S.astype(np.float64))
    assert np.array_equal(st.sumsq.cpu().numpy(), Q.astype(np.float64))
    assert np.array_equal(st.counts.cpu().numpy(), n.astype(np.float64))
    assert st.status.cpu().tolist() == [bad, oor]


@pytest.mark.parametrize("V,G,k", [(1, 1, 1), (40, 3, 15), (256, 1, 100), (1000, 32, 200),
                                   (5000, 4, 300), (16384, 2, 64)])
def test_device_fin_matches_host_fin(V, G, k):
    """Device scoring + top-k (bitonic sort) == host FIN == the oracle's
    select_features / train_tables (pinned to the reference) at every V."""
    rng = np.random.default_rng(V + G)
    S = rng.integers(0, 50, size=(G, 2, V)) * (rng.random((G, 2, V)) < 0.7)
    half = V // 2
    S[:, :, 1:2 * half:2] = S[:, :, 0:2 * half:2]                 # plenty of score ties
    n = rng.integers(0, 12, size=(G, 2))
    if G > 2:
        S[1, 1] = 0                                                # insufficient malware
    st = dense.FitStats(torch.from_numpy(S.astype(np.float64)).cuda(), None,
                        torch.from_numpy(n.astype(np.float64)).cuda(),
                        torch.zeros(2, dtype=torch.int64, device="cuda"))
    dev = dense.fin_train_device(st, k=k, alpha=1.0, min_per_class=3)
    host = dense.fin_train(S.astype(np.float64), n.astype(np.float64), k=k, alpha=1.0,
                           min_per_class=3)
    assert dev.state.tolist() == host.state.tolist()
    assert dev.n_features.tolist() == host.n_features.tolist()
    for g in range(G):
        F = int(host.n_features[g])
        assert dev.features[g, :F].tolist() == host.features[g, :F].tolist()
    assert dev.log_prior.tobytes() == host.log_prior.tobytes()
    assert dev.log_lik.tobytes() == host.log_lik.tobytes()
    # the oracle: (benign, malware) class order, exact integer sums
    for g in range(G):
        if host.state[g] == 0:
            assert O.trainable(n[g:g + 1].astype(np.int64), 3) == []
            continue
        if host.state[g] < 0:
            with pytest.raises(O.OracleError):
                O.select_features(S[g].astype(np.int64), k, g)
            continue
        feats, _ = O.select_features(S[g].astype(np.int64), k, g)
        F = int(host.n_features[g])
        assert feats.tolist() == dev.features[g, :F].tolist()
        t = O.train_tables(S[g].astype(np.int64), n[g].astype(np.int64), feats, 1.0, g)
        assert t.log_prior.tobytes() == dev.log_prior[g].tobytes()
        assert t.log_lik.tobytes() == np.ascontiguousarray(dev.log_lik[g, :, :F]).tobytes()


def test_library_comms_allreduce_single_device():
    """gnb_comms_* / gnb_fit_allreduce (NCCL, dlopen'ed) on the one GPU of this
    box: local communicator and rank communicator of size 1; the SUM of one
    device's statistics is those statistics, bit for bit."""
    from paper_1905_13746_b200.sharding import Comms
    dev = torch.device("cuda")
    x, size, lab = dense.generate(5000, 64, n_classes=3, seed=5, device=dev)
    st = dense.fit_stats(x, size, lab, n_classes=3, group_size_bytes=5120, max_size_bytes=5120)
    want = st.packed().clone()
    c = Comms.local([torch.cuda.current_device()])
    assert len(c) == 1
    c.allreduce([st])
    torch.cuda.synchronize()
    assert torch.equal(st.packed(), want)
    c.close()
    r = Comms.rank(1, 0, Comms.unique_id(), torch.cuda.current_device())
    r.allreduce([st])
    torch.cuda.synchronize()
    assert torch.equal(st.packed(), want)
    r.close()
