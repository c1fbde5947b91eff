"""Randomised K-PRED / K-FIT parity sweep on the GPU against the C oracle.

Every shape draws its own kernel path: row box (1-D bulk or 2-D tile,
resident or staged tables, 13- and 26-quad register staging), 128-B box (one
or two chunks per stage), gather4 after a slot sort, the generic L1 kernel;
int32 / uint16 / uint8 storage; 2..16 classes; packed or padded pitches;
grouped, shuffled and out-of-range sizes.  Bar: labels identical and
log-posteriors bit-identical (exact mode); fit statistics exact.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_1905_13746_b200 import dense  # noqa: E402

_DT = {0: (torch.int32, np.int32, 2**20), 1: (torch.uint16, np.uint16, 65536),
       2: (torch.uint8, np.uint8, 256)}


def _case(seed):
    rng = np.random.default_rng(seed)
    F = int(rng.choice([1, 3, 13, 31, 50, 52, 64, 77, 100, 104, 129, 200, 256, 300, 353, 500,
                        700, 1000]))
    C = int(rng.choice([2, 2, 2, 3, 4, 5, 8, 16]))
    S = int(rng.choice([1, 1, 2, 5, 29, 64]))
    G = max(S, int(rng.integers(1, 40)))
    width = int(rng.integers(1, 500))
    n = int(rng.choice([1, 127, 128, 129, 1000, 4099, 20000]))
    dk = int(rng.integers(0, 3))
    tdt, ndt, hi = _DT[dk]
    eb = np.dtype(ndt).itemsize
    q = 16 // eb
    pad = int(rng.choice([0, 0, q, 3 * q]))
    ldx = (F + q - 1) // q * q + pad
    order = str(rng.choice(["grouped", "shuffled", "sorted"]))
    return rng, F, C, S, G, width, n, tdt, ndt, hi, ldx, order


@pytest.mark.parametrize("seed", range(60))
def test_predict_fuzz(seed):
    rng, F, C, S, G, width, n, tdt, ndt, hi, ldx, order = _case(seed)
    limit = width * G
    prior = np.log(rng.dirichlet(np.ones(C), size=S))
    ll = np.log(rng.dirichlet(np.ones(F), size=(S, C)))
    route = rng.integers(0, S, size=G).astype(np.int32)
    x = rng.poisson(float(rng.choice([0.3, 2.0, 40.0])), size=(n, F)).clip(0, hi - 1).astype(ndt)
    size = rng.integers(0, limit, size=n)
    if order == "grouped":
        size = np.sort(size)
    bad = rng.random(n) < 0.02
    size[bad] = rng.choice([-1, limit, limit + 7, 2**31 - 1], size=int(bad.sum()))
    size = size.astype(np.int32)
    dev = torch.device("cuda")
    base = torch.zeros((n, ldx), dtype=tdt, device=dev)
    base[:, :F] = torch.from_numpy(x).to(dev)
    xd = base[:, :F]
    sd = torch.from_numpy(size).to(dev)
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=limit)
    perm = dense.slot_sort(sd, t) if order == "sorted" else None
    lab, lp = dense.predict(xd, sd, t, perm=perm)
    torch.cuda.synchronize()
    want, wlp = O.c_predict(x, size, route, prior, ll, width=width, limit=limit, threads=4)
    got = lab.cpu().numpy()
    assert got.tolist() == want.tolist(), (F, C, S, n, ldx, order, tdt)
    ok = want >= 0
    assert lp.cpu().numpy()[ok].tobytes() == wlp[ok].tobytes(), (F, C, S, n, ldx, order, tdt)


@pytest.mark.parametrize("seed", range(20))
def test_fit_fuzz(seed):
    rng = np.random.default_rng(1000 + seed)
    V = int(rng.choice([16, 64, 112, 128, 256, 512]))  # 16-B row pitch in every storage
    C = int(rng.choice([2, 3, 16]))
    G = int(rng.choice([1, 4, 32, 100]))
    width = int(rng.integers(1, 300))
    limit = width * G
    n = int(rng.choice([1, 127, 1000, 30000]))
    dk = int(rng.integers(0, 3))
    tdt, ndt, hi = _DT[dk]
    x = rng.poisson(float(rng.choice([0.5, 5.0])), size=(n, V)).clip(0, hi - 1).astype(np.int32)
    size = rng.integers(-3, limit + 3, size=n).astype(np.int32)
    lab = rng.integers(-1, C + 1, size=n).astype(np.int32)
    dev = torch.device("cuda")
    st = dense.fit_stats(torch.from_numpy(x).to(dev).to(tdt), torch.from_numpy(size).to(dev),
                         torch.from_numpy(lab).to(dev), n_classes=C, group_size_bytes=width,
                         max_size_bytes=limit)
    torch.cuda.synchronize()
    S, Q, cnt, _, _ = O.fit_stats(x, size, lab, C, width, limit)
    assert np.array_equal(st.sums.cpu().numpy(), S)
    assert np.array_equal(st.sumsq.cpu().numpy(), Q)
    assert np.array_equal(st.counts.cpu().numpy(), cnt)
