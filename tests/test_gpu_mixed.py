"""Mixed-slot K-PRED (predict_mixed_kernel): rows of many size groups in any
order, every slot's table resident in shared memory, each tile's rows sorted by
routed slot inside the CTA.  Bit-exact against the oracle (pinned to the
reference's per-file loop, engine.py:198-205 / classifier.py:132-158).
"""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_1905_13746_b200 import dense  # noqa: E402
from paper_1905_13746_b200._native import lib  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tables(rng, S, C, F, G):
    prior = np.log(rng.dirichlet(np.ones(C), size=S))
    ll = np.log(rng.dirichlet(np.ones(F), size=(S, C)))
    route = rng.integers(0, S, size=G).astype(np.int32)
    route[:S] = np.arange(S)  # every slot reachable
    return prior, ll, route


def _check(x, size, prior, ll, route, width, limit, dtype=torch.int32, ldx=None):
    dev = torch.device("cuda")
    N, F = x.shape
    ld = ldx or F
    base = torch.zeros((N, ld), dtype=torch.int64, device=dev)
    base[:, :F] = torch.from_numpy(x.astype(np.int64)).to(dev)
    xd = base.to(dtype)[:, :F]
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=limit)
    lab, lp = dense.predict(xd, torch.from_numpy(size.astype(np.int32)).to(dev), t)
    torch.cuda.synchronize()
    lab, lp = lab.cpu().numpy(), lp.cpu().numpy()
    want, wlp = O.predict_dense(np.clip(x, 0, None), size, route, prior, ll, width=width,
                                limit=limit)
    neg = (x < 0).any(axis=1)
    want = np.where(neg & (want >= 0), -2, want)
    assert lab.tolist() == want.tolist()
    ok = want >= 0
    assert lp[ok].tobytes() == wlp[ok].tobytes()
    assert np.isnan(lp[want == -1]).all()
    return lab


def _mixed_rows(F, x_type, C, S):
    return lib.gnb_predict_mixed_rows(F, x_type, C, S)


@pytest.mark.parametrize("S,F", [(2, 105), (5, 200), (29, 200), (64, 128), (200, 33 * 4)])
@pytest.mark.parametrize("N", [1, 255, 256, 257, 20_000])
def test_shuffled_many_slots(S, F, N):
    """Rows of S slots shuffled; sizes out of range on both sides; partial last tile."""
    rng = np.random.default_rng(S * 1000 + F + N)
    G = S + 3
    width = 100
    prior, ll, route = _tables(rng, S, 2, F, G)
    size = rng.integers(-30, G * width + 30, size=N)
    x = rng.poisson(2.0, size=(N, F))
    _check(x, size, prior, ll, route, width, G * width, ldx=(F + 3) // 4 * 4)


@pytest.mark.parametrize("S,F,dtype", [(29, 200, torch.int32), (7, 105, torch.int32),
                                         (40, 300, torch.uint8), (3, 33, torch.int32),
                                         (72, 105, torch.int32)])
def test_many_tiles_per_cta(S, F, dtype):
    """Several tiles per persistent CTA (the header ring and the stage ring wrap
    many times): every row of a shuffled ragged batch vs the C oracle."""
    rng = np.random.default_rng(S + F)
    G, width = S + 2, 100
    prior, ll, route = _tables(rng, S, 2, F, G)
    N = 148 * 256 * 5 + 77
    size = rng.integers(-10, G * width + 10, size=N)
    hi = 255 if dtype == torch.uint8 else 40
    x = rng.integers(0, hi, size=(N, F))
    x[rng.random((N, F)) < 0.5] = 0
    dev = torch.device("cuda")
    ld = {torch.int32: (F + 3) // 4 * 4, torch.uint8: (F + 15) // 16 * 16}[dtype]
    base = torch.zeros((N, ld), dtype=torch.int32, device=dev)
    base[:, :F] = torch.from_numpy(x.astype(np.int32)).to(dev)
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=G * width)
    lab, lp = dense.predict(base.to(dtype)[:, :F], torch.from_numpy(size.astype(np.int32)).to(dev), t)
    want, wlp = O.c_predict(x.astype(np.int32), size.astype(np.int32), route, prior, ll,
                            width=width, limit=G * width, threads=8)
    lab, lp = lab.cpu().numpy(), lp.cpu().numpy()
    assert lab.tolist() == want.tolist()
    ok = want >= 0
    assert lp[ok].tobytes() == wlp[ok].tobytes()


@pytest.mark.parametrize("order_hint", ["auto", "grouped", "mixed"])
@pytest.mark.parametrize("rows", ["grouped", "shuffled", "one_slot_mixed"])
def test_order_hints_give_identical_results(order_hint, rows):
    """GNB_ORDER_AUTO (device tile-mix count gating the two kernels), GROUPED
    and MIXED hints, on grouped and shuffled rows: all equal the oracle."""
    rng = np.random.default_rng(17)
    S, G, F, width = 29, 32, 200, 100
    prior, ll, route = _tables(rng, S, 2, F, G)
    N = 148 * 256 * 2 + 99
    size = np.sort(rng.integers(-5, G * width + 5, size=N))
    if rows == "shuffled":
        size = rng.permutation(size)
    if rows == "one_slot_mixed":  # all rows in one group except a few strays
        size = np.full(N, 50)
        size[rng.choice(N, 40, replace=False)] = 250
    x = rng.integers(0, 30, size=(N, F))
    dev = torch.device("cuda")
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=G * width)
    lab, lp = dense.predict(torch.from_numpy(x.astype(np.int32)).to(dev),
                            torch.from_numpy(size.astype(np.int32)).to(dev), t, order=order_hint)
    want, wlp = O.c_predict(x.astype(np.int32), size.astype(np.int32), route, prior, ll,
                            width=width, limit=G * width, threads=8)
    lab, lp = lab.cpu().numpy(), lp.cpu().numpy()
    assert lab.tolist() == want.tolist()
    ok = want >= 0
    assert lp[ok].tobytes() == wlp[ok].tobytes()


def test_mixed_hint_sorts_when_kernel_does_not_apply():
    """order="mixed" on a shape without the mixed-slot kernel (C = 3) takes the
    device slot sort + gather4 path; same results as the oracle."""
    rng = np.random.default_rng(23)
    S, G, F, width = 5, 8, 200, 100
    prior, ll, route = _tables(rng, S, 3, F, G)
    N = 20_000
    size = rng.integers(-5, G * width + 5, size=N)
    x = rng.integers(0, 30, size=(N, F))
    dev = torch.device("cuda")
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=G * width)
    assert dense.needs_slot_sort(torch.int32, t)
    lab, lp = dense.predict(torch.from_numpy(x.astype(np.int32)).to(dev),
                            torch.from_numpy(size.astype(np.int32)).to(dev), t, order="mixed")
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=width, limit=G * width)
    lab, lp = lab.cpu().numpy(), lp.cpu().numpy()
    assert lab.tolist() == want.tolist()
    ok = want >= 0
    assert lp[ok].tobytes() == wlp[ok].tobytes()


def test_order_hint_rejected():
    t = dense.DeviceTables.build(np.log([[0.5, 0.5]]), np.log(np.full((1, 2, 4), 0.25)),
                                 np.zeros(1, np.int32), group_size_bytes=10, max_size_bytes=10)
    x = torch.zeros((4, 4), dtype=torch.int32, device="cuda")
    s = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(Exception):
        dense.predict(x, s, t, order="sorted")


def test_kernel_is_taken_for_these_shapes():
    """The shapes above run the mixed-slot kernel (not the row box / sort paths)."""
    I32 = 0
    assert _mixed_rows(200, I32, 2, 29) == 256
    assert _mixed_rows(105, I32, 2, 72) == 256     # the most slots that fit at F=105: a
    assert _mixed_rows(105, I32, 2, 75) == 0       # 73-bin histogram, 3 warp-wide scan passes
    assert _mixed_rows(105, I32, 2, 2) == 256
    assert _mixed_rows(200, I32, 2, 1) == 0        # one slot: uniform tiles, 6-CTA kernel
    assert _mixed_rows(200, I32, 3, 29) == 0       # C > 2: other class pads
    assert _mixed_rows(2000, I32, 2, 64) == 0      # tables do not fit: sort + gather path


@pytest.mark.parametrize("dtype,hi,F", [(torch.uint16, 60000, 300), (torch.uint8, 255, 300),
                                        (torch.uint8, 255, 700), (torch.int32, 2**31 - 1, 150)])
def test_narrow_storage_and_extremes(dtype, hi, F):
    rng = np.random.default_rng(F)
    S, G, width = 7, 10, 1000
    prior, ll, route = _tables(rng, S, 2, F, G)
    N = 3000
    size = rng.integers(0, G * width, size=N)
    x = rng.integers(0, hi, size=(N, F), dtype=np.int64)
    x[rng.random((N, F)) < 0.6] = 0
    ld = {torch.int32: (F + 3) // 4 * 4, torch.uint16: (F + 7) // 8 * 8,
          torch.uint8: (F + 15) // 16 * 16}[dtype]
    _check(x, size, prior, ll, route, width, G * width, dtype=dtype, ldx=ld)


def test_negative_counts_and_statuses():
    rng = np.random.default_rng(3)
    S, G, F, width = 9, 12, 160, 1000
    prior, ll, route = _tables(rng, S, 2, F, G)
    N = 1000
    size = rng.integers(0, G * width, size=N)
    size[[0, 10, 500, 999]] = [-1, G * width, 2**31 - 1, -2**31]
    x = rng.poisson(1.0, size=(N, F))
    x[[3, 300, 777], [0, 159, 80]] = -1
    lab = _check(x, size, prior, ll, route, width, G * width, ldx=F)
    assert lab[[0, 10, 500, 999]].tolist() == [-1] * 4
    assert lab[[3, 300, 777]].tolist() == [-2] * 3


def test_fma_mode():
    rng = np.random.default_rng(11)
    S, G, F, width = 13, 16, 256, 1000
    prior, ll, route = _tables(rng, S, 2, F, G)
    N = 4000
    size = rng.integers(0, G * width, size=N)
    x = rng.integers(0, 3000, size=(N, F))
    dev = torch.device("cuda")
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=G * width)
    xd = torch.from_numpy(x.astype(np.int32)).to(dev)
    sd = torch.from_numpy(size.astype(np.int32)).to(dev)
    _, lp = dense.predict(xd, sd, t, mode="fma")
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=width, limit=G * width)
    rel = np.abs(lp.cpu().numpy() - wlp) / np.abs(wlp)
    assert rel.max() < 1e-11


_AB = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1905_13746_b200 import dense
rng = np.random.default_rng(5)
S, G, F, N, width = int(sys.argv[2]), 40, 200, 50_000, 100
prior = np.log(rng.dirichlet(np.ones(2), size=S))
ll = np.log(rng.dirichlet(np.ones(F), size=(S, 2)))
route = (np.arange(G) % S).astype(np.int32)
size = rng.integers(-5, G * width + 5, size=N).astype(np.int32)
x = rng.poisson(2.0, size=(N, F)).astype(np.int32)
t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=G * width)
lab, lp = dense.predict(torch.from_numpy(x).cuda(), torch.from_numpy(size).cuda(), t)
sys.stdout.buffer.write(lab.cpu().numpy().tobytes() + lp.cpu().numpy().tobytes())
"""


@pytest.mark.parametrize("S", [1, 29])
def test_same_bytes_with_and_without_mixed_kernel(S):
    """GNB_PRED_MIXED=0 (6-CTA kernel, L1 tables on mixed tiles), 1 (default) and
    2 (mixed kernel even for one slot) give byte-identical outputs."""
    outs = []
    for mode in ("0", "1", "2"):
        env = dict(os.environ, GNB_PRED_MIXED=mode)
        r = subprocess.run([sys.executable, "-c", _AB, ROOT, str(S)], env=env,
                           capture_output=True, timeout=300)
        assert r.returncode == 0, r.stderr.decode()[-2000:]
        outs.append(r.stdout)
    assert outs[0] == outs[1] == outs[2]


def test_auto_gate_from_concurrent_host_threads():
    """GNB_ORDER_AUTO from several host threads at once, on one shared stream and
    on per-thread streams: each call's count -> gated-kernel sequence stays its
    own (results equal the single-threaded ones)."""
    import threading
    rng = np.random.default_rng(31)
    S, G, F, width = 12, 14, 200, 100
    prior, ll, route = _tables(rng, S, 2, F, G)
    dev = torch.device("cuda")
    t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=width, max_size_bytes=G * width)
    cases = []
    for i in range(4):
        N = 60_000 + 1000 * i
        size = np.sort(rng.integers(0, G * width, size=N))
        if i % 2:
            size = rng.permutation(size)      # odd threads: shuffled -> mixed-slot kernel
        x = torch.from_numpy(rng.integers(0, 20, size=(N, F)).astype(np.int32)).to(dev)
        sd = torch.from_numpy(size.astype(np.int32)).to(dev)
        lab, lp = dense.predict(x, sd, t)
        torch.cuda.synchronize()
        cases.append((x, sd, lab.clone(), lp.clone()))
    for per_thread_stream in (False, True):
        errors = []  # filled by the worker threads

        def work(i):
            try:
                x, sd, lab0, lp0 = cases[i]
                s = torch.cuda.Stream() if per_thread_stream else torch.cuda.current_stream()
                with torch.cuda.stream(s):
                    for _ in range(15):
                        lab, lp = dense.predict(x, sd, t, stream=s)
                        s.synchronize()
                        if not (torch.equal(lab, lab0) and torch.equal(lp.view(torch.int64),
                                                                       lp0.view(torch.int64))):
                            errors.append((i, "mismatch"))
                            return
            except Exception as e:  # noqa: BLE001 -- reported by the assert below
                errors.append((i, repr(e)))

        th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
        for h in th:
            h.start()
        for h in th:
            h.join()
        assert not errors, errors
