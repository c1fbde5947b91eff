"""Multi-GPU product paths on the device(s) this box has: the single-process
sharded fit (K-FIT per device + the library's NCCL all-reduce) and predict,
the host-buffer sharded entry points, and bench.py's self-launched multi-rank
mode (--gpus 2 with gloo: ranks share the GPU; a functional check, not a
measurement)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_1905_13746_b200 import dense  # noqa: E402
from paper_1905_13746_b200 import _native as N  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _devs():
    return list(range(torch.cuda.device_count()))


def test_fit_and_predict_sharded_equal_single_device():
    devs = _devs()
    n, V = 300_001, 64
    x, size, lab = dense.generate(n, V, divergence=0.3, seed=5)
    one = dense.fit_stats(x, size, lab, n_classes=2, group_size_bytes=5120, max_size_bytes=5120)
    bounds = [(n * i // len(devs), n * (i + 1) // len(devs)) for i in range(len(devs))]
    xs = [x[a:b].to(f"cuda:{d}") for (a, b), d in zip(bounds, devs)]
    ss = [size[a:b].to(f"cuda:{d}") for (a, b), d in zip(bounds, devs)]
    ls = [lab[a:b].to(f"cuda:{d}") for (a, b), d in zip(bounds, devs)]
    sh = dense.fit_stats_sharded(xs, ss, ls, n_classes=2, group_size_bytes=5120,
                                 max_size_bytes=5120)
    for st in sh:
        assert torch.equal(st.sums.cpu(), one.sums.cpu())
        assert torch.equal(st.sumsq.cpu(), one.sumsq.cpu())
        assert torch.equal(st.counts.cpu(), one.counts.cpu())
    fin = dense.fin_train(one.sums.cpu().numpy(), one.counts.cpu().numpy(), k=40, alpha=1.0,
                          min_per_class=6)
    F = int(fin.n_features[0])
    cols = torch.from_numpy(fin.features[0, :F].astype(np.int64))
    tabs = [dense.DeviceTables.build(fin.log_prior[:1], fin.log_lik[:1, :, :F],
                                     np.zeros(1, np.int32), group_size_bytes=5120,
                                     max_size_bytes=5120, device=f"cuda:{d}") for d in devs]
    outs = dense.predict_sharded([xx[:, cols.to(xx.device)].contiguous() for xx in xs], ss, tabs)
    lab_all = torch.cat([o[0].cpu() for o in outs]).numpy()
    lp_all = torch.cat([o[1].cpu() for o in outs]).numpy()
    want, wlp = O.predict_dense(x.cpu().numpy()[:, fin.features[0, :F]], size.cpu().numpy(),
                                np.zeros(1, np.int32), fin.log_prior[:1], fin.log_lik[:1, :, :F],
                                width=5120, limit=5120)
    assert lab_all.tolist() == want.tolist() and lp_all.tobytes() == wlp.tobytes()


@pytest.mark.parametrize("x_type", ["int32", "uint8"])
def test_host_sharded_entry_points(x_type):
    """gnb_predict_host_sharded / gnb_fit_stats_host_sharded with 1-3 shards
    (shards may share a device) == the single-device calls == the oracle."""
    rng = np.random.default_rng(3)
    n, F = 50_003, 100
    x = rng.poisson(1.5, size=(n, F)).astype(np.int32)
    size = rng.integers(-10, 3 * 1000 + 10, size=n).astype(np.int32)
    label = rng.integers(-1, 2, size=n).astype(np.int32)
    prior = np.log(rng.dirichlet(np.ones(2), size=3))
    ll = np.log(rng.dirichlet(np.ones(F), size=(3, 2)))
    route = np.array([2, 0, 1], np.int32)
    want, wlp = O.predict_dense(x, size, route, prior, ll, width=1000, limit=3000)
    S, Q, cnt, bad, oor = O.fit_stats(x, size, label, 2, 1000, 3000)
    xh = x.astype(x_type)
    xt = N.X_I32 if x_type == "int32" else N.X_U8
    for nd in (1, 2, 3):
        devs = np.array([i % torch.cuda.device_count() for i in range(nd)], np.int32)
        lab = np.empty(n, np.int32)
        lp = np.empty((n, 2))
        el = np.zeros(1, np.int64)
        N.check(N.lib.gnb_predict_host_sharded(
            xh.ctypes.data, xt, n, F, F, size.ctypes.data, 1000, 3000, route.ctypes.data, 3, 2,
            prior.ctypes.data, ll.ctypes.data, lab.ctypes.data, lp.ctypes.data, nd,
            devs.ctypes.data, el.ctypes.data))
        assert lab.tolist() == want.tolist()
        ok = want >= 0
        assert lp[ok].tobytes() == wlp[ok].tobytes() and el[0] > 0
        Sd, Qd, nd_ = np.zeros((3, 2, F)), np.zeros((3, 2, F)), np.zeros((3, 2))
        st = np.zeros(2, np.uint64)
        N.check(N.lib.gnb_fit_stats_host_sharded(
            x.ctypes.data, n, F, F, size.ctypes.data, label.ctypes.data, 1000, 3000, 2,
            Sd.ctypes.data, Qd.ctypes.data, nd_.ctypes.data, st.ctypes.data, nd,
            devs.ctypes.data))
        assert np.array_equal(Sd, S) and np.array_equal(Qd, Q) and np.array_equal(nd_, cnt)
        assert st.tolist() == [bad, oor]
    bad_dev = np.array([0, 99], np.int32)
    with pytest.raises(Exception):
        N.check(N.lib.gnb_predict_host_sharded(
            xh.ctypes.data, xt, n, F, F, size.ctypes.data, 1000, 3000, route.ctypes.data, 3, 2,
            prior.ctypes.data, ll.ctypes.data, lab.ctypes.data, lp.ctypes.data, 2,
            bad_dev.ctypes.data, el.ctypes.data))


@pytest.mark.timeout(600)
def test_bench_self_launches_ranks():
    """`python bench.py --gpus 2` re-execs itself under torch.distributed.run:
    2 ranks (gloo, sharing this box's GPU), strong-scaled cfg4 rows split between
    them, one JSON line with n_gpus 2."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dist-backend",
           "gloo", "--rows", "2000000", "--steps", "3", "--warmup", "3", "--no-e2e",
           "--no-cpu-baseline", "--no-object-api"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=500)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["scaling"] == "strong"
    assert out["config"]["rows_total"] == 2_000_000
    assert out["config"]["rows_per_gpu"] == 1_000_000
