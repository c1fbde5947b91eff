"""Fixed per-launch cost of K-PRED on short launches (cfg2-sized, L2 flushed).

Times the row-box K-PRED (F=50 int32) at several row counts and, for scale,
a device-to-device copy of the same rows, both with bench.py's flush + event
method.  The intercept of time vs. bytes is the fixed cost (launch + ramp +
tail).

  gpurun -- 'python tools/short_launch_probe.py'
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_1905_13746_b200 import dense  # noqa: E402


def main() -> None:
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    F = int(os.environ.get("PROBE_F", "50"))
    out = {"F": F, "rows": []}
    nmax = 16_000_000
    x, size, lab = dense.generate(nmax, F, divergence=0.8, seed=0, device=dev)
    prior = np.log(np.array([[0.5, 0.5]]))
    ll = np.log(np.full((1, 2, F), 1.0 / F))
    t = dense.DeviceTables.build(prior, ll, np.zeros(1, np.int32), group_size_bytes=5120,
                                 max_size_bytes=5120, device=dev)
    label = torch.empty(nmax, dtype=torch.int32, device=dev)
    lp = torch.empty((nmax, 2), dtype=torch.float64, device=dev)
    base = x.as_strided((nmax, x.stride(0)), (x.stride(0), 1))
    for n in (250_000, 500_000, 1_000_000, 2_000_000, 4_000_000, 16_000_000):
        ms, _ = bench._timed_launches(
            lambda: dense.predict(x[:n], size[:n], t, label_out=label[:n],
                                  logpost_out=lp[:n]), 20, 3)
        nbytes = n * (4 * F + 24)
        xs = base[:n].reshape(-1)
        dst = torch.empty_like(xs)
        ms_cp, _ = bench._timed_launches(lambda: dst.copy_(xs), 20, 3)
        del dst
        out["rows"].append({
            "n": n, "kpred_us": round(ms * 1e3, 2),
            "kpred_gbs": round(nbytes / (ms / 1e3) / 1e9, 1),
            "d2d_copy_us": round(ms_cp * 1e3, 2),
            "d2d_copy_gbs": round(2 * xs.numel() * 4 / (ms_cp / 1e3) / 1e9, 1)})
        print(json.dumps(out["rows"][-1]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
