"""e2e host-pipeline probe: gnb_predict_host_typed on 8M x 256 pinned rows stored
uint4 / uint8, wall time per call (3 calls after one warm call).  Run once per
GNB_HOST_CHUNK_MB setting (the knob is read once per process):
  gpurun -- 'for c in 8 16 32 64; do GNB_HOST_CHUNK_MB=$c python tools/e2e_chunk_probe.py; done'"""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_13746_b200 import _native as N  # noqa: E402
from paper_1905_13746_b200 import dense  # noqa: E402

m, F, width = 8_000_000, 256, 5120
g = torch.Generator().manual_seed(0)
x = torch.randint(0, 3, (m, F), dtype=torch.uint8, generator=g)
size = torch.randint(0, width, (m,), dtype=torch.int32, generator=g).pin_memory()
prior = np.log(np.array([[0.5, 0.5]]))
lik = np.ascontiguousarray(-np.random.default_rng(0).random((1, 2, F)) * 10)
route = np.zeros(1, np.int32)
lab = torch.empty(m, dtype=torch.int32).pin_memory()
lp = torch.empty((m, 2), dtype=torch.float64).pin_memory()
out = {"chunk_mb": os.environ.get("GNB_HOST_CHUNK_MB", "default")}
for name in ("uint4", "uint8"):
    if name == "uint4":
        xh = torch.empty((m, (F + 15) // 16 * 8), dtype=torch.uint8).pin_memory()
        for i in range(0, m, 1 << 20):
            dense.pack_u4(x[i:i + (1 << 20)], out=xh[i:i + (1 << 20)])
        xt, ldx = N.X_U4, 2 * xh.shape[1]
    else:
        xh, xt, ldx = x.pin_memory(), N.X_U8, F

    def call():
        N.check(N.lib.gnb_predict_host_typed(xh.data_ptr(), xt, m, F, ldx, size.data_ptr(), width,
                                             width, route.ctypes.data, 1, 2, prior.ctypes.data,
                                             lik.ctypes.data, lab.data_ptr(), lp.data_ptr(), 0,
                                             None), "predict_host_typed")
    call()
    t = time.perf_counter()
    for _ in range(3):
        call()
    dt = (time.perf_counter() - t) / 3
    out[name] = {"samples_per_s": round(m / dt), "ms": round(dt * 1e3, 2),
                 "h2d_gbs": round(m * (ldx // (2 if name == "uint4" else 1) + 4) / dt / 1e9, 1)}
print(json.dumps(out))
