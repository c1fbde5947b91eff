"""Host read bandwidth of the int32 e2e rows: pinned vs pageable source, and the
library's int32 e2e with each (narrowing reads the rows on host threads, so the
caller's buffer need not be pinned).  One JSON line."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_13746_b200 import _native as N  # noqa: E402

torch.set_num_threads(os.cpu_count())
m, F = 8_000_000, 256
out = {}
for pinned in (False, True):
    src = torch.randint(0, 16, (m, F), dtype=torch.int32)
    if pinned:
        src = src.pin_memory()
    dst = torch.empty((m, F), dtype=torch.uint8)
    dst.copy_(src)
    t = time.perf_counter()
    for _ in range(3):
        dst.copy_(src)
    out[f"torch_narrow_gbs_{'pinned' if pinned else 'pageable'}"] = round(
        3 * m * F * 4 / (time.perf_counter() - t) / 1e9, 1)
    size = torch.randint(0, 5120, (m,), dtype=torch.int32)
    lab = torch.empty(m, dtype=torch.int32, pin_memory=True)
    lp = torch.empty((m, 2), dtype=torch.float64, pin_memory=True)
    prior = np.log(np.array([[0.5, 0.5]]))
    lik = np.log(np.full((1, 2, F), 1.0 / F))
    route = np.zeros(1, np.int32)
    el = ctypes.c_int64()

    def step():
        N.check(N.lib.gnb_predict_host_typed(
            src.data_ptr(), N.X_I32, m, F, F, size.data_ptr(), 5120, 5120, route.ctypes.data,
            1, 2, prior.ctypes.data, lik.ctypes.data, lab.data_ptr(), lp.data_ptr(), 0,
            ctypes.addressof(el)))
    step()
    t = time.perf_counter()
    for _ in range(3):
        step()
    out[f"e2e_int32_{'pinned' if pinned else 'pageable'}_rows_per_s"] = round(
        3 * m / (time.perf_counter() - t), 1)
    del src, dst
print(json.dumps(out), flush=True)
