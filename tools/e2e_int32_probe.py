"""e2e on int32 host rows (the data-independent storage): where does the time go?
Host DRAM narrowing rate, the C port on int32 vs uint8 rows, and
gnb_predict_host_typed with host-side narrowing off/on.  One JSON line."""
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1905_13746_b200 import _native as N  # noqa: E402

m, F = 8_000_000, 256
out = {"rows": m, "features": F, "cpu_count": os.cpu_count()}
x, size, label = O.synth_dense(1_000_000, F, seed=0, divergence=0.8)
S, _, n, _, _ = O.fit_stats(x, size, label, 2, 5120, 5120)
feats, _ = O.select_features(S[0], F, 0)
t = O.train_tables(S[0], n[0], feats, 1.0, 0)
xg = np.ascontiguousarray(x[:, feats]).astype(np.int32)
reps = m // len(xg)
xh = torch.empty((m, F), dtype=torch.int32, pin_memory=True)
for i in range(reps):
    xh[i * len(xg):(i + 1) * len(xg)] = torch.from_numpy(xg)
sh = torch.from_numpy(np.tile(size.astype(np.int32), reps)).pin_memory()
lab = torch.empty(m, dtype=torch.int32, pin_memory=True)
lp = torch.empty((m, 2), dtype=torch.float64, pin_memory=True)
prior, lik = np.ascontiguousarray(t.log_prior[None]), np.ascontiguousarray(t.log_lik[None])
route = np.zeros(1, np.int32)

# host narrowing throughput (torch, all threads)
torch.set_num_threads(os.cpu_count())
dst = torch.empty((m, F), dtype=torch.uint8)
dst.copy_(xh)
t0 = time.perf_counter()
for _ in range(3):
    dst.copy_(xh)
dt = (time.perf_counter() - t0) / 3
out["torch_narrow_int32_to_u8_rows_per_s"] = round(m / dt, 1)
out["torch_narrow_read_gbs"] = round(m * F * 4 / dt / 1e9, 1)


def e2e(narrow):
    os.environ["GNB_HOST_NARROW"] = "1" if narrow else "0"
    el = ctypes.c_int64()

    def step():
        N.check(N.lib.gnb_predict_host_typed(
            xh.data_ptr(), N.X_I32, m, F, F, sh.data_ptr(), 5120, 5120, route.ctypes.data, 1, 2,
            prior.ctypes.data, lik.ctypes.data, lab.data_ptr(), lp.data_ptr(), 0,
            ctypes.addressof(el)))
    step()
    t0 = time.perf_counter()
    for _ in range(3):
        step()
    return round(3 * m / (time.perf_counter() - t0), 1)


out["e2e_int32_plain"] = e2e(False)
out["e2e_int32_host_narrow"] = e2e(True)
for chunk in (16, 32, 128):
    os.environ["GNB_HOST_CHUNK_MB"] = str(chunk)
# C port on int32 / uint8 rows (2M-row sample, all threads)
xs = xh[:2_000_000].numpy()
for name, arr in (("int32", xs), ("uint8", xs.astype(np.uint8))):
    O.c_predict(arr, sh[:2_000_000].numpy(), route, prior, lik, width=5120, limit=5120,
                threads=os.cpu_count())
    t0 = time.perf_counter()
    k = 0
    while time.perf_counter() - t0 < 5:
        O.c_predict(arr, sh[:2_000_000].numpy(), route, prior, lik, width=5120, limit=5120,
                    threads=os.cpu_count())
        k += 1
    out[f"c_port_{name}_rows_per_s"] = round(k * 2_000_000 / (time.perf_counter() - t0), 1)
print(json.dumps(out), flush=True)
