"""K-PRED on uint8 rows (cfg4 shape, 16M rows): one warm launch, then one more
for ncu (`-k regex:predict_tma -s 1 -c 1`).  Prints the plain timing of 10
launches when run without ncu.  gpurun -- python tools/u8_probe.py [--fma] [--u16]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1905_13746_b200 import dense  # noqa: E402

n, V, width = 16_000_000, 256, 5120
dev = torch.device("cuda")
x, size, lab = dense.generate(n, V, divergence=0.8, seed=0, device=dev)
st = dense.fit_stats(x, size, lab, n_classes=2, group_size_bytes=width, max_size_bytes=width)
fin = dense.fin_train(st.sums.cpu().numpy(), st.counts.cpu().numpy(), k=V, alpha=1.0,
                      min_per_class=6)
F = int(fin.n_features[0])
dense.generate(n, F, divergence=0.8, seed=0, col_map=fin.features[0, :F].copy(),
               out=(x[:, :F], size, lab), device=dev)
xdt = torch.uint16 if "--u16" in sys.argv else torch.uint8
xg = x[:, :F].to(xdt)
del x
t = dense.DeviceTables.build(fin.log_prior[:1], fin.log_lik[:1, :, :F], np.zeros(1, np.int32),
                             group_size_bytes=width, max_size_bytes=width, device=dev)
label = torch.empty(n, dtype=torch.int32, device=dev)
lp = torch.empty((n, 2), dtype=torch.float64, device=dev)
mode = "fma" if "--fma" in sys.argv else "exact"
for _ in range(2):
    dense.predict(xg, size, t, logpost=True, label_out=label, logpost_out=lp, mode=mode)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    dense.predict(xg, size, t, logpost=True, label_out=label, logpost_out=lp, mode=mode)
b.record()
b.synchronize()
ms = a.elapsed_time(b) / 10
print(f"{str(xdt)[6:]} {mode}: {ms:.3f} ms/launch, {n / ms / 1e6:.2f} G samples/s, "
      f"{n * (F * xg.element_size() + 24) / ms / 1e6:.0f} GB/s")
