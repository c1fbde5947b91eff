"""Mixed-slot K-PRED probe: N rows x F int32 features, S slots (G = S+3 size
groups, 0.9^g weights), grouped or shuffled order; prints ms and fraction of
the measured HBM peak for the default dispatch.  Env knobs (GNB_PRED_MIXED,
GNB_MIXED_STAGES) select the kernel / ring depth for A/B runs."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1905_13746_b200 import dense  # noqa: E402

N, F, S = (int(a) for a in sys.argv[1:4])
order = sys.argv[4] if len(sys.argv) > 4 else "shuffled"
peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6532.2) if os.path.exists(
    "MEASURED_PEAKS.json") else 6532.2
rng = np.random.default_rng(0)
G = S + 3
w = 0.9 ** np.arange(G)
counts = np.floor(N * w / w.sum()).astype(np.int64)
counts[0] += N - counts.sum()
route = (np.arange(G) % S).astype(np.int32)
prior = np.log(rng.dirichlet(np.ones(2), size=S))
ll = np.log(rng.dirichlet(np.ones(F), size=(S, 2)))
dev = torch.device("cuda")
size = torch.from_numpy(np.concatenate(
    [g * 100 + rng.integers(0, 100, size=c) for g, c in enumerate(counts)]).astype(np.int32)).to(dev)
x = torch.randint(0, 8, (N, F), dtype=torch.int32, device=dev)
if order == "shuffled":
    size = size[torch.randperm(N, device=dev)].contiguous()
t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=100, max_size_bytes=G * 100)
lab = torch.empty(N, dtype=torch.int32, device=dev)
lp = torch.empty((N, 2), dtype=torch.float64, device=dev)
for _ in range(3):
    dense.predict(x, size, t, label_out=lab, logpost_out=lp)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ms = []
for _ in range(10):
    ev[0].record()
    dense.predict(x, size, t, label_out=lab, logpost_out=lp)
    ev[1].record()
    torch.cuda.synchronize()
    ms.append(ev[0].elapsed_time(ev[1]))
m = float(np.median(ms))
print(json.dumps({"N": N, "F": F, "S": S, "order": order, "ms": round(m, 4),
                  "frac": round(N * (4 * F + 24) / (m / 1e3) / 1e9 / peak, 4),
                  "mixed": os.environ.get("GNB_PRED_MIXED", "1"),
                  "stages": os.environ.get("GNB_MIXED_STAGES", "auto")}))
