"""A/B of K-PRED on a SHUFFLED ragged batch (cfg3 rows in random order): the
device slot sort and the permuted predict timed separately (CUDA events, L2
flushed before each launch).  Geometry via the GNB_* environment knobs; one
JSON line per run.  Usage: python tools/gather_ab.py [label]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import _timed_launches  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1905_13746_b200 import dense  # noqa: E402

dev = torch.device("cuda")
G, V, N = 32, 200, 4_194_304
w = 0.9 ** np.arange(G)
counts = np.floor(N * w / w.sum()).astype(np.int64)
counts[0] += N - counts.sum()
width, limit = 5120, G * 5120
x, size, lab = dense.generate(N, V, group_rows=counts, divergence=0.8, seed=0, device=dev)
st = dense.fit_stats(x, size, lab, n_classes=2, group_size_bytes=width, max_size_bytes=limit)
fin = dense.fin_train(st.sums.cpu().numpy(), st.counts.cpu().numpy(), k=V, alpha=1.0,
                      min_per_class=6)
trained = [g for g in range(G) if fin.state[g] == 1 and g not in (5, 8, 17)]
slot = {g: i for i, g in enumerate(trained)}
route = np.array([slot[int(g)] for g in O.route_table(trained, G)], np.int32)
F = int(max(fin.n_features[g] for g in trained))
t = dense.DeviceTables.build(fin.log_prior[trained], fin.log_lik[trained][:, :, :F], route,
                             group_size_bytes=width, max_size_bytes=limit, device=dev)
xg = dense.gather_features(x, size, t, fin.features[trained][:, :F].astype(np.int32),
                           fin.n_features[trained].astype(np.int32))
del x
shuf = torch.randperm(N, device=dev, generator=torch.Generator(device=dev).manual_seed(0))
xs, ss = xg[shuf].contiguous(), size[shuf].contiguous()
label = torch.empty(N, dtype=torch.int32, device=dev)
lp = torch.empty((N, 2), dtype=torch.float64, device=dev)
perm = dense.slot_sort(ss, t)
sort_ms, _ = _timed_launches(lambda: dense.slot_sort(ss, t), 20, 3)
pred_ms, _ = _timed_launches(lambda: dense.predict(xs, ss, t, label_out=label, logpost_out=lp,
                                                   perm=perm), 20, 3)
ref_lab = torch.empty_like(label)
ref_lp = torch.empty_like(lp)
dense.predict(xs, ss, t, label_out=ref_lab, logpost_out=ref_lp)
dense.predict(xs, ss, t, label_out=label, logpost_out=lp, perm=perm)
same = bool(torch.equal(label, ref_lab) and torch.equal(lp, ref_lp))
peak = 6532.2
bps = 4 * F + 24
env = {k: v for k, v in os.environ.items() if k.startswith("GNB_")}
print(json.dumps({"label": sys.argv[1] if len(sys.argv) > 1 else "", "env": env, "F": F,
                  "sort_ms": round(sort_ms, 4), "predict_ms": round(pred_ms, 4),
                  "predict_frac": round(N * bps / (pred_ms / 1e3) / 1e9 / peak, 4),
                  "total_frac": round(N * bps / ((pred_ms + sort_ms) / 1e3) / 1e9 / peak, 4),
                  "identical_to_unpermuted": same}), flush=True)
