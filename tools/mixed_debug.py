"""Mixed-slot K-PRED full-size parity diagnostic: every row vs the C oracle,
grouped and shuffled order, with mismatch positions (tile, CTA round, lane)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import oracle as O
from paper_1905_13746_b200 import dense

rng = np.random.default_rng(0)
G, F, N = 32, 200, int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
counts = (N * 0.9 ** np.arange(G) / (0.9 ** np.arange(G)).sum()).astype(int)
counts[0] += N - counts.sum()
trained = [g for g in range(G) if g not in (5, 8, 17)]
S = len(trained)
prior = np.log(rng.dirichlet(np.ones(2), size=S))
ll = np.log(rng.dirichlet(np.ones(F), size=(S, 2)))
route = np.array([trained.index(t) for t in O.route_table(trained, G)], dtype=np.int32)
size = np.concatenate([g * 5120 + rng.integers(0, 5120, size=c) for g, c in enumerate(counts)])
x = rng.poisson(1.0, size=(N, F)).astype(np.int32)
t = dense.DeviceTables.build(prior, ll, route, group_size_bytes=5120, max_size_bytes=G * 5120)
want, wlp = O.c_predict(x, size.astype(np.int32), route, prior, ll, width=5120, limit=G * 5120,
                        threads=16)
for name, order in (("grouped", np.arange(N)), ("shuffled", rng.permutation(N))):
    lab, lp = dense.predict(torch.from_numpy(x[order]).cuda(),
                            torch.from_numpy(size[order].astype(np.int32)).cuda(), t)
    lab, lp = lab.cpu().numpy(), lp.cpu().numpy()
    bad = np.nonzero((lab != want[order]) |
                     (lp.view(np.int64) != wlp[order].view(np.int64)).any(axis=1))[0]
    print(name, "rows", N, "mismatch", len(bad))
    if len(bad):
        tile = bad // 256
        print("  first", bad[:10].tolist())
        print("  tiles", np.unique(tile)[:20].tolist(), "n tiles bad", len(np.unique(tile)))
        print("  cta round", np.bincount(tile // 148)[:10].tolist())
        print("  pos in tile", np.bincount(bad % 256, minlength=256)[:64].tolist())
