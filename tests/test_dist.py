"""N>1 host logic on CPU with gloo, world_size 2, through the repo's own sharded
drivers (sharding.fit_distributed / train_distributed / gather_rows): sharded fit
stats + one all-reduce + host FIN give the single-process statistics and the
identical model; sharded predict outputs gather to the single-process result.
Only the per-rank kernels are stood in by the CPU oracle (no GPU here)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_1905_13746_b200.sharding import allreduce_stats, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _cpu_fit(x, size, label, *, n_classes, group_size_bytes, max_size_bytes, sumsq=True):
    """The local statistics producer on CPU (K-FIT needs a GPU): the oracle's
    counts, in the repo's own FitStats container."""
    from paper_1905_13746_b200.dense import FitStats
    S, Q, n, bad, oor = O.fit_stats(x, size, label, n_classes, group_size_bytes, max_size_bytes)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))  # noqa: E731
    return FitStats(t(S), t(Q) if sumsq else None, t(n), torch.tensor([bad, oor]))


def _worker(rank, world, port, out):
    from paper_1905_13746_b200.sharding import fit_distributed, gather_rows, train_distributed
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, size, label = O.synth_dense(5003, 40, seed=1, divergence=0.3)
    lo, hi = shard_bounds(len(size), world, rank)
    # the repo's sharded drivers: local stats -> the one all-reduce (-> host FIN)
    st = fit_distributed(x[lo:hi], size[lo:hi], label[lo:hi], n_classes=2,
                         group_size_bytes=5120, max_size_bytes=5120, fit=_cpu_fit)
    fin = train_distributed(x[lo:hi], size[lo:hi], label[lo:hi], k=30, alpha=1.0,
                            group_size_bytes=5120, max_size_bytes=5120, min_per_class=6,
                            fit=_cpu_fit)
    F = int(fin.n_features[0])
    feats = fin.features[0, :F]
    lab, lp = O.predict_dense(x[lo:hi][:, feats], size[lo:hi], np.zeros(1, np.int32),
                              fin.log_prior[:1], fin.log_lik[:1, :, :F], width=5120, limit=5120)
    all_lab = gather_rows(torch.from_numpy(lab.astype(np.int32)))
    all_lp = gather_rows(torch.from_numpy(np.ascontiguousarray(lp)))
    if rank == 0:
        out.put((st.sums.numpy().tobytes(), st.sumsq.numpy().tobytes(), st.counts.numpy().tobytes(),
                 feats.tolist(), fin.log_lik[0, :, :F].tobytes(), all_lab.numpy().tolist(),
                 all_lp.numpy().tobytes()))
    dist.destroy_process_group()


def test_shard_bounds_cover_rows():
    for n in (0, 1, 7, 100, 101):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


@pytest.mark.timeout(180)
def test_gloo_world2_fit_allreduce_and_predict():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=150)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    S2, Q2, n2, feats2, ll2, all_lab, all_lp = res
    x, size, label = O.synth_dense(5003, 40, seed=1, divergence=0.3)
    S, Q, n, _, _ = O.fit_stats(x, size, label, 2, 5120, 5120)
    assert S.astype(np.float64).tobytes() == S2
    assert Q.astype(np.float64).tobytes() == Q2
    assert n.astype(np.float64).tobytes() == n2
    feats, _ = O.select_features(S[0], 30, 0)
    t = O.train_tables(S[0], n[0], feats, 1.0, 0)
    assert feats.tolist() == feats2 and t.log_lik.tobytes() == ll2
    lab, lp = O.predict_dense(x[:, feats], size, np.zeros(1, np.int32), t.log_prior[None],
                              t.log_lik[None], width=5120, limit=5120)
    assert all_lab == lab.tolist()
    assert all_lp == lp.tobytes()
