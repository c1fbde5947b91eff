"""N>1 host logic on CPU with gloo, world_size 2: sharded fit stats + one all-reduce
give the single-process statistics and the identical bundle; sharded predict
concatenates to the single-process result."""

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


class _CpuStats:
    """FitStats stand-in holding CPU tensors (the GPU fit is tested on the GPU)."""

    def __init__(self, S, Q, n):
        self.sums, self.sumsq, self.counts = (torch.from_numpy(a.astype(np.float64))
                                              for a in (S, Q, n))

    def packed(self):
        return torch.cat([self.sums.reshape(-1), self.sumsq.reshape(-1), self.counts.reshape(-1)])

    def unpack_(self, flat):
        o = 0
        for t in (self.sums, self.sumsq, self.counts):
            t.copy_(flat[o:o + t.numel()].view_as(t))
            o += t.numel()
        return self


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, size, label = O.synth_dense(5003, 40, seed=1, divergence=0.3)
    lo, hi = shard_bounds(len(size), world, rank)
    S, Q, n, _, _ = O.fit_stats(x[lo:hi], size[lo:hi], label[lo:hi], 2, 5120, 5120)
    st = allreduce_stats(_CpuStats(S, Q, n))
    feats, _ = O.select_features(st.sums.numpy()[0].astype(np.int64), 30, 0)
    t = O.train_tables(st.sums.numpy()[0].astype(np.int64), st.counts.numpy()[0].astype(np.int64),
                       feats, 1.0, 0)
    lab, lp = O.predict_dense(x[lo:hi][:, feats], size[lo:hi], np.zeros(1, np.int32),
                              t.log_prior[None], t.log_lik[None], width=5120, limit=5120)
    gl = [None] * world
    dist.all_gather_object(gl, (lab.tolist(), lp.tobytes()))
    if rank == 0:
        out.put((st.sums.numpy().tobytes(), st.sumsq.numpy().tobytes(), st.counts.numpy().tobytes(),
                 feats.tolist(), t.log_lik.tobytes(), gl))
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
    S2, Q2, n2, feats2, ll2, parts = res
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
    assert sum((p[0] for p in parts), []) == lab.tolist()
    assert b"".join(p[1] for p in parts) == lp.tobytes()
