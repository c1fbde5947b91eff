#!/usr/bin/env python
"""Benchmark of the group-wise Naive Bayes predict hot path (BASELINE.json metric:
samples classified/s and achieved HBM GB/s, % of roofline, at 1/2/4/8 B200).

Workload (BASELINE.json configs[3]): 100M samples x 256 opcode features per
GPU, 2 classes, one size group; one K-PRED launch per step over the whole
HBM-resident shard (label + both log-posteriors written).  Inputs (102 GB)
are far larger than L2, so every step streams X from HBM.  Synthetic data
follows the reference's law (GEN, counter-based, identical under sharding);
the model is FITTED on that data with K-FIT (+ NCCL all-reduce of the stats
for N > 1) and FIN, then X is re-materialised in the model's FeatureSet
order (the predict layout) -- all outside the timed region.

    python bench.py [--gpus N --steps K --warmup W]     # our sm_100a kernels
    python bench.py --impl reference ...                 # CPU reference arm
    torchrun --nproc-per-node N bench.py --gpus N ...    # one rank per GPU

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "samples classified/sec (predict, fused argmax)"
UNIT = "samples/s"
DEFAULT_ROWS = 100_000_000
DEFAULT_F = 256


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--rows", type=int, default=DEFAULT_ROWS,
                    help="cfg4 samples: the job total (strong scaling, default) or per GPU "
                         "(--scaling weak)")
    ap.add_argument("--scaling", choices=("strong", "weak"), default="strong",
                    help="strong = BASELINE cfg4 (100M samples sharded over the GPUs); "
                         "weak = --rows per GPU")
    ap.add_argument("--features", type=int, default=DEFAULT_F)
    ap.add_argument("--e2e-rows", type=int, default=8_000_000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-object-api", action="store_true")
    ap.add_argument("--object-rows", type=int, default=100_000)
    ap.add_argument("--no-logpost", action="store_true")
    ap.add_argument("--fit-rows", type=int, default=1_000_000_000)
    ap.add_argument("--ref-rows", type=int, default=2_000_000,
                    help="CPU reference arm: rows scored per step (bounded sample)")
    ap.add_argument("--ref-py-samples", type=int, default=20_000,
                    help="reference arm: samples for the unmodified Python reference "
                         "(classify_sequential / classify_parallel); 0 skips it")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="gloo: exercise the multi-rank path with ranks sharing one GPU "
                         "(host-side collectives only; testing, not a bench number)")
    ap.add_argument("--x-dtype", choices=("int32", "uint16", "uint8"), default="int32",
                    help="storage of the predict matrix (same counts; narrower = fewer bytes)")
    ap.add_argument("--workload", choices=("predict", "sweep", "ragged", "fit", "fin"),
                    default="predict",
                    help="predict = cfg4 (driver default); sweep = cfg2 F sweep at 1M rows; "
                         "ragged = cfg3 32 size groups in one launch; fit = cfg5 1B x 128, C=16")
    ap.add_argument("--flush", choices=("clean", "write"), default="clean",
                    help="secondary workloads' L2 flush before each launch: write = 512 MB "
                         "write only (leaves ~126 MB of dirty lines that the timed kernel "
                         "then writes back); clean = the write followed by a 256 MB read "
                         "of another buffer, so L2 holds only clean lines")
    ap.add_argument("--pitch", choices=("packed", "line"), default="packed",
                    help="sweep/ragged int32 row pitch: packed = 16-B multiple, line = "
                         "128-B multiple (pad columns are never read)")
    return ap.parse_args()


SPEC_HBM_GBS = 8000.0  # B200 HBM3e spec (DGX figure), the north star's denominator


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def live_copy_gbs():
    """This box's device copy bandwidth, measured the way MEASURED_PEAKS.json's
    hbm_gbs is (b.copy_(a) over 1 Gi bf16 elements, read + write bytes, best of
    10, CUDA events): reported beside `peak` so a frac above 1 (a box faster than
    the pod's figure) can be read against the same box."""
    import torch
    try:
        a = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda")
        b = torch.empty_like(a)
        b.copy_(a)
        best = None
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            b.copy_(a)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        del a, b
        torch.cuda.empty_cache()
        return 2 * (1 << 30) * 2 / (best / 1e3) / 1e9
    except Exception:
        return None


def ncu_traffic():
    """Per-sample DRAM bytes of K-PRED from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_predict.json")) as fh:
            d = json.load(fh)
        return float(d["dram_bytes_per_sample"]), d
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (clocks + throttle reasons)."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), line.strip()))

    def mark(self, begin: bool):
        if begin:
            self.t0 = time.time()
        else:
            self.t1 = time.time()

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.15)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        inside = [r for t, r in self.rows if self.t0 - 0.06 <= t <= self.t1 + 0.06] or \
            [r for _, r in self.rows]
        sm, mx, reasons, power = [], [], set(), []
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in inside:
            parts = [p.strip() for p in r.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                power.append(float(parts[7]))
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": statistics.median(power) if power else None}


# ---------------------------------------------------------------- distributed plumbing
def relaunch_if_needed(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec this command
    under torch.distributed.run with one rank per GPU, so the driver's plain
    invocation and its torchrun invocation measure the same thing."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_init(args):
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        backend = args.dist_backend if args.impl == "ours" else "gloo"
        if args.impl == "ours":
            if backend == "gloo":          # test mode: every rank may share GPU 0
                local = local % max(torch.cuda.device_count(), 1)
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def _coll_device(device):
    """Collectives run where the backend can: CUDA tensors for NCCL, CPU for gloo."""
    import torch.distributed as dist
    return device if dist.get_backend() == "nccl" else "cpu"


def barrier_max(value: float, world: int, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier_sum(value: float, world: int, device=None) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


# ---------------------------------------------------------------- our arm
def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1905_13746_b200 import _native as N
    from paper_1905_13746_b200 import dense
    from paper_1905_13746_b200.sharding import allreduce_stats

    from paper_1905_13746_b200.sharding import shard_bounds

    dev = torch.device("cuda", torch.cuda.current_device())
    V = args.features
    width = 5120
    # contiguous shard of the global index space (engine.py:264-268 chunking):
    # strong scaling = BASELINE cfg4, 100M samples over all GPUs
    total = args.rows if args.scaling == "strong" else args.rows * world
    offset, hi = shard_bounds(total, world, rank)
    n = hi - offset
    group_rows = [total]

    # ---- data + model (outside the timed region)
    x, size, lab = dense.generate(n, V, group_rows=group_rows, divergence=0.8, seed=0,
                                  row_offset=offset, device=dev)
    st = dense.fit_stats(x, size, lab, n_classes=2, group_size_bytes=width,
                         max_size_bytes=width)
    allreduce_stats(st)                     # NCCL over NVLink: the fit's only exchange
    fin = dense.fin_train(st.sums.cpu().numpy(), st.counts.cpu().numpy(), k=V, alpha=1.0,
                          min_per_class=6)
    assert fin.state[0] == 1, "synthetic group must be trainable"
    F = int(fin.n_features[0])
    feats = fin.features[0, :F].copy()
    # the same samples gathered into FeatureSet order: the predict input layout
    dense.generate(n, F, group_rows=group_rows, divergence=0.8, seed=0, row_offset=offset,
                   col_map=feats, out=(x[:, :F], size, lab), device=dev)
    xg = x[:, :F]
    if args.x_dtype != "int32":
        assert int(xg.max()) < (256 if args.x_dtype == "uint8" else 65536), "counts do not fit"
        xg = xg.to(getattr(torch, args.x_dtype))   # lossless: every count fits
        del x
        torch.cuda.empty_cache()
    tables = dense.DeviceTables.build(fin.log_prior[:1], fin.log_lik[:1, :, :F],
                                      np.zeros(1, np.int32), group_size_bytes=width,
                                      max_size_bytes=width, device=dev)
    label = torch.empty(n, dtype=torch.int32, device=dev)
    logpost = None if args.no_logpost else torch.empty((n, 2), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        dense.predict(xg, size, tables, logpost=logpost is not None, label_out=label,
                      logpost_out=logpost)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark(True)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for a, b in evs:
        a.record(stream)
        step()
        b.record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    clocks.mark(False)
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t0.elapsed_time(t1)
    launch_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = barrier_max(total_ms, world, dev)
    mean_launch_ms = barrier_max(sum(launch_ms) / len(launch_ms), world, dev)
    ms_per_step = total_ms / args.steps
    value = total * args.steps / (total_ms / 1e3)     # every rank's rows / slowest rank

    # ---- the same rows stored as uint8 (lossless here): 4x fewer bytes per sample
    narrow = None

    def timed(xx, mode):
        for _ in range(3):
            dense.predict(xx, size, tables, logpost=logpost is not None, label_out=label,
                          logpost_out=logpost, mode=mode)
        a8, b8 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a8.record(stream)
        for _ in range(args.steps):
            dense.predict(xx, size, tables, logpost=logpost is not None, label_out=label,
                          logpost_out=logpost, mode=mode)
        b8.record(stream)
        b8.synchronize()
        return barrier_max(a8.elapsed_time(b8) / args.steps, world, dev)

    if args.x_dtype == "int32" and int(xg.max()) < 256:
        x8 = xg.to(torch.uint8)
        ms8 = timed(x8, "exact")
        bps8 = F + 4 + (4 + (16 if logpost is not None else 0))
        narrow = {"x_dtype": "uint8", "value": round(total / (ms8 / 1e3), 1),
                  "ms_per_step": round(ms8, 4), "bytes_per_sample": f"F+24 = {bps8}",
                  "achieved_gbs": round(n * bps8 / (ms8 / 1e3) / 1e9, 1),
                  "note": "same rows, counts < 256: K-PRED is FP64/I2F-bound, not HBM-bound"}
        # GNB_MODE_FMA (one rounding per term; not bit-exact, ~1e-12 relative):
        # halves the FP64 work where K-PRED is compute-bound
        ms8f = timed(x8, "fma")
        narrow["fma_mode"] = {"value": round(total / (ms8f / 1e3), 1),
                              "ms_per_step": round(ms8f, 4)}
        del x8

    # the narrow / fma timings above reused the output buffers: restore the
    # exact-mode int32 results that the parity check below compares
    step()
    torch.cuda.synchronize()

    # ---- correctness spot check of this run (labels vs generator classes)
    acc = float((label[:1_000_000] == lab[:1_000_000]).float().mean().item())

    # ---- roofline of the dominant (only) kernel
    out_bytes = 4 + (16 if logpost is not None else 0)
    eb = xg.element_size()
    bytes_per_sample = eb * F + 4 + out_bytes
    achieved = n * bytes_per_sample / (mean_launch_ms / 1e3) / 1e9
    peak, peak_kind = peaks()
    tps, ncu = ncu_traffic()
    # the committed capture is of cfg4 (int32, F=256, C=2): per-sample traffic
    # carries over to any row count of that shape, not to other shapes
    if not (F == 256 and eb == 4):
        tps, ncu = None, None
    wq = ((F * eb + 15) // 16) | 1
    kernel = ("gnb::predict_rowbox_kernel<2,T,2>" if wq <= 26 and wq * 16 // eb <= 256
              else "gnb::predict_tma_kernel<2,T,1,4,2>")
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "peak_source": peak_kind,
                "traffic": round(tps * n) if tps else None,
                "algorithmic_bytes_per_launch": n * bytes_per_sample,
                "bytes_per_sample": f"{eb}F+4+{out_bytes} = {bytes_per_sample}",
                "kernel": kernel,
                # report the 8.0 TB/s spec figure beside the measured peak
                "peak_spec": SPEC_HBM_GBS, "frac_spec": round(achieved / SPEC_HBM_GBS, 4)}
    if ncu:
        roofline["traffic_source"] = ncu.get("source")
    live = live_copy_gbs()
    if live:
        roofline["live_copy_gbs"] = round(live, 1)
        roofline["frac_live_copy"] = round(achieved / live, 4)

    # ---- end to end through the C ABI with host (pinned) buffers
    e2e = None
    xmax = _max_count(xg)
    host_dtype = "uint8" if xmax < 256 else ("uint16" if xmax < 65536 else "int32")
    if not args.no_e2e:
        # rows per rank: the e2e number is a throughput; keep the job's pinned
        # host memory bounded as ranks are added (all ranks share one host)
        m = min(max(args.e2e_rows // world, 1_000_000), n)
        sh = torch.empty(m, dtype=torch.int32, pin_memory=True)
        sh.copy_(size[:m])
        lh = torch.empty(m, dtype=torch.int32, pin_memory=True)
        ph = torch.empty((m, 2), dtype=torch.float64, pin_memory=True)
        prior = np.ascontiguousarray(fin.log_prior[:1])
        lik = np.ascontiguousarray(fin.log_lik[:1, :, :F])
        route = np.zeros(1, np.int32)
        el = ctypes.c_int64()

        def e2e_run(dtype_name, narrow=True, raw_every=None):
            xt = {"int32": N.X_I32, "uint16": N.X_U16, "uint8": N.X_U8, "uint4": N.X_U4}[dtype_name]
            if dtype_name == "uint4":    # two counts per byte, unpacked on the device
                pb = (F + 15) // 16 * 8
                xh = torch.empty((m, pb), dtype=torch.uint8, pin_memory=True)
                for i in range(0, m, 1 << 20):
                    j = min(i + (1 << 20), m)
                    dense.pack_u4(xg[i:j].cpu(), out=xh[i:j])
                ldx, row_b = 2 * pb, pb
            else:
                xh = torch.empty((m, F), dtype=getattr(torch, dtype_name), pin_memory=True)
                xh.copy_(xg[:m])
                ldx, row_b = F, xh.element_size() * F
            h2d_x = m * row_b
            if dtype_name == "int32" and narrow:
                # the library narrows int32 chunks losslessly on host threads (nibbles
                # if every count < 16, else bytes / half-words); from page-locked
                # memory every 3rd chunk goes raw by DMA meanwhile (api.cu,
                # kHostRawEvery) -- the exact wire bytes of that schedule:
                nb = ((F + 15) // 16 * 8 if xmax < 16 else (F + 15) // 16 * 16 if xmax < 256
                      else (F + 7) // 8 * 16 if xmax < 65536 else row_b)
                ld4 = (F + 3) // 4 * 4 * 4
                per = max(1024, (64 << 20) // ld4)
                per = (per + 127) // 128 * 128
                every = 3 if raw_every is None else raw_every
                h2d_x = 0
                for k, r0 in enumerate(range(0, m, per)):
                    cnt = min(per, m - r0)
                    h2d_x += cnt * (ld4 if every > 0 and k % every == every - 1 else nb)
            os.environ["GNB_HOST_NARROW"] = "1" if narrow else "0"
            if raw_every is not None:
                os.environ["GNB_HOST_RAW_EVERY"] = str(raw_every)

            def step():
                N.check(N.lib.gnb_predict_host_typed(
                    xh.data_ptr(), xt, m, F, ldx, sh.data_ptr(), width, width, route.ctypes.data,
                    1, 2, prior.ctypes.data, lik.ctypes.data, lh.data_ptr(), ph.data_ptr(), local,
                    ctypes.addressof(el)), "gnb_predict_host_typed")

            step()
            if world > 1:
                dist.barrier()
            t = time.perf_counter()
            for _ in range(args.e2e_steps):
                step()
            dt = barrier_max(time.perf_counter() - t, world, dev)
            os.environ.pop("GNB_HOST_NARROW", None)
            os.environ.pop("GNB_HOST_RAW_EVERY", None)
            ok = bool(torch.equal(lh, label[:m].cpu()))
            del xh
            return {"value": round(world * m * args.e2e_steps / dt, 1), "unit": UNIT,
                    "h2d_bytes_per_step": h2d_x + m * 4, "d2h_bytes_per_step": m * (4 + 16),
                    "host_x_bytes_per_step": m * row_b,
                    "rows_per_step_per_gpu": m, "x_host_dtype": dtype_name,
                    "api": "gnb_predict_host_typed (C ABI, pinned host buffers; int32 rows "
                           "narrowed on host threads / every 3rd chunk raw by DMA, H2D of X + "
                           "sizes, kernel, D2H of labels + log-posteriors, all inside the "
                           "timed region)",
                    "matches_device_labels": ok}

        # headline: the canonical int32 host rows, any counts; the
        # library picks the wire storage per chunk (lossless) -- data-independent
        # API, bound by host DRAM reads of the int32 rows, like the C port's
        e2e = e2e_run("int32")
        if world == 1:
            legs = {"int32_host_rows_no_narrowing": ("int32", False),
                    "int32_host_rows_narrowing_only": ("int32", True, 0)}
            if host_dtype != "int32":
                legs[f"{host_dtype}_host_rows"] = (host_dtype, True)
            if _max_count(xg[:m]) < 16:
                legs["uint4_host_rows_caller_packed"] = ("uint4", True)
            for name, leg in legs.items():
                e2e[name] = {k: v for k, v in e2e_run(*leg).items()
                             if k in ("value", "h2d_bytes_per_step")}
        del sh, lh, ph
        # the e2e rooflines: int32 host rows are read once by the host threads
        # that narrow them (host DRAM read bound); the narrowed rows then cross
        # PCIe (against a plain pinned 1 GiB torch copy on the same link)
        e2e["host_read"] = host_read_roofline(e2e, F, dev)
        e2e["pcie"] = pcie_roofline(e2e, dev)

    # ---- CPU baseline: C oracle on the box's host cores (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_from(xg, size, fin, F, width, args.cpu_seconds, "int32",
                                label=label, logpost=logpost)

    # ---- the reference-shaped object API (SampleRecord in, TimedRun out), rank 0, N=1
    obj = None
    if rank == 0 and world == 1 and not args.no_object_api:
        obj = object_api_leg(args.object_rows, V, local)

    return {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (reference synth law, GEN kernel, seed 0); model fitted on it",
        "config": {"workload": ("cfg4: predict 100M samples x 256 features sharded over the "
                                "GPUs, 2 classes, 1 size group")
                   if (total == DEFAULT_ROWS and V == DEFAULT_F and args.scaling == "strong")
                   else f"predict {total} samples x {V} features ({args.scaling} scaling), "
                        "2 classes",
                   "rows_total": total, "rows_per_gpu": n, "features": F, "classes": 2,
                   "x_dtype": args.x_dtype,
                   "outputs": "label int32 + log-posterior fp64 x2" if logpost is not None
                   else "label int32", "parity": "bit-exact vs reference (exact mode)",
                   "l2": "inputs (%.1f GB/GPU) >> 126 MB L2; no flush needed" % (n * 4 * F / 1e9),
                   "parallelism": f"dp{world} (row shards, no predict collective)"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "narrow_storage": narrow,
        "object_api": obj,
        "gpu_launches": args.steps * world, "clocks": clk,
        "accuracy_vs_generator_labels": round(acc, 4),
        "mean_launch_ms": round(mean_launch_ms, 4),
    }


def cpu_baseline_from(xg, size, fin, F, width, seconds, host_dtype="int32", label=None,
                      logpost=None):
    """C oracle (reference algorithm, exact) on a bounded sample of the same rows,
    stored like the e2e host rows (same storage on both sides): 2M rows taken at
    an even stride over the whole job, so the timed sample spans every part of
    the matrix.  As the checker, its outputs are also compared with the
    device's labels / log-posteriors of those rows (bit-exact expected)."""
    import numpy as np
    import torch
    from oracle import oracle as O
    n = xg.shape[0]
    sample = min(2_000_000, n)
    idx = torch.arange(sample, dtype=torch.int64, device=xg.device) * (n - 1) // max(sample - 1, 1)
    xs = xg[idx].cpu().numpy().astype(host_dtype)
    ss = size[idx].cpu().numpy()
    threads = os.cpu_count() or 1
    prior, lik = fin.log_prior[:1], fin.log_lik[:1, :, :F]
    route = np.zeros(1, np.int32)
    done, t = 0, time.perf_counter()
    out = None
    while True:
        out = O.c_predict(xs, ss, route, prior, lik, width=width, limit=width, threads=threads)
        done += sample
        if time.perf_counter() - t >= seconds:
            break
    dt = time.perf_counter() - t
    res = {"value": round(done / dt, 1), "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{sample} rows of this workload (even stride over all {n} rows), "
                     f"{done // sample} passes in {dt:.1f}s",
           "impl": "oracle/gnb_oracle.c (exact mul-then-add, pthreads)",
           "x_host_dtype": host_dtype, "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count()}
    if label is not None:
        want_lab, want_lp = out
        res["device_labels_equal"] = bool(np.array_equal(label[idx].cpu().numpy(), want_lab))
        if logpost is not None:
            res["device_logpost_bit_equal"] = (logpost[idx].cpu().numpy().tobytes() ==
                                               np.ascontiguousarray(want_lp).tobytes())
    return res


# ---------------------------------------------------------------- reference arm
def run_reference(args, world, rank):
    """The reference algorithm on the box's host cores (oracle port: the reference
    is pure Python and cannot be compiled)."""
    import numpy as np
    from oracle import oracle as O
    if rank != 0:
        return None
    V = args.features
    sample = args.ref_rows
    x, size, label = O.synth_dense(sample, V, seed=0, divergence=0.8)
    S, _, n, _, _ = O.fit_stats(x, size, label, 2, 5120, 5120)
    feats, _ = O.select_features(S[0], V, 0)
    t = O.train_tables(S[0], n[0], feats, 1.0, 0)
    xg = np.ascontiguousarray(x[:, feats])
    host_dtype = "int32"            # the storage of our e2e headline (int32 host rows)
    xg = xg.astype(host_dtype)
    route = np.zeros(1, np.int32)
    threads = os.cpu_count() or 1

    def step():
        O.c_predict(xg, size, route, t.log_prior[None], t.log_lik[None], width=5120,
                    limit=5120, threads=threads)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = sample * args.steps / dt
    ref_py = reference_python_leg(args.ref_py_samples, V) if args.ref_py_samples > 0 else None
    return {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "impl": "reference",
        "data": "synthetic (reference synth law, numpy)",
        "config": {"workload": "cfg4: predict 100M samples x 256 features per GPU, 2 classes, "
                               "1 size group (CPU: bounded sample per step)",
                   "rows_per_step": sample, "features": V, "classes": 2,
                   "x_host_dtype": host_dtype},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": threads,
                         "kind": "port", "sample": f"{sample} rows per step",
                         "impl": "oracle/gnb_oracle.c", "cpu_model": cpu_model(),
                         "os_cpu_count": os.cpu_count()},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_python": ref_py,
    }


def host_read_roofline(e2e, F, dev):
    """Achieved host DRAM read GB/s of the int32 e2e rows vs this host's own
    ceiling for the same two readers at once: all cores streaming an int32 ->
    uint8 narrow (torch copy, 2 GiB) while the copy engine DMAs a pinned
    1 GiB buffer to the device in a loop (the e2e path reads the int32 rows
    with both)."""
    import torch
    n = (2 << 30) // (4 * F)
    src = torch.ones((n, F), dtype=torch.int32)
    dst = torch.empty((n, F), dtype=torch.uint8)
    h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    threads = torch.get_num_threads()
    torch.set_num_threads(os.cpu_count() or 1)
    dst.copy_(src)
    stream = torch.cuda.Stream(dev)
    done = threading.Event()
    dma = {"bytes": 0}

    def pump():
        with torch.cuda.stream(stream):
            while not done.is_set():
                d.copy_(h, non_blocking=True)
                stream.synchronize()
                dma["bytes"] += 1 << 30

    th = threading.Thread(target=pump, daemon=True)
    th.start()
    t = time.perf_counter()
    for _ in range(3):
        dst.copy_(src)
    dt = time.perf_counter() - t
    done.set()
    th.join()
    cpu_gbs = 3 * n * F * 4 / dt / 1e9
    dma_gbs = dma["bytes"] / dt / 1e9
    torch.set_num_threads(threads)
    rows_per_s = e2e["value"] / max(int(os.environ.get("WORLD_SIZE", "1")), 1)
    achieved = rows_per_s * e2e["host_x_bytes_per_step"] / e2e["rows_per_step_per_gpu"] / 1e9
    peak = cpu_gbs + dma_gbs
    del src, dst, h, d
    return {"bound": "host_dram_read", "achieved_gbs": round(achieved, 1),
            "peak_gbs": round(peak, 1), "frac": round(achieved / peak, 3),
            "peak_source": "all-core torch int32->uint8 copy (%.1f GB/s) concurrent with a "
                           "pinned H2D DMA loop (%.1f GB/s)" % (cpu_gbs, dma_gbs)}


def pcie_roofline(e2e, dev):
    """Achieved H2D GB/s of the e2e leg vs a pinned 1 GiB host->device copy."""
    import torch
    h = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    b.record()
    b.synchronize()
    peak = 3 * (1 << 30) / (a.elapsed_time(b) / 1e3) / 1e9
    rows_per_s = e2e["value"] / max(int(os.environ.get("WORLD_SIZE", "1")), 1)
    achieved = rows_per_s * e2e["h2d_bytes_per_step"] / e2e["rows_per_step_per_gpu"] / 1e9
    del h, d
    return {"bound": "pcie_h2d", "achieved_gbs": round(achieved, 1),
            "copy_gbs": round(peak, 1), "frac": round(achieved / peak, 3)}


def cpu_model() -> str:
    """The host CPU's model name (lscpu's "Model name"), from /proc/cpuinfo."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def object_api_leg(n, V, device):
    """The drop-in a reference user calls: train_bundle + classify_parallel on n
    SampleRecords of the synthetic law (1 size group, V opcodes, k = V), wall
    time of each call (ADAPT walk + device + TimedRun objects) and the device
    share (TimedRun.elapsed_ns, the reference's own classification clock).
    Compare with `reference_python` in the --impl reference line."""
    import numpy as np
    import paper_1905_13746_b200 as gnb
    rng = np.random.default_rng(0)
    vocab = [f"op{i:03d}" for i in range(V)]
    label = np.arange(n) % 2
    size = rng.integers(0, 5120, size=n)
    w = np.where(np.arange(V)[None, :] < V // 2, 1.0, 0.2)
    p = np.where(label[:, None] == 1, w, w[:, ::-1])
    x = rng.poisson((64 + size // 64)[:, None] * (p / p.sum(1, keepdims=True)))
    samples = []
    for i in range(n):
        nz = np.nonzero(x[i])[0]
        samples.append(gnb.SampleRecord(
            f"s{i}", gnb.Label.MALWARE if label[i] else gnb.Label.BENIGN, int(size[i]),
            gnb.OpcodeHistogram.from_counts({vocab[j]: int(x[i, j]) for j in nz})))
    grouped, _ = gnb.partition_by_group(samples, gnb.GroupingConfig())
    gnb.train_bundle(grouped, V, created_at="bench", device=device)        # warm
    t = time.perf_counter()
    bundle = gnb.train_bundle(grouped, V, created_at="bench", device=device)
    fit_s = time.perf_counter() - t
    wl = gnb.Workload(tuple(samples), lanes=os.cpu_count() or 1)
    gnb.classify_parallel(bundle, wl, device=device)                      # warm
    t = time.perf_counter()
    run = gnb.classify_parallel(bundle, wl, warmup=False, device=device)
    cls_s = time.perf_counter() - t
    acc = float(np.mean([(p.label == gnb.Label.MALWARE) == bool(label[i])
                         for i, p in enumerate(run.predictions)]))
    return {"api": "paper_1905_13746_b200.train_bundle / classify_parallel (reference "
                   "signatures, SampleRecord in, TimedRun out)",
            "samples": n, "features": V, "k": V,
            "train_bundle_samples_per_s": round(n / fit_s, 1),
            "classify_parallel_wall_samples_per_s": round(n / cls_s, 1),
            "classify_parallel_elapsed_samples_per_s": round(n / (run.elapsed_ns / 1e9), 1),
            "accuracy": round(acc, 4)}


def _max_count(t):
    """Largest count of a device row block (torch has no max kernel for uint16)."""
    import torch
    return int((t.to(torch.int32) if t.dtype == torch.uint16 else t).max())


def reference_python_leg(n, V):
    """The UNMODIFIED reference package (baseline/_ref, pip-installed from
    /root/reference) through its own public API on a bounded sample: Tc =
    classify_sequential (1 core), Tp = classify_parallel (all cores), both by the
    reference's own elapsed_ns.  Reported beside the C port."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "groupnb")):
        return {"unavailable": "baseline/_ref not installed (see DESIGN.md section 5)"}
    try:
        if ref not in sys.path:
            sys.path.insert(0, ref)
        from groupnb.corpus import GroupingConfig, partition_by_group
        from groupnb.engine import Workload, classify_parallel, classify_sequential, train_bundle
        from groupnb.synth import SyntheticSpec, generate_synthetic
        t0 = time.perf_counter()
        spec = SyntheticSpec(group_count=1, samples_per_group_per_class=n // 2,
                             vocabulary_size=V, divergence=0.8, seed=0)
        samples = generate_synthetic(spec)
        grouped, _ = partition_by_group(samples, GroupingConfig())
        t1 = time.perf_counter()
        bundle = train_bundle(grouped, k=V)
        t2 = time.perf_counter()
        work = tuple(samples)
        lanes = os.cpu_count() or 1
        tc = classify_sequential(bundle, Workload(work, 1), warmup=False)
        tp = classify_parallel(bundle, Workload(work, lanes), warmup=False)
        return {"impl": "groupnb (reference pkg, unmodified)", "samples": len(work),
                "features": V, "classes": 2,
                "Tc_samples_per_s": round(len(work) / (tc.elapsed_ns / 1e9), 1),
                "Tp_samples_per_s": round(len(work) / (tp.elapsed_ns / 1e9), 1),
                "Tp_lanes": lanes,
                "fit_samples_per_s": round(len(work) / (t2 - t1), 1),
                "generate_s": round(t1 - t0, 2),
                "labels_equal_Tc_Tp": [p.label for p in tc.predictions] ==
                                      [p.label for p in tp.predictions]}
    except Exception as e:  # reported, never fatal for the C-port arm
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}


# ---------------------------------------------------------------- secondary workloads
FLUSH_MODE = "clean"


def _pitch(args, F):
    """int32 row pitch (elements): 16-B multiple ("packed") or 128-B line ("line")."""
    return (F + 31) // 32 * 32 if args.pitch == "line" else (F + 3) // 4 * 4


def _timed_launches(fn, steps, warmup, flush_bytes=512 << 20):
    """Mean device time (ms) of fn() over `steps` launches, L2 flushed before each
    (a 512 MB write, > 126 MB L2; in "clean" mode followed by a 256 MB read of a
    second buffer so the flush's dirty lines are written back before the timed
    region, not inside it), CUDA events on the launching stream, with the
    launch already queued behind a short device sleep when the first event fires."""
    import torch
    flush = torch.empty(flush_bytes // 4, dtype=torch.int32, device="cuda")
    clean = torch.ones(flush_bytes // 8, dtype=torch.int32, device="cuda")
    sink = torch.empty((), dtype=torch.int64, device="cuda")
    for _ in range(warmup):
        fn()
    # and at least ~0.3 s of back-to-back work, so SM/memory clocks have left
    # any idle state before the first timed launch of a short kernel
    torch.cuda.synchronize()
    t_end = time.perf_counter() + 0.3
    while time.perf_counter() < t_end:
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
    times = []
    s = torch.cuda.current_stream()
    # `warmup` untimed rounds of the exact measured sequence (flush, clean
    # read, sleep, launch) first: the first rounds on freshly allocated
    # buffers ran ~8 % slower than every later one
    for it in range(warmup + steps):
        flush.zero_()
        if FLUSH_MODE == "clean":
            torch.sum(clean, 0, out=sink)
        # keep the GPU busy ~50 us so the host has enqueued fn()'s launch before
        # event a fires: the events then bracket device time only, not the
        # Python/ctypes launch path of a 40-700 us kernel
        torch.cuda._sleep(100_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        if it >= warmup:
            times.append(a.elapsed_time(b))
    return sum(times) / len(times), statistics.median(times)


def run_sweep(args, world, rank, local):
    """cfg2: F = 50/100/200/500/1000 at 1M samples, 2 classes, 1 B200."""
    import numpy as np
    import torch
    from oracle import oracle as O
    from paper_1905_13746_b200 import dense
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n = 1_000_000
    peak, kind = peaks()
    rows = []
    for F in (50, 100, 200, 500, 1000):
        x, size, lab = dense.generate(n, F, divergence=0.8, seed=0, device=dev,
                                      ldx=_pitch(args, F))
        st = dense.fit_stats(x, size, lab, n_classes=2, group_size_bytes=5120,
                             max_size_bytes=5120)
        fin = dense.fin_train(st.sums.cpu().numpy(), st.counts.cpu().numpy(), k=F, alpha=1.0,
                              min_per_class=6)
        nf = int(fin.n_features[0])
        feats = fin.features[0, :nf].copy()
        dense.generate(n, nf, divergence=0.8, seed=0, col_map=feats,
                       out=(x[:, :nf], size, lab), device=dev)
        t = dense.DeviceTables.build(fin.log_prior[:1], fin.log_lik[:1, :, :nf],
                                     np.zeros(1, np.int32), group_size_bytes=5120,
                                     max_size_bytes=5120, device=dev)
        label = torch.empty(n, dtype=torch.int32, device=dev)
        lp = torch.empty((n, 2), dtype=torch.float64, device=dev)
        mean_ms, med_ms = _timed_launches(
            lambda: dense.predict(x[:, :nf], size, t, label_out=label, logpost_out=lp),
            args.steps, max(args.warmup, 3))
        bps = 4 * nf + 24
        # parity spot check of this launch: the C oracle on a strided subsample
        idx = torch.arange(0, n, 97, device=dev)
        want, wlp = O.c_predict(x[:, :nf][idx].cpu().numpy(), size[idx].cpu().numpy(),
                                np.zeros(1, np.int32), fin.log_prior[:1],
                                fin.log_lik[:1, :, :nf], width=5120, limit=5120, threads=8)
        exact = bool(np.array_equal(label[idx].cpu().numpy(), want) and
                     lp[idx].cpu().numpy().tobytes() == wlp.tobytes())
        # the same byte count through a plain device copy (half read, half
        # written) timed identically (flush, sleep, events): what ONE isolated
        # launch of this size can reach at all (launch + ramp + wave tail)
        half = n * bps // 2 // 4
        src = torch.ones(half, dtype=torch.int32, device=dev)
        dst = torch.empty_like(src)
        copy_ms, _ = _timed_launches(lambda: dst.copy_(src), args.steps, max(args.warmup, 3))
        del src, dst
        rows.append({"F": nf, "ldx": int(x.stride(0)), "ms": round(mean_ms, 4),
                     "samples_per_s": round(n / (mean_ms / 1e3), 1),
                     "achieved_gbs": round(n * bps / (mean_ms / 1e3) / 1e9, 1),
                     "frac": round(n * bps / (mean_ms / 1e3) / 1e9 / peak, 4),
                     "copy_same_bytes": {"ms": round(copy_ms, 4),
                                         "frac": round(n * bps / (copy_ms / 1e3) / 1e9 / peak, 4)},
                     "frac_of_copy": round(copy_ms / mean_ms, 4),
                     "bit_exact_subsample_vs_oracle": exact})
        del x, size, lab, label, lp
    return {"metric": METRIC, "workload": "cfg2: F sweep at 1M samples, 2 classes, L2 flushed "
            "before every launch", "flush": FLUSH_MODE, "pitch": args.pitch, "unit": UNIT, "peak_gbs": peak, "peak_source": kind,
            "bytes_per_sample": "4F+24", "rows": rows, "steps": args.steps}


def run_ragged(args, world, rank, local):
    """cfg3: 4,194,304 samples in 32 ragged size groups (n_g ~ 0.9^g), F=200, groups
    {5, 8, 17} untrained (routed), one K-PRED launch for all groups."""
    import numpy as np
    import torch
    from oracle import oracle as O
    from paper_1905_13746_b200 import _native as N_
    from paper_1905_13746_b200 import dense
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    G, V, N = 32, 200, 4_194_304
    w = 0.9 ** np.arange(G)
    counts = np.floor(N * w / w.sum()).astype(np.int64)
    counts[0] += N - counts.sum()
    width, limit = 5120, G * 5120
    x, size, lab = dense.generate(N, V, group_rows=counts, divergence=0.8, seed=0, device=dev,
                                  ldx=_pitch(args, V))
    st = dense.fit_stats(x, size, lab, n_classes=2, group_size_bytes=width, max_size_bytes=limit)
    fin = dense.fin_train(st.sums.cpu().numpy(), st.counts.cpu().numpy(), k=V, alpha=1.0,
                          min_per_class=6)
    trained = [g for g in range(G) if fin.state[g] == 1 and g not in (5, 8, 17)]
    slot = {g: i for i, g in enumerate(trained)}
    route = np.array([slot[int(g)] for g in O.route_table(trained, G)], np.int32)
    F = int(max(fin.n_features[g] for g in trained))
    prior = fin.log_prior[trained]
    lik = fin.log_lik[trained][:, :, :F]
    feats = fin.features[trained][:, :F].astype(np.int32)
    nfeat = fin.n_features[trained].astype(np.int32)
    t = dense.DeviceTables.build(prior, lik, route, group_size_bytes=width, max_size_bytes=limit,
                                 device=dev)
    xg = dense.gather_features(x, size, t, feats, nfeat)
    label = torch.empty(N, dtype=torch.int32, device=dev)
    lp = torch.empty((N, 2), dtype=torch.float64, device=dev)
    mean_ms, med_ms = _timed_launches(
        lambda: dense.predict(xg, size, t, label_out=label, logpost_out=lp),
        args.steps, max(args.warmup, 3))
    # parity spot check against the C oracle on a strided subsample
    idx = np.arange(0, N, 97)
    xs, ss = xg.cpu().numpy()[idx], size.cpu().numpy()[idx]
    want, wlp = O.c_predict(xs, ss, route, prior, lik, width=width, limit=limit, threads=8)
    ok = bool((label.cpu().numpy()[idx] == want).all() and
              lp.cpu().numpy()[idx].tobytes() == wlp.tobytes())
    peak, kind = peaks()
    bps = 4 * F + 24
    shuf = torch.randperm(N, device=dev)
    xs_, ss_ = xg[shuf].contiguous(), size[shuf].contiguous()
    lab_g, lp_g = label.clone(), lp.clone()   # grouped-order outputs (oracle-checked above)
    mix_ms, _ = _timed_launches(
        lambda: dense.predict(xs_, ss_, t, label_out=label, logpost_out=lp), args.steps, 3)
    hint_ms, _ = _timed_launches(
        lambda: dense.predict(xs_, ss_, t, label_out=label, logpost_out=lp, order="mixed"),
        args.steps, 3)
    # shuffled outputs == grouped outputs at the same rows (bit for bit)
    mix_ok = bool(torch.equal(label, lab_g[shuf]) and
                  torch.equal(lp.view(torch.int64), lp_g[shuf].view(torch.int64)))
    mixed_rows = int(N_.lib.gnb_predict_mixed_rows(F, N_.X_I32, 2, len(trained)))
    # same shuffled batch, device slot sort + gather4 K-PRED (both inside the timed launch)
    srt_ms, _ = _timed_launches(
        lambda: dense.predict(xs_, ss_, t, label_out=label, logpost_out=lp,
                              perm=dense.slot_sort(ss_, t)), args.steps, 3)
    lab_srt = label.clone()
    dense.predict(xs_, ss_, t, label_out=label, logpost_out=lp)
    srt_ok = bool(torch.equal(lab_srt, label))
    return {"metric": METRIC, "workload": "cfg3: 4,194,304 samples, 32 ragged size groups "
            "(0.9^g), F=200, groups 5/8/17 untrained -> routed, single launch",
            "flush": FLUSH_MODE, "pitch": args.pitch, "unit": UNIT, "value": round(N / (mean_ms / 1e3), 1), "ms": round(mean_ms, 4),
            "achieved_gbs": round(N * bps / (mean_ms / 1e3) / 1e9, 1),
            "frac": round(N * bps / (mean_ms / 1e3) / 1e9 / peak, 4), "peak_gbs": peak,
            "trained_groups": len(trained), "bit_exact_subsample_vs_oracle": ok,
            "shuffled_rows": {"ms": round(mix_ms, 4),
                              "value": round(N / (mix_ms / 1e3), 1),
                              "frac": round(N * bps / (mix_ms / 1e3) / 1e9 / peak, 4),
                              "bit_exact_vs_grouped_order": mix_ok,
                              "kernel": ("predict_mixed_kernel (all slot tables resident in "
                                         "smem, in-tile slot sort, no device sort)"
                                         if mixed_rows else "predict_tma_kernel (L1 tables)"),
                              "order_hint_mixed": {"ms": round(hint_ms, 4),
                                                   "frac": round(N * bps / (hint_ms / 1e3) / 1e9 / peak, 4)},
                              "note": "same rows in random order, one plain predict call "
                                      "(order auto: a device count of the tiles that mix "
                                      "models gates the kernel choice, timed)"},
            "shuffled_rows_slot_sorted": {
                "ms": round(srt_ms, 4), "value": round(N / (srt_ms / 1e3), 1),
                "frac": round(N * bps / (srt_ms / 1e3) / 1e9 / peak, 4),
                "labels_equal_unsorted_path": srt_ok,
                "note": "gnb_slot_sort (device counting sort by routed slot) + K-PRED with "
                        "TMA tile::gather4, both timed"}}


def run_fit(args, world, rank, local):
    """cfg5: fit statistics (S, Q, n) over 1B samples x 128 features, 16 classes,
    rows sharded over the ranks, generated in 100M-row chunks (512 GB total does
    not fit one GPU), fit kernel timed per chunk, one NCCL all-reduce at the end."""
    import numpy as np
    import torch
    from paper_1905_13746_b200 import dense
    from paper_1905_13746_b200.sharding import allreduce_stats, shard_bounds
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    total, V, C = args.fit_rows, 128, 16
    lo, hi = shard_bounds(total, world, rank)
    chunk = min(100_000_000, hi - lo)
    x, size, lab = dense.generate(chunk, V, n_classes=C, group_rows=[total], divergence=0.8,
                                  seed=0, row_offset=lo, device=dev)
    xt = getattr(torch, args.x_dtype)
    xs = x if args.x_dtype == "int32" else torch.empty((chunk, V), dtype=xt, device=dev)
    # warm-up launch (module load, tensor-map path) outside the timed region
    dense.fit_stats(xs[:1024], size[:1024], lab[:1024], n_classes=C, group_size_bytes=5120,
                    max_size_bytes=5120)
    st = None
    ms = 0.0
    s = torch.cuda.current_stream()
    for r0 in range(lo, hi, chunk):
        n = min(chunk, hi - r0)
        dense.generate(n, V, n_classes=C, group_rows=[total], divergence=0.8, seed=0,
                       row_offset=r0, out=(x[:n], size[:n], lab[:n]), device=dev)
        if args.x_dtype != "int32":        # same counts, narrower storage (lossless check)
            assert int(x[:n].max()) < (256 if args.x_dtype == "uint8" else 65536)
            xs[:n].copy_(x[:n])
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        st = dense.fit_stats(xs[:n], size[:n], lab[:n], n_classes=C, group_size_bytes=5120,
                             max_size_bytes=5120, out=st, accumulate=st is not None)
        b.record(s)
        b.synchronize()
        ms += a.elapsed_time(b)
    # parity spot check on this workload's data: the first 1M rows of the last
    # chunk fitted again and compared with the C oracle's exact integer counts
    from oracle import oracle as O
    m = min(1_000_000, n)
    chk = dense.fit_stats(xs[:m], size[:m], lab[:m], n_classes=C, group_size_bytes=5120,
                          max_size_bytes=5120)
    So, Qo, no, bado, ooro = O.c_fit_stats(x[:m].cpu().numpy(), size[:m].cpu().numpy(),
                                           lab[:m].cpu().numpy(), C, 5120, 5120)
    exact = bool(np.array_equal(chk.sums.cpu().numpy(), So.astype(np.float64)) and
                 np.array_equal(chk.sumsq.cpu().numpy(), Qo.astype(np.float64)) and
                 np.array_equal(chk.counts.cpu().numpy(), no.astype(np.float64)) and
                 chk.status.cpu().tolist() == [bado, ooro])
    del chk
    if world > 1:
        torch.distributed.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    allreduce_stats(st)
    b.record(s)
    b.synchronize()
    ar_ms = a.elapsed_time(b)
    ms = barrier_max(ms, world, dev)
    peak, kind = peaks()
    bps = xs.element_size() * V + 8
    rows_here = hi - lo
    n_total = float(st.counts.sum().item())
    return {"metric": "samples fitted/sec (sums, sums of squares, counts)", "unit": UNIT,
            "workload": (f"cfg5: fit {total:,} samples x 128 features, 16 classes, 1 size group"
                         if total == 1_000_000_000 else
                         f"fit {total:,} samples x 128 features, 16 classes"),
            "value": round(total / ((ms + ar_ms) / 1e3), 1), "fit_kernel_ms": round(ms, 3),
            "allreduce_ms": round(ar_ms, 4), "n_gpus": world,
            "achieved_gbs_per_gpu": round(rows_here * bps / (ms / 1e3) / 1e9, 1),
            "frac": round(rows_here * bps / (ms / 1e3) / 1e9 / peak, 4), "peak_gbs": peak,
            "bytes_per_sample": f"{xs.element_size()}V+8", "x_dtype": args.x_dtype,
            "rows_counted": n_total, "bit_exact_chunk_vs_oracle": exact,
            "stats_bytes_allreduced": int(st.packed().numel() * 8)}


def run_fin(args, world, rank, local):
    """FIN: feature scoring + top-k + logs for every size
    group from the fitted statistics, host C++ (gnb_fin_train) vs device
    (gnb_fin_train_device, scoring + bitonic top-k on the GPU, logs on the
    host); outputs must be identical.  Wall time per call, median of `steps`."""
    import numpy as np
    import torch
    from paper_1905_13746_b200 import dense
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    rows = []
    for G, V, k in ((32, 256, 100), (32, 1024, 200), (8, 16384, 256)):
        n = 20_000 * G if V <= 1024 else 4_000 * G
        x, size, lab = dense.generate(n, V, group_rows=[n // G] * G, divergence=0.8, seed=1,
                                      device=dev)
        st = dense.fit_stats(x, size, lab, n_classes=2, group_size_bytes=5120,
                             max_size_bytes=5120 * G)
        S, cnt = st.sums.cpu().numpy(), st.counts.cpu().numpy()
        del x, size, lab

        def host():
            return dense.fin_train(S, cnt, k=k, alpha=1.0, min_per_class=6)

        def device():
            r = dense.fin_train_device(st, k=k, alpha=1.0, min_per_class=6)
            torch.cuda.synchronize()
            return r

        h, d = host(), device()
        same = all(np.array_equal(getattr(h, f), getattr(d, f))
                   for f in ("state", "n_features", "features", "log_prior", "log_lik"))
        # the oracle (pinned to the reference) on the first trained group
        from oracle import oracle as O
        g0 = int(np.nonzero(h.state == 1)[0][0])
        feats, _ = O.select_features(S[g0].astype(np.int64), k, g0)
        tt = O.train_tables(S[g0].astype(np.int64), cnt[g0].astype(np.int64), feats, 1.0, g0)
        F0 = int(d.n_features[g0])
        oracle_ok = (feats.tolist() == d.features[g0, :F0].tolist() and
                     tt.log_lik.tobytes() == np.ascontiguousarray(d.log_lik[g0, :, :F0]).tobytes())
        th, td = [], []
        for _ in range(max(args.steps, 5)):
            t0 = time.perf_counter()
            host()
            th.append(time.perf_counter() - t0)
            t0 = time.perf_counter()
            device()
            td.append(time.perf_counter() - t0)
        rows.append({"groups": G, "vocab": V, "k": k, "host_ms": round(statistics.median(th) * 1e3, 3),
                     "device_ms": round(statistics.median(td) * 1e3, 3), "identical": same,
                     "bit_exact_group_vs_oracle": oracle_ok})
        del st
    return {"metric": "FIN wall time per call (feature scoring + top-k + log tables, all groups)",
            "workload": "fin: G groups x V vocabulary statistics from K-FIT on synthetic rows",
            "unit": "ms", "rows": rows}


def main():
    global FLUSH_MODE
    args = parse()
    FLUSH_MODE = args.flush
    relaunch_if_needed(args)
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        out = run_reference(args, world, rank)
    elif args.workload == "sweep":
        out = run_sweep(args, world, rank, local)
    elif args.workload == "ragged":
        out = run_ragged(args, world, rank, local)
    elif args.workload == "fin":
        out = run_fin(args, world, rank, local)
    elif args.workload == "fit":
        out = run_fit(args, world, rank, local)
    else:
        out = run_ours(args, world, rank, local)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
