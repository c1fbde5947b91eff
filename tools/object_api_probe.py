#!/usr/bin/env python
"""Where the object-level drop-in (classify_parallel on SampleRecords) spends
its wall time: ADAPT gather, the device call (warm), TimedRun construction.

    gpurun -- python tools/object_api_probe.py [--rows N]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1905_13746_b200 as gnb  # noqa: E402
from paper_1905_13746_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=200_000)
    ap.add_argument("--vocab", type=int, default=256)
    ap.add_argument("--k", type=int, default=100)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    n, V = a.rows, a.vocab
    vocab = [f"op{i:03d}" for i in range(V)]
    label = rng.integers(0, 2, size=n)
    size = rng.integers(0, 32 * 5120, size=n)
    w = np.where(np.arange(V)[None, :] < V // 2, 1.0, 0.2)
    p = np.where(label[:, None] == 1, w, w[:, ::-1])
    p = p / p.sum(1, keepdims=True)
    x = rng.poisson((64 + size // 64)[:, None] * p)
    samples = []
    for i in range(n):
        nz = np.nonzero(x[i])[0]
        samples.append(gnb.SampleRecord(
            f"s{i}", gnb.Label.MALWARE if label[i] else gnb.Label.BENIGN, int(size[i]),
            gnb.OpcodeHistogram.from_counts({vocab[j]: int(x[i, j]) for j in nz})))
    cfg = gnb.GroupingConfig()
    grouped, _ = gnb.partition_by_group(samples, cfg)
    out = {"rows": n, "vocab": V, "k": a.k}
    gnb.train_bundle(grouped, a.k, created_at="p")
    t = time.perf_counter()
    bundle = gnb.train_bundle(grouped, a.k, created_at="p")
    out["fit_object_s"] = round(time.perf_counter() - t, 3)
    wl = gnb.Workload(tuple(samples), lanes=8)
    gnb.classify_parallel(bundle, wl)                       # buffers, context
    t = time.perf_counter()
    packed = api._PackedBundle(bundle, api._ns.of(bundle))
    out["pack_s"] = round(time.perf_counter() - t, 4)
    t = time.perf_counter()
    xg, sz = api._gather(samples, packed, cfg)
    out["adapt_gather_s"] = round(time.perf_counter() - t, 4)
    t = time.perf_counter()
    lab, lp, el = api._predict_host(xg, sz, packed, cfg.group_count, [0])
    out["device_call_s"] = round(time.perf_counter() - t, 4)
    out["device_elapsed_s"] = round(el / 1e9, 4)
    t = time.perf_counter()
    run = gnb.classify_parallel(bundle, wl, warmup=False)
    out["classify_parallel_s"] = round(time.perf_counter() - t, 3)
    out["classify_parallel_samples_per_s"] = round(n / out["classify_parallel_s"], 1)
    out["elapsed_ns"] = run.elapsed_ns
    out["timedrun_build_s_est"] = round(out["classify_parallel_s"] - out["adapt_gather_s"]
                                        - out["device_call_s"] - out["pack_s"], 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
