#!/usr/bin/env python
"""End-to-end wall time of the reference-shaped pipelines on one GPU.

    python tools/e2e_pipeline.py [--rows N] [--vocab V] [--k K]

(1) object API: SampleRecords -> train_bundle -> classify_parallel (ADAPT + C ABI)
(2) JSONL API:  text -> read_corpus -> train_bundle_corpus -> classify_corpus
                -> predictions_jsonl (C++ ingest / writer + device kernels)
Prints one JSON line (seconds and samples/s per stage).
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_1905_13746_b200 as gnb  # noqa: E402
from paper_1905_13746_b200 import ingest  # noqa: E402
from paper_1905_13746_b200.api import classify_corpus, train_bundle_corpus  # noqa: E402


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
    lines = []
    for i in range(n):
        nz = np.nonzero(x[i])[0]
        lines.append(json.dumps({"id": f"s{i}", "label": "malware" if label[i] else "benign",
                                 "size_bytes": int(size[i]),
                                 "opcodes": {vocab[j]: int(x[i, j]) for j in nz}}))
    text = "\n".join(lines) + "\n"
    cfg = gnb.GroupingConfig()
    out = {"rows": n, "vocab": V, "k": a.k, "jsonl_mb": round(len(text) / 1e6, 1)}

    t = time.perf_counter()
    corpus = ingest.read_corpus(text)
    out["ingest_s"] = round(time.perf_counter() - t, 3)
    train_bundle_corpus(corpus, cfg, a.k, created_at="e2e")   # first CUDA use
    t = time.perf_counter()
    bundle = train_bundle_corpus(corpus, cfg, a.k, created_at="e2e")
    out["fit_corpus_s"] = round(time.perf_counter() - t, 3)
    classify_corpus(bundle, corpus, warmup=False)   # CUDA context / module load
    t = time.perf_counter()
    lab, lp, eff, errors, elapsed = classify_corpus(bundle, corpus, warmup=False)
    out["classify_corpus_s"] = round(time.perf_counter() - t, 3)
    out["classify_corpus_device_s"] = round(elapsed / 1e9, 4)
    t = time.perf_counter()
    text_out = corpus.predictions_jsonl(lab, lp, eff, cfg.max_size_bytes)
    out["write_s"] = round(time.perf_counter() - t, 3)
    total = out["ingest_s"] + out["fit_corpus_s"] + out["classify_corpus_s"] + out["write_s"]
    out["jsonl_pipeline_samples_per_s"] = round(n / total, 1)
    out["accuracy"] = round(float((lab == label).mean()), 4)

    samples = corpus.records()
    grouped, _ = gnb.partition_by_group(samples, cfg)
    t = time.perf_counter()
    b2 = gnb.train_bundle(grouped, a.k, created_at="e2e")
    out["fit_object_s"] = round(time.perf_counter() - t, 3)
    gnb.classify_parallel(b2, gnb.Workload(tuple(samples), lanes=8), warmup=False)  # warm
    t = time.perf_counter()
    run = gnb.classify_parallel(b2, gnb.Workload(tuple(samples), lanes=8), warmup=False)
    out["classify_object_s"] = round(time.perf_counter() - t, 3)
    out["classify_object_elapsed_ns"] = run.elapsed_ns
    same = all(p is not None and p.label == (gnb.Label.MALWARE if l == 1 else gnb.Label.BENIGN)
               for p, l in zip(run.predictions, lab))
    out["object_equals_corpus_path"] = bool(same) and b2 == bundle
    print(json.dumps(out))


if __name__ == "__main__":
    main()
