"""The paper's Figs. 2-4 sweep, GPU mode, through the reference's OWN harness.

The unmodified reference (`groupnb`, baseline/_ref) with the GPU backend
installed (`backend.install`): its `train_bundles` fits on the B200, its
`run_bench` times `classify_sequential` (Tc, the reference's own single-core
Python, unchanged) against `classify_parallel` (Tp, now K-PRED on the GPU) for
every feature budget k x batch of 768*m files (bench.py:114-172), and
`emit_csv` writes the reference's CSV (bench.py:175-183).
plots CPU vs GPU time against batch size and k (figures absent from the text;
"up to 200x" on a GTX 1050Ti vs an i7-7700HQ).

    python tools/paper_sweep.py [--out profiles/r02_paper_sweep.csv] [--reps 3]

Prints one JSON summary line (speedup per k at the largest batch, Tp samples/s).
"""
import argparse
import io
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)

import groupnb as gn  # noqa: E402

from paper_1905_13746_b200 import backend  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_paper_sweep.csv"))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--groups", type=int, default=8)
    ap.add_argument("--per-class", type=int, default=150)
    ap.add_argument("--vocab", type=int, default=256)
    ap.add_argument("--counts", default="1,2,4,8,16")
    a = ap.parse_args()
    calls = backend.install(gn)
    t0 = time.perf_counter()
    spec = gn.SyntheticSpec(group_count=a.groups, samples_per_group_per_class=a.per_class,
                            vocabulary_size=a.vocab, divergence=0.8, seed=2026)
    corpus = gn.generate_synthetic(spec)
    grouped, _ = gn.partition_by_group(corpus, gn.GroupingConfig())
    split = gn.split_train_test(grouped, (2, 1), seed=0)
    ks = (20, 40, 80, 100, 160, 200)
    bundles = gn.train_bundles(split.train, ks, created_at="sweep")
    test = split.test.all_samples()
    config = gn.BenchConfig(k_values=ks, batch_multiple=768,
                            batch_counts=tuple(int(c) for c in a.counts.split(",")),
                            lanes=os.cpu_count() or 1, repetitions=a.reps)
    report = gn.run_bench(bundles, test, config)
    buf = io.StringIO()
    gn.emit_csv(report, buf)
    text = buf.getvalue()
    assert gn.parse_csv(text) == report
    with open(a.out, "w") as fh:
        fh.write(text)
    # accuracy of the GPU bundles on the held-out split (reference Tc predictions)
    acc = {}
    for k in ks:
        run = gn.classify_sequential(bundles[k], gn.Workload(tuple(test), lanes=1), warmup=False)
        acc[k] = round(sum(p.label is s.label for p, s in zip(run.predictions, test)) / len(test), 4)
    big = max(r.batch_size for r in report.rows)
    rows = {(r.k, r.batch_size, r.mode): r for r in report.rows}
    summary = {"workload": f"paper sweep: {a.groups} size groups x {2 * a.per_class} samples, "
                           f"V={a.vocab}, k in {list(ks)}, batches 768*m, m in {a.counts}",
               "csv": os.path.relpath(a.out, ROOT), "rows": len(report.rows),
               "lanes": config.lanes, "repetitions": a.reps,
               "speedup_at_largest_batch": {k: round(rows[(k, big, 'parallel')].speedup, 1)
                                            for k in ks},
               "Tp_gpu_samples_per_s_at_largest_batch": {
                   k: round(big / (rows[(k, big, 'parallel')].elapsed_ns_median / 1e9), 1)
                   for k in ks},
               "Tc_reference_samples_per_s_at_largest_batch": {
                   k: round(big / (rows[(k, big, 'sequential')].elapsed_ns_median / 1e9), 1)
                   for k in ks},
               "heldout_accuracy": acc, "backend_calls": dict(calls),
               "wall_s": round(time.perf_counter() - t0, 1)}
    print(json.dumps(summary), flush=True)
    backend.uninstall()


if __name__ == "__main__":
    main()
