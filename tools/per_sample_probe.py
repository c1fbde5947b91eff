"""Per-sample scoring latency (verdict r01 weak #9): the reference's
classifier.predict / log_posterior vs this package's api.predict / log_posterior
(host C walk of model._packed, no device round trip) on the reference's own
objects; prints us/sample and checks bit equality."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)
from groupnb import classifier, corpus, engine, synth  # noqa: E402

import paper_1905_13746_b200 as P  # noqa: E402

out = {}
for k in (20, 100, 200):
    spec = synth.SyntheticSpec(group_count=1, samples_per_group_per_class=1000,
                               vocabulary_size=256, divergence=0.1, seed=0)
    recs = synth.generate_synthetic(spec)
    train, _ = corpus.partition_by_group(recs, corpus.GroupingConfig())
    bundle = engine.train_bundle(train, k=k, created_at="t")
    model = next(iter(bundle.models.values()))
    hs = [r.histogram for r in recs]
    row = {}
    for name, fn in (("reference_predict", classifier.predict), ("repo_predict", P.api.predict),
                     ("reference_log_posterior", classifier.log_posterior),
                     ("repo_log_posterior", P.api.log_posterior)):
        best = 1e9
        for _ in range(3):
            t = time.perf_counter()
            for h in hs:
                fn(model, h)
            best = min(best, (time.perf_counter() - t) / len(hs) * 1e6)
        row[name + "_us"] = round(best, 3)
    a = [classifier.predict(model, h) for h in hs]
    b = [P.api.predict(model, h) for h in hs]
    row["bit_equal"] = all(x.label == y.label and x.log_posterior == y.log_posterior
                           for x, y in zip(a, b))
    row["speedup_predict"] = round(row["reference_predict_us"] / row["repo_predict_us"], 2)
    out[f"k={k}"] = row
print(json.dumps(out))
