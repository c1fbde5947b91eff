import json, sys
tag = sys.argv[1]
for l in open(f"gpurun_out/{tag}_sweep.json"):
    if l.startswith("{"):
        for r in json.loads(l)["rows"]:
            print(r["F"], r["ms"], r["frac"], r["copy_same_bytes"]["frac"], r["frac_of_copy"], r["bit_exact_subsample_vs_oracle"])
for l in open(f"gpurun_out/{tag}_ragged.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print("ragged grouped", d["frac"], "shuffled", d["shuffled_rows"]["frac"], d["shuffled_rows"]["order_hint_mixed"]["frac"])
for l in open(f"gpurun_out/{tag}_cfg4.json"):
    if l.startswith("{"):
        d = json.loads(l)
        print("cfg4", d["value"], d["roofline"]["frac"])
