"""SASS evidence per hot kernel of libgnb.so (cuobjdump -sass): counts of the
mnemonics that prove TMA (UTMALDG, UTMALDG...GATHER4, UBLKCP), mbarriers
(SYNCS.*), the exact FP64 arithmetic (DMUL / DADD, no DFMA in exact mode),
conversions and shared-memory traffic, plus registers / spills
(cuobjdump -res-usage).  Writes profiles/<name>.json.

    python tools/sass_summary.py [out.json]
"""
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1905_13746_b200", "libgnb.so")
KEYS = ("UTMALDG", "UTMALDG.2D.GATHER4", "UBLKCP", "SYNCS", "DMUL", "DADD", "DFMA", "I2F.F64",
        "LDS", "LDS.128", "STG", "RED", "ATOMS", "MATCH", "SHFL", "REDUX", "UTMAPF")


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                             text=True).stdout.splitlines()
        return dict(zip(names, out))
    except Exception:
        return {n: n for n in names}


def main():
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles",
                                                                   "r02_sass_summary.json")
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", LIB], capture_output=True, text=True).stdout
    regs = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)",
                         res):
        regs[m.group(1)] = {"registers": int(m.group(2)), "stack": int(m.group(3)),
                            "local_spill_bytes": int(m.group(5))}
    funcs = re.split(r"\n\s+Function : ", sass)[1:]
    names = [f.split("\n", 1)[0].strip() for f in funcs]
    dm = demangle(names)
    out = {}
    for name, body in zip(names, funcs):
        ops = re.findall(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", body)
        c = collections.Counter(ops)
        counts = {}
        for k in KEYS:
            n = sum(v for op, v in c.items() if op == k or op.startswith(k + "."))
            if k == "LDS.128":
                n = c.get("LDS.128", 0)
            if n:
                counts[k] = n
        out[dm.get(name, name)] = {"instructions": len(ops), **counts, **regs.get(name, {})}
    hot = {k: v for k, v in out.items()
           if any(s in k for s in ("predict_tma_kernel<2, int, 1, 4, 2, false, 1, false>",
                                   "predict_tma_kernel<2, int, 1, 4, 2, true, 1, false>",
                                   "predict_rowbox_kernel<2, int, 2, false, 13, 4, true>",
                                   "predict_rowbox_kernel<2, int, 2, false, 26, 2, false>",
                                   "predict_mixed_kernel<int, 8, 2, false>",
                                   "tile_mix_kernel",
                                   "fit_tma_kernel", "gather_kernel<int>", "unpack_u4",
                                   "slot_sort", "fin_select"))}
    doc = {"library": "paper_1905_13746_b200/libgnb.so (sm_100a)",
           "how": "python tools/sass_summary.py (cuobjdump -sass / -res-usage)",
           "hot_kernels": hot, "all_kernels": len(out)}
    with open(out_path, "w") as fh:
        json.dump(doc, fh, indent=1)
    for k, v in hot.items():
        print(k[:110], {kk: vv for kk, vv in v.items() if kk in ("instructions", "UTMALDG", "UBLKCP", "SYNCS", "DMUL", "DADD", "DFMA", "local_spill_bytes")})


if __name__ == "__main__":
    main()
