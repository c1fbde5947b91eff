#!/usr/bin/env python
"""Static SASS check of stage releases: SYNCS.ARRIVE carries no implicit wait on
earlier shared-memory loads, so a consumer that releases a stage (the TMA may
then overwrite it) must have WAITED on every LDS it issued from that stage.

For every `SYNCS.ARRIVE...A1T0` (a plain arrive: consumer releases and the
producer's own arrives) this walks the instruction stream backwards to the
stage acquire that precedes it (`SYNCS.PHASECHK`) and checks that every LDS in
between has its write scoreboard waited on (wait mask in the control bits) by
some instruction at or before the arrive.  A hit means the release can overtake
the load -- the TMA-refill WAR race found in round 2 (profiles/r02_tuning.md).

    python tools/sass_release_check.py paper_1905_13746_b200/libgnb.so [--kernel REGEX]
"""

import argparse
import json
import re
import subprocess
import sys
from collections import defaultdict

INSN = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]{16}) \*/")
CTRL = re.compile(r"^\s*/\* (0x[0-9a-f]{16}) \*/\s*$")


def parse(sass_text):
    """{function: [(addr, text, ctrl_word), ...]}"""
    funcs = defaultdict(list)
    cur = None
    pending = None
    for line in sass_text.splitlines():
        if "Function :" in line:
            cur = line.split("Function :")[1].strip()
            continue
        m = INSN.search(line)
        if m and cur:
            pending = (int(m.group(1), 16), m.group(2).strip(), int(m.group(3), 16))
            continue
        c = CTRL.match(line)
        if c and pending is not None:
            addr, text, _lo = pending
            funcs[cur].append((addr, text, int(c.group(1), 16)))
            pending = None
    return funcs


def ctrl_fields(hi):
    c = hi >> 41
    return {"wbar": (c >> 5) & 7, "wait": (c >> 11) & 63}


def check(insns, window=4000):
    """List of (arrive_addr, lds_addr) pairs where the LDS is not waited on."""
    bad = []
    n_rel = 0
    for i, (addr, text, hi) in enumerate(insns):
        if "SYNCS.ARRIVE" not in text or "A1T0" not in text:
            continue
        n_rel += 1
        loads = []  # (index, sb)
        j = i - 1
        while j >= 0 and i - j < window:
            t = insns[j][1]
            if "SYNCS.PHASECHK" in t:
                break
            if re.search(r"\bLDS(\.|\s)", t) and not t.startswith("@!PT"):
                sb = ctrl_fields(insns[j][2])["wbar"]
                if sb != 7:
                    loads.append((j, sb))
            j -= 1
        for (k, sb) in loads:
            waited = any(ctrl_fields(insns[m][2])["wait"] >> sb & 1 for m in range(k + 1, i + 1))
            if not waited:
                bad.append((hex(addr), hex(insns[k][0]), insns[k][1]))
    return n_rel, bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("binary")
    ap.add_argument("--kernel", default="predict_|fit_")
    ap.add_argument("--out")
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.binary], capture_output=True, text=True,
                          check=True).stdout
    report = {}
    for fn, insns in parse(sass).items():
        if not re.search(a.kernel, fn):
            continue
        n_rel, bad = check(insns)
        if n_rel:
            report[fn] = {"releases": n_rel, "unwaited_lds_before_release": bad}
    flagged = {k: v for k, v in report.items() if v["unwaited_lds_before_release"]}
    summary = {"kernels_checked": len(report), "kernels_flagged": len(flagged),
               "flagged": flagged}
    text = json.dumps(summary, indent=1)
    if a.out:
        open(a.out, "w").write(text + "\n")
    print(text[:4000])
    return 1 if flagged else 0


if __name__ == "__main__":
    sys.exit(main())
