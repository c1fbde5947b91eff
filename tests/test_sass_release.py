"""Static SASS check (CPU, cuobjdump): every stage release (SYNCS.ARRIVE) in the
built K-PRED / K-FIT kernels waits on the shared-memory loads issued from that
stage first -- the TMA-refill WAR race of round 2 cannot come back unnoticed
(tools/sass_release_check.py; it flags the racy build, profiles/r02_tuning.md)."""

import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1905_13746_b200", "libgnb.so")


@pytest.mark.skipif(shutil.which("cuobjdump") is None or not os.path.exists(LIB),
                    reason="needs cuobjdump and a built libgnb.so")
def test_no_stage_release_overtakes_its_loads():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sass_release_check.py"), LIB],
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert '"kernels_flagged": 0' in r.stdout
