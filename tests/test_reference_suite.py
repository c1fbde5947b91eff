"""The reference's OWN test suite, run with the GPU backend installed.

`backend.install()` rebinds groupnb's train_bundle / train_group /
train_bundles / classify_parallel to the sm_100a path (classify_sequential, the
Tc baseline, stays the reference's Python).  The unmodified reference tests
(pkg/tests, 205 tests: engine, classifier, acceptance C1-C9, bench sweep, CLI,
...) must then pass as they do on the reference itself -- in particular C4
(GPU Tp bit-identical to the reference's Tc on 50 random workloads), C7
(exclusion + fallback routing), bundle JSON round trips of GPU-trained bundles
and the CLI's byte-identical parallel/sequential prediction files.

The suite lives next to the pip-installed reference in baseline/_ref
(git-ignored, copied by tools/install_reference.sh; never committed)."""

import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(REF, "tests")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.isdir(TESTS),
                                 reason="baseline/_ref/tests missing (tools/install_reference.sh)")]


@pytest.mark.timeout(1500)
def test_reference_suite_on_gpu_backend():
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF, ROOT]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "paper_1905_13746_b200.pytest_backend",
           "-p", "no:cacheprovider", "--rootdir", REF, TESTS]
    r = subprocess.run(cmd, cwd=REF, env=env, capture_output=True, text=True, timeout=1400)
    tail = r.stdout[-6000:] + r.stderr[-3000:]
    assert r.returncode == 0, tail
    m = re.search(r"\[gnb-backend\] (.*)", r.stdout)
    assert m, tail
    calls = dict(kv.split("=") for kv in m.group(1).split())
    # the GPU operations really ran (and often): fit and Tp
    assert int(calls.get("classify_parallel", 0)) >= 50, calls
    assert int(calls.get("train_bundle", 0)) >= 50, calls
    assert int(calls.get("train_group", 0)) >= 10, calls
    assert int(calls.get("train_bundles", 0)) >= 1, calls
    passed = re.search(r"(\d+) passed", r.stdout)
    assert passed and int(passed.group(1)) >= 200, tail
