"""the reference's own bench sweep (run_bench / emit_csv,
bench.py:114-183) in GPU mode -- tools/paper_sweep.py at a small size: the
reference CSV round-trips, every (k, batch) cell has a sequential (reference
Tc) and a parallel (GPU Tp) row, and the GPU path really ran."""

import json
import os
import subprocess
import sys

import pytest

from refpkg import groupnb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(groupnb() is None, reason="baseline/_ref not installed")]


@pytest.mark.timeout(600)
def test_paper_sweep_gpu_mode(tmp_path):
    out = tmp_path / "sweep.csv"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "paper_sweep.py"),
                        "--out", str(out), "--reps", "1", "--groups", "3", "--per-class", "40",
                        "--counts", "1,2"], capture_output=True, text=True, timeout=500)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["rows"] == 6 * 2 * 2
    assert d["backend_calls"]["classify_parallel"] == 6 * 2
    assert d["backend_calls"]["train_bundles"] == 1
    lines = out.read_text().splitlines()
    assert lines[0] == "k,batch_size,mode,lanes,elapsed_ns_median,elapsed_ns_min,speedup"
    assert len(lines) == 1 + 24
    assert all(v > 0.9 for v in d["heldout_accuracy"].values())
