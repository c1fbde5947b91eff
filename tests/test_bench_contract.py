"""bench.py JSON contract: the CPU reference arm here, the GPU arm on a B200."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1", "--ref-rows", "20000",
              "--ref-py-samples", "2000"], 300)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    ref = d["reference_python"]   # the unmodified reference pkg, when installed
    assert "unavailable" in ref or (ref["Tc_samples_per_s"] > 0 and ref["labels_equal_Tc_Tp"])


@pytest.mark.gpu
@pytest.mark.timeout(600)
def test_gpu_arm_contract():
    d = _run(["--rows", "2000000", "--steps", "5", "--warmup", "3", "--e2e-rows", "1000000",
              "--e2e-steps", "1", "--cpu-seconds", "1", "--object-rows", "20000"], 550)
    assert BASE_KEYS <= set(d)
    assert {"roofline", "cpu_baseline", "gpu_launches", "clocks"} <= set(d)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert d["gpu_launches"] == 5 and d["e2e"]["matches_device_labels"] is True
    assert d["accuracy_vs_generator_labels"] > 0.9
    o = d["object_api"]
    assert o["samples"] == 20000 and o["accuracy"] > 0.9
    assert o["classify_parallel_elapsed_samples_per_s"] > 0
