"""bench.py's JSON contract on CPU: the reference arm (the oracle port timed
on the host cores) prints one line with the keys the driver reads; the
GPU arm's line is exercised by the gpu-marked test."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args, timeout=600):
    r = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, capture_output=True, text=True,
                       timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--chi", "128")
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["config"]["chi"] == 128 and "workload" in d["config"]
    assert d["scaling"] in ("weak", "strong")


@pytest.mark.gpu
def test_gpu_arm_line():
    d = _run("--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--chi", "128", "--qubits", "64")
    assert BASE_KEYS <= set(d)
    for k in ("roofline", "e2e", "gpu_launches", "clocks", "e2e_pipeline"):
        assert k in d
    assert d["gpu_launches"] > 0 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and 0 < r["frac"] < 1 and r["unit"] == "TFLOP/s"
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["clocks"]["samples"] > 0
    assert d["e2e_pipeline"]["gates"] > 0
