"""bench.py's JSON-line contract (the driver parses it): the --impl reference arm (the
oracle, CPU) runs here; the torus arm runs on a GPU (-m gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"]


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run(["--impl", "reference", "--steps", "2", "--warmup", "1"])
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["value"] > 0 and d["gpu_launches"] == 0


@pytest.mark.gpu
def test_torus_arm_json_line():
    d = _run(["--steps", "20", "--warmup", "3", "--no-cpu"])
    for k in REQUIRED + ["roofline", "e2e", "gpu_launches", "clocks", "cpu_baseline"]:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 20
    r = d["roofline"]
    assert r["bound"] == "hbm" and 0 < r["frac"] < 1.5 and r["peak"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["sanity"]["equals_cast_roundtrip"]
