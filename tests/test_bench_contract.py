"""bench.py's JSON-line contract (the driver parses it): the reference arm (the oracle on the
host, CPU) and the GPU arm on the smallest workload.  Keys and types only -- the numbers are the
bench's business."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "3"], 300)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["unit"] == "iters/s" and d["higher_is_better"] is True
    assert d["config"]["workload"] == "tiny"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run(["--config", "tiny", "--steps", "3", "--warmup", "3", "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["value"] > 0 and d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["config"]["workload"] == "tiny"
    assert d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    for k in ("roofline", "roofline_step", "clocks"):
        assert k in d
    r = d["roofline"]
    assert r["bound"] in ("hbm", "alu", "tensor") and r["peak"] > 0 and 0 < r["frac"] and r["achieved"] > 0
