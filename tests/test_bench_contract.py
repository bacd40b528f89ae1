"""bench.py's one-line JSON contract (the task statement's bench rules; DESIGN.md
§7): the keys and their types for the reference arm (the CPU oracle, runs
here) and for the library arm (`-m gpu`), on the small C1 config."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def check_common(d, steps, warmup):
    assert d["metric"] == "rank-k PCA wall time (s)" and d["unit"] == "s"
    assert d["higher_is_better"] is False
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] == warmup
    assert d["value"] > 0 and abs(d["ms_per_step"] - 1e3 * d["value"]) <= 1e-6 * d["ms_per_step"] + 1e-9
    assert d["scaling"] in ("strong", "weak")
    assert d["vs_baseline"] is None  # BASELINE.md has no number for this metric on this workload
    assert d["data"] == "synthetic" and d["dtype"] == "f64"
    assert d["config"]["workload"].startswith("C1")
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "C1", "--steps", "2", "--warmup", "3")
    check_common(d, 2, 3)
    assert d["impl"] == "reference"
    assert d["e2e"] == {"value": d["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["value"] == d["value"]


@pytest.mark.gpu
def test_library_arm_line():
    d = run_bench("--config", "C1", "--steps", "3", "--warmup", "3")
    check_common(d, 3, 3)
    assert "impl" not in d or d["impl"] != "reference"
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and r["unit"] in ("GB/s", "TFLOP/s")
    assert r["achieved"] > 0 and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == "s" and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert c["sm_mhz"] > 0 and c["sm_max_mhz"] > 0 and isinstance(c["reasons"], list)
