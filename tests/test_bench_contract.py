"""bench.py output contract (the JSON line the round driver parses), on the
small BASELINE configs[0] workload so it runs in seconds.

* reference arm (CPU, runs anywhere the compiled reference exists): one line
  with impl = "reference", a cpu_baseline and an e2e object;
* our arm (GPU): every key of the contract, a roofline with a positive
  fraction, the CUDA-graph note, clocks and a launch count.
"""
import json
import os
import subprocess
import sys

import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
             "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, cwd=ROOT,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    if not oracle.available("reference"):
        pytest.skip("oracle/_ref not built")
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_our_arm_contract(cuda):
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3"])
    assert BASE_KEYS <= set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["scaling"] == "weak" and d["vs_baseline"] is None
    assert "workload" in d["config"] and d["config"]["cuda_graph"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    # per step: stage 1, stage 2 + Adam (fused at one rank), Y build, apply
    assert d["gpu_launches"] >= 4 * 3
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
