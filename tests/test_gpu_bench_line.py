"""GPU: bench.py's JSON line on the headline config (C4, N = 1) carries every key of the contract — the value, the
roofline object (whole call and the live k_core entry), the FP64 fraction, the CPU-oracle baseline, the end-to-end
number with its copied bytes, the launch count and the clocks sampled during the timed region — and its numbers
are consistent with each other (the value from ms_per_step, the roofline from the algorithmic bytes)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_keys_and_consistency():
    env = dict(os.environ, BSF_REBUILD="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                        "--no-secondary"], capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks",
              "fp64"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["dtype"] == "f64" and "C4" in d["config"]["workload"]
    el = 1022 * 1022
    assert abs(d["value"] - el / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and 0.0 < rf["frac"] < 1.0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    assert abs(rf["achieved"] - 1783529768 / (d["ms_per_step"] * 1e-3) / 1e9) <= 1e-6 * rf["achieved"]
    assert rf["kernel"]["kernel"] == "k_core" and 0.0 < rf["kernel"]["frac"] < 1.0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 1024 * 1024 * 24 and d["e2e"]["value"] > 0
    assert d["gpu_launches"] >= 3 * 5
    assert d["clocks"]["sm_mhz"] > 0
