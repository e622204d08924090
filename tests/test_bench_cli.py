"""bench.py's contract on a CPU-only machine: the reference arm (the CPU oracle) prints one JSON line with the
required keys on the headline config; the GPU arm's helpers (algorithmic bytes / flops, peaks) are consistent
with SURVEY §8(d)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["unit"] == "elements/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and "C4" in line["config"]["workload"]


def test_algorithmic_model_matches_survey():
    import bench
    # C4 1784 MB per call, C2 27.5 MB per state; nnzb closed form 23 S^2 + 48 S + 8
    assert bench.reduced_nnzb(1024) == 24072196 and bench.reduced_nnzb(128) == 371204
    assert abs(bench.algorithmic_bytes(1024 * 1024, bench.reduced_nnzb(1024)) / 1e6 - 1783.5) < 0.1
    assert abs(bench.algorithmic_bytes(128 * 128, bench.reduced_nnzb(128)) / 1e6 - 27.51) < 0.01
    # SURVEY §8(d) flop table: C4 4.37 GFLOP (symmetric model) from the point counts 2,109,394 and 1,046,525
    assert abs(bench.algorithmic_flops(2109394, 1046525) / 1e9 - 4.32) < 0.06


def test_reference_arm_under_torchrun_two_ranks():
    """--gpus 2 without a torchrun environment re-launches bench.py under torch.distributed.run (127.0.0.1); in the
    reference arm rank 0 alone runs and prints one JSON line, rank 1 exits 0 without work."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0
