"""k_core phase matrix on C4 (one 1024^2 sheet): the kernel's live duration (CUDA events around its launch,
bsf_set_kernel_timing) with its profiling switches BSF_CORE_DEBUG = 1 (no point phase after the prologue),
2 (no gather), 4 (no staging stores / bulk stores), 8 (no bulk copies) and combinations.  Each setting runs in
its own process (the switch is read once per process)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, statistics
sys.path.insert(0, %r)
import torch, workloads as W, paper_2506_18867_b200 as B
sh = W.make_c4()
h = B.Sheet.from_sheet(sh)
x = torch.from_numpy(sh.x).cuda()
E, g, v = h.alloc_outputs()
for _ in range(3): h.eval_all(x, E, g, v, B.PROJECT_PSD)
torch.cuda.synchronize()
h.set_kernel_timing(10)
for _ in range(10): h.eval_all(x, E, g, v, B.PROJECT_PSD)
torch.cuda.synchronize()
c, b = h.kernel_timing(10)
print(statistics.median(c) * 1e3)
"""

if __name__ == "__main__":
    out = {}
    for dbg in sys.argv[1:] or ["0", "1", "2", "4", "8", "3", "6", "5"]:
        env = dict(os.environ, BSF_CORE_DEBUG=dbg, BSF_REBUILD="0")
        r = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True)
        out[dbg] = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-300:]
        print(json.dumps({"BSF_CORE_DEBUG": dbg, "k_core_us": out[dbg]}), flush=True)
