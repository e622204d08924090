"""Demo: a 128x128 control-point sheet hanging by its top edge under gravity, integrated with implicit Euler
(one projected-Newton solve per step on the device: bsf_eval_ip_batch + bsf_pcg).  Prints per-step Newton /
PCG iterations, energy and wall time.  usage: python scripts/hanging_sheet.py [steps] [n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import workloads as W
import paper_2506_18867_b200 as B
from paper_2506_18867_b200.newton import implicit_euler_step

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n = int(sys.argv[2]) if len(sys.argv) > 2 else 128
sh = W.make_sheet(n, 1.0, 3)          # flat rest = initial state
s = B.Sheet.from_sheet(sh)
dt = 1e-2
pinned = np.zeros((n, n), bool)
pinned[-1, :] = True                  # top edge fixed
s.set_inertia(areal_density=0.1, dt=dt, gravity=(0.0, 0.0, -9.81), pinned=pinned)
x = torch.from_numpy(sh.x).cuda()
v = torch.zeros_like(x)
t0 = time.time()
for k in range(steps):
    torch.cuda.synchronize()
    a = time.time()
    x, v, st = implicit_euler_step(s, x, v, dt, tol=1e-6)
    torch.cuda.synchronize()
    print(f"step {k}: newton {st.iterations} pcg {sum(st.pcg_iterations)} E {st.energies[-1]:+.6e} "
          f"min z {float(x[..., 2].min()):+.4f} m  {1e3 * (time.time() - a):.1f} ms", flush=True)
print(f"{steps} steps of a {n}x{n} sheet in {time.time() - t0:.2f} s")
