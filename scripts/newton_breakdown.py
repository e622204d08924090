"""Per-Newton-iteration time breakdown on the device, in the terms of the paper's ablation figure (PAPER.md:1384-1395:
runtime decomposition per Newton iteration): the incremental-potential assembly (energy + gradient + PSD-projected
Hessian, bsf_eval_ip_batch), one line-search energy evaluation (the energy-only call), and the linear solve
(block-Jacobi PCG to 1e-10, or the banded Cholesky factor + solve).  A sheet hanging by its top edge (implicit
Euler, dt = 10 ms), one Newton iteration of the first step, CUDA events, median of 5.

usage: python scripts/newton_breakdown.py [out.json]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


rows = []
for n in (128, 226):
    sh = W.make_sheet(n, 1.0 if n == 128 else 2.0, 3)
    s = B.Sheet.from_sheet(sh)
    dt = 1e-2
    pinned = np.zeros((n, n), bool)
    pinned[-1, :] = True
    s.set_inertia(areal_density=0.1, dt=dt, gravity=(0.0, 0.0, -9.81), pinned=pinned)
    x = torch.from_numpy(sh.x).cuda().unsqueeze(0).contiguous()
    xhat = x.clone()
    E = torch.zeros(1, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(x)
    V = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    for _ in range(3):
        s.eval_ip_batch(x, xhat, E, G, V, flags=B.PROJECT_PSD)
    t_asm, _ = timed(lambda: s.eval_ip_batch(x, xhat, E, G, V, flags=B.PROJECT_PSD))
    t_e, _ = timed(lambda: s.eval_ip_batch(x, xhat, E, None, None, flags=B.PROJECT_PSD))
    t_pcg, res = timed(lambda: s.pcg(V[0], -G[0], max_iter=5000, rtol=1e-10))
    t_fac, _ = timed(lambda: s.chol_factor(V[0]), reps=3)
    t_sol, _ = timed(lambda: s.chol_solve(-G[0]))
    row = {"sheet": f"{n}x{n}", "dofs": 3 * n * n, "assembly_ms": t_asm, "energy_only_ms": t_e,
           "pcg_ms": t_pcg, "pcg_iterations": int(res[1]), "chol_factor_ms": t_fac, "chol_solve_ms": t_sol,
           "assembly_share_pcg_iteration": t_asm / (t_asm + t_pcg + 3 * t_e),
           "assembly_share_chol_iteration": t_asm / (t_asm + t_fac + t_sol + 3 * t_e),
           "note": "one Newton iteration = assembly + solve + the line search's energy evaluations (3 assumed)"}
    rows.append(row)
    print(json.dumps(row), flush=True)
    s.close()
if len(sys.argv) > 1:
    json.dump({"config": "hanging sheet, implicit Euler dt = 10 ms, first Newton iteration, one B200", "rows": rows},
              open(sys.argv[1], "w"), indent=1)
