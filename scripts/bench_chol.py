"""Direct solve of the Newton system (bsf_chol_factor / bsf_chol_solve) on the C2 (128^2) and C3
(226^2, the paper's largest scene size) incremental-potential Hessians, beside block-Jacobi PCG to 1e-10 on the same
system.  Device time with CUDA events (the factorisation synchronises once at its end to read the pivots).
Prints one JSON line per config."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

for name, sh in (("C2", W.make_c2(state=0)), ("C3", W.make_c3())):
    s = B.Sheet.from_sheet(sh)
    s.set_inertia(0.15, 2e-3, gravity=(0.0, 0.0, -9.81))
    x = torch.from_numpy(sh.x).cuda().unsqueeze(0)
    xh = x + 1e-3 * torch.randn_like(x)
    E = torch.zeros(1, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(x)
    V = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_ip_batch(x, xh, E, G, V, flags=B.PROJECT_PSD)
    torch.cuda.synchronize()
    v, b = V[0], -G[0]
    s.chol_factor(v)   # first call: band allocation, cuBLAS / cuSOLVER handles
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    s.chol_factor(v)
    ev[1].record()
    xs = s.chol_solve(b)
    ev[2].record()
    torch.cuda.synchronize()
    res = float((b - s.spmv(v, xs)).norm() / b.norm())
    sol = torch.zeros_like(b)
    s.pcg(v, b, sol, max_iter=5, rtol=1e-10)
    sol.zero_()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    sol, it, rr = s.pcg(v, b, sol, max_iter=20000, rtol=1e-10)
    t1.record()
    torch.cuda.synchronize()
    n = 3 * sh.n_u * sh.n_v
    kd = 6 * sh.n_u + 5
    print(json.dumps({"config": name, "dofs": n, "half_bandwidth": kd, "factor_ms": ev[0].elapsed_time(ev[1]),
                      "solve_ms": ev[1].elapsed_time(ev[2]), "chol_relres": res,
                      "factor_gflop_model": n * kd * kd / 1e9,
                      "pcg_iters": it, "pcg_relres": rr, "pcg_ms": t0.elapsed_time(t1)}), flush=True)
