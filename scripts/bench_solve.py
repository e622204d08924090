"""BSR SpMV bandwidth and block-Jacobi PCG on the C2 / C4 incremental-potential Hessian (one state).
Prints one JSON line per config.  usage: python scripts/bench_solve.py"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W, paper_2506_18867_b200 as B

for name, sh in (("C2", W.make_c2(state=0)), ("C4", W.make_c4())):
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
    y = s.spmv(v, x[0])
    for _ in range(3):
        s.spmv(v, x[0], y)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(20):
        s.spmv(v, x[0], y)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 20
    bytes_ = s.nnzb * (72 + 4) + (s.n_u * s.n_v) * (24 + 24 + 4)   # blocks + col idx, x + y + row ptr
    lo, hi = s.gershgorin(v)
    sol = torch.zeros_like(b)
    s.pcg(v, b, sol, max_iter=5, rtol=1e-10)   # warm
    sol.zero_()
    torch.cuda.synchronize()
    t0.record()
    sol, it, rr = s.pcg(v, b, sol, max_iter=5000, rtol=1e-10)
    t1.record()
    torch.cuda.synchronize()
    print(json.dumps({"config": name, "nnzb": s.nnzb, "spmv_ms": ms, "spmv_GBps": bytes_ / (ms * 1e-3) / 1e9,
                      "gershgorin": [lo, hi], "pcg_iters": it, "pcg_relres": rr, "pcg_ms": t0.elapsed_time(t1),
                      "pcg_ms_per_iter": t0.elapsed_time(t1) / max(it, 1)}))
