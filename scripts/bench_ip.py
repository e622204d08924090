"""Incremental-potential call (bsf_eval_ip_batch) vs the elastic call on C2 (100 states): device time per
call (CUDA events, warm, outputs > L2), the epilogue's share, and its bandwidth against the measured copy
peak.  Prints one JSON line.  usage: python scripts/bench_ip.py [states]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W, paper_2506_18867_b200 as B

nst = int(sys.argv[1]) if len(sys.argv) > 1 else 100
sheets = [W.make_c2(state=k) for k in range(nst)]
h = B.Sheet.from_sheet(sheets[0])
pinned = np.zeros((h.n_v, h.n_u), bool)
pinned[-1, :] = True
h.set_inertia(0.15, 1e-3, gravity=(0.0, 0.0, -9.81), pinned=pinned)
X = torch.stack([torch.from_numpy(s.x) for s in sheets]).cuda()
XH = X + 1e-3 * torch.randn_like(X)
E = torch.zeros(nst, dtype=torch.float64, device="cuda")
G = torch.zeros_like(X)
V = torch.zeros((nst, h.nnzb, 3, 3), dtype=torch.float64, device="cuda")


def timed(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


t_el = timed(lambda: h.eval_all_batch(X, E, G, V, B.PROJECT_PSD))
t_ip = timed(lambda: h.eval_ip_batch(X, XH, E, G, V, B.PROJECT_PSD))
n_cp = h.n_u * h.n_v
el = (h.n_u - 2) * (h.n_v - 2) * nst
# epilogue bytes actually moved per control point: x 24 + xhat 24 + m 8 + diag index 4 + gradient 48 (RMW)
# + 3 diagonal doubles 48 (RMW); pinned elimination is a few rows
epi_bytes = nst * n_cp * (24 + 24 + 8 + 4 + 48 + 48)
print(json.dumps({"states": nst, "elastic_ms": t_el, "ip_ms": t_ip, "epilogue_ms": t_ip - t_el,
                  "ip_elements_per_s": el / (t_ip * 1e-3), "elastic_elements_per_s": el / (t_el * 1e-3),
                  "epilogue_GBps": epi_bytes / ((t_ip - t_el) * 1e-3) / 1e9 if t_ip > t_el else None,
                  "launches_ip": h.last_launch_count()}))
