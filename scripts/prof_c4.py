"""Timing of the tile kernels on C4 (1024^2, interior dominated) and C2 (128^2)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads as W, paper_2506_18867_b200 as B
def run(sh, nst, label):
    h = B.Sheet.from_sheet(sh)
    X = torch.from_numpy(sh.x).cuda().unsqueeze(0).repeat(nst, 1, 1, 1).contiguous()
    E = torch.zeros(nst, dtype=torch.float64, device="cuda")
    G = torch.zeros((nst,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
    V = torch.zeros((nst, h.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    for _ in range(2): h.eval_all_batch(X, E, G, V, 1)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(3): h.eval_all_batch(X, E, G, V, 1)
    t1.record(); torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 3
    ncp = sh.n_u * sh.n_v * nst
    alg = (72 * h.nnzb + 48 * sh.n_u * sh.n_v) * nst
    print(f"{label}: {ms*1e3/nst:.1f} us/sheet, {ncp/ms/1e6:.3f} Gcp/s, {alg/ms/1e6:.0f} GB/s")
run(W.make_c4(), 4, "C4 x4")
run(W.make_c2(0), 100, "C2 x100")
