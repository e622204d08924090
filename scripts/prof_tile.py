"""Small driver for ncu: C2 states through bsf_eval_all_batch (tile or generic path)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads as W, paper_2506_18867_b200 as B
nst = int(sys.argv[1]) if len(sys.argv) > 1 else 20
flags = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sheets = [W.make_c2(state=k) for k in range(nst)]
h = B.Sheet.from_sheet(sheets[0])
X = torch.stack([torch.from_numpy(s.x) for s in sheets]).cuda()
E = torch.zeros(nst, dtype=torch.float64, device="cuda")
G = torch.zeros((nst,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
V = torch.zeros((nst, h.nnzb, 3, 3), dtype=torch.float64, device="cuda")
for _ in range(3):
    h.eval_all_batch(X, E, G, V, flags)
torch.cuda.synchronize()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(5):
    h.eval_all_batch(X, E, G, V, flags)
t1.record(); torch.cuda.synchronize()
ms = t0.elapsed_time(t1) / 5
print(f"{nst} states: {ms:.3f} ms/call, {ms*1e3/nst:.2f} us/state, launches={h.last_launch_count()}")
if os.environ.get("PROF_KT"):   # per-kernel live times (bsf_set_kernel_timing): k_core and k_band of the call
    h.set_kernel_timing(5)
    for _ in range(5):
        h.eval_all_batch(X, E, G, V, flags)
    torch.cuda.synchronize()
    c, b = h.kernel_timing(5)
    import statistics
    print(f"k_core {statistics.median(c):.3f} ms, k_band {statistics.median(b):.3f} ms (live, beside each other)")
