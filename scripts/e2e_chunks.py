"""e2e (host-buffer call) time per 100 C2 states vs the upload chunk size."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, workloads as W, paper_2506_18867_b200 as B
sheets = [W.make_c2(state=k) for k in range(100)]
h = B.Sheet.from_sheet(sheets[0])
Xh = torch.stack([torch.from_numpy(s.x) for s in sheets]).pin_memory()
X = Xh.cuda()
E = torch.zeros(100, dtype=torch.float64, device="cuda"); Eh = torch.zeros(100, dtype=torch.float64).pin_memory()
G = torch.zeros((100,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
V = torch.zeros((100, h.nnzb, 3, 3), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for ch in (0, 10, 20, 25, 34, 50, 100):
    for _ in range(2): h.eval_all_batch_host(Xh, X, E, Eh, G, V, flags=1, chunk=ch, stream=st)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(5): h.eval_all_batch_host(Xh, X, E, Eh, G, V, flags=1, chunk=ch, stream=st)
    b.record(st); torch.cuda.synchronize()
    print(f"chunk {ch}: {a.elapsed_time(b)/5:.3f} ms")
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(5): X.copy_(Xh, non_blocking=True)
b.record(st); torch.cuda.synchronize()
print(f"H2D alone: {a.elapsed_time(b)/5:.3f} ms")
