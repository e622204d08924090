"""Per-phase cycle breakdown of k_tile (library built with -DBSF_PHASE_TIMERS, BSF_LIB_PATH set)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, workloads as W, paper_2506_18867_b200 as B
sh = W.make_c4() if "--c4" in sys.argv else W.make_c2(0)
nst = 2 if "--c4" in sys.argv else 50
h = B.Sheet.from_sheet(sh)
X = torch.from_numpy(sh.x).cuda().unsqueeze(0).repeat(nst, 1, 1, 1).contiguous()
E = torch.zeros(nst, dtype=torch.float64, device="cuda")
G = torch.zeros((nst,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
V = torch.zeros((nst, h.nnzb, 3, 3), dtype=torch.float64, device="cuda")
h.eval_all_batch(X, E, G, V, 1); torch.cuda.synchronize()
L = B.lib()
buf = (C.c_ulonglong * 16)()
L.bsf_debug_phase_timers(buf, 1)
h.eval_all_batch(X, E, G, V, 1); torch.cuda.synchronize()
L.bsf_debug_phase_timers(buf, 1)
v = np.array(list(buf), dtype=np.float64)
steps = v[10]
print("gather steps (all CTAs):", int(steps))
print("per step cycles: pos+bookkeeping %.0f | point phase %.0f | gather phase (to barrier) %.0f" % (v[0] / steps, v[1] / steps, v[9] / steps))
print("per-warp gather busy cycles:", " ".join("w%d=%.0f" % (k, v[2 + k] / steps) for k in range(7)))
