"""Per-iteration cycle breakdown of k_core (library built with -DBSF_PHASE_TIMERS, BSF_LIB_PATH set)."""
import sys, os, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, workloads as W, paper_2506_18867_b200 as B
sh = W.make_c4() if "--c4" in sys.argv else W.make_c3() if "--c3" in sys.argv else W.make_c2(0)
nst = 1 if ("--c4" in sys.argv or "--c3" in sys.argv or "--single" in sys.argv) else 100
h = B.Sheet.from_sheet(sh)
X = torch.from_numpy(sh.x).cuda().unsqueeze(0).repeat(nst, 1, 1, 1).contiguous()
E = torch.zeros(nst, dtype=torch.float64, device="cuda")
G = torch.zeros((nst,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
V = torch.zeros((nst, h.nnzb, 3, 3), dtype=torch.float64, device="cuda")
h.eval_all_batch(X, E, G, V, 1); torch.cuda.synchronize()
L = B.lib()
buf = (C.c_ulonglong * 48)()
L.bsf_debug_core_timers(buf, 1)
h.eval_all_batch(X, E, G, V, 1); torch.cuda.synchronize()
L.bsf_debug_core_timers(buf, 1)
v = np.array(list(buf), dtype=np.float64)
n = v[6]
print("iterations:", int(n))
print("point eval %.0f | point-warp gather %.0f | warp0 gather %.0f | warp2 gather %.0f | wait_all %.0f | barrier %.0f | iteration %.0f"
      % (v[0] / n, v[7] / n, v[1] / n, v[2] / n, v[3] / n, v[4] / n, v[5] / n))
c = v[10]
print("CTAs %d: setup %.0f | loop %.0f (prologue %.0f) | whole %.0f cycles per CTA" % (c, v[8] / c, v[9] / c, v[12] / c, v[11] / c))
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record()
for _ in range(5): h.eval_all_batch(X, E, G, V, 1)
t1.record(); torch.cuda.synchronize()
print("call ms", t0.elapsed_time(t1) / 5)
print("section (d): tid0 %.0f  tid32 %.0f" % (v[13] / n, v[14] / n))
print("per-warp busy (T0->before barrier):", " ".join("w%d=%.0f" % (w, v[16 + w] / n) for w in range(16)))
