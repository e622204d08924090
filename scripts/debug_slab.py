import sys, os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import oracle as O, workloads as W, paper_2506_18867_b200 as B
sh = W.make_c2(state=1)
for (r0, r1) in [(41, 90), (41, 73), (73, 90), (40, 90), (41, 91)]:
    o = O.Oracle.from_sheet(sh, r0=r0, r1=r1)
    Er, gr, vr = o.eval(sh.x, flags=1)
    s = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1)
    xd = torch.from_numpy(np.ascontiguousarray(sh.x[s.x_row_begin:s.x_row_end])).cuda()
    E, g, v = s(xd, 1); torch.cuda.synchronize(); g = g.cpu().numpy(); v = v.cpu().numpy()
    dg = np.linalg.norm(g - gr, axis=2); nb = np.linalg.norm(gr, axis=2)
    bad = np.argwhere(dg > 1e-9 * nb.max())
    dv = np.linalg.norm((v - vr).reshape(-1, 9), axis=1)
    print((r0, r1), "E rel %.1e" % (abs(E.item() - Er) / Er), "bad g cps:", len(bad), bad[:6].tolist(), "max dH/max %.1e" % (dv.max() / np.abs(vr).max()))
