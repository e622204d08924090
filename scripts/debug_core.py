"""GPU debug: core+frame path vs tile-only vs the oracle on one C2 state; prints worst offenders."""
import sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import oracle as O, workloads as W
import paper_2506_18867_b200 as B
from parity import diag_block_norms, rel_grad, rel_hess, rel_energy

n = int(sys.argv[1]) if len(sys.argv) > 1 else 0
sh = W.make_c2(state=3) if n == 0 else W.make_sheet(n, 1.0, 5, n_modes=4, amp=5e-3, lam=0.2)
flags = B.PROJECT_PSD
t0 = time.time()
s = B.Sheet.from_sheet(sh)
print("create", time.time() - t0, "core rect", s.core_rect())
xd = torch.from_numpy(sh.x).cuda()
res = {}
for name, f in [("core", flags), ("tile", flags | B.TILE_ONLY)]:
    E, g, v = s(xd, f)
    torch.cuda.synchronize()
    res[name] = (float(E.item()), g.cpu().numpy(), v.cpu().numpy())
o = O.Oracle.from_sheet(sh)
Er, gr, vr = o.eval(sh.x, flags=1)
rp, ci = o.pattern()
va = o.eval(sh.x, flags=1 | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
hd = diag_block_norms(vr, rp, ci, 0, sh.n_u)
cm = np.abs(sh.x).max()
for name, (E, g, v) in res.items():
    print(name, "E", rel_energy(E, Er), "g", rel_grad(g, gr, hd, cm), "H", rel_hess(v, vr, va))
E, g, v = res["core"]
vv, vr2 = v.reshape(-1, 9), np.asarray(vr).reshape(-1, 9)
n_ = np.linalg.norm(vr2, axis=1)
fl = np.maximum(1e-2 * np.linalg.norm(np.asarray(va).reshape(-1, 9), axis=1), 1e-300)
err = np.linalg.norm(vv - vr2, axis=1) / np.maximum(n_, fl)
bad = np.argsort(-err)[:8]
rows = np.searchsorted(rp, bad, side="right") - 1
for b, r in zip(bad, rows):
    print("blk", b, "row", (r % sh.n_u, r // sh.n_u), "col", (ci[b] % sh.n_u, ci[b] // sh.n_u), "err", err[b])
    print("   got", vv[b].round(6), "\n   ref", vr2[b].round(6))
ge = np.linalg.norm(g.reshape(-1, 3) - np.asarray(gr).reshape(-1, 3), axis=1)
wb = np.argsort(-ge)[:5]
print("worst g", [(int(a % sh.n_u), int(a // sh.n_u), float(ge[a])) for a in wb])
