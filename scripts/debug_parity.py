"""Diagnostic: per-path parity errors against the oracle with the worst block / cp located."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle as O, workloads as W, paper_2506_18867_b200 as B
from parity import diag_block_norms, rel_grad, rel_hess, rel_energy

def run(name, sh, flags):
    mu = O.material_from_young(sh.E, sh.nu, sh.h)
    o = O.Oracle.from_sheet(sh, mu=mu)
    Er, gr, vr = o.eval(sh.x, flags=flags)
    rp, ci = o.pattern()
    s = B.Sheet.from_sheet(sh)
    xd = torch.from_numpy(sh.x).cuda()
    n = sh.n_u
    for path in (0, B.GENERIC_PATH):
        E, g, v = s(xd, flags | path); torch.cuda.synchronize()
        g, v = g.cpu().numpy(), v.cpu().numpy()
        V, Vr = v.reshape(-1, 9), vr.reshape(-1, 9)
        nr = np.linalg.norm(Vr, axis=1); d = np.linalg.norm(V - Vr, axis=1)
        rel = d / np.maximum(nr, 1e-9 * nr.max())
        k = int(np.argmax(rel)); a = int(np.searchsorted(rp, k, side="right") - 1); b = int(ci[k])
        print(f"{name} flags={flags} path={'generic' if path else 'tile'}: E {rel_energy(E.item(), Er):.1e} "
              f"g {rel_grad(g, gr, diag_block_norms(vr, rp, ci, 0, n), np.abs(sh.x).max()):.1e} H {rel.max():.1e} "
              f"worst block a=({a % n},{a // n}) b=({b % n},{b // n}) |H|/max={nr[k] / nr.max():.2e} |dH|/max={d[k] / nr.max():.2e}")
        # distribution of relative errors of blocks above 1e-6 max
        big = nr > 1e-6 * nr.max()
        print("   blocks>1e-6max: max rel %.2e ; median %.2e" % (rel[big].max(), np.median(rel[big])))

run("C1", W.make_c1(), 0)
run("C2s3", W.make_c2(state=3), 0)
run("C2s3", W.make_c2(state=3), 1)
sh = W.make_c2(state=3); sh.x = np.ascontiguousarray(np.concatenate([sh.rest_xy, np.zeros((128,128,1))], -1) + np.random.default_rng(0).normal(0, 1e-3, (128,128,3)))
run("C2-unrotated-noise", sh, 0)
