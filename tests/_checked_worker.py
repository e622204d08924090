"""Worker of tests/test_gpu_checked.py: runs in its own process with BSF_LIB_PATH pointing at the checked library
(-DBSF_CHECKED: every kernel fills its shared memory with NaN first).  For each case it pre-fills the outputs
with NaN inside guard zones of a sentinel pattern, calls the library three times, and writes a JSON report:
guards intact (no write outside the outputs), outputs finite (every entry written, no read of unwritten
shared memory), repeated calls bit-identical, and the oracle comparison (north-star tolerance)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402
from parity import diag_block_norms, rel_energy, rel_grad, rel_hess  # noqa: E402

GUARD = 4096
SENT = -1.2345678901234567e300


def guarded(n):
    buf = torch.full((n + 2 * GUARD,), SENT, dtype=torch.float64, device="cuda")
    buf[GUARD:GUARD + n] = float("nan")
    return buf, buf[GUARD:GUARD + n]


def case(name, sh, mrule=0, brule=0, flags=B.PROJECT_PSD, r0=0, r1=None, x=None, env=None):
    x = sh.x if x is None else x
    r1 = sh.n_v if r1 is None else r1
    s = B.Sheet.from_sheet(sh, mrule, brule, row_begin=r0, row_end=r1)
    xd = torch.from_numpy(np.ascontiguousarray(x[s.x_row_begin:s.x_row_end])).cuda()
    gbuf, g = guarded((r1 - r0) * sh.n_u * 3)
    vbuf, v = guarded(s.nnzb * 9)
    ebuf, E = guarded(1)
    outs = []
    for _ in range(3):
        s.eval_all(xd, E, g.view(r1 - r0, sh.n_u, 3), v.view(s.nnzb, 3, 3), flags)
        torch.cuda.synchronize()
        outs.append((E.clone(), g.clone(), v.clone()))
    guards = all(bool((b[:GUARD] == SENT).all()) and bool((b[-GUARD:] == SENT).all()) for b in (gbuf, vbuf, ebuf))
    finite = all(bool(torch.isfinite(t).all()) for t in outs[0])
    determ = all(torch.equal(a, b) for o in outs[1:] for a, b in zip(o, outs[0]))
    mu = O.material_from_young(sh.E, sh.nu, sh.h)
    o = O.Oracle.from_sheet(sh, mrule, brule, r0=r0, r1=r1, mu=mu)
    Er, gr, vr = o.eval(x, flags=flags & 7)
    rp, ci = o.pattern()
    va = o.eval(x, flags=(flags & 7) | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    gn, vn = outs[0][1].cpu().numpy(), outs[0][2].cpu().numpy()
    rep = {"case": name, "launches": s.last_launch_count(), "guards_intact": guards, "finite": finite,
           "deterministic": determ, "rel_E": rel_energy(float(outs[0][0].item()), Er),
           "rel_g": rel_grad(gn, gr, diag_block_norms(vr, rp, ci, r0, sh.n_u), np.abs(x).max()),
           "rel_H": rel_hess(vn, vr, va)}
    print(json.dumps(rep), flush=True)
    return rep


def main(out):
    assert "checked" in B._build.LIB, B._build.LIB
    reps = []
    c1, c2 = W.make_c1(), W.make_c2(state=3)
    s40 = W.make_sheet(40, 1.0, 8, n_modes=4, amp=5e-3)
    reps.append(case("C1 core+band+frame", c1))
    reps.append(case("C2 core+band+frame", c2))
    reps.append(case("C2 tile only", c2, flags=B.PROJECT_PSD | B.TILE_ONLY))
    reps.append(case("C1 generic", c1, flags=B.PROJECT_PSD | B.GENERIC_PATH))
    reps.append(case("n40 G3-FULL (k_g3)", s40, 2, 2))
    reps.append(case("n40 G2-INT (tile)", s40, 1, 1))
    reps.append(case("C2 slab [40,90)", c2, r0=40, r1=90))
    reps.append(case("C2 exact Hessian", c2, flags=0))
    n = 24
    rest = W.make_curved_rest(n, n, seed=6)
    xc = np.concatenate([rest, np.zeros((n, n, 1))], -1) * 1.02 + np.random.default_rng(1).normal(0, 2e-3, (n, n, 3))
    shc = W.Sheet(n, n, W.open_uniform_knots(n), W.open_uniform_knots(n), rest, xc, 1e5, 0.3, 3e-4)
    reps.append(case("n24 curved rest (tile)", shc))
    with open(out, "w") as f:
        json.dump(reps, f)


if __name__ == "__main__":
    main(sys.argv[1])
