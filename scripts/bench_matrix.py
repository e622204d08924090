"""Secondary measurement rows of SURVEY §8(d): every config x {exact Hessian, PSD-projected} x {reduced
rules, G3-FULL}, one B200, device-resident inputs, CUDA events around K back-to-back calls.

  C1  16^2, one sheet (launch-bound: reported, not graded)
  C2  128^2, the 100 seeded states in one bsf_eval_all_batch call (the bench's launch)
  C3  226^2, E = 1e5, one sheet (its outputs fit in L2: the rate is an upper bound)
  C4  1024^2, one sheet
  C5  64 sheets of 256^2 with per-sheet L, E, nu in one bsf_eval_all_batch_params call (all 64; the
      bench's per-GPU share is 8)

Per row: ms per call, elements/s, algorithmic bytes per call (24 N_cp + 24 N_cp + 72 nnzb + 8
per sheet) / time as a fraction of the measured HBM copy peak.  G3-FULL rows are FP64-bound:
their fraction is also given against the FP64 peak measured by scripts/ubench/fp64 when its JSON is passed.
Round 2 groups: "g2" = the G2-INTERIOR rule (the paper's ablation (A), 2x2 Gauss on the
interior spans) beside the reduced rule (B) on C2 and C4; "curved" = a non-affine (curved)
rest grid of C2 and C4 size on the general path, whose per-point rest tables (G, w: 40 B per membrane point; w and
the five Laplacian coefficients: 48 B per bending point) are counted as extra algorithmic bytes.
usage: python scripts/bench_matrix.py [out.json] [fp64.json] [groups: base,g2,curved]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import workloads as W
import paper_2506_18867_b200 as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HBM = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
FP64 = json.load(open(sys.argv[2]))["fp64_tflops"] if len(sys.argv) > 2 and sys.argv[2] != "-" else None
GROUPS = (sys.argv[3] if len(sys.argv) > 3 else "base").split(",")


def alg_bytes(n_cp, nnzb):
    return 24 * n_cp + 24 * n_cp + 72 * nnzb + 8


def g3_flops_per_call(n_cp, n_u, n_v):
    """SURVEY §8(d) flop model for G3-FULL: 9 S^2 membrane points with k = 9 (3.83 kflop each) and 9 S^2
    bending points with k = 9 (10 k + 6 + 4 k (k + 1) / 2 = 276 flop)."""
    S2 = (n_u - 2) * (n_v - 2)
    return 9 * S2 * (24 * 9 + 194 + 76 * 45) + 9 * S2 * (10 * 9 + 6 + 4 * 45)


def run(name, sheets, rule, flags, steps=10, warmup=3, params=None, tables=False):
    s = B.Sheet.from_sheet(sheets[0], rule, rule)
    nb = len(sheets)
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    E = torch.zeros(nb, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((nb, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    P = None
    if params is not None:
        P = torch.from_numpy(np.stack(params)).cuda()

    def call():
        if P is None:
            s.eval_all_batch(X, E, G, V, flags)
        else:
            s.eval_all_batch_params(X, P, E, G, V, flags)

    for _ in range(warmup):
        call()
    torch.cuda.synchronize()
    t = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        call()
        b.record()
        b.synchronize()
        t.append(a.elapsed_time(b))
    ms = float(np.median(t))
    q = sheets[0]
    n_cp = q.n_u * q.n_v
    el = (q.n_u - 2) * (q.n_v - 2) * nb
    byt = alg_bytes(n_cp, s.nnzb) * nb
    tb = 0
    if tables:   # per-point rest tables read per call: the tile kernel's (G, w: 40 B per membrane point; w and five
        # Laplacian coefficients: 48 B per bending point) on the frame, and k_core's on the interior rectangle
        # (per knot: two membrane points x 5 doubles and one bending point x 10; per cp: 23 bending blocks + 8
        # bending weights), chol.hpp-style counts from the pattern sizes
        i0, i1, j0, j1 = s.core_rect()
        q = sheets[0]
        core_cp = (i1 - i0) * (j1 - j0)
        frac_core = core_cp / (q.n_u * q.n_v)
        tb = (40 * s.n_membrane + 48 * s.n_bending) * (1.0 - frac_core) + \
            8 * ((q.n_u - 1) * (q.n_v - 1) * 20 + core_cp * 31)
        tb = int(tb) * nb
    rule_name = {B.RULE_REDUCED: "reduced", B.RULE_G2_INTERIOR: "g2_interior", B.RULE_G3_FULL: "g3_full"}[rule]
    row = {"config": name, "rule": rule_name,
           "flags": "psd" if flags & B.PROJECT_PSD else "exact", "sheets": nb, "ms_per_call": round(ms, 4),
           "elements_per_s": el / ms * 1e3, "alg_bytes": byt, "hbm_frac": byt / (ms * 1e-3) / (HBM * 1e9),
           "launches": s.last_launch_count(), "core": s.core_rect()[1] > 0}
    if tables:
        row["table_bytes"] = tb
        row["hbm_frac_with_tables"] = (byt + tb) / (ms * 1e-3) / (HBM * 1e9)
    if rule == B.RULE_G3_FULL:
        fl = g3_flops_per_call(n_cp, q.n_u, q.n_v) * nb
        row["model_gflop"] = fl / 1e9
        if FP64:
            row["fp64_frac"] = fl / (ms * 1e-3) / (FP64 * 1e12)
    del X, G, V, E
    s.close()
    torch.cuda.empty_cache()
    return row


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    rows = []
    c5 = W.make_c5()
    c5p = [B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h)) for q in c5]
    cases = [("C1", [W.make_c1()], None),
             ("C2", [W.make_c2(state=k) for k in range(100)], None),
             ("C3", [W.make_c3(1e5)], None),
             ("C4", [W.make_c4()], None),
             ("C5", c5, c5p)]

    def emit(r, t0):
        r["wall_s"] = round(time.time() - t0, 1)
        print(json.dumps(r), flush=True)
        rows.append(r)
    if "base" in GROUPS:
        for name, sheets, params in cases:
            for rule in (B.RULE_REDUCED, B.RULE_G3_FULL):
                for flags in (B.PROJECT_PSD, 0):
                    t0 = time.time()
                    emit(run(name, sheets, rule, flags, params=params), t0)
    if "g2" in GROUPS:   # ablation (A) G2-INTERIOR vs (B) reduced
        for name, sheets, params in (cases[1], cases[3]):
            for rule in (B.RULE_G2_INTERIOR, B.RULE_REDUCED):
                t0 = time.time()
                emit(run(name, sheets, rule, B.PROJECT_PSD), t0)
    if "curved" in GROUPS:   # non-affine rest grids on the general path (per-point rest tables)
        for name, n, nst in (("C2-curved", 128, 100), ("C4-curved", 1024, 1)):
            rest = W.make_curved_rest(n, n, seed=7)
            ku = W.open_uniform_knots(n)
            rng = np.random.default_rng(11)
            base = np.concatenate([rest, np.zeros((n, n, 1))], -1)
            sheets = [W.Sheet(n, n, ku, ku, rest, base * 1.01 + rng.normal(0, 1e-3 / n * 16, (n, n, 3)), 1e5, 0.3, 3e-4)
                      for _ in range(nst)]
            t0 = time.time()
            emit(run(name, sheets, B.RULE_REDUCED, B.PROJECT_PSD, tables=True), t0)
    if out:
        with open(out, "w") as f:
            json.dump({"hbm_gbs": HBM, "fp64_tflops": FP64, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
