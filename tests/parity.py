"""Comparison helpers: the north star's tolerance (relative error <= 1e-10 in fp64 for energy,
gradient and every Hessian block; pattern bit-exact), with the floors of SURVEY §8(c).6 /
DESIGN.md §"Tolerance":
  energy:    |dE| / |E|                       (absolute 1e-30 floor for an exact-zero energy)
  gradient:  |dg_a| / max(|g_a|, 1e-4 |H_aa|_F |C|_max)          per control point
  Hessian:   |dH_blk|_F / max(|H_blk|_F, 1e-2 |S_blk|_F)          per 3x3 block
where S_blk = sum_q |H_q,blk| (entrywise) is the block's cancellation scale (oracle FLAG_ABS_SUM).
Blocks that vanish in exact arithmetic are sums of cancelling terms (e.g. two bending points
contributing -1/4 and +1/4 w mu c^2); their fp64 noise is ~4e-14 S_blk in the oracle itself (its
affine second-order inverse-map terms are pure rounding), so they are measured against 1% of
their term scale.
The gradient floor scales with the local stiffness |H_aa| times the position magnitude |C|_max:
F = sum_a C_a b_a is formed from absolute positions, so the absolute fp64 accuracy of g_a is
~u |H_aa| |C|_max (the oracle disagrees with ITSELF by 1.9e-10 per control point under an exact
rigid motion of C2 with a 1e-12 g_max floor, and by <= 3e-12 with this floor).
"""
import numpy as np

TOL = 1e-10
HESS_FLOOR = 1e-2


def rel_energy(E, Eref):
    return abs(E - Eref) / max(abs(Eref), 1e-30)


GRAD_FLOOR = 1e-4


def diag_block_norms(vals, row_ptr, col_idx, row_begin, n_u):
    """|H_aa|_F of the diagonal block of every (owned) block row."""
    vals = np.asarray(vals).reshape(-1, 9)
    row_ptr, col_idx = np.asarray(row_ptr, np.int64), np.asarray(col_idx, np.int64)
    nrows = len(row_ptr) - 1
    rows = np.repeat(np.arange(nrows, dtype=np.int64), np.diff(row_ptr))
    k = np.flatnonzero(col_idx == rows + row_begin * n_u)   # one diagonal block per row, in row order
    assert len(k) == nrows, "pattern without a diagonal block"
    return np.linalg.norm(vals[k], axis=1)


def rel_grad(g, gref, hdiag, cmax):
    """hdiag: |H_aa|_F per control point (from the oracle), cmax: max |C| over the positions."""
    g, gref = np.asarray(g).reshape(-1, 3), np.asarray(gref).reshape(-1, 3)
    n = np.linalg.norm(gref, axis=1)
    floor = np.maximum(GRAD_FLOOR * np.asarray(hdiag) * cmax, 1e-300)
    return float((np.linalg.norm(g - gref, axis=1) / np.maximum(n, floor)).max(initial=0.0))


def rel_hess(v, vref, vabs):
    """vabs: sum_q |H_q,blk| per block (oracle eval with FLAG_ABS_SUM)."""
    v, vref = np.asarray(v).reshape(-1, 9), np.asarray(vref).reshape(-1, 9)
    n = np.linalg.norm(vref, axis=1)
    floor = np.maximum(HESS_FLOOR * np.linalg.norm(np.asarray(vabs).reshape(-1, 9), axis=1), 1e-300)
    return float((np.linalg.norm(v - vref, axis=1) / np.maximum(n, floor)).max(initial=0.0))


def assert_parity(E, g, v, Eref, gref, vref, tol=TOL, what="", hdiag=None, cmax=None, vabs=None):
    if E is not None:
        assert rel_energy(E, Eref) <= tol, f"{what} energy rel err {rel_energy(E, Eref):.3e}"
    if g is not None:
        assert hdiag is not None and cmax is not None, "gradient parity needs the oracle's |H_aa| and |C|_max"
        r = rel_grad(g, gref, hdiag, cmax)
        assert r <= tol, f"{what} gradient rel err {r:.3e}"
    if v is not None:
        assert vabs is not None, "Hessian parity needs the oracle's per-block absolute sums"
        r = rel_hess(v, vref, vabs)
        assert r <= tol, f"{what} Hessian rel err {r:.3e}"
