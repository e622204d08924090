"""Comparison helpers: the north star's tolerance (relative error <= 1e-10 in fp64 for energy,
gradient and every Hessian block; pattern bit-exact), with the floors of SURVEY §8(c).6 /
DESIGN.md §"Tolerance":
  energy:    |dE| / |E|                       (absolute 1e-30 floor for an exact-zero energy)
  gradient:  |dg_a| / max(|g_a|, 1e-12 max_b |g_b|)            per control point
  Hessian:   |dH_blk|_F / max(|H_blk|_F, 1e-9 max |H_blk|_F)   per 3x3 block
The Hessian floor is 1e-9 (not SURVEY's 1e-12): blocks that vanish in exact arithmetic are sums of
terms up to ~1e-6 of the largest block that cancel (measured on C1: sum|terms| = 9.4e-7 max), so
their fp64 noise (~1e-22 max) already equals a 1e-12 floor's allowance.
"""
import numpy as np

TOL = 1e-10
HESS_FLOOR = 1e-9


def rel_energy(E, Eref):
    return abs(E - Eref) / max(abs(Eref), 1e-30)


def rel_grad(g, gref):
    g, gref = np.asarray(g).reshape(-1, 3), np.asarray(gref).reshape(-1, 3)
    n = np.linalg.norm(gref, axis=1)
    floor = 1e-12 * max(n.max(initial=0.0), 1e-300)
    return float((np.linalg.norm(g - gref, axis=1) / np.maximum(n, floor)).max(initial=0.0))


def rel_hess(v, vref):
    v, vref = np.asarray(v).reshape(-1, 9), np.asarray(vref).reshape(-1, 9)
    n = np.linalg.norm(vref, axis=1)
    floor = HESS_FLOOR * max(n.max(initial=0.0), 1e-300)
    return float((np.linalg.norm(v - vref, axis=1) / np.maximum(n, floor)).max(initial=0.0))


def assert_parity(E, g, v, Eref, gref, vref, tol=TOL, what=""):
    if E is not None:
        assert rel_energy(E, Eref) <= tol, f"{what} energy rel err {rel_energy(E, Eref):.3e}"
    if g is not None:
        assert rel_grad(g, gref) <= tol, f"{what} gradient rel err {rel_grad(g, gref):.3e}"
    if v is not None:
        assert rel_hess(v, vref) <= tol, f"{what} Hessian rel err {rel_hess(v, vref):.3e}"
