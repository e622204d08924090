"""Pins of the oracle's contact pullback: the contact mesh is embedded in the
sheet (x^alpha = sum_ij N_ij(u_alpha, v_alpha) C^ij, Eq. `eq: trig mesh node from control points`) and a barrier's
gradient / Hessian on the mesh vertices is pulled back to the control points by the chain rule (Eq. `eq: gradient
and hessian of contact barrier`).  Pinned against what the mathematics fixes:
  * the weights: partition of unity, and linear precision (a Greville rest grid maps (u, v) to the affine rest
    position exactly), the closed-form (1/2, 1/2) x (1/2, 1/2) weights at an interior knot point;
  * the Hessian: energy second differences of a quadratic pair energy B(x(C)) (exact for a quadratic, an
    independent route: no chain rule written out), symmetry, and translation invariance of a spring-like pair;
  * the gradient: energy first differences of the same energy.
"""
import numpy as np

import oracle as O
import workloads as W


def _sheet(n=9, L=1.0):
    return W.make_sheet(n, L, 3, n_modes=2, amp=5e-3)


def _oracle(sh):
    return O.Oracle.from_sheet(sh)


def test_weights_partition_of_unity_and_linear_precision():
    sh = _sheet(9, 1.3)
    o = _oracle(sh)
    S = sh.n_u - 2
    rng = np.random.default_rng(0)
    uv = np.concatenate([rng.uniform(0, S, (40, 2)), [[0, 0], [S, S], [3.0, 2.0], [0.5, S]]])
    Wt = o.contact_weights(uv)
    np.testing.assert_allclose(Wt.sum(1), 1.0, atol=1e-14)
    assert (Wt >= -1e-15).all()
    # Greville rest grid: X(u, v) = (L u / S, L v / S) exactly (quadratic B-splines reproduce linear maps)
    X = Wt @ sh.rest_xy.reshape(-1, 2)
    np.testing.assert_allclose(X, 1.3 * uv / S, atol=1e-14)


def test_weights_at_an_interior_knot():
    sh = _sheet(9)
    o = _oracle(sh)
    Wt = o.contact_weights(np.array([[3.0, 4.0]]))[0].reshape(sh.n_v, sh.n_u)
    # right limits at a knot: N_p(p) = N_{p+1}(p) = 1/2, so four control points weigh 1/4
    nz = np.argwhere(Wt > 0)
    assert sorted(map(tuple, nz)) == [(4, 3), (4, 4), (5, 3), (5, 4)]
    np.testing.assert_allclose(Wt[Wt > 0], 0.25, atol=1e-15)


def _pairs(rng, nvert, npairs, obstacle=True):
    verts = rng.integers(0, nvert, (npairs, 4)).astype(np.int32)
    if obstacle:
        verts[npairs // 2:, 1:] = -1   # point-obstacle pairs: one cloth vertex
    A = rng.normal(size=(npairs, 12, 12))
    H = A @ A.transpose(0, 2, 1)       # symmetric PSD pair Hessians
    g = rng.normal(size=(npairs, 12))
    return verts, H, g


def test_pullback_equals_energy_second_differences():
    sh = _sheet(8)
    o = _oracle(sh)
    rng = np.random.default_rng(1)
    S = sh.n_u - 2
    uv = rng.uniform(0, S, (30, 2))
    verts, H, g = _pairs(rng, 30, 12)
    Hcp, gcp = o.contact_pullback(uv, verts, H, g)
    Wt = o.contact_weights(uv)
    x0 = rng.normal(size=(30, 3))

    def energy(C):   # B = sum_c 1/2 dx_c . H_c dx_c + g_c . x_c over the pair's valid slots, x = W C
        x = Wt @ C.reshape(-1, 3)
        e = 0.0
        for c in range(len(verts)):
            m = verts[c] >= 0
            idx = np.repeat(m, 3)
            d = np.zeros(12)
            xx = np.zeros(12)
            d[idx] = (x[verts[c][m]] - x0[verts[c][m]]).reshape(-1)
            xx[idx] = x[verts[c][m]].reshape(-1)
            e += 0.5 * d @ H[c] @ d + g[c] @ xx
        return e

    C0 = rng.normal(size=(sh.n_u * sh.n_v * 3))
    h = 0.5   # a quadratic energy: second differences are exact for any step
    for _ in range(6):
        d1, d2 = rng.normal(size=C0.shape), rng.normal(size=C0.shape)
        fd = (energy(C0 + h * d1 + h * d2) - energy(C0 + h * d1 - h * d2) - energy(C0 - h * d1 + h * d2)
              + energy(C0 - h * d1 - h * d2)) / (4 * h * h)
        assert abs(fd - d1 @ Hcp @ d2) <= 1e-9 * max(1.0, abs(fd))
    np.testing.assert_allclose(Hcp, Hcp.T, atol=1e-12 * np.abs(Hcp).max())
    assert gcp.shape == (sh.n_v, sh.n_u, 3)


def test_gradient_equals_energy_first_differences():
    sh = _sheet(7)
    o = _oracle(sh)
    rng = np.random.default_rng(2)
    S = sh.n_u - 2
    uv = rng.uniform(0, S, (20, 2))
    verts, _, g = _pairs(rng, 20, 10)
    H0 = np.zeros((10, 12, 12))
    _, gcp = o.contact_pullback(uv, verts, H0, g)
    Wt = o.contact_weights(uv)

    def energy(C):   # linear energy sum_c g_c . x_c: its C-gradient is exact from one first difference
        x = Wt @ C.reshape(-1, 3)
        e = 0.0
        for c in range(len(verts)):
            for sa in range(4):
                if verts[c][sa] >= 0:
                    e += g[c][3 * sa:3 * sa + 3] @ x[verts[c][sa]]
        return e

    C0 = rng.normal(size=(sh.n_u * sh.n_v * 3))
    for _ in range(5):
        d = rng.normal(size=C0.shape)
        fd = (energy(C0 + d) - energy(C0 - d)) / 2.0
        assert abs(fd - gcp.reshape(-1) @ d) <= 1e-11 * max(1.0, abs(fd))


def test_spring_pair_is_translation_invariant():
    sh = _sheet(9)
    o = _oracle(sh)
    rng = np.random.default_rng(3)
    S = sh.n_u - 2
    uv = rng.uniform(0, S, (10, 2))
    verts = np.array([[0, 1, -1, -1], [2, 7, -1, -1], [4, 5, -1, -1]], np.int32)
    H = np.zeros((3, 12, 12))
    for c in range(3):
        k = rng.uniform(1, 3)
        blk = k * np.eye(3)
        H[c, 0:3, 0:3], H[c, 3:6, 3:6], H[c, 0:3, 3:6], H[c, 3:6, 0:3] = blk, blk, -blk, -blk
    Hcp, _ = o.contact_pullback(uv, verts, H)
    t = np.tile(rng.normal(size=3), sh.n_u * sh.n_v)   # a rigid translation of every control point
    np.testing.assert_allclose(Hcp @ t, 0.0, atol=1e-12 * np.abs(Hcp).max())
