"""Pins of the CPU oracle against what the paper and mathematics fix (not against itself).

Each test names the pin and the passage it comes from.  Parity status per oracle function:
  basis (Cox–de Boor)          pinned: partition of unity, textbook pieces, Marsden identity, C1, FD
  gauss                        pinned: numpy leggauss (library special case), polynomial exactness
  membrane/bending rules       pinned: TikZ coordinates of Fig. 4/5 (tests/golden), counts, sum of weights
  inverse map (b, L, w)        pinned: identity-map invariants, Newton-inverted finite differences
  membrane energy              pinned: closed forms (uniform stretch, simple shear, rigid motion)
  bending energy               pinned: paraboloid / cylinder / twist closed forms; Navier plate
  gradient                     pinned: complex step of the energy, translation / rotation properties
  Hessian                      pinned: complex step of the gradient, symmetry, null space, covariance
  PSD projection (D7)          pinned: numpy eigh clamp per FBW term, closed-form spectra
  pattern                      pinned: closed-form nnzb, completeness vs complex-step Hessian
  slab mode                    pinned: bit-identical to the unpartitioned oracle
  material_from_young mu_st/mu_sh: "parity unpinned" (naming convention D6); mu_bd pinned by the plate.
"""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W


# ----------------------------------------------------------------------------- basis
def test_basis_partition_of_unity_and_derivative_sums():
    """SPEC.md:80 / PAPER.md:172: sum N = 1, sum N' = 0, sum N'' = 0; N >= 0."""
    rng = np.random.default_rng(0)
    for n in (3, 4, 7, 20):
        k = W.open_uniform_knots(n)
        for x in rng.uniform(0, n - 2, 300):
            N, dN, ddN = O.basis_all(k, x)
            assert abs(N.sum() - 1) < 1e-14
            assert abs(dN.sum()) < 1e-12 and abs(ddN.sum()) < 1e-12
            assert (N >= 0).all()
            assert np.count_nonzero(N) <= 3


def test_basis_midpoint_and_knot_values():
    """(1/8, 3/4, 1/8) at a uniform span midpoint; (1/2, 1/2) at an interior knot."""
    k = W.open_uniform_knots(10)
    N, _, _ = O.basis_all(k, 4.5)
    nz = N[N != 0]
    np.testing.assert_allclose(nz, [1 / 8, 3 / 4, 1 / 8], rtol=0, atol=1e-15)
    N, dN, _ = O.basis_all(k, 4.0)
    assert np.count_nonzero(N) == 2
    np.testing.assert_allclose(N[N != 0], [0.5, 0.5], atol=1e-15)


def test_basis_textbook_pieces():
    """Uniform quadratic B-spline pieces (textbook): on local t in [0,3]:
    t^2/2, (-2t^2+6t-3)/2, (3-t)^2/2; open-end basis N_0 = (1-u)^2 on [0,1]."""
    n = 12
    k = W.open_uniform_knots(n)
    rng = np.random.default_rng(1)
    for x in rng.uniform(0, n - 2, 200):
        N, dN, ddN = O.basis_all(k, x)
        for i in range(2, n - 2):          # bases with uniform knots (i-2, ..., i+1)
            t = x - (i - 2)
            if 0 <= t < 1:
                ref, d, dd = t * t / 2, t, 1.0
            elif 1 <= t < 2:
                ref, d, dd = (-2 * t * t + 6 * t - 3) / 2, -2 * t + 3, -2.0
            elif 2 <= t < 3:
                ref, d, dd = (3 - t) ** 2 / 2, -(3 - t), 1.0
            else:
                ref, d, dd = 0.0, 0.0, 0.0
            assert abs(N[i] - ref) < 1e-14 and abs(dN[i] - d) < 1e-13 and abs(ddN[i] - dd) < 1e-13
        if x < 1:
            assert abs(N[0] - (1 - x) ** 2) < 1e-14 and abs(dN[0] + 2 * (1 - x)) < 1e-13


def test_basis_marsden_reproduction():
    """Quadratic precision (Marsden identity / blossoms): sum_i N_i(x) (xi_{i+1}+xi_{i+2})/2 = x and
    sum_i N_i(x) xi_{i+1} xi_{i+2} = x^2 for p = 2 (SPEC.md:68 affine reproduction)."""
    n = 9
    k = W.open_uniform_knots(n)
    g = 0.5 * (k[1:n + 1] + k[2:n + 2])
    b = k[1:n + 1] * k[2:n + 2]
    for x in np.linspace(0, n - 2, 101):
        N, dN, ddN = O.basis_all(k, x)
        assert abs(N @ g - x) < 1e-13 and abs(dN @ g - 1) < 1e-12 and abs(ddN @ g) < 1e-12
        assert abs(N @ b - x * x) < 1e-12 and abs(dN @ b - 2 * x) < 1e-11 and abs(ddN @ b - 2) < 1e-11


def test_basis_c1_and_finite_differences():
    """C1 continuity at interior knots and derivatives vs central FD."""
    n = 8
    k = W.open_uniform_knots(n)
    for p in range(1, n - 2):
        _, dl, _ = O.basis_all(k, p - 1e-9)
        _, dr, _ = O.basis_all(k, p)
        assert np.abs(dl - dr).max() < 1e-8
    h = 1e-5
    for x in np.random.default_rng(2).uniform(0.01, n - 2.01, 50):
        N, dN, ddN = O.basis_all(k, x)
        Np, dNp, _ = O.basis_all(k, x + h)
        Nm, dNm, _ = O.basis_all(k, x - h)
        if np.floor(x + h) != np.floor(x - h):
            continue
        assert np.abs((Np - Nm) / (2 * h) - dN).max() < 1e-8
        assert np.abs((dNp - dNm) / (2 * h) - ddN).max() < 1e-7


def test_basis_right_limit_second_derivative_at_knots():
    """Half-open indicator of Eq. `eq: B-spline basis` => right limits at knots:
    (1,-2,1) on interior spans and (1,-3,2) on the last span (D4)."""
    n = 9
    S = n - 2
    k = W.open_uniform_knots(n)
    for p in range(1, S):
        _, _, dd = O.basis_all(k, float(p))
        nz = dd[np.abs(dd) > 0]
        idx = np.nonzero(dd)[0]
        assert list(idx) == [p, p + 1, p + 2]
        expect = [1, -3, 2] if p == S - 1 else ([2, -3, 1] if p == 0 else [1, -2, 1])
        np.testing.assert_allclose(nz, expect, atol=1e-14)


# ----------------------------------------------------------------------------- gauss
@pytest.mark.parametrize("m", [1, 2, 3])
def test_gauss_vs_numpy_and_exactness(m):
    x, w = O.gauss(m, 2.0, 3.5)
    xr, wr = np.polynomial.legendre.leggauss(m)
    np.testing.assert_allclose(x, 2.75 + 0.75 * xr, atol=1e-15)
    np.testing.assert_allclose(w, 0.75 * wr, atol=1e-15)
    for d in range(2 * m):
        exact = (3.5 ** (d + 1) - 2.0 ** (d + 1)) / (d + 1)
        assert abs((w * x ** d).sum() - exact) < 1e-12 * max(1, exact)
    d = 2 * m
    exact = (3.5 ** (d + 1) - 2.0 ** (d + 1)) / (d + 1)
    assert abs((w * x ** d).sum() - exact) > 1e-8


# ----------------------------------------------------------------------------- rules
def _close_set(A, B, tol):
    A, B = np.asarray(A, float), np.asarray(B, float)
    assert len(A) == len(B), (len(A), len(B))
    used = np.zeros(len(B), bool)
    for a in A:
        d = np.abs(B - a).max(axis=1)
        d[used] = np.inf
        j = int(np.argmin(d))
        assert d[j] <= tol, (a, B[j], d[j])
        used[j] = True


def test_membrane_rule_matches_fig4_interior(golden):
    """Interior-region membrane points for S=5 equal PAPER.md:381-408 at the drawn precision."""
    u, v, w, _ = O.rule(O.RULE_REDUCED, False, 5, 5)
    sel = (u >= 1) & (u <= 4) & (v >= 1) & (v <= 4)
    drawn = np.array([[float(a), float(b)] for a, b in golden("fig4_membrane_interior_S5.txt")])
    _close_set(np.stack([u[sel], v[sel]], 1), drawn, 6e-4)


def test_membrane_rule_matches_fig4_reference_cells(golden):
    """Boundary spans follow the reference cells of PAPER.md:409-435 (drawn at 1.25 scale)."""
    rows = golden("fig4_reference_cells.txt")
    origin = {"corner": (6, 4), "bottomtop": (6, 2), "leftright": (6, 0)}
    cells = {c: [] for c in origin}
    for c, x, y in rows:
        x0, y0 = origin[c]
        cells[c].append([(float(x) - x0) / 1.25, (float(y) - y0) / 1.25])
    S = 5
    u, v, w, _ = O.rule(O.RULE_REDUCED, False, S, S)
    for (i, j), c in [((0, 0), "corner"), ((4, 4), "corner"), ((0, 4), "corner"), ((2, 0), "bottomtop"),
                      ((1, 4), "bottomtop"), ((0, 2), "leftright"), ((4, 3), "leftright")]:
        sel = (u > i) & (u < i + 1) & (v > j) & (v < j + 1)
        _close_set(np.stack([u[sel] - i, v[sel] - j], 1), cells[c], 2e-3)


def test_bending_rule_matches_fig4(golden):
    u, v, w, _ = O.rule(O.RULE_REDUCED, True, 5, 5)
    drawn = np.array([[float(a), float(b)] for a, b in golden("fig4_bending_S5.txt")])
    _close_set(np.stack([u, v], 1), drawn, 1e-12)


@pytest.mark.parametrize("S", [3, 4, 5, 8, 13])
def test_rule_counts_and_weights(S):
    """Counts 2S^2+20S-14 (membrane) and S^2+2S-3 (bending);
    sum of parametric weights = S^2 (no overlap/gap); all weights > 0."""
    for bend, cnt in ((False, 2 * S * S + 20 * S - 14), (True, S * S + 2 * S - 3)):
        u, v, w, st = O.rule(O.RULE_REDUCED, bend, S, S)
        assert len(u) == cnt
        assert abs(w.sum() - S * S) < 1e-12 and (w > 0).all()
    for kind in (O.RULE_G2_INTERIOR, O.RULE_G3_FULL):
        for bend in (False, True):
            u, v, w, _ = O.rule(kind, bend, S, S)
            assert abs(w.sum() - S * S) < 1e-12


def test_rule_polynomial_exactness():
    """Composite exactness: reduced rules integrate 1, u, v exactly over the
    domain but not u^2; G3-FULL is exact for u^a v^b, a,b <= 5."""
    S = 7
    for bend in (False, True):
        u, v, w, _ = O.rule(O.RULE_REDUCED, bend, S, S)
        assert abs((w * u).sum() - S ** 3 / 2) < 1e-11 and abs((w * v).sum() - S ** 3 / 2) < 1e-11
        assert abs((w * u * u).sum() - S ** 4 / 3) > 1e-6
    u, v, w, _ = O.rule(O.RULE_G3_FULL, False, S, S)
    for a in range(6):
        for b in range(6):
            ex = S ** (a + 1) / (a + 1) * S ** (b + 1) / (b + 1)
            assert abs((w * u ** a * v ** b).sum() - ex) < 1e-11 * ex


def test_rule_dual_cell_exactness():
    """Within one full interior dual cell the 2-point Gauss pair integrates cubics along its
    direction exactly (1x2 / 2x1 Gauss)."""
    S = 8
    u, v, w, _ = O.rule(O.RULE_REDUCED, False, S, S)
    p, q = 3, 3  # even -> along v
    sel = (u == p) & (np.abs(v - q) <= 0.5)
    assert sel.sum() == 2
    for d in range(4):
        ex = ((q + 0.5) ** (d + 1) - (q - 0.5) ** (d + 1)) / (d + 1)
        assert abs((w[sel] * v[sel] ** d).sum() - ex) < 1e-12


def test_fig5_support_points(golden):
    """The 12 membrane points in an interior control point's support and the
    8 bending points (D4)."""
    S = 9
    u, v, w, st = O.rule(O.RULE_REDUCED, False, S, S)
    i, j = 5, 5           # interior cp with i + j even: its support [i-2, i+1] x [j-2, j+1]
    pts = [(u[k] - (i - 2), v[k] - (j - 2)) for k in range(len(u)) if any((s == [i, j]).all() for s in st[k])]
    drawn = np.array([[float(a), float(b)] for a, b in golden("fig5_support_points.txt")])
    _close_set(pts, drawn, 6e-4)
    ub, vb, wb, stb = O.rule(O.RULE_REDUCED, True, S, S)
    nb = sum(1 for k in range(len(ub)) if any((s == [i, j]).all() for s in stb[k]))
    assert nb == 8


def test_stencil_completeness_by_basis_values():
    """Every cp whose N, N_u, N_v (membrane) or second derivatives (bending) are nonzero at a
    point lies in that point's structural stencil."""
    S = 6
    n = S + 2
    k = W.open_uniform_knots(n)
    for bend in (False, True):
        for kind in (0, 1, 2):
            u, v, w, st = O.rule(kind, bend, S, S)
            for q in range(len(u)):
                Nu, dNu, ddNu = O.basis_all(k, u[q])
                Nv, dNv, ddNv = O.basis_all(k, v[q])
                A = np.abs(np.outer(dNv, Nu)) + np.abs(np.outer(Nv, dNu))   # [j, i]
                if bend:
                    A = A + np.abs(np.outer(Nv, ddNu)) + np.abs(np.outer(ddNv, Nu)) + np.abs(np.outer(dNv, dNu))
                need = {(ii, jj) for jj, ii in zip(*np.nonzero(A))}
                have = {tuple(s) for s in st[q]}
                assert need <= have
                assert len(have) <= 9


def test_rule_errors():
    with pytest.raises(RuntimeError):
        O.rule(O.RULE_REDUCED, False, 2, 5)
    rest = W.greville_grid(5, 5, 1.0)
    bad = W.open_uniform_knots(5).copy()
    bad[3] = 0.5
    with pytest.raises(RuntimeError):
        O.Oracle(5, 5, bad, W.open_uniform_knots(5), rest, np.ones(4))
    flip = rest.copy()
    flip[..., 0] *= -1   # mirrored map: det J < 0
    with pytest.raises(RuntimeError):
        O.Oracle(5, 5, W.open_uniform_knots(5), W.open_uniform_knots(5), flip, np.ones(4))


# ----------------------------------------------------------------------------- inverse map
def _surface(k, Xc, u, v):
    Nu, dNu, ddNu = O.basis_all(k, u)
    Nv, dNv, ddNv = O.basis_all(k, v)
    X = np.einsum("j,i,jic->c", Nv, Nu, Xc)
    J = np.stack([np.einsum("j,i,jic->c", Nv, dNu, Xc), np.einsum("j,i,jic->c", dNv, Nu, Xc)], 1)
    return X, J


def test_inverse_map_identity_invariants():
    """For ANY material map: the identity world map has F = I (sum_a X_a b_a^T = I), Laplacian 0
    (sum_a L_a X_a = 0), and translations are null (sum b_a = 0, sum L_a = 0)."""
    n = 9
    rest = W.make_curved_rest(n, n, seed=3)
    o = O.Oracle(n, n, W.open_uniform_knots(n), W.open_uniform_knots(n), rest, np.ones(4))
    Xf = rest.reshape(-1, 2)
    for kpt in range(o.n_membrane + o.n_bending):
        P = o.point(kpt)
        Xa = Xf[P["cps"]]
        if P["bending"]:
            assert abs(P["coef"].sum()) < 1e-9 * np.abs(P["coef"]).max()
            assert np.abs(P["coef"] @ Xa).max() < 1e-9 * np.abs(P["coef"]).max()
        else:
            np.testing.assert_allclose(Xa.T @ P["coef"], np.eye(2), atol=1e-12)
            assert np.abs(P["coef"].sum(0)).max() < 1e-12


def test_inverse_map_vs_newton_finite_differences():
    """b_a = grad_X N_a and L_a = Lap_X N_a, through the inverse function theorem (PAPER.md:287,
    568), against central differences of N_a(u(X), v(X)) with (u, v)(X) found by Newton."""
    n = 8
    S = n - 2
    k = W.open_uniform_knots(n)
    rest = W.make_curved_rest(n, n, seed=5, bend=0.1)
    o = O.Oracle(n, n, k, k, rest, np.ones(4))
    u, v, w, _ = O.rule(O.RULE_REDUCED, False, S, S)
    ub, vb, wb, _ = O.rule(O.RULE_REDUCED, True, S, S)
    us, vs = np.concatenate([u, ub]), np.concatenate([v, vb])

    def uv_of(X, guess):
        uv = np.array(guess, float)
        for _ in range(50):
            Xc, J = _surface(k, rest, *uv)
            step = np.linalg.solve(J, X - Xc)
            uv = uv + step
            if np.abs(step).max() < 1e-15:
                break
        return uv

    def Na(a, X, guess, side):
        uu, vv = uv_of(X, guess)
        # stay on the side of the knot that the point's right-limit convention uses
        Nu, _, _ = O.basis_all(k, uu)
        Nv, _, _ = O.basis_all(k, vv)
        i, j = a % n, a // n
        return Nu[i] * Nv[j]

    rng = np.random.default_rng(0)
    pts = rng.choice(len(us), 25, replace=False)

    def richardson(D, h):
        return (4 * D(h / 2) - D(h)) / 3      # O(h^4) central differences

    checked = 0
    for kp in pts:
        P = o.point(int(kp))
        uq, vq = us[kp], vs[kp]
        if uq == int(uq) or vq == int(vq):
            continue  # knot-line points: one-sided limits; covered by the identity invariants
        X0, _ = _surface(k, rest, uq, vq)
        for t, a in enumerate(P["cps"]):
            f = lambda dx, dy: Na(a, X0 + np.array([dx, dy]), (uq, vq), 0)
            g1 = richardson(lambda h: (f(h, 0) - f(-h, 0)) / (2 * h), 2e-3)
            g2 = richardson(lambda h: (f(0, h) - f(0, -h)) / (2 * h), 2e-3)
            if P["bending"]:
                lap = richardson(lambda h: (f(h, 0) + f(-h, 0) + f(0, h) + f(0, -h) - 4 * f(0, 0)) / (h * h), 4e-3)
                assert abs(lap - P["coef"][t]) < 1e-6 * np.abs(P["coef"]).max()
            else:
                assert abs(g1 - P["coef"][t, 0]) < 1e-8 * S and abs(g2 - P["coef"][t, 1]) < 1e-8 * S
            checked += 1
    assert checked > 20


def test_affine_rest_weights():
    """Greville flat L x L sheet: det J = (L/S)^2 so w = w_hat (L/S)^2 and sum w = L^2 (Q7)."""
    n, L = 10, 1.7
    sh = W.make_sheet(n, L, 0)
    o = O.Oracle.from_sheet(sh)
    tot = sum(o.point(k)["w"] for k in range(o.n_membrane))
    assert abs(tot - L * L) < 1e-12
    tot = sum(o.point(k)["w"] for k in range(o.n_membrane, o.n_membrane + o.n_bending))
    assert abs(tot - L * L) < 1e-12


# ----------------------------------------------------------------------------- energies
MU = np.array([3.0, 5.0, 0.7, 0.0])


def _affine_world(rest, M, t=(0, 0, 0)):
    return np.einsum("ab,jib->jia", M, rest) + np.asarray(t)


@pytest.mark.parametrize("rule", [O.RULE_REDUCED, O.RULE_G2_INTERIOR, O.RULE_G3_FULL])
def test_membrane_uniform_stretch_and_shear(rule):
    """F constant => E = A * Psi(F) for every rule: uniform stretch lambda:
    A (mu1 + mu2)(lambda-1)^2; simple shear F=[[1,g],[0,1],[0,0]]:
    A [mu2 (sqrt(1+g^2)-1)^2 + mu_sh g^2]."""
    n, L = 9, 1.3
    sh = W.make_sheet(n, L, 0)
    o = O.Oracle(n, n, sh.knots_u, sh.knots_v, sh.rest_xy, MU, rule, rule)
    A = L * L
    for lam in (0.8, 1.0, 1.25):
        M = np.array([[lam, 0], [0, lam], [0, 0]])
        E, _, _ = o.eval(_affine_world(sh.rest_xy, M), flags=O.FLAG_NO_BENDING, gradient=False, hessian=False)
        assert abs(E - A * (MU[0] + MU[1]) * (lam - 1) ** 2) < 1e-12 * max(1, E)
    g = 0.3
    M = np.array([[1, g], [0, 1], [0, 0]])
    E, _, _ = o.eval(_affine_world(sh.rest_xy, M), flags=O.FLAG_NO_BENDING, gradient=False, hessian=False)
    assert abs(E - A * (MU[1] * (math.sqrt(1 + g * g) - 1) ** 2 + MU[2] * g * g)) < 1e-12


def test_rigid_motion_zero_energy_and_gradient():
    """Rigid motions: E = 0 and g = 0 (frame indifference of FBW and of |Lap phi|^2)."""
    sh = W.make_sheet(12, 1.0, 0)
    mu = np.array([3.0, 5.0, 0.7, 0.2])
    o = O.Oracle.from_sheet(sh, mu=mu)
    R = W.random_rotation(np.random.default_rng(4))
    x = np.einsum("ab,jib->jia", R, np.concatenate([sh.rest_xy, np.zeros((12, 12, 1))], -1)) + [0.3, -1, 2]
    E, g, _ = o.eval(x, hessian=False)
    assert abs(E) < 1e-26 and np.abs(g).max() < 1e-12 * mu.max()


def _blossom_paraboloid(sh, kx, ky):
    """Control points of z = kx X1^2/2 + ky X2^2/2 on a Greville flat sheet (Marsden identity)."""
    n, L = sh.n_u, sh.rest_xy[0, -1, 0]
    S = n - 2
    k = sh.knots_u
    bu = k[1:n + 1] * k[2:n + 2] * (L / S) ** 2
    x = np.concatenate([sh.rest_xy, np.zeros((n, n, 1))], -1)
    x[..., 2] = 0.5 * kx * bu[None, :] + 0.5 * ky * bu[:, None]
    return x


@pytest.mark.parametrize("rule", [O.RULE_REDUCED, O.RULE_G2_INTERIOR, O.RULE_G3_FULL])
def test_bending_closed_forms(rule):
    """Paraboloid z = k|X|^2/2: Lap phi = (0,0,2k) => E_bd = 2 mu_bd k^2 A; cylinder z = k X1^2/2:
    E_bd = mu_bd k^2 A / 2; twist z = k X1 X2: E_bd = 0."""
    n, L = 10, 1.5
    sh = W.make_sheet(n, L, 0)
    mu = np.array([0.0, 0.0, 0.0, 2.5])
    o = O.Oracle(n, n, sh.knots_u, sh.knots_v, sh.rest_xy, mu, rule, rule)
    A, kap = L * L, 0.7
    E, _, _ = o.eval(_blossom_paraboloid(sh, kap, kap), flags=O.FLAG_NO_MEMBRANE, gradient=False, hessian=False)
    assert abs(E - 2 * mu[3] * kap ** 2 * A) < 1e-11 * E
    E, _, _ = o.eval(_blossom_paraboloid(sh, kap, 0), flags=O.FLAG_NO_MEMBRANE, gradient=False, hessian=False)
    assert abs(E - 0.5 * mu[3] * kap ** 2 * A) < 1e-11 * E
    x = np.concatenate([sh.rest_xy, np.zeros((n, n, 1))], -1)
    x[..., 2] = kap * sh.rest_xy[..., 0] * sh.rest_xy[..., 1]
    E, _, _ = o.eval(x, flags=O.FLAG_NO_MEMBRANE, gradient=False, hessian=False)
    assert abs(E) < 1e-24


def test_navier_plate_pins_bending_stiffness():
    """simply supported square plate, uniform load B: w_max =
    0.048744 B a^4 (1-nu^2)/(E h^3) = 0.0040620 B a^4 / D.  Solving the oracle's bending Hessian
    with mu_bd = E h^3/(12(1-nu^2)) (D6) reproduces it under refinement."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    E, nu, h, a, B = 2e6, 0.03, 0.01, 1.0, 9.81
    exact = 0.048744 * B * a ** 4 * (1 - nu * nu) / (E * h ** 3)
    errs = []
    for n in (18, 34):
        sh = W.make_sheet(n, a, 0, E=E, nu=nu, h=h)
        mu = O.material_from_young(E, nu, h)
        o = O.Oracle.from_sheet(sh, mu=mu)
        x0 = np.concatenate([sh.rest_xy, np.zeros((n, n, 1))], -1)
        _, _, vals = o.eval(x0, flags=O.FLAG_NO_MEMBRANE, energy=False, gradient=False)
        rp, ci = o.pattern()
        K = sp.csr_matrix((vals[:, 2, 2], ci, rp), shape=(n * n, n * n))
        # consistent load f_a = B * integral N_a = B (L/S)^2 * (xi_{i+3}-xi_i)/3 * (xi_{j+3}-xi_j)/3
        k = sh.knots_u
        S = n - 2
        s1 = (k[3:n + 3] - k[0:n]) / 3 * (a / S)
        f = B * np.outer(s1, s1).ravel()
        free = np.ones((n, n), bool)
        free[0, :] = free[-1, :] = free[:, 0] = free[:, -1] = False
        fr = free.ravel()
        z = np.zeros(n * n)
        z[fr] = spl.spsolve(K[fr][:, fr].tocsc(), f[fr])
        # deflection at the plate centre, evaluated on the surface
        N, _, _ = O.basis_all(k, S / 2)
        wmax = N @ z.reshape(n, n) @ N
        errs.append(abs(wmax - exact) / exact)
    assert errs[1] < errs[0] and errs[1] < 0.01, errs


# ----------------------------------------------------------------------------- derivatives
def _tiny(n, seed, curved=False, rule=O.RULE_REDUCED, amp=0.05):
    sh = W.make_sheet(n, 1.0, seed)
    rng = np.random.default_rng(seed + 7)
    rest = W.make_curved_rest(n, n, seed) if curved else sh.rest_xy
    x = np.concatenate([rest, np.zeros((n, n, 1))], -1) * 1.1 + rng.normal(0, amp, (n, n, 3))
    mu = np.array([3.0, 4.0, 1.5, 0.05])
    o = O.Oracle(n, n, sh.knots_u, sh.knots_v, rest, mu, rule, rule)
    return o, x


@pytest.mark.parametrize("n,curved,rule", [(5, False, 0), (6, True, 0), (7, False, 1), (5, True, 2)])
def test_gradient_complex_step(n, curved, rule):
    """dE/dC_k = Im E(C + i h e_k)/h, h = 1e-30, <= 1e-12 relative."""
    o, x = _tiny(n, 11 + n, curved, rule)
    E, g, _ = o.eval(x, hessian=False)
    gc = np.zeros_like(x)
    hh = 1e-30
    for idx in np.ndindex(x.shape):
        xi = np.zeros_like(x)
        xi[idx] = hh
        gc[idx] = o.energy_cplx(x, xi).imag / hh
    assert np.abs(g - gc).max() < 1e-12 * np.abs(gc).max()
    assert abs(o.energy_cplx(x, np.zeros_like(x)).real - E) < 1e-14 * E
    # translation: sum of gradients vanishes
    assert np.abs(g.reshape(-1, 3).sum(0)).max() < 1e-12 * np.abs(g).max()


def test_gradient_rotation_covariance_and_fd():
    o, x = _tiny(6, 3)
    _, g, _ = o.eval(x, hessian=False)
    R = W.random_rotation(np.random.default_rng(9))
    _, gR, _ = o.eval(x @ R.T, hessian=False)
    assert np.abs(gR - g @ R.T).max() < 1e-12 * np.abs(g).max()
    h = 1e-6
    for idx in [(1, 2, 0), (3, 3, 2), (0, 5, 1)]:
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fd = (o.eval(xp, hessian=False, gradient=False)[0] - o.eval(xm, hessian=False, gradient=False)[0]) / (2 * h)
        assert abs(fd - g[idx]) < 1e-6 * np.abs(g).max()


@pytest.mark.parametrize("n,curved,rule", [(5, False, 0), (6, True, 0), (5, False, 2), (6, False, 1)])
def test_hessian_complex_step_and_structure(n, curved, rule):
    """Unprojected H = complex step of the analytic gradient (dense), every nonzero inside the
    pattern, symmetric, block rows sum to 0, rotation covariant."""
    o, x = _tiny(n, 20 + n, curved, rule)
    H = o.dense_hessian(x)
    N = n * n
    Hc = np.zeros((3 * N, 3 * N))
    hh = 1e-30
    for k in range(3 * N):
        xi = np.zeros(3 * N)
        xi[k] = hh
        Hc[:, k] = (o.gradient_cplx(x, xi.reshape(x.shape)).imag / hh).ravel()
    scale = np.abs(Hc).max()
    assert np.abs(H - Hc).max() < 1e-12 * scale
    # completeness: every structural nonzero of the complex-step Hessian is in the pattern
    rp, ci = o.pattern()
    mask = np.zeros((N, N), bool)
    for a in range(N):
        mask[a, ci[rp[a]:rp[a + 1]]] = True
    blk = np.abs(Hc).reshape(N, 3, N, 3).max(axis=(1, 3))
    assert not ((blk > 1e-13 * scale) & ~mask).any()
    assert np.abs(H - H.T).max() < 1e-13 * scale
    assert np.abs(H.reshape(3 * N, N, 3).sum(1)).max() < 1e-11 * scale
    R = W.random_rotation(np.random.default_rng(n))
    HR = o.dense_hessian(x @ R.T)
    Rb = np.kron(np.eye(N), R)
    assert np.abs(HR - Rb @ H @ Rb.T).max() < 1e-11 * scale


def test_projection_matches_eigh_clamp_per_term():
    """D7: A_proj = PSD(H_st1) + PSD(H_st2) + PSD(H_sh), each term's F-space Hessian clamped by its
    eigen-decomposition (numpy eigh as the library special case)."""
    rng = np.random.default_rng(0)
    mu = np.array([2.0, 3.0, 0.8, 0.0])
    for _ in range(50):
        f1, f2 = rng.normal(size=3) * rng.uniform(0.3, 1.5), rng.normal(size=3) * rng.uniform(0.3, 1.5)
        tot = np.zeros((6, 6))
        for m in ([mu[0], 0, 0, 0], [0, mu[1], 0, 0], [0, 0, mu[2], 0]):
            Ht = O.membrane_A(np.array(m, float), f1, f2, False)
            lam, V = np.linalg.eigh(Ht)
            tot += (V * np.maximum(lam, 0)) @ V.T
        Ap = O.membrane_A(mu, f1, f2, True)
        assert np.abs(Ap - tot).max() < 1e-12 * np.abs(tot).max()
        assert np.linalg.eigvalsh(Ap).min() > -1e-12 * np.abs(Ap).max()
        # closed-form stretch spectrum: 2mu along f, 2mu(1-1/|f|) (x2) across
        Hs = O.membrane_A(np.array([mu[0], 0, 0, 0]), f1, f2, False)[:3, :3]
        nf = np.linalg.norm(f1)
        np.testing.assert_allclose(np.sort(np.linalg.eigvalsh(Hs)),
                                   np.sort([2 * mu[0], 2 * mu[0] * (1 - 1 / nf), 2 * mu[0] * (1 - 1 / nf)]),
                                   atol=1e-12 * 2 * mu[0] / min(nf, 1))


def test_projection_special_cases():
    """Stretched (lambda >= 1) with I6 = 0: projection is a no-op; compressed (lambda < 1) with
    I6 = 0: each stretch block becomes exactly 2 mu f^ f^T."""
    mu = np.array([2.0, 3.0, 0.8, 0.0])
    f1, f2 = np.array([1.2, 0, 0]), np.array([0, 1.1, 0])
    np.testing.assert_allclose(O.membrane_A(mu, f1, f2, True), O.membrane_A(mu, f1, f2, False), atol=1e-14)
    f1, f2 = np.array([0.7, 0, 0]), np.array([0, 0.9, 0])
    A = O.membrane_A(np.array([mu[0], mu[1], 0, 0]), f1, f2, True)
    np.testing.assert_allclose(A[:3, :3], 2 * mu[0] * np.diag([1, 0, 0]), atol=1e-14)
    np.testing.assert_allclose(A[3:, 3:], 2 * mu[1] * np.diag([0, 1, 0]), atol=1e-14)


def test_projected_hessian_psd_and_nullspace():
    o, x = _tiny(6, 40, amp=0.2)
    H = o.dense_hessian(x, flags=O.FLAG_PROJECT)
    s = np.abs(H).max()
    assert np.linalg.eigvalsh(0.5 * (H + H.T)).min() > -1e-12 * s
    assert np.abs(H.reshape(H.shape[0], -1, 3).sum(1)).max() < 1e-11 * s
    Hb = o.dense_hessian(x, flags=O.FLAG_NO_MEMBRANE)
    Hb2 = o.dense_hessian(x * 1.3 + 0.1, flags=O.FLAG_NO_MEMBRANE)
    assert np.array_equal(Hb, Hb2)   # bending Hessian is constant in C


# ----------------------------------------------------------------------------- pattern / slabs
@pytest.mark.parametrize("S", [3, 4, 5, 9, 16])
def test_pattern_closed_forms(S):
    n = S + 2
    sh = W.make_sheet(n, 1.0, 0)
    o = O.Oracle.from_sheet(sh)
    assert o.nnzb == 23 * S * S + 48 * S + 8
    og = O.Oracle.from_sheet(sh, mrule=O.RULE_G3_FULL, brule=O.RULE_G3_FULL)
    assert og.nnzb == (5 * n - 6) ** 2
    rp, ci = o.pattern()
    assert (np.diff(rp) <= 25).all()
    if S >= 7:
        a = (n // 2) * n + n // 2
        cols = ci[rp[a]:rp[a + 1]] - a
        offs = {(int(c % n + n // 2) - n // 2 - 0, 0) for c in []}
        di = [((c + n // 2 + 2 * n) % n) - n // 2 for c in cols]
        dj = [int(np.round((c - d) / n)) for c, d in zip(cols, di)]
        got = set(zip(di, dj))
        expect = {(p, q) for p in range(-2, 3) for q in range(-2, 3)} - {(2, 2), (-2, -2)}
        assert got == expect
    for r in range(n * n):
        row = ci[rp[r]:rp[r + 1]]
        assert (np.diff(row) > 0).all() and r in row


def test_slab_mode_bit_identical():
    """Row slabs with 2-row halos reproduce the unpartitioned oracle bit for bit."""
    sh = W.make_c1()
    full = O.Oracle.from_sheet(sh)
    E, g, vals = full.eval(sh.x, flags=O.FLAG_PROJECT)
    rp, ci = full.pattern()
    Es, gs, vs, cis = [], [], [], []
    for r0, r1 in ((0, 5), (5, 6), (6, 11), (11, 16)):
        o = O.Oracle.from_sheet(sh, r0=r0, r1=r1)
        e, gg, vv = o.eval(sh.x, flags=O.FLAG_PROJECT)
        Es.append(e); gs.append(gg); vs.append(vv)
        cis.append(o.pattern()[1])
    assert np.array_equal(np.concatenate(cis), ci)
    assert np.array_equal(np.concatenate(gs), g)
    assert np.array_equal(np.concatenate(vs), vals)
    assert abs(sum(Es) - E) < 1e-14 * E


def test_thread_count_independent():
    sh = W.make_c1()
    o = O.Oracle.from_sheet(sh)
    a = o.eval(sh.x, threads=1)
    b = o.eval(sh.x, threads=4)
    assert a[0] == b[0] and np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])


def test_rigid_motion_self_consistency_within_tolerance():
    """The oracle is frame-indifferent up to fp64 noise; that noise, measured with the parity metric
    of tests/parity.py, stays 30x below the 1e-10 tolerance — the calibration of the
    gradient floor 1e-4 |H_aa| |C|_max and the Hessian floor 1e-2 sum_q |H_q,blk|."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from parity import diag_block_norms, rel_grad, rel_hess
    sh = W.make_c2(state=3)
    o = O.Oracle.from_sheet(sh)
    rp, ci = o.pattern()
    E, g, v = o.eval(sh.x, flags=O.FLAG_PROJECT)
    R = W.random_rotation(np.random.default_rng(5))
    E2, g2, v2 = o.eval(sh.x @ R.T + np.array([0.0625, -0.125, 0.03125]), flags=O.FLAG_PROJECT)
    v2 = np.einsum("ab,kbc,dc->kad", R.T, v2, R.T)
    va = o.eval(sh.x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    assert abs(E2 - E) / E < 1e-13
    assert rel_grad(g2 @ R, g, diag_block_norms(v, rp, ci, 0, sh.n_u), np.abs(sh.x).max()) < 1e-11
    assert rel_hess(v2, v, va) < 1e-11
    # the abs-sum scale dominates every block and equals |H| for single-term blocks
    assert (np.linalg.norm(va.reshape(-1, 9), axis=1) >= np.linalg.norm(v.reshape(-1, 9), axis=1) * (1 - 1e-14)).all()
