"""Pins of the oracle's incremental-potential terms (CPU only).

  lumped mass   pinned: closed form R0 h^2 (t_{i+3}-t_i)/3 (t_{j+3}-t_j)/3 on an
                                            affine sheet; total = R0 * area of a curved rest shape (area by
                                            Green's theorem on the boundary curve); slab rows = full rows
  inertia / gravity energy   pinned: uniform offset -> M|d|^2/(2dt^2); flat sheet at height c
                                            -> -M g_z c
  gradient / Hessian increments             pinned: central differences of the energy increment (exact for a
                                            quadratic), Hessian increment diagonal and equal to m/dt^2
  pinned control points (Q14)     pinned: zero gradient rows, identity diagonal blocks, zero rows and
                                            columns, untouched elsewhere
"""
import numpy as np
import pytest

import oracle as O
import workloads as W


def _knot_integrals(n):
    """int N_i du over the open uniform knot vector of n bases: (t_{i+3} - t_i) / 3."""
    S = n - 2
    t = np.concatenate([[0, 0], np.arange(S + 1), [S, S]]).astype(float)
    return (t[3:n + 3] - t[0:n]) / 3.0


@pytest.mark.parametrize("n,L", [(8, 1.0), (16, 2.5)])
def test_lumped_mass_closed_form(n, L):
    sh = W.make_sheet(n, L, 3)
    o = O.Oracle.from_sheet(sh)
    R0 = 0.37
    m = o.lumped_mass(R0)
    h = L / (n - 2)
    ku = _knot_integrals(n)
    ref = R0 * h * h * np.outer(ku, ku)
    assert np.max(np.abs(m - ref)) < 1e-14 * R0 * L * L
    assert abs(m.sum() - R0 * L * L) < 1e-13 * R0 * L * L


def _boundary_area(rest, n_u, n_v, samples=20000):
    """Area enclosed by the rest map's boundary curve (Green's theorem, fine polyline), via the textbook
    open-uniform quadratic basis of numpy-independent closed form on each span."""
    def curve(P, s):   # quadratic B-spline curve with open uniform knots, parameter s in [0, S]
        S = len(P) - 2
        sp = np.minimum(np.floor(s).astype(int), S - 1)
        x = s - sp
        # span-local bases (uniform middle piece, modified at the two end spans)
        out = np.zeros((len(s), 2))
        for k in range(len(s)):
            i, t = sp[k], x[k]
            if S == 1:
                b = [(1 - t) ** 2, 2 * t * (1 - t), t * t]
            elif i == 0:
                b = [(1 - t) ** 2, 2 * t - 1.5 * t * t, 0.5 * t * t]
            elif i == S - 1:
                b = [0.5 * (1 - t) ** 2, -1.5 * t * t + t + 0.5, t * t]
            else:
                b = [0.5 * (1 - t) ** 2, -t * t + t + 0.5, 0.5 * t * t]
            out[k] = b[0] * P[i] + b[1] * P[i + 1] + b[2] * P[i + 2]
        return out
    s_u = np.linspace(0, n_u - 2, samples)
    s_v = np.linspace(0, n_v - 2, samples)
    pts = np.concatenate([curve(rest[0, :, :], s_u), curve(rest[:, -1, :], s_v),
                          curve(rest[-1, ::-1, :], s_u), curve(rest[::-1, 0, :], s_v)])
    x, y = pts[:, 0], pts[:, 1]
    return 0.5 * abs(np.sum(x * np.roll(y, -1) - np.roll(x, -1) * y))


def test_lumped_mass_total_curved_rest():
    n = 12
    sh = W.make_sheet(n, 1.0, 4)
    rest = W.make_curved_rest(n, n, 11)
    sh2 = W.Sheet(n, n, sh.knots_u, sh.knots_v, rest, sh.x, sh.E, sh.nu, sh.h)
    o = O.Oracle.from_sheet(sh2)
    R0 = 1.3
    area = _boundary_area(rest, n, n)
    assert abs(o.lumped_mass(R0).sum() - R0 * area) < 1e-6 * R0 * area


def test_lumped_mass_slabs_match_full():
    sh = W.make_c1()
    full = O.Oracle.from_sheet(sh).lumped_mass(1.0)
    for r0, r1 in [(0, 5), (5, 6), (6, 16)]:
        part = O.Oracle.from_sheet(sh, r0=r0, r1=r1).lumped_mass(1.0)
        assert np.array_equal(part, full[r0:r1])


def _setup(seed=1):
    sh = W.make_c1()
    o = O.Oracle.from_sheet(sh)
    rng = np.random.default_rng(seed)
    m = o.lumped_mass(0.2)
    xhat = sh.x + rng.normal(0, 2e-3, sh.x.shape)
    return sh, o, m, xhat


def test_ip_energy_closed_forms():
    sh, o, m, _ = _setup()
    dt = 1e-2
    d = np.array([1e-3, -2e-3, 5e-4])
    E0 = o.eval(sh.x, energy=True, gradient=False, hessian=False)[0]
    E = o.eval_ip(sh.x, sh.x - d, m, dt, gradient=False, hessian=False)[0]
    assert abs((E - E0) - m.sum() * d.dot(d) / (2 * dt * dt)) < 1e-12 * abs(E - E0)
    flat = sh.x.copy()
    flat[..., 2] = 0.25   # the sheet translated to height 0.25 (elastic energy unchanged)
    g = np.array([0.0, 0.0, -9.81])
    E0 = o.eval(flat, gradient=False, hessian=False)[0]
    E = o.eval_ip(flat, flat, m, dt, gravity=g, gradient=False, hessian=False)[0]
    assert abs((E - E0) - m.sum() * 9.81 * 0.25) < 1e-12 * m.sum() * 9.81 * 0.25


def test_ip_gradient_and_hessian_increments_by_differences():
    sh, o, m, xhat = _setup(2)
    dt, grav = 3e-3, np.array([0.3, -9.81, 1.2])
    x = sh.x
    def inc(xx):   # energy, gradient and Hessian of the IP terms alone
        Ee, ge, ve = o.eval(xx)
        Ei, gi, vi = o.eval_ip(xx, xhat, m, dt, grav)
        return Ei - Ee, gi - ge, vi - ve
    _, gI, vI = inc(x)
    rng = np.random.default_rng(5)
    h = 1e-4
    for _ in range(6):
        j, i, c = rng.integers(0, sh.n_v), rng.integers(0, sh.n_u), rng.integers(0, 3)
        xp, xm = x.copy(), x.copy()
        xp[j, i, c] += h
        xm[j, i, c] -= h
        fd = (inc(xp)[0] - inc(xm)[0]) / (2 * h)
        assert abs(fd - gI[j, i, c]) < 1e-7 * max(1.0, abs(gI[j, i, c]))
        gp, gm = inc(xp)[1], inc(xm)[1]
        col = (gp - gm) / (2 * h)   # column (j,i,c) of the Hessian increment: m_a/dt^2 on the diagonal only
        expect = np.zeros_like(col)
        expect[j, i, c] = m[j, i] / dt ** 2
        assert np.max(np.abs(col - expect)) < 1e-6 * m[j, i] / dt ** 2
    rp, ci = o.pattern()
    for a in range(sh.n_u * sh.n_v):
        for k in range(rp[a], rp[a + 1]):
            exp = (m.flat[a] / dt ** 2) * np.eye(3) if ci[k] == a else np.zeros((3, 3))
            assert np.allclose(vI[k], exp, rtol=1e-12, atol=1e-12 * m.max() / dt ** 2)


def test_ip_pinned_masking():
    sh, o, m, xhat = _setup(3)
    dt = 1e-2
    pinned = np.zeros((sh.n_v, sh.n_u), bool)
    pinned[-1, :] = True          # top edge
    pinned[0, 0] = True           # one corner
    E, g, v = o.eval_ip(sh.x, xhat, m, dt, (0, 0, -9.81))
    Ep, gp, vp = o.eval_ip(sh.x, xhat, m, dt, (0, 0, -9.81), pinned=pinned)
    assert Ep == E
    assert np.all(gp[pinned] == 0) and np.array_equal(gp[~pinned], g[~pinned])
    rp, ci = o.pattern()
    pf = pinned.ravel()
    for a in range(sh.n_u * sh.n_v):
        for k in range(rp[a], rp[a + 1]):
            b = ci[k]
            if pf[a] or pf[b]:
                assert np.array_equal(vp[k], np.eye(3) if a == b else np.zeros((3, 3)))
            else:
                assert np.array_equal(vp[k], v[k])


@pytest.mark.parametrize("case", ["c1", "slab", "curved"])
def test_library_host_lumped_mass_matches_oracle(case):
    """bsf_set_inertia computes the masses on the host (also for a host-only handle, device = -1); they
    equal the oracle's row-summed consistent mass to rounding."""
    import paper_2506_18867_b200 as B
    sh = W.make_c1()
    r0, r1 = (3, 9) if case == "slab" else (0, sh.n_v)
    if case == "curved":
        sh = W.Sheet(sh.n_u, sh.n_v, sh.knots_u, sh.knots_v, W.make_curved_rest(sh.n_u, sh.n_v, 2), sh.x, sh.E,
                     sh.nu, sh.h)
    s = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1, device=-1)
    s.set_inertia(0.7, 1e-3, gravity=(0, 0, -9.81))
    m = s.lumped_mass()
    ref = O.Oracle.from_sheet(sh, r0=r0, r1=r1).lumped_mass(0.7)
    assert np.max(np.abs(m - ref)) < 1e-14 * ref.max()
