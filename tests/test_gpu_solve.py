"""GPU: linear algebra on the assembled Hessian against the oracle's matrix.

  bsf_bsr_spmv    vs scipy.sparse BSR product of the oracle's values (same pattern), 1e-13 relative
  bsf_gershgorin  contains numpy's eigenvalues of the oracle's dense matrix (small sheet)
  bsf_pcg         Newton step of the incremental potential: |b - Hx| <= rtol |b| re-measured on the host with
                  the oracle's matrix, and the solution vs scipy's sparse direct solve
"""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_18867_b200 as B  # noqa: E402


def _bsr(o, vals, n_cols):
    rp, ci = o.pattern()
    return sp.bsr_matrix((np.asarray(vals), ci, rp), shape=(3 * (len(rp) - 1), 3 * n_cols)).tocsr()


def _ip_system(sh, R0=0.15, dt=2e-3):
    o = O.Oracle.from_sheet(sh)
    m = o.lumped_mass(R0)
    rng = np.random.default_rng(3)
    xhat = sh.x + rng.normal(0, 1e-3, sh.x.shape)
    E, g, v = o.eval_ip(sh.x, xhat, m, dt, (0, 0, -9.81), flags=O.FLAG_PROJECT)
    return o, m, xhat, g, v


@pytest.mark.parametrize("case", ["c1", "c2", "slab"])
def test_spmv_matches_scipy(case):
    sh = W.make_c1() if case == "c1" else W.make_c2(state=1)
    r0, r1 = (30, 70) if case == "slab" else (0, sh.n_v)
    o = O.Oracle.from_sheet(sh, r0=r0, r1=r1)
    _, _, v = o.eval(sh.x, flags=O.FLAG_PROJECT)
    s = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1)
    rng = np.random.default_rng(9)
    xv = rng.normal(size=(sh.n_v, sh.n_u, 3))
    y = s.spmv(torch.from_numpy(v).cuda(), torch.from_numpy(np.ascontiguousarray(xv[s.x_row_begin:s.x_row_end])).cuda())
    torch.cuda.synchronize()
    ref = (_bsr(o, v, sh.n_u * sh.n_v) @ xv.reshape(-1)).reshape(r1 - r0, sh.n_u, 3)
    assert np.max(np.abs(y.cpu().numpy() - ref)) <= 1e-13 * np.max(np.abs(ref))


def test_gershgorin_contains_spectrum():
    sh = W.make_c1()
    o, m, xhat, g, v = _ip_system(sh)
    s = B.Sheet.from_sheet(sh)
    lo, hi = s.gershgorin(torch.from_numpy(v).cuda())
    lam = np.linalg.eigvalsh(_bsr(o, v, sh.n_u * sh.n_v).toarray())
    assert lo <= lam.min() * (1 + 1e-12) and lam.max() <= hi * (1 + 1e-12)
    # and the bound is a real Gershgorin bound (tight up to the disc radii): lo <= min diagonal entry
    assert lo <= np.min(np.diag(_bsr(o, v, sh.n_u * sh.n_v).toarray()))


@pytest.mark.parametrize("case", ["c1", "c2"])
def test_pcg_newton_step(case):
    sh = W.make_c1() if case == "c1" else W.make_c2(state=2)
    o, m, xhat, g, v = _ip_system(sh)
    s = B.Sheet.from_sheet(sh)
    V = torch.from_numpy(v).cuda()
    b = torch.from_numpy(-g).cuda()
    x, it, rr = s.pcg(V, b, max_iter=2000, rtol=1e-11)
    torch.cuda.synchronize()
    A = _bsr(o, v, sh.n_u * sh.n_v)
    xs = x.cpu().numpy().reshape(-1)
    res = np.linalg.norm(-g.reshape(-1) - A @ xs) / np.linalg.norm(g)
    assert rr <= 1e-11 and res <= 2e-11, (it, rr, res)
    ref = spla.spsolve(A.tocsc(), -g.reshape(-1))
    assert np.linalg.norm(xs - ref) <= 1e-8 * np.linalg.norm(ref), (it, np.linalg.norm(xs - ref) / np.linalg.norm(ref))
    assert 0 < it < 2000


def test_pcg_rejects_indefinite():
    sh = W.make_c1()
    o = O.Oracle.from_sheet(sh)
    _, g, v = o.eval(sh.x)        # no projection, no inertia: singular / indefinite
    v = v.copy()
    rp, ci = o.pattern()
    for a in range(len(rp) - 1):  # flip the sign of the diagonal blocks: certainly not SPD
        for k in range(rp[a], rp[a + 1]):
            if ci[k] == a:
                v[k] = -np.eye(3)
    s = B.Sheet.from_sheet(sh)
    with pytest.raises(B.BsfError):
        s.pcg(torch.from_numpy(v).cuda(), torch.from_numpy(np.ones_like(g)).cuda(), max_iter=50, rtol=1e-10)


def test_solve_and_ip_edge_cases():
    """b = 0 converges at once to x = 0; max_iter = 0 leaves the initial guess; invalid inertia settings and
    PCG on a slab handle are refused; an empty batch is a no-op."""
    sh = W.make_c1()
    o, m, xhat, g, v = _ip_system(sh)
    s = B.Sheet.from_sheet(sh)
    V = torch.from_numpy(v).cuda()
    zero = torch.zeros((sh.n_v, sh.n_u, 3), dtype=torch.float64, device="cuda")
    x, it, rr = s.pcg(V, zero.clone(), max_iter=100, rtol=1e-10)
    assert it == 0 and rr == 0.0 and torch.count_nonzero(x) == 0
    x0 = torch.ones_like(zero)
    x, it, rr = s.pcg(V, torch.from_numpy(-g).cuda(), x=x0.clone(), max_iter=0, rtol=1e-10)
    assert torch.equal(x, x0)
    with pytest.raises(B.BsfError):
        s.set_inertia(0.1, 0.0)
    with pytest.raises(B.BsfError):
        s.set_inertia(-1.0, 1e-3)
    slab = B.Sheet.from_sheet(sh, row_begin=4, row_end=10)
    _, _, vs = O.Oracle.from_sheet(sh, r0=4, r1=10).eval(sh.x, flags=O.FLAG_PROJECT)
    with pytest.raises(B.BsfError):
        slab.pcg(torch.from_numpy(vs).cuda(), torch.zeros((6, sh.n_u, 3), dtype=torch.float64, device="cuda"))
    s.set_inertia(0.1, 1e-3)
    X = torch.zeros((0,) + s.x_shape(), dtype=torch.float64, device="cuda")
    s.eval_ip_batch(X, torch.zeros((0, sh.n_v, sh.n_u, 3), dtype=torch.float64, device="cuda"))


def _gpu_ip_hessian(sh, R0=0.15, dt=2e-3):
    """The library's incremental-potential Hessian (PSD-projected elastic + inertia) on the device."""
    s = B.Sheet.from_sheet(sh)
    rng = np.random.default_rng(3)
    xhat = sh.x + rng.normal(0, 1e-3, sh.x.shape)
    s.set_inertia(R0, dt, gravity=np.array([0.0, 0.0, -9.81]))
    X = torch.from_numpy(sh.x).cuda().unsqueeze(0).contiguous()
    XH = torch.from_numpy(xhat).cuda().unsqueeze(0).contiguous()
    E = torch.zeros(1, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_ip_batch(X, XH, E, G, V, B.PROJECT_PSD)
    torch.cuda.synchronize()
    return s, G[0], V[0]


def _csr(s, vals):
    rp, ci = s.pattern()
    n = s.n_rows
    return sp.bsr_matrix((vals.cpu().numpy(), ci, rp), shape=(3 * n, 3 * n)).tocsr()


@pytest.mark.parametrize("case", ["c1", "c2", "c3"])
def test_chol_factor_solve_matches_scipy(case):
    """bsf_chol_factor + bsf_chol_solve (banded Cholesky on the device) on the Newton matrix of the
    incremental potential: the solution against scipy's sparse direct solve of the same matrix (1e-10 relative)
    and the residual |b - Hx| re-measured with the library's SpMV."""
    sh = {"c1": W.make_c1, "c2": lambda: W.make_c2(state=2), "c3": W.make_c3}[case]()
    s, g, v = _gpu_ip_hessian(sh)
    s.chol_factor(v)
    b = -g
    x = s.chol_solve(b)
    torch.cuda.synchronize()
    ref = spla.spsolve(_csr(s, v).tocsc(), b.cpu().numpy().reshape(-1)).reshape(x.shape)
    xn = x.cpu().numpy()
    assert np.linalg.norm(xn - ref) <= 1e-10 * np.linalg.norm(ref)
    r = b - s.spmv(v, x)
    torch.cuda.synchronize()
    assert float(r.norm() / b.norm()) <= 1e-12
    x2 = s.chol_solve(b, b.clone())   # in-place solve
    torch.cuda.synchronize()
    assert torch.equal(x2, x)


def test_chol_rejects_indefinite():
    sh = W.make_c1()
    s, g, v = _gpu_ip_hessian(sh)
    with pytest.raises(B.BsfError) as e:
        s.chol_factor(-v)
    assert e.value.status == -1 and "not positive definite" in str(e.value)
    with pytest.raises(B.BsfError):
        B.Sheet.from_sheet(sh, row_begin=0, row_end=8).chol_factor(v[:10])   # slab handles: whole sheets only


def test_neumann_split_gated_by_gershgorin():
    """(D + B) x = b by the Neumann series on the factorised D: D the incremental-potential
    Hessian, B a symmetric coupling in the same pattern (here a scaled elastic Hessian of another state, standing in
    for the off-diagonal contact Hessian, which is out of scope).  The gate bound lambda_max(B)/lambda_min(D) comes
    from Gershgorin discs: below 1 the series converges to scipy's direct solve of D + B; at or above 1 the call
    refuses (factorise D + B instead)."""
    sh = W.make_c2(state=4)
    s, g, v = _gpu_ip_hessian(sh, dt=1e-4)   # inertia-dominated D: a positive Gershgorin lower bound
    s.chol_factor(v)
    sh2 = W.make_c2(state=9)
    E2, g2, vb = s(torch.from_numpy(sh2.x).cuda(), 0)   # exact elastic Hessian of another state (symmetric)
    torch.cuda.synchronize()
    lo_d, _ = s.gershgorin(v)
    assert lo_d > 0.0
    lo_b, hi_b = s.gershgorin(vb)
    eps = 0.3 * lo_d / max(abs(lo_b), abs(hi_b))
    Bv = eps * vb
    b = -g
    x, gate, terms = s.neumann_solve(Bv, b, max_terms=200, rtol=1e-14)
    torch.cuda.synchronize()
    assert 0.0 < gate < 1.0 and abs(gate - 0.3) < 1e-9 and 1 <= terms <= 200
    ref = spla.spsolve((_csr(s, v) + _csr(s, Bv)).tocsc(), b.cpu().numpy().reshape(-1)).reshape(x.shape)
    assert np.linalg.norm(x.cpu().numpy() - ref) <= 1e-10 * np.linalg.norm(ref)
    with pytest.raises(B.BsfError) as e:
        s.neumann_solve(Bv * (4.0 / 0.3), b)
    assert e.value.status == -1 and "gate" in str(e.value)
