"""GPU: one implicit-Euler step by projected Newton (paper_2506_18867_b200/newton.py) against the same
algorithm run on the CPU oracle (oracle.eval_ip + scipy's sparse direct solve + the same backtracking line
search): both converge to the same minimiser of the incremental potential."""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle as O
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_18867_b200 as B  # noqa: E402
from paper_2506_18867_b200.newton import implicit_euler_step  # noqa: E402


def _oracle_step(sh, x, v, dt, R0, grav, pinned, tol, max_iter=50):
    o = O.Oracle.from_sheet(sh)
    m = o.lumped_mass(R0)
    rp, ci = o.pattern()
    xhat = x + dt * v
    xk = x.copy()
    vscale = 1.0 + np.abs(v).max()
    for _ in range(max_iter):
        E, g, vals = o.eval_ip(xk, xhat, m, dt, grav, pinned, flags=O.FLAG_PROJECT)
        A = sp.bsr_matrix((vals, ci, rp), shape=(3 * sh.n_u * sh.n_v,) * 2).tocsc()
        d = spla.spsolve(A, -g.reshape(-1)).reshape(g.shape)
        if np.abs(d).max() <= tol * dt * vscale:
            break
        gd = float((g * d).sum())
        alpha = 1.0
        while True:
            xt = xk + alpha * d
            Et = o.eval_ip(xt, xhat, m, dt, grav, pinned, flags=O.FLAG_PROJECT, gradient=False, hessian=False)[0]
            if Et <= E + 1e-4 * alpha * gd + 1e-14 * abs(E) or alpha < 1e-8:
                break
            alpha *= 0.5
        xk = xt
    return xk


@pytest.mark.parametrize("n", [16, 24])
@pytest.mark.parametrize("solver", ["chol", "pcg"])
def test_hanging_sheet_step_matches_oracle(n, solver):
    sh = W.make_sheet(n, 1.0, 5, n_modes=3, amp=2e-3, lam=0.3)
    R0, dt, grav = 0.2, 1e-2, np.array([0.0, 0.0, -9.81])
    pinned = np.zeros((n, n), bool)
    pinned[-1, :] = True                       # hang by the top edge
    rng = np.random.default_rng(n)
    v = rng.normal(0, 1e-2, sh.x.shape)
    v[pinned] = 0.0
    s = B.Sheet.from_sheet(sh)
    s.set_inertia(R0, dt, gravity=grav, pinned=pinned)
    x_gpu, v_gpu, st = implicit_euler_step(s, torch.from_numpy(sh.x).cuda(), torch.from_numpy(v).cuda(), dt,
                                           tol=1e-7, solver=solver)
    assert st.converged and st.iterations < 10, st
    assert all(e1 <= e0 + 1e-12 * abs(e0) for e0, e1 in zip(st.energies, st.energies[1:])), st.energies
    x_ref = _oracle_step(sh, sh.x, v, dt, R0, grav, pinned, tol=1e-7)
    xg = x_gpu.cpu().numpy()
    assert np.array_equal(xg[pinned], sh.x[pinned])            # pinned points did not move
    step = np.abs(x_ref - sh.x).max()
    assert np.abs(xg - x_ref).max() <= 1e-6 * step, (np.abs(xg - x_ref).max(), step)
