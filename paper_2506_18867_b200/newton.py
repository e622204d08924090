"""One implicit-Euler time step by projected Newton on the device.

The step minimises the incremental potential (Eq. `eq:incremental_potential`)
    E(x) = E_elastic(x) + sum_a m_a/(2 dt^2) |x_a - xhat_a|^2 - sum_a m_a g.x_a,   xhat = x^n + dt v^n,
with the paper's solver structure: the per-term PSD-projected Hessian (projected Newton), a linear solve for
the search direction (here block-Jacobi PCG on the device instead of the paper's Cholesky), and a
backtracking line search on the energy; it stops when the search direction is small.
Energies, gradients, Hessians and the linear solve come from the library's kernels (bsf_eval_ip_batch,
bsf_pcg); this module sequences the calls and does the line search's vector updates (x + alpha d) and its
scalar logic with plain torch operations on the device (SURVEY §8(f) #3 is a driver around the hot path).  Pinned control points (set_inertia(pinned=...)) stay fixed:
their gradient rows are zero and their Hessian rows are identity, so the direction vanishes there.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import paper_2506_18867_b200 as B


@dataclass
class NewtonStats:
    iterations: int = 0
    pcg_iterations: list = field(default_factory=list)
    energies: list = field(default_factory=list)
    steps: list = field(default_factory=list)
    converged: bool = False


def implicit_euler_step(sheet: "B.Sheet", x, v, dt: float, flags: int = B.PROJECT_PSD, tol: float = 1e-6,
                        max_iter: int = 50, pcg_rtol: float = 1e-10, pcg_max_iter: int = 5000,
                        armijo: float = 1e-4, solver: str = "pcg"):
    """x, v: CUDA float64 [n_v, n_u, 3] (whole-sheet handle with set_inertia(...) called for this dt).
    Returns (x_new, v_new, NewtonStats).  tol: stop when max_a |d_a| <= tol * dt * (1 + max_a |v_a|)
    (the direction in units of a velocity change, as IPC-style solvers do).  solver: "pcg" (block-Jacobi PCG) or
    "chol" (the device banded Cholesky, the paper's direct solve; C2 128^2: 48 ms factor + 16 ms
    solve per Newton iteration, slower than PCG at these sizes, independent of the conditioning)."""
    import torch
    if sheet.row_begin != 0 or sheet.row_end != sheet.n_v:
        raise ValueError("implicit_euler_step needs a whole-sheet handle")
    xhat = (x + dt * v).unsqueeze(0).contiguous()
    xk = x.clone().unsqueeze(0)
    E = torch.zeros(1, dtype=torch.float64, device=x.device)
    G = torch.zeros_like(xk)
    V = torch.zeros((1, sheet.nnzb, 3, 3), dtype=torch.float64, device=x.device)
    Et = torch.zeros_like(E)
    stats = NewtonStats()
    vscale = 1.0 + float(v.abs().max())
    for it in range(max_iter):
        sheet.eval_ip_batch(xk, xhat, E, G, V, flags=flags)
        if solver == "chol":
            sheet.chol_factor(V[0])
            d = sheet.chol_solve(-G[0])
            stats.pcg_iterations.append(0)
        else:
            d, n_pcg, _ = sheet.pcg(V[0], -G[0], max_iter=pcg_max_iter, rtol=pcg_rtol)
            stats.pcg_iterations.append(n_pcg)
        e0 = float(E.item())
        stats.energies.append(e0)
        stats.iterations = it + 1
        if float(d.abs().max()) <= tol * dt * vscale:
            stats.converged = True
            break
        gd = float((G[0] * d).sum())   # directional derivative (< 0 for an SPD system)
        alpha = 1.0
        while True:
            xt = xk + alpha * d.unsqueeze(0)
            sheet.eval_ip_batch(xt, xhat, Et, None, None, flags=flags)
            # Armijo with a rounding allowance (near the minimiser E changes by less than its last bits)
            if float(Et.item()) <= e0 + armijo * alpha * gd + 1e-14 * abs(e0) or alpha < 1e-8:
                break
            alpha *= 0.5
        stats.steps.append(alpha)
        xk = xt
    x_new = xk[0]
    return x_new, (x_new - x) / dt, stats
