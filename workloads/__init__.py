"""Seeded synthetic inputs for the B-spline cloth assembly path.

This module is shared by the CPU oracle tests and the CUDA path. It holds NO arithmetic of the
method (no basis functions, quadrature, energies or derivatives): it only builds knot vectors,
rest control grids and deformed control-point positions from seeded random numbers, following
the recipe in SURVEY.md §8(d) / DESIGN.md §"Input recipe".

Stand-ins: the paper's scenes (Table 1) are its own assets and are not
available; these synthetic sheets stand in for them.  C3 takes the paper's largest scene size
(~51K control points).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

__all__ = [
    "Sheet", "open_uniform_knots", "greville_grid", "wrinkle_field", "random_rotation",
    "make_config", "make_c1", "make_c2", "make_c3", "make_c4", "make_c5", "make_sheet",
    "CONFIG_SEEDS",
]

CONFIG_SEEDS = {"C1": 1001, "C2": 1002, "C3": 1003, "C4": 1004, "C5": 1005}


@dataclasses.dataclass
class Sheet:
    """One sheet: parametric knots, rest (material) grid, deformed (world) grid, material."""
    n_u: int
    n_v: int
    knots_u: np.ndarray      # [n_u + 3] f64
    knots_v: np.ndarray      # [n_v + 3] f64
    rest_xy: np.ndarray      # [n_v, n_u, 2] f64, material control points X^alpha
    x: np.ndarray            # [n_v, n_u, 3] f64, world control points C^alpha
    E: float                 # Young's modulus (Pa)
    nu: float                # Poisson ratio
    h: float                 # thickness (m)
    name: str = ""

    @property
    def spans(self) -> int:
        return (self.n_u - 2) * (self.n_v - 2)


def open_uniform_knots(n: int) -> np.ndarray:
    """Open uniform integer knot vector for n quadratic control points:
    (0,0,0,1,...,S-1,S,S,S), S = n-2."""
    S = n - 2
    if S < 1:
        raise ValueError("need n >= 3 control points")
    return np.concatenate([[0.0, 0.0], np.arange(0, S + 1, dtype=np.float64), [S, S]]).astype(np.float64)


def greville_grid(n_u: int, n_v: int, Lx: float, Ly: float | None = None) -> np.ndarray:
    """Flat Lx x Ly rest sheet with control points at the Greville abscissae of the knots
    (reading Q7): X_ij = (Lx*g_i/S_u, Ly*g_j/S_v), g_i = (xi_{i+1}+xi_{i+2})/2."""
    Ly = Lx if Ly is None else Ly
    ku, kv = open_uniform_knots(n_u), open_uniform_knots(n_v)
    gu = 0.5 * (ku[1:n_u + 1] + ku[2:n_u + 2]) / (n_u - 2)
    gv = 0.5 * (kv[1:n_v + 1] + kv[2:n_v + 2]) / (n_v - 2)
    X = np.empty((n_v, n_u, 2), dtype=np.float64)
    X[:, :, 0] = Lx * gu[None, :]
    X[:, :, 1] = Ly * gv[:, None]
    return X


def wrinkle_field(rng: np.random.Generator, XY: np.ndarray, n_modes: int, amp, lam) -> np.ndarray:
    """Sum of sinusoidal modes A_m sin(2 pi d_m.X / lambda_m + phi_m) evaluated at XY[...,2].
    amp / lam: callables rng->value or scalars."""
    z = np.zeros(XY.shape[:-1], dtype=np.float64)
    for _ in range(n_modes):
        A = amp(rng) if callable(amp) else float(amp)
        L = lam(rng) if callable(lam) else float(lam)
        th = rng.uniform(0.0, 2.0 * math.pi)
        ph = rng.uniform(0.0, 2.0 * math.pi)
        d = np.array([math.cos(th), math.sin(th)])
        z += A * np.sin(2.0 * math.pi * (XY @ d) / L + ph)
    return z


def random_rotation(rng: np.random.Generator) -> np.ndarray:
    """Uniformly distributed rotation matrix (normalised Gaussian quaternion)."""
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def _embed(X: np.ndarray) -> np.ndarray:
    Y = np.zeros(X.shape[:-1] + (3,), dtype=np.float64)
    Y[..., :2] = X
    return Y


def make_sheet(n: int, L: float, seed: int, *, noise: float = 0.0, n_modes: int = 0,
               amp=0.0, lam=0.1, stretch: float = 1.0, rigid: bool = False,
               E: float = 1e5, nu: float = 0.3, h: float = 3e-4, name: str = "") -> Sheet:
    rng = np.random.default_rng(seed)
    X = greville_grid(n, n, L)
    Y = _embed(X)
    Y[..., :2] = stretch * X
    if n_modes:
        Y[..., 2] += wrinkle_field(rng, X, n_modes, amp, lam)
    if noise:
        Y += rng.normal(0.0, noise, size=Y.shape)
    if rigid:
        R = random_rotation(rng)
        c = np.array([0.5 * L, 0.5 * L, 0.0])
        t = rng.normal(0.0, 0.1, size=3)
        Y = (Y - c) @ R.T + c + t
    k = open_uniform_knots(n)
    return Sheet(n, n, k, k.copy(), X, np.ascontiguousarray(Y), E, nu, h, name)


def make_c1(seed: int = CONFIG_SEEDS["C1"]) -> Sheet:
    """C1: 16x16 cps, flat 1 m square, rest + N(0, 1e-3^2) on all coordinates, E=1e5."""
    return make_sheet(16, 1.0, seed, noise=1e-3, name="C1")


def make_c2(state: int = 0, seed0: int = 2001) -> Sheet:
    """C2: 128x128, 8 wrinkle modes (A=5e-3, lambda~U(0.05,0.3)) + rigid rotation/translation.
    State k uses seed 2001+k (100 states)."""
    return make_sheet(128, 1.0, seed0 + state, n_modes=8, amp=5e-3,
                      lam=lambda r: r.uniform(0.05, 0.3), rigid=True, name="C2")


def make_c3(E: float = 1e5, seed: int = CONFIG_SEEDS["C3"]) -> Sheet:
    """C3: 226x226 (~51K cps), flat 2 m square stretched 5% biaxially, 8 modes A=1e-2."""
    return make_sheet(226, 2.0, seed, n_modes=8, amp=1e-2, lam=lambda r: r.uniform(0.05, 0.5),
                      stretch=1.05, E=E, name="C3")


def _loguniform(lo, hi):
    return lambda r: float(math.exp(r.uniform(math.log(lo), math.log(hi))))


def make_c4(seed: int = CONFIG_SEEDS["C4"], n: int = 1024) -> Sheet:
    """C4: 1024x1024 (~1M cps), L=4 m, 32 multi-scale modes (A log-U[1e-3,2e-2],
    lambda log-U[0.02,2])."""
    return make_sheet(n, 4.0, seed, n_modes=32, amp=_loguniform(1e-3, 2e-2),
                      lam=_loguniform(0.02, 2.0), name="C4")


def make_c5(seed: int = CONFIG_SEEDS["C5"], count: int = 64, n: int = 256) -> list[Sheet]:
    """C5: batch of 64 independent 256x256 sheets with per-sheet L, E, nu."""
    rng = np.random.default_rng(seed)
    out = []
    for s in range(count):
        L = float(rng.uniform(0.5, 2.0))
        E = float(math.exp(rng.uniform(math.log(1e4), math.log(1e6))))
        nu = float(rng.uniform(0.2, 0.45))
        sub = int(rng.integers(0, 2**31 - 1))
        out.append(make_sheet(n, L, sub, n_modes=8, amp=5e-3,
                              lam=lambda r: r.uniform(0.05, 0.3), E=E, nu=nu, name=f"C5[{s}]"))
    return out


def make_curved_rest(n_u: int, n_v: int, seed: int, L: float = 1.0, bend: float = 0.08) -> np.ndarray:
    """A non-affine (curved) rest grid for the general inverse-map path: Greville grid plus a
    smooth in-plane displacement small enough to keep the map injective."""
    rng = np.random.default_rng(seed)
    X = greville_grid(n_u, n_v, L)
    a = rng.uniform(-bend, bend, size=4) * L
    s, t = X[..., 0] / L, X[..., 1] / L
    X = X.copy()
    X[..., 0] += a[0] * np.sin(math.pi * t) * s + a[1] * s * s
    X[..., 1] += a[2] * np.sin(math.pi * s) * t + a[3] * t * s
    return X


def make_config(name: str, **kw):
    return {"C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5}[name](**kw)


@dataclasses.dataclass
class ContactSet:
    """Synthetic contact inputs for the pullback: the embedded mesh's vertex parameters uv
    [n_vert, 2] and the active pairs' vertex slots verts [n, 4] (-1 = an obstacle vertex without DOFs), barrier
    Hessians H [n, 12, 12] (symmetric PSD) and gradients g [n, 12]."""
    uv: np.ndarray
    verts: np.ndarray
    H: np.ndarray
    g: np.ndarray


def make_contact(sh: Sheet, res: int, n_pairs: int, seed: int, obstacle_frac: float = 0.5,
                 scale: float = 1.0) -> ContactSet:
    """The contact mesh of a cloth sheet: a regular triangle mesh with `res` vertices per knot span along each
    parameter direction (vertex params on a grid, so some lie exactly on knot lines), as when the sheet is
    tessellated for collision.  Pairs are local, like proximity pairs: self-contact pairs
    (edge-edge / point-triangle) take 4 vertices within a few mesh steps; a fraction are cloth-vertex vs obstacle
    (point-triangle with the triangle on a static obstacle: 3 slots -1), as for a sheet falling on a cube."""
    rng = np.random.default_rng(seed)
    Su, Sv = sh.n_u - 2, sh.n_v - 2
    mu, mv = Su * res + 1, Sv * res + 1
    gu, gv = np.meshgrid(np.linspace(0.0, Su, mu), np.linspace(0.0, Sv, mv))
    uv = np.stack([gu.reshape(-1), gv.reshape(-1)], axis=1)
    n_vert = len(uv)
    a = rng.integers(0, n_vert, n_pairs)
    ia, ja = a % mu, a // mu
    verts = np.empty((n_pairs, 4), np.int64)
    verts[:, 0] = a
    for s in range(1, 4):
        di, dj = rng.integers(-3, 4, n_pairs), rng.integers(-3, 4, n_pairs)
        verts[:, s] = np.clip(ja + dj, 0, mv - 1) * mu + np.clip(ia + di, 0, mu - 1)
    n_obs = int(round(obstacle_frac * n_pairs))
    obs = rng.permutation(n_pairs)[:n_obs]
    verts[obs, 1:] = -1
    A = rng.normal(size=(n_pairs, 12, 12))
    H = scale * (A @ A.transpose(0, 2, 1)) / 12.0
    g = scale * rng.normal(size=(n_pairs, 12))
    return ContactSet(uv, verts.astype(np.int32), H, g)
