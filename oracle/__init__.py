"""CPU oracle (TEST INFRASTRUCTURE ONLY) — ctypes wrapper around oracle/bsf_oracle.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` leg may
import this package.  The product path (paper_2506_18867_b200) never does.

Every function here is argument marshalling; the arithmetic lives in bsf_oracle.cpp, which
cites the paper passage each step follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bsf_oracle.cpp")
# BSF_ORACLE_SANITIZE=1: an AddressSanitizer + UBSan build (liboracle_asan.so; run the process with
# LD_PRELOAD of libasan, see profiles/r02_sanitizers.md); otherwise the optimised build.
_SANITIZE = os.environ.get("BSF_ORACLE_SANITIZE") == "1"
_LIB = os.path.join(_HERE, "liboracle_asan.so" if _SANITIZE else "liboracle.so")
_lock = threading.Lock()
_lib = None

RULE_REDUCED, RULE_G2_INTERIOR, RULE_G3_FULL = 0, 1, 2
FLAG_PROJECT, FLAG_NO_MEMBRANE, FLAG_NO_BENDING, FLAG_ABS_SUM = 1, 2, 4, 8


def build(force: bool = False) -> str:
    """Compile the oracle (g++ -O3 -march=native -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        cmd = ["g++", "-std=c++17", "-O3", "-march=native", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-o", tmp, _SRC]
        if _SANITIZE:
            cmd[2:3] = ["-O1", "-g", "-fsanitize=address,undefined", "-fno-sanitize-recover=undefined",
                        "-fno-omit-frame-pointer"]
        subprocess.check_call(cmd)
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            dp, ip, vp = C.POINTER(C.c_double), C.POINTER(C.c_int32), C.c_void_p
            L.oracle_last_error.restype = C.c_char_p
            L.oracle_basis_all.argtypes = [dp, C.c_int, C.c_double, dp, dp, dp]
            L.oracle_gauss.argtypes = [C.c_int, C.c_double, C.c_double, dp, dp]
            L.oracle_rule.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, dp, dp, dp, ip, ip]
            L.oracle_material_from_young.argtypes = [C.c_double] * 5 + [dp]
            L.oracle_create.restype = vp
            L.oracle_create.argtypes = [C.c_int, C.c_int, dp, dp, dp, dp, C.c_int, C.c_int, C.c_int, C.c_int]
            L.oracle_destroy.argtypes = [vp]
            L.oracle_nnzb.restype = C.c_int64
            L.oracle_nnzb.argtypes = [vp]
            L.oracle_num_points.argtypes = [vp, ip, ip]
            L.oracle_pattern.argtypes = [vp, ip, ip]
            L.oracle_point.argtypes = [vp, C.c_int, dp, ip, ip, dp]
            L.oracle_eval.argtypes = [vp, dp, C.c_int, dp, dp, dp, C.c_int]
            L.oracle_energy_cplx.argtypes = [vp, dp, dp, C.c_int, dp, dp]
            L.oracle_gradient_cplx.argtypes = [vp, dp, dp, C.c_int, dp, dp]
            L.oracle_membrane_A.argtypes = [dp, dp, C.c_int, dp]
            L.oracle_lumped_mass.argtypes = [vp, C.c_double, dp]
            L.oracle_eval_ip.argtypes = [vp, dp, dp, dp, C.c_double, dp, C.POINTER(C.c_uint8), C.c_int, dp, dp, dp,
                                         C.c_int]
            L.oracle_contact_weights.argtypes = [vp, C.c_int, dp, dp]
            L.oracle_contact_pullback.argtypes = [vp, C.c_int, dp, C.c_int, ip, dp, dp, dp, dp]
            _lib = L
    return _lib


def _p(a, t=C.c_double):
    return a.ctypes.data_as(C.POINTER(t))


def _check(rc):
    if rc < 0:
        raise RuntimeError(f"oracle error {rc}: {lib().oracle_last_error().decode()}")
    return rc


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def basis_all(knots, x):
    knots = np.ascontiguousarray(knots, dtype=np.float64)
    n = len(knots) - 3
    N, dN, ddN = np.zeros(n), np.zeros(n), np.zeros(n)
    _check(lib().oracle_basis_all(_p(knots), len(knots), float(x), _p(N), _p(dN), _p(ddN)))
    return N, dN, ddN


def gauss(m, a, b):
    x, w = np.zeros(m), np.zeros(m)
    _check(lib().oracle_gauss(m, float(a), float(b), _p(x), _p(w)))
    return x, w


def rule(kind: int, bending: bool, Su: int, Sv: int):
    """Return (u, v, w_hat, stencils) where stencils is a list of (k,2) int arrays of (i, j)."""
    n = _check(lib().oracle_rule(kind, int(bending), Su, Sv, 0, None, None, None, None, None))
    u, v, w = np.zeros(n), np.zeros(n), np.zeros(n)
    st_n = np.zeros(n, np.int32)
    st = np.zeros(n * 18, np.int32)
    _check(lib().oracle_rule(kind, int(bending), Su, Sv, n, _p(u), _p(v), _p(w), _p(st_n, C.c_int32),
                             _p(st, C.c_int32)))
    sts = [st[k * 18:k * 18 + 2 * st_n[k]].reshape(-1, 2).copy() for k in range(n)]
    return u, v, w, sts


def material_from_young(E, nu, h, shear_E=-1.0, bend_E=-1.0) -> np.ndarray:
    mu = np.zeros(4)
    _check(lib().oracle_material_from_young(E, nu, h, shear_E, bend_E, _p(mu)))
    return mu


def membrane_A(mu4, f1, f2, project=False):
    mu4 = np.ascontiguousarray(mu4, dtype=np.float64)
    f = np.ascontiguousarray(np.concatenate([f1, f2]), dtype=np.float64)
    A = np.zeros(36)
    lib().oracle_membrane_A(_p(mu4), _p(f), int(project), _p(A))
    return A.reshape(6, 6)


class Oracle:
    """Oracle handle for one sheet (optionally one owned row slab [r0, r1) of control points)."""

    def __init__(self, n_u, n_v, knots_u, knots_v, rest_xy, mu4, mrule=RULE_REDUCED, brule=RULE_REDUCED,
                 r0=0, r1=None):
        L = lib()
        r1 = n_v if r1 is None else r1
        self.n_u, self.n_v, self.r0, self.r1 = n_u, n_v, r0, r1
        self.lo, self.hi = max(0, r0 - 2), min(n_v, r1 + 2)
        ku = np.ascontiguousarray(knots_u, dtype=np.float64)
        kv = np.ascontiguousarray(knots_v, dtype=np.float64)
        rest = np.ascontiguousarray(rest_xy, dtype=np.float64)
        mu = np.ascontiguousarray(mu4, dtype=np.float64)
        self.mu = mu
        self._h = L.oracle_create(n_u, n_v, _p(ku), _p(kv), _p(rest), _p(mu), mrule, brule, r0, r1)
        if not self._h:
            raise RuntimeError(f"oracle_create failed: {L.oracle_last_error().decode()}")
        self.nnzb = int(L.oracle_nnzb(self._h))
        nm, nb = C.c_int32(), C.c_int32()
        L.oracle_num_points(self._h, C.byref(nm), C.byref(nb))
        self.n_membrane, self.n_bending = nm.value, nb.value

    @classmethod
    def from_sheet(cls, sh, mrule=RULE_REDUCED, brule=RULE_REDUCED, r0=0, r1=None, mu=None):
        mu = material_from_young(sh.E, sh.nu, sh.h) if mu is None else mu
        return cls(sh.n_u, sh.n_v, sh.knots_u, sh.knots_v, sh.rest_xy, mu, mrule, brule, r0, r1)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                lib().oracle_destroy(h)
            except TypeError:   # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    def pattern(self):
        nrows = (self.r1 - self.r0) * self.n_u
        rp = np.zeros(nrows + 1, np.int32)
        ci = np.zeros(self.nnzb, np.int32)
        lib().oracle_pattern(self._h, _p(rp, C.c_int32), _p(ci, C.c_int32))
        return rp, ci

    def point(self, k):
        w = C.c_double()
        n = C.c_int32()
        cps = np.zeros(9, np.int32)
        coef = np.zeros(18)
        bend = _check(lib().oracle_point(self._h, k, C.byref(w), C.byref(n), _p(cps, C.c_int32), _p(coef)))
        k_ = n.value
        return dict(bending=bool(bend), w=w.value, cps=cps[:k_].copy(),
                    coef=(coef[:k_].copy() if bend else coef[:2 * k_].reshape(k_, 2).copy()))

    def _xslab(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape[0] == self.n_v and (self.lo, self.hi) != (0, self.n_v):
            x = np.ascontiguousarray(x[self.lo:self.hi])
        assert x.shape == (self.hi - self.lo, self.n_u, 3), x.shape
        return x

    def eval(self, x, flags=0, energy=True, gradient=True, hessian=True, threads=None):
        x = self._xslab(x)
        E = np.zeros(1)
        g = np.zeros((self.r1 - self.r0, self.n_u, 3)) if gradient else None
        vals = np.zeros((self.nnzb, 3, 3)) if hessian else None
        threads = max_threads() if threads is None else threads
        lib().oracle_eval(self._h, _p(x), flags, _p(E) if energy else None,
                          _p(g) if gradient else None, _p(vals) if hessian else None, threads)
        return (float(E[0]) if energy else None), g, vals

    def lumped_mass(self, R0):
        """Lumped mass of the owned control points [owned rows, n_u]: consistent M by 3x3 Gauss per span,
        row sums."""
        m = np.zeros((self.r1 - self.r0, self.n_u))
        _check(lib().oracle_lumped_mass(self._h, float(R0), _p(m)))
        return m

    def eval_ip(self, x, xhat, m, dt, gravity=(0.0, 0.0, 0.0), pinned=None, flags=0, energy=True, gradient=True,
                hessian=True, threads=None):
        """Incremental potential: elastic + sum m/(2dt^2)|x-xhat|^2 - sum m g.x, with
        pinned control points masked (pinned: bool [n_v, n_u] over all rows, or None)."""
        x = self._xslab(x)
        xhat = np.ascontiguousarray(xhat, dtype=np.float64).reshape(self.r1 - self.r0, self.n_u, 3)
        m = np.ascontiguousarray(m, dtype=np.float64).reshape(self.r1 - self.r0, self.n_u)
        grav = np.ascontiguousarray(gravity, dtype=np.float64)
        pin = None if pinned is None else np.ascontiguousarray(pinned, dtype=np.uint8).reshape(self.n_v, self.n_u)
        E = np.zeros(1)
        g = np.zeros((self.r1 - self.r0, self.n_u, 3)) if gradient else None
        vals = np.zeros((self.nnzb, 3, 3)) if hessian else None
        threads = max_threads() if threads is None else threads
        _check(lib().oracle_eval_ip(self._h, _p(x), _p(xhat), _p(m), float(dt), _p(grav),
                                    None if pin is None else pin.ctypes.data_as(C.POINTER(C.c_uint8)), flags,
                                    _p(E) if energy else None, _p(g) if gradient else None,
                                    _p(vals) if hessian else None, threads))
        return (float(E[0]) if energy else None), g, vals

    def contact_weights(self, uv):
        """Dense weights W [n_vert, n_v * n_u] of the contact-mesh vertices at parametric points uv [n_vert, 2]
        (x^alpha = W[alpha] @ C)."""
        uv = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
        W = np.zeros((len(uv), self.n_u * self.n_v))
        _check(lib().oracle_contact_weights(self._h, len(uv), _p(uv), _p(W)))
        return W

    def contact_pullback(self, uv, verts, H, g=None):
        """Chain rule of the contact barrier to the control points: pairs verts [n, 4] (-1 = no
        DOFs), Hessians H [n, 12, 12], gradients g [n, 12] -> dense Hcp [3 n_cp, 3 n_cp] and gcp [n_v, n_u, 3]."""
        uv = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
        verts = np.ascontiguousarray(verts, dtype=np.int32).reshape(-1, 4)
        H = np.ascontiguousarray(H, dtype=np.float64).reshape(-1, 12, 12)
        n3 = 3 * self.n_u * self.n_v
        Hcp = np.zeros((n3, n3))
        gcp = np.zeros((self.n_v, self.n_u, 3))
        gg = None if g is None else np.ascontiguousarray(g, dtype=np.float64).reshape(-1, 12)
        _check(lib().oracle_contact_pullback(self._h, len(uv), _p(uv), len(verts), _p(verts, C.c_int32), _p(H),
                                             None if gg is None else _p(gg), _p(Hcp), _p(gcp)))
        return Hcp, (gcp if g is not None else None)

    def energy_cplx(self, x_re, x_im, flags=0):
        x_re, x_im = self._xslab(x_re), self._xslab(x_im)
        er, ei = C.c_double(), C.c_double()
        lib().oracle_energy_cplx(self._h, _p(x_re), _p(x_im), flags, C.byref(er), C.byref(ei))
        return complex(er.value, ei.value)

    def gradient_cplx(self, x_re, x_im, flags=0):
        x_re, x_im = self._xslab(x_re), self._xslab(x_im)
        shape = (self.r1 - self.r0, self.n_u, 3)
        gr, gi = np.zeros(shape), np.zeros(shape)
        lib().oracle_gradient_cplx(self._h, _p(x_re), _p(x_im), flags, _p(gr), _p(gi))
        return gr + 1j * gi

    def dense_hessian(self, x, flags=0):
        """Dense 3N x 3N Hessian (owned rows x all columns) from the BSR output (tiny grids)."""
        _, _, vals = self.eval(x, flags, energy=False, gradient=False)
        rp, ci = self.pattern()
        N = self.n_u * self.n_v
        nrows = len(rp) - 1
        H = np.zeros((3 * nrows, 3 * N))
        for a in range(nrows):
            for k in range(rp[a], rp[a + 1]):
                b = ci[k]
                H[3 * a:3 * a + 3, 3 * b:3 * b + 3] = vals[k]
        return H
