"""B200-native FP64 assembly of quadratic B-spline cloth energies (arXiv 2506.18867).

Thin ctypes binding over libbsfem.so (include/bsfem.h).  Argument marshalling only: every step of
the hot path runs in the library's CUDA kernels.  There is NO CPU fallback — if the extension is
missing or no CUDA device is present the compute calls raise.

PyTorch is used only for device memory and streams.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

__all__ = ["Sheet", "Material", "material_from_young", "affine_params", "lib", "RULE_REDUCED", "RULE_G2_INTERIOR",
           "RULE_G3_FULL", "PROJECT_PSD", "NO_MEMBRANE", "NO_BENDING", "GENERIC_PATH", "TILE_ONLY", "BsfError"]

RULE_REDUCED, RULE_G2_INTERIOR, RULE_G3_FULL = 0, 1, 2
PROJECT_PSD, NO_MEMBRANE, NO_BENDING, GENERIC_PATH, TILE_ONLY = 1, 2, 4, 8, 16
ASYNC_STAGE = 32   # eval_all_batch_host: upload waits only for the last call that read the same stage

_STATUS = {0: "OK", -1: "INVALID_ARG", -2: "KNOTS", -3: "TOO_SMALL", -4: "DEGENERATE_GEOMETRY",
           -5: "SINGULAR_STRETCH", -6: "CUDA", -7: "OOM", -8: "NCCL", -9: "NO_DEVICE"}

SYMBOLS = ["bsf_material_from_young", "bsf_create", "bsf_destroy", "bsf_set_material", "bsf_get_sizes",
           "bsf_get_pattern", "bsf_eval_all_batch", "bsf_eval_all_batch_params", "bsf_eval_energy", "bsf_eval_gradient", "bsf_assemble_hessian", "bsf_eval_all",
           "bsf_halo_exchange", "bsf_nccl_get_unique_id", "bsf_nccl_comm_init", "bsf_nccl_comm_destroy",
           "bsf_allreduce_sum", "bsf_get_core_rect", "bsf_eval_all_batch_host", "bsf_set_inertia",
           "bsf_get_lumped_mass", "bsf_eval_ip_batch", "bsf_bsr_spmv", "bsf_gershgorin", "bsf_pcg",
           "bsf_eval_all_slab", "bsf_set_kernel_timing", "bsf_get_kernel_timing",
           "bsf_last_launch_count", "bsf_poll_status", "bsf_affine_params", "bsf_halo_plan", "bsf_chol_factor",
           "bsf_chol_solve", "bsf_neumann_solve", "bsf_contact_mesh", "bsf_contact_positions",
           "bsf_contact_assemble", "bsf_contact_get", "bsf_contact_neumann_solve", "bsf_last_error"]


class BsfError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"bsf error {status} ({_STATUS.get(status, '?')}): {msg}")
        self.status = status


class Material(C.Structure):
    _fields_ = [("mu_st1", C.c_double), ("mu_st2", C.c_double), ("mu_sh", C.c_double), ("mu_bd", C.c_double)]

    def as_array(self):
        return np.array([self.mu_st1, self.mu_st2, self.mu_sh, self.mu_bd])


_lib = None


def lib():
    """Load (building in-tree if stale) libbsfem.so; raises if it cannot be built/loaded."""
    global _lib
    if _lib is None:
        path = _build.LIB
        if not os.path.exists(path) or os.environ.get("BSF_REBUILD", "1") == "1":
            path = _build.build()
        L = C.CDLL(path)
        dp, vp, ip = C.POINTER(C.c_double), C.c_void_p, C.POINTER(C.c_int32)
        i64p = C.POINTER(C.c_int64)
        L.bsf_last_error.restype = C.c_char_p
        L.bsf_material_from_young.argtypes = [C.c_double] * 5 + [C.POINTER(Material)]
        L.bsf_create.argtypes = [C.c_int, C.c_int, dp, dp, dp, C.POINTER(Material), C.c_int, C.c_int, C.c_int,
                                 C.c_int, C.c_int, C.POINTER(vp)]
        L.bsf_destroy.argtypes = [vp]
        L.bsf_set_material.argtypes = [vp, C.POINTER(Material)]
        L.bsf_get_sizes.argtypes = [vp, i64p, i64p, i64p, i64p]
        L.bsf_get_pattern.argtypes = [vp, ip, ip]
        L.bsf_eval_all.argtypes = [vp, vp, vp, vp, vp, C.c_int, vp]
        L.bsf_eval_all_batch.argtypes = [vp, C.c_int, vp, C.c_int64, vp, vp, C.c_int64, vp, C.c_int64, C.c_int, vp]
        L.bsf_eval_all_batch_params.argtypes = [vp, C.c_int, vp, C.c_int64, vp, vp, vp, C.c_int64, vp, C.c_int64,
                                                C.c_int, vp]
        L.bsf_eval_energy.argtypes = [vp, vp, vp, C.c_int, vp]
        L.bsf_eval_gradient.argtypes = [vp, vp, vp, C.c_int, vp]
        L.bsf_assemble_hessian.argtypes = [vp, vp, vp, C.c_int, vp]
        L.bsf_halo_exchange.argtypes = [vp, vp, vp, C.c_int, C.c_int, vp]
        L.bsf_nccl_get_unique_id.argtypes = [vp]
        L.bsf_nccl_comm_init.argtypes = [C.c_int, vp, C.c_int, C.c_int, C.POINTER(vp)]
        L.bsf_nccl_comm_destroy.argtypes = [vp]
        L.bsf_allreduce_sum.argtypes = [vp, C.c_int64, vp, vp]
        L.bsf_last_launch_count.argtypes = [vp]
        L.bsf_get_core_rect.argtypes = [vp, ip]
        L.bsf_eval_all_batch_host.argtypes = [vp, C.c_int, vp, C.c_int64, vp, vp, vp, vp, vp, C.c_int64, vp,
                                              C.c_int64, C.c_int, C.c_int, vp]
        L.bsf_set_inertia.argtypes = [vp, C.c_double, C.c_double, dp, C.POINTER(C.c_uint8)]
        L.bsf_get_lumped_mass.argtypes = [vp, dp]
        L.bsf_eval_ip_batch.argtypes = [vp, C.c_int, vp, C.c_int64, vp, C.c_int64, vp, vp, vp, C.c_int64, vp,
                                        C.c_int64, C.c_int, vp]
        L.bsf_set_kernel_timing.argtypes = [vp, C.c_int]
        L.bsf_get_kernel_timing.argtypes = [vp, C.POINTER(C.c_float), C.POINTER(C.c_float), C.c_int]
        L.bsf_eval_all_slab.argtypes = [vp, vp, vp, C.c_int, C.c_int, vp, vp, vp, C.c_int, vp]
        L.bsf_bsr_spmv.argtypes = [vp, vp, vp, vp, vp]
        L.bsf_gershgorin.argtypes = [vp, vp, dp, dp, vp]
        L.bsf_pcg.argtypes = [vp, vp, vp, vp, C.c_int, C.c_double, C.POINTER(C.c_int), dp, vp]
        L.bsf_poll_status.argtypes = [vp]
        L.bsf_chol_factor.argtypes = [vp, vp, vp]
        L.bsf_chol_solve.argtypes = [vp, vp, vp, vp]
        L.bsf_neumann_solve.argtypes = [vp, vp, vp, vp, C.c_int, C.c_double, dp, C.POINTER(C.c_int), vp]
        L.bsf_halo_plan.argtypes = [vp, C.c_int, C.c_int, i64p]
        L.bsf_contact_mesh.argtypes = [vp, C.c_int, dp]
        L.bsf_contact_positions.argtypes = [vp, vp, vp, vp]
        L.bsf_contact_assemble.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp, i64p, vp]
        L.bsf_contact_get.argtypes = [vp, vp, vp, vp, vp]
        L.bsf_contact_neumann_solve.argtypes = [vp, vp, vp, C.c_int, C.c_double, dp, C.POINTER(C.c_int), vp]
        L.bsf_affine_params.argtypes = [C.c_int, C.c_int, dp, C.POINTER(Material), dp]
        for s in SYMBOLS:
            getattr(L, s).restype = C.c_int if s not in ("bsf_last_error",) else C.c_char_p
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise BsfError(rc, lib().bsf_last_error().decode())


def material_from_young(E, nu, h, shear_E=-1.0, bend_E=-1.0) -> Material:
    m = Material()
    _check(lib().bsf_material_from_young(E, nu, h, shear_E, bend_E, C.byref(m)))
    return m


def _dp(a):
    return np.ascontiguousarray(a, dtype=np.float64).ctypes.data_as(C.POINTER(C.c_double))


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return C.c_void_p(t.data_ptr())


def _hptr(t):
    """Host tensor pointer (contiguous CPU float64; page-locked for asynchronous copies)."""
    if t is None:
        return None
    if t.is_cuda or not t.is_contiguous():
        raise ValueError("expected a contiguous CPU tensor")
    return C.c_void_p(t.data_ptr())


def _item(t):
    """Elements per batch item of a [B, ...] tensor (0 if None; valid for B == 0)."""
    if t is None:
        return 0
    n = 1
    for d in t.shape[1:]:
        n *= int(d)
    return n


def _stream(stream):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def affine_params(rest_xy, material) -> np.ndarray:
    """Per-item parameters of bsf_eval_all_batch_params (G00 G01 G10 G11 det J mu_st1 mu_st2 mu_sh mu_bd)
    of a flat affine rest sheet rest_xy [n_v, n_u, 2], computed by the library (bsf_affine_params)."""
    rest = np.ascontiguousarray(rest_xy, dtype=np.float64)
    if rest.ndim != 3 or rest.shape[2] != 2:
        raise ValueError("rest_xy must be [n_v, n_u, 2]")
    if not isinstance(material, Material):
        material = Material(*[float(v) for v in material])
    out = np.zeros(9)
    _check(lib().bsf_affine_params(rest.shape[1], rest.shape[0], rest.ctypes.data_as(C.POINTER(C.c_double)),
                                   C.byref(material), out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


class Sheet:
    """Handle for one sheet (or one owned row slab [row_begin, row_end) of control points)."""

    def __init__(self, n_u, n_v, knots_u, knots_v, rest_xy, material, membrane_rule=RULE_REDUCED,
                 bending_rule=RULE_REDUCED, row_begin=0, row_end=None, device=0):
        L = lib()
        row_end = n_v if row_end is None else row_end
        if not isinstance(material, Material):
            material = Material(*[float(v) for v in material])
        self.n_u, self.n_v, self.row_begin, self.row_end = n_u, n_v, row_begin, row_end
        self.x_row_begin, self.x_row_end = max(0, row_begin - 2), min(n_v, row_end + 2)
        self.device = device
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (knots_u, knots_v, rest_xy)]
        h = C.c_void_p()
        _check(L.bsf_create(n_u, n_v, self._keep[0].ctypes.data_as(C.POINTER(C.c_double)),
                            self._keep[1].ctypes.data_as(C.POINTER(C.c_double)),
                            self._keep[2].ctypes.data_as(C.POINTER(C.c_double)), C.byref(material),
                            membrane_rule, bending_rule, row_begin, row_end, device, C.byref(h)))
        self._h = h
        a, b, c, d = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(L.bsf_get_sizes(h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        self.n_rows, self.nnzb, self.n_membrane, self.n_bending = a.value, b.value, c.value, d.value
        self._pattern = None

    @classmethod
    def from_sheet(cls, sh, membrane_rule=RULE_REDUCED, bending_rule=RULE_REDUCED, row_begin=0, row_end=None,
                   device=0, material=None):
        mat = material_from_young(sh.E, sh.nu, sh.h) if material is None else material
        return cls(sh.n_u, sh.n_v, sh.knots_u, sh.knots_v, sh.rest_xy, mat, membrane_rule, bending_rule,
                   row_begin, row_end, device)

    def close(self):
        if getattr(self, "_h", None):
            try:
                lib().bsf_destroy(self._h)
            except TypeError:   # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    __del__ = close

    def set_material(self, material):
        if not isinstance(material, Material):
            material = Material(*[float(v) for v in material])
        _check(lib().bsf_set_material(self._h, C.byref(material)))

    def pattern(self):
        """(row_ptr int32 [n_rows+1], col_idx int32 [nnzb]) as numpy arrays (host)."""
        if self._pattern is None:
            rp = np.zeros(self.n_rows + 1, np.int32)
            ci = np.zeros(self.nnzb, np.int32)
            _check(lib().bsf_get_pattern(self._h, rp.ctypes.data_as(C.POINTER(C.c_int32)),
                                         ci.ctypes.data_as(C.POINTER(C.c_int32))))
            self._pattern = (rp, ci)
        return self._pattern

    def x_shape(self):
        return (self.x_row_end - self.x_row_begin, self.n_u, 3)

    def alloc_outputs(self, energy=True, gradient=True, hessian=True):
        import torch
        dev = torch.device("cuda", self.device)
        E = torch.zeros(1, dtype=torch.float64, device=dev) if energy else None
        g = torch.zeros((self.row_end - self.row_begin, self.n_u, 3), dtype=torch.float64, device=dev) if gradient else None
        v = torch.zeros((self.nnzb, 3, 3), dtype=torch.float64, device=dev) if hessian else None
        return E, g, v

    def eval_all(self, x, energy=None, grad=None, vals=None, flags=0, stream=None):
        """Enqueue the fused E/g/H pass on `stream` (default: torch's current stream).  Outputs are
        caller-owned CUDA tensors (None to skip)."""
        if tuple(x.shape) != self.x_shape() or x.dtype.itemsize != 8:
            raise ValueError(f"x must be float64 of shape {self.x_shape()}")
        _check(lib().bsf_eval_all(self._h, _ptr(x), _ptr(energy), _ptr(grad), _ptr(vals), int(flags),
                                  _stream(stream)))

    def eval_all_batch(self, x, energy=None, grad=None, vals=None, flags=0, stream=None):
        """Batched pass: x [B, *x_shape()], energy [B], grad [B, rows, n_u, 3], vals [B, nnzb, 3, 3]
        (contiguous CUDA float64; any output may be None)."""
        B = x.shape[0]
        if tuple(x.shape[1:]) != self.x_shape():
            raise ValueError(f"x must be [B, {self.x_shape()}]")
        gs = _item(grad)
        vs = _item(vals)
        _check(lib().bsf_eval_all_batch(self._h, int(B), _ptr(x), _item(x), _ptr(energy), _ptr(grad), gs,
                                        _ptr(vals), vs, int(flags), _stream(stream)))

    def set_inertia(self, areal_density, dt, gravity=None, pinned=None):
        """Incremental-potential terms (Q13/Q14): areal density R0, time step dt, gravity (3,)
        and an optional pinned mask (bool [n_v, n_u] over all rows).  Works on host-only handles."""
        g = None if gravity is None else np.ascontiguousarray(gravity, dtype=np.float64)
        pin = None if pinned is None else np.ascontiguousarray(pinned, dtype=np.uint8).reshape(self.n_v, self.n_u)
        _check(lib().bsf_set_inertia(self._h, float(areal_density), float(dt),
                                     None if g is None else g.ctypes.data_as(C.POINTER(C.c_double)),
                                     None if pin is None else pin.ctypes.data_as(C.POINTER(C.c_uint8))))
        self._ip_keep = (g, pin)

    def lumped_mass(self):
        """Lumped masses of the owned control points (numpy [rows, n_u]) of the last set_inertia."""
        m = np.zeros((self.row_end - self.row_begin, self.n_u))
        _check(lib().bsf_get_lumped_mass(self._h, m.ctypes.data_as(C.POINTER(C.c_double))))
        return m

    def eval_ip_batch(self, x, xhat, energy=None, grad=None, vals=None, flags=0, stream=None, params=None):
        """Incremental potential for a batch: x [B, *x_shape()], xhat [B, rows, n_u, 3] (CUDA float64);
        outputs as eval_all_batch."""
        B = x.shape[0]
        if tuple(x.shape[1:]) != self.x_shape() or tuple(xhat.shape) != (B, self.row_end - self.row_begin, self.n_u, 3):
            raise ValueError("x must be [B, *x_shape()] and xhat [B, rows, n_u, 3]")
        gs = _item(grad)
        vs = _item(vals)
        _check(lib().bsf_eval_ip_batch(self._h, int(B), _ptr(x), _item(x), _ptr(xhat), _item(xhat),
                                       _ptr(params), _ptr(energy), _ptr(grad), gs, _ptr(vals), vs, int(flags),
                                       _stream(stream)))

    def eval_all_slab(self, x, energy=None, grad=None, vals=None, comm=None, rank=0, nranks=1, flags=0, stream=None):
        """Halo exchange (NCCL communicator handle `comm`, nranks > 1) overlapped with the assembly of the
        interior rows; outputs as eval_all."""
        _check(lib().bsf_eval_all_slab(self._h, _ptr(x), comm, int(rank), int(nranks), _ptr(energy), _ptr(grad),
                                       _ptr(vals), int(flags), _stream(stream)))

    def set_kernel_timing(self, ncalls):
        """Record CUDA events around k_core / k_band in each of the next calls (ring of `ncalls`)."""
        _check(lib().bsf_set_kernel_timing(self._h, int(ncalls)))

    def kernel_timing(self, n):
        """(core_ms, band_ms) lists of the last min(n, recorded) calls (synchronises)."""
        c, b = (C.c_float * max(n, 1))(), (C.c_float * max(n, 1))()
        k = lib().bsf_get_kernel_timing(self._h, c, b, int(n))
        return list(c[:k]), list(b[:k])

    def spmv(self, vals, x, y=None, stream=None):
        """y = H x with the BSR values `vals` [nnzb, 3, 3]; x in the position layout (x_shape()), y [rows, n_u, 3]."""
        import torch
        if y is None:
            y = torch.empty((self.row_end - self.row_begin, self.n_u, 3), dtype=torch.float64, device=x.device)
        _check(lib().bsf_bsr_spmv(self._h, _ptr(vals), _ptr(x), _ptr(y), _stream(stream)))
        return y

    def gershgorin(self, vals, stream=None):
        """(lo, hi): the spectrum of H lies in [lo, hi] (Gershgorin discs of the scalar rows)."""
        lo, hi = C.c_double(), C.c_double()
        _check(lib().bsf_gershgorin(self._h, _ptr(vals), C.byref(lo), C.byref(hi), _stream(stream)))
        return lo.value, hi.value

    def pcg(self, vals, b, x=None, max_iter=1000, rtol=1e-10, stream=None):
        """Block-Jacobi PCG for H x = b (whole-sheet handle, SPD H); returns (x, iterations, relative residual)."""
        import torch
        x = torch.zeros_like(b) if x is None else x
        it, rr = C.c_int(), C.c_double()
        _check(lib().bsf_pcg(self._h, _ptr(vals), _ptr(b), _ptr(x), int(max_iter), float(rtol), C.byref(it),
                             C.byref(rr), _stream(stream)))
        return x, it.value, rr.value

    def chol_factor(self, vals, stream=None):
        """Banded Cholesky of the SPD matrix with BSR values `vals` [nnzb, 3, 3] (whole-sheet handle); synchronises."""
        _check(lib().bsf_chol_factor(self._h, _ptr(vals), _stream(stream)))

    def chol_solve(self, b, x=None, stream=None):
        """x = D^-1 b with the last factorisation; b, x [n_v, n_u, 3] (CUDA float64)."""
        import torch
        x = torch.empty_like(b) if x is None else x
        _check(lib().bsf_chol_solve(self._h, _ptr(b), _ptr(x), _stream(stream)))
        return x

    def neumann_solve(self, vals_B, b, x=None, max_terms=100, rtol=1e-13, stream=None):
        """(D + B) x = b by the Gershgorin-gated Neumann series on the factorised D; returns
        (x, gate bound, terms).  Raises BsfError(INVALID_ARG) if the gate bound is >= 1."""
        import torch
        x = torch.empty_like(b) if x is None else x
        g, t = C.c_double(), C.c_int()
        _check(lib().bsf_neumann_solve(self._h, _ptr(vals_B), _ptr(b), _ptr(x), int(max_terms), float(rtol),
                                       C.byref(g), C.byref(t), _stream(stream)))
        return x, g.value, t.value

    # ---- contact pullback (Alg. 1)
    def contact_mesh(self, uv):
        """Embed a contact mesh: vertex parameters uv [n_vert, 2] (host, in [0, S_u] x [0, S_v])."""
        uv = np.ascontiguousarray(uv, dtype=np.float64).reshape(-1, 2)
        self._n_vert = len(uv)
        _check(lib().bsf_contact_mesh(self._h, len(uv), uv.ctypes.data_as(C.POINTER(C.c_double))))

    def contact_positions(self, x, xv=None, stream=None):
        """Mesh vertex positions [n_vert, 3] of control points x [n_v, n_u, 3] (CUDA float64)."""
        import torch
        xv = torch.empty((self._n_vert, 3), dtype=torch.float64, device=x.device) if xv is None else xv
        _check(lib().bsf_contact_positions(self._h, _ptr(x), _ptr(xv), _stream(stream)))
        return xv

    def contact_assemble(self, verts, H, g=None, grad=None, vals=None, stream=None):
        """Pull the pairs' barrier Hessians H [n, 12, 12] (and gradients g [n, 12]) of mesh vertices verts [n, 4]
        (CUDA int32, -1 = no DOFs) back to the control points: grad (CUDA [n_v, n_u, 3]) += gradient, vals (the
        handle's BSR values) diagonal blocks += the diagonal blocks; returns the number of off-diagonal blocks
        (fetch them with contact_get())."""
        import torch
        if verts.dtype != torch.int32 or H.dtype != torch.float64 or (g is not None and g.dtype != torch.float64):
            raise ValueError("verts must be int32 and H / g float64")
        n = int(verts.shape[0])
        nnz = C.c_int64()
        _check(lib().bsf_contact_assemble(self._h, n, _ptr(verts), _ptr(H), _ptr(g), _ptr(grad), _ptr(vals),
                                          C.byref(nnz), _stream(stream)))
        self._contact_nnz = nnz.value
        return nnz.value

    def contact_get(self, device=None, stream=None):
        """The off-diagonal contact matrix of the last contact_assemble as CUDA (row_ptr, col_idx, vals[nnz, 3, 3])."""
        import torch
        dev = device or torch.device("cuda", torch.cuda.current_device())
        nnz = self._contact_nnz
        rp = torch.empty(self.n_u * self.n_v + 1, dtype=torch.int32, device=dev)
        ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        va = torch.empty((max(nnz, 1), 3, 3), dtype=torch.float64, device=dev)
        _check(lib().bsf_contact_get(self._h, _ptr(rp), _ptr(ci), _ptr(va), _stream(stream)))
        return rp, ci[:nnz], va[:nnz]

    def contact_neumann_solve(self, b, x=None, max_terms=100, rtol=1e-13, stream=None):
        """(D + B_contact) x = b, D the last chol_factor matrix, B the last contact assembly's off-diagonal blocks
        (PAPER.md:879-882); returns (x, gate bound, terms)."""
        import torch
        x = torch.empty_like(b) if x is None else x
        gt, t = C.c_double(), C.c_int()
        _check(lib().bsf_contact_neumann_solve(self._h, _ptr(b), _ptr(x), int(max_terms), float(rtol), C.byref(gt),
                                               C.byref(t), _stream(stream)))
        return x, gt.value, t.value

    def eval_all_batch_host(self, x_host, x_stage, energy=None, energy_host=None, grad=None, vals=None, params=None,
                            flags=0, chunk=0, stream=None):
        """End-to-end batched pass from HOST positions: x_host [B, *x_shape()] (CPU float64, pinned for
        overlap) is uploaded chunk by chunk into x_stage (CUDA, same shape) while earlier chunks compute;
        energies land in `energy` (CUDA [B]) and, if given, in `energy_host` (CPU [B], valid after the
        stream synchronises)."""
        B = x_host.shape[0]
        if tuple(x_host.shape[1:]) != self.x_shape() or tuple(x_stage.shape) != tuple(x_host.shape):
            raise ValueError(f"x_host / x_stage must be [B, {self.x_shape()}]")
        if x_host.is_cuda or not x_stage.is_cuda:
            raise ValueError("x_host must be a CPU tensor and x_stage a CUDA tensor")
        gs = _item(grad)
        vs = _item(vals)
        _check(lib().bsf_eval_all_batch_host(self._h, int(B), _hptr(x_host), _item(x_host), _ptr(x_stage),
                                             _ptr(params), _hptr(energy_host), _ptr(energy), _ptr(grad), gs,
                                             _ptr(vals), vs, int(flags), int(chunk), _stream(stream)))

    def eval_all_batch_params(self, x, params, energy=None, grad=None, vals=None, flags=0, stream=None):
        """Batch of different affine sheets on this handle's grid: params [B, 9] (CUDA float64,
        see affine_params())."""
        B = x.shape[0]
        if tuple(x.shape[1:]) != self.x_shape() or tuple(params.shape) != (B, 9):
            raise ValueError("x must be [B, *x_shape()] and params [B, 9]")
        gs = _item(grad)
        vs = _item(vals)
        _check(lib().bsf_eval_all_batch_params(self._h, int(B), _ptr(x), _item(x), _ptr(params), _ptr(energy),
                                               _ptr(grad), gs, _ptr(vals), vs, int(flags), _stream(stream)))

    def eval_energy(self, x, energy, flags=0, stream=None):
        _check(lib().bsf_eval_energy(self._h, _ptr(x), _ptr(energy), int(flags), _stream(stream)))

    def eval_gradient(self, x, grad, flags=0, stream=None):
        _check(lib().bsf_eval_gradient(self._h, _ptr(x), _ptr(grad), int(flags), _stream(stream)))

    def assemble_hessian(self, x, vals, flags=0, stream=None):
        _check(lib().bsf_assemble_hessian(self._h, _ptr(x), _ptr(vals), int(flags), _stream(stream)))

    def halo_plan(self, rank, nranks):
        """The library's halo exchange plan [(peer, send_off, recv_off, count) below, (...) above], offsets and
        counts in doubles of the position buffer (bsf_halo_plan)."""
        p = (C.c_int64 * 8)()
        _check(lib().bsf_halo_plan(self._h, int(rank), int(nranks), p))
        return [tuple(p[0:4]), tuple(p[4:8])]

    def poll_status(self):
        """Raise BsfError(SINGULAR_STRETCH) if a completed earlier call met |F e_beta| < 1e-12 at a membrane point
        (synchronise its stream first); the report is consumed."""
        _check(lib().bsf_poll_status(self._h))

    def last_launch_count(self) -> int:
        return int(lib().bsf_last_launch_count(self._h))

    def core_rect(self):
        """(i0, i1, j0, j1): control points whose rows the interior core kernel writes; zeros if none."""
        r = (C.c_int32 * 4)()
        _check(lib().bsf_get_core_rect(self._h, r))
        return tuple(int(v) for v in r)

    def __call__(self, x, flags=0):
        """Convenience: allocate outputs, run, return (E tensor[1], grad, vals)."""
        E, g, v = self.alloc_outputs()
        self.eval_all(x, E, g, v, flags)
        return E, g, v
