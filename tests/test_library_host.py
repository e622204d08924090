"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol that
include/bsfem.h declares, validates its inputs, and its independently built pattern equals the
oracle's bit for bit (host-only handles, device = -1)."""
import os
import re

import numpy as np
import pytest

import oracle as O
import paper_2506_18867_b200 as B
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "bsfem.h")).read()
    declared = set(re.findall(r"^\s*(?:bsf_status|int|const char\*)\s+(bsf_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 12
    L = B.lib()
    for s in declared:
        assert hasattr(L, s), s
    assert declared == set(B.SYMBOLS)


def test_material_map_matches_oracle():
    """D6 material map, two independent implementations."""
    for args in [(1e5, 0.3, 3e-4), (2e6, 0.03, 0.01), (1e4, 0.45, 1e-3)]:
        m = B.material_from_young(*args).as_array()
        np.testing.assert_allclose(m, O.material_from_young(*args), rtol=1e-15)
    m = B.material_from_young(1e5, 0.3, 3e-4, shear_E=500.0, bend_E=1e3).as_array()
    np.testing.assert_allclose(m, O.material_from_young(1e5, 0.3, 3e-4, 500.0, 1e3), rtol=1e-15)
    with pytest.raises(B.BsfError):
        B.material_from_young(-1, 0.3, 1e-3)


@pytest.mark.parametrize("n_u,n_v", [(5, 5), (6, 9), (16, 16), (33, 17)])
@pytest.mark.parametrize("rules", [(0, 0), (1, 1), (2, 2), (0, 2)])
def test_pattern_bit_exact_vs_oracle(n_u, n_v, rules):
    ku, kv = W.open_uniform_knots(n_u), W.open_uniform_knots(n_v)
    rest = W.greville_grid(n_u, n_v, 1.0, 0.7)
    mu = np.ones(4)
    s = B.Sheet(n_u, n_v, ku, kv, rest, mu, rules[0], rules[1], device=-1)
    o = O.Oracle(n_u, n_v, ku, kv, rest, mu, rules[0], rules[1])
    rp, ci = s.pattern()
    rpo, cio = o.pattern()
    assert np.array_equal(rp, rpo) and np.array_equal(ci, cio)
    assert (s.n_membrane, s.n_bending) == (o.n_membrane, o.n_bending)


@pytest.mark.parametrize("slab", [(0, 3), (3, 10), (10, 20), (19, 20), (0, 20)])
def test_slab_pattern_bit_exact(slab):
    sh = W.make_sheet(20, 1.0, 0)
    s = B.Sheet.from_sheet(sh, row_begin=slab[0], row_end=slab[1], device=-1)
    o = O.Oracle.from_sheet(sh, r0=slab[0], r1=slab[1])
    assert np.array_equal(s.pattern()[0], o.pattern()[0]) and np.array_equal(s.pattern()[1], o.pattern()[1])
    assert s.n_rows == (slab[1] - slab[0]) * 20


def test_pattern_c2_size_and_closed_form():
    sh = W.make_c2()
    s = B.Sheet.from_sheet(sh, device=-1)
    S = 126
    assert s.nnzb == 23 * S * S + 48 * S + 8 == 371204
    assert (s.n_membrane, s.n_bending) == (2 * S * S + 20 * S - 14, S * S + 2 * S - 3)


def test_create_errors():
    n = 8
    k = W.open_uniform_knots(n)
    rest = W.greville_grid(n, n, 1.0)
    bad = k.copy()
    bad[4] += 0.5
    with pytest.raises(B.BsfError) as e:
        B.Sheet(n, n, bad, k, rest, np.ones(4), device=-1)
    assert e.value.status == -2
    k4 = W.open_uniform_knots(4)
    with pytest.raises(B.BsfError) as e:
        B.Sheet(4, 4, k4, k4, W.greville_grid(4, 4, 1.0), np.ones(4), device=-1)
    assert e.value.status == -3
    B.Sheet(4, 4, k4, k4, W.greville_grid(4, 4, 1.0), np.ones(4), 2, 2, device=-1)  # G3-FULL allows S = 2
    flip = rest.copy()
    flip[..., 1] *= -1
    with pytest.raises(B.BsfError) as e:
        B.Sheet(n, n, k, k, flip, np.ones(4), device=-1)
    assert e.value.status == -4
    with pytest.raises(B.BsfError) as e:
        B.Sheet(n, n, k, k, rest, np.ones(4), row_begin=5, row_end=3, device=-1)
    assert e.value.status == -1


def test_host_only_handle_refuses_compute():
    import torch
    sh = W.make_c1()
    s = B.Sheet.from_sheet(sh, device=-1)
    with pytest.raises((B.BsfError, ValueError)):
        s.eval_all(torch.zeros(s.x_shape(), dtype=torch.float64))


def test_host_only_handle_refuses_every_compute_entry_point():
    """Every device entry point returns BSF_E_NO_DEVICE on a host-only handle (device = -1) without touching
    its (dummy, non-null) pointers; the host-side inertia set-up and mass query still work."""
    import ctypes as C
    sh = W.make_c1()
    s = B.Sheet.from_sheet(sh, device=-1)
    L = B.lib()
    p = C.c_void_p(16)   # never dereferenced
    no_dev = -9
    assert L.bsf_eval_all(s._h, p, p, p, p, 0, None) == no_dev
    assert L.bsf_eval_all_batch(s._h, 1, p, 0, p, p, 0, p, 0, 0, None) == no_dev
    assert L.bsf_eval_all_slab(s._h, p, None, 0, 1, p, p, p, 0, None) == no_dev
    assert L.bsf_bsr_spmv(s._h, p, p, p, None) == no_dev
    lo, hi = C.c_double(), C.c_double()
    assert L.bsf_gershgorin(s._h, p, C.byref(lo), C.byref(hi), None) == no_dev
    it, rr = C.c_int(), C.c_double()
    assert L.bsf_pcg(s._h, p, p, p, 10, 1e-8, C.byref(it), C.byref(rr), None) == no_dev
    assert L.bsf_set_kernel_timing(s._h, 4) == no_dev
    # round-2 entry points: device work refused (NO_DEVICE); calls that need an earlier device result
    # (a factorisation, a contact mesh / assembly) refuse with INVALID_ARG, pointers untouched
    assert L.bsf_chol_factor(s._h, p, None) == no_dev
    assert L.bsf_chol_solve(s._h, p, p, None) == -1
    g, t = C.c_double(), C.c_int()
    assert L.bsf_neumann_solve(s._h, p, p, p, 10, 1e-10, C.byref(g), C.byref(t), None) == -1
    uv = np.array([[0.5, 0.5]])
    assert L.bsf_contact_mesh(s._h, 1, uv.ctypes.data_as(C.POINTER(C.c_double))) == no_dev
    assert L.bsf_contact_positions(s._h, p, p, None) == -1
    n = C.c_int64()
    assert L.bsf_contact_assemble(s._h, 1, p, p, p, p, p, C.byref(n), None) == -1
    assert L.bsf_contact_get(s._h, p, p, p, None) == -1
    assert L.bsf_contact_neumann_solve(s._h, p, p, 10, 1e-10, C.byref(g), C.byref(t), None) == -1
    s.set_inertia(0.2, 1e-3, gravity=(0, 0, -9.81))
    assert s.lumped_mass().shape == (sh.n_v, sh.n_u)
    assert L.bsf_eval_ip_batch(s._h, 1, p, 0, p, 0, None, p, p, 0, p, 0, 0, None) == no_dev
    assert L.bsf_eval_ip_batch(s._h, 0, None, 0, None, 0, None, None, None, 0, None, 0, 0, None) == 0   # empty batch


def test_affine_params_closed_form():
    """bsf_affine_params (step a2 in the library) against the closed form of a Greville sheet:
    X(u, v) = R diag(L_u/S_u, L_v/S_v) (u, v) + X0, so J = R diag(.), G = J^-1, det J = L_u L_v / (S_u S_v)."""
    mu = B.Material(1.0, 2.0, 3.0, 4.0)
    for n_u, n_v, Lu, Lv, th in [(16, 16, 1.0, 1.0, 0.0), (9, 23, 0.7, 2.5, 0.0), (40, 12, 1.3, 0.4, 0.61)]:
        rest = W.greville_grid(n_u, n_v, Lu, Lv)
        R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        rest = rest @ R.T + np.array([0.3, -1.1])
        J = R @ np.diag([Lu / (n_u - 2), Lv / (n_v - 2)])
        G = np.array([[J[1, 1], -J[0, 1]], [-J[1, 0], J[0, 0]]]) / (J[0, 0] * J[1, 1] - J[0, 1] * J[1, 0])
        p = B.affine_params(rest, mu)
        np.testing.assert_allclose(p[:4], G.ravel(), rtol=1e-12, atol=1e-12 * np.abs(G).max())
        np.testing.assert_allclose(p[4], Lu * Lv / ((n_u - 2) * (n_v - 2)), rtol=1e-12)
        np.testing.assert_array_equal(p[5:], [1.0, 2.0, 3.0, 4.0])
    # a curved rest grid is not affine; a mirrored one has det J < 0
    with pytest.raises(B.BsfError) as e:
        B.affine_params(W.make_curved_rest(16, 16, 3), mu)
    assert e.value.status == -1
    with pytest.raises(B.BsfError) as e:
        B.affine_params(W.greville_grid(16, 16, 1.0, 1.0)[:, ::-1].copy(), mu)
    assert e.value.status == -4


def test_binding_does_no_rest_arithmetic():
    """The binding marshals arguments only: no inverse-map arithmetic on rest data."""
    src = open(os.path.join(ROOT, "paper_2506_18867_b200", "__init__.py")).read()
    assert "np.linalg" not in src and "rest_xy[" not in src and "inv(" not in src


def test_halo_plan():
    """bsf_halo_plan (the rows bsf_halo_exchange sends / receives), on host-only slab handles."""
    n = 40
    sh = W.make_sheet(n, 1.0, 0)
    row = n * 3
    mid = B.Sheet.from_sheet(sh, row_begin=10, row_end=20, device=-1)   # buffer rows [8, 22)
    assert mid.halo_plan(1, 3) == [(0, 2 * row, 0, 2 * row), (2, 10 * row, 12 * row, 2 * row)]
    first = B.Sheet.from_sheet(sh, row_begin=0, row_end=10, device=-1)   # buffer rows [0, 12)
    assert first.halo_plan(0, 3) == [(-1, 0, 0, 0), (1, 8 * row, 10 * row, 2 * row)]
    last = B.Sheet.from_sheet(sh, row_begin=20, row_end=40, device=-1)   # buffer rows [18, 40)
    assert last.halo_plan(2, 3) == [(1, 2 * row, 0, 2 * row), (-1, 0, 0, 0)]
    whole = B.Sheet.from_sheet(sh, device=-1)
    assert whole.halo_plan(0, 1) == [(-1, 0, 0, 0), (-1, 0, 0, 0)]
    with pytest.raises(B.BsfError):
        B.Sheet.from_sheet(sh, row_begin=10, row_end=11, device=-1).halo_plan(1, 3)
