"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on identical seeded inputs.

Tolerance: relative 1e-10 per the north star (tests/parity.py gives the per-quantity definition
and floors); pattern bit-exact.  Both the fused tile path and the generic gather path are checked.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W
from parity import TOL, assert_parity, diag_block_norms, rel_energy

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_18867_b200 as B  # noqa: E402

PATHS = [0, B.TILE_ONLY, B.GENERIC_PATH]   # core + frame tile kernels, tile kernel alone, generic


def _gpu(sheet_obj, x, flags):
    xd = torch.from_numpy(np.ascontiguousarray(x[sheet_obj.x_row_begin:sheet_obj.x_row_end])).cuda()
    E, g, v = sheet_obj(xd, flags)
    torch.cuda.synchronize()
    return float(E.item()), g.cpu().numpy(), v.cpu().numpy()


def _check(sh, x=None, mrule=0, brule=0, flags=0, r0=0, r1=None, rest=None, mu=None):
    x = sh.x if x is None else x
    if rest is not None:
        sh = W.Sheet(sh.n_u, sh.n_v, sh.knots_u, sh.knots_v, rest, x, sh.E, sh.nu, sh.h)
    mu = O.material_from_young(sh.E, sh.nu, sh.h) if mu is None else mu
    o = O.Oracle.from_sheet(sh, mrule, brule, r0=r0, r1=r1, mu=mu)
    Er, gr, vr = o.eval(x, flags=flags & 7)
    rp, ci = o.pattern()
    hd = diag_block_norms(vr, rp, ci, r0, sh.n_u)
    if flags & 6:   # one energy switched off: scale the floor with the full Hessian's diagonal
        hd = diag_block_norms(o.eval(x, flags=flags & 1, energy=False, gradient=False)[2], rp, ci, r0, sh.n_u)
    va = o.eval(x, flags=(flags & 7) | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    s = B.Sheet.from_sheet(sh, mrule, brule, row_begin=r0, row_end=r1, material=B.Material(*mu))
    assert np.array_equal(s.pattern()[1], ci) and np.array_equal(s.pattern()[0], rp)
    for path in PATHS:
        E, g, v = _gpu(s, x, flags | path)
        assert_parity(E, g, v, Er, gr, vr, what=f"path={path} flags={flags} rules={mrule},{brule}",
                      hdiag=hd, cmax=np.abs(x).max(), vabs=va)
    return s, (Er, gr, vr)


@pytest.mark.parametrize("rules", [(0, 0), (1, 1), (2, 2)])
@pytest.mark.parametrize("flags", [0, B.PROJECT_PSD])
def test_c1_all_rules(rules, flags):
    _check(W.make_c1(), mrule=rules[0], brule=rules[1], flags=flags)


@pytest.mark.parametrize("flags", [0, B.PROJECT_PSD, B.NO_BENDING, B.NO_MEMBRANE])
def test_c2_state(flags):
    _check(W.make_c2(state=3), flags=flags)


@pytest.mark.parametrize("E", [1e4, 1e6])
def test_c3_material_sweep(E):
    _check(W.make_c3(E=E), flags=B.PROJECT_PSD)


def test_curved_rest_general_path():
    n = 24
    sh = W.make_sheet(n, 1.0, 5, n_modes=4, amp=5e-3, lam=0.2)
    rest = W.make_curved_rest(n, n, seed=6)
    x = np.concatenate([rest, np.zeros((n, n, 1))], -1) * 1.02 + np.random.default_rng(1).normal(0, 2e-3, (n, n, 3))
    for flags in (0, B.PROJECT_PSD):
        _check(sh, x=x, rest=rest, flags=flags)
        _check(sh, x=x, rest=rest, flags=flags, mrule=2, brule=2)


@pytest.mark.parametrize("n", [40, 128])
def test_curved_rest_core_kernel(n):
    """A curved (non-affine) rest grid runs its interior on k_core with per-point rest tables (G, w, Laplacian
    coefficients; per-cp bending blocks) and its frame on the tile kernel; parity with the oracle,
    projected and exact, and the core rectangle is in use."""
    sh = W.make_sheet(n, 1.0, 5, n_modes=4, amp=5e-3, lam=0.2)
    rest = W.make_curved_rest(n, n, seed=11)
    rng = np.random.default_rng(n)
    x = np.concatenate([rest, np.zeros((n, n, 1))], -1) * 1.02 + rng.normal(0, 0.2 / n, (n, n, 3))
    for flags in (B.PROJECT_PSD, 0):
        s, _ = _check(sh, x=x, rest=rest, flags=flags)
        assert s.core_rect()[1] > 0, s.core_rect()


@pytest.mark.parametrize("n_u,n_v", [(5, 5), (7, 6), (37, 19), (130, 9)])
def test_ragged_and_small(n_u, n_v):
    ku, kv = W.open_uniform_knots(n_u), W.open_uniform_knots(n_v)
    rest = W.greville_grid(n_u, n_v, 1.3, 0.9)
    rng = np.random.default_rng(n_u * 100 + n_v)
    x = np.concatenate([rest, np.zeros((n_v, n_u, 1))], -1) + rng.normal(0, 1e-2, (n_v, n_u, 3))
    sh = W.Sheet(n_u, n_v, ku, kv, rest, x, 1e5, 0.3, 3e-4)
    for flags in (0, B.PROJECT_PSD):
        _check(sh, flags=flags)


def test_g3_full_smallest():
    n = 4
    ku = W.open_uniform_knots(n)
    rest = W.greville_grid(n, n, 1.0)
    x = np.concatenate([rest, np.zeros((n, n, 1))], -1) + np.random.default_rng(0).normal(0, 1e-2, (n, n, 3))
    _check(W.Sheet(n, n, ku, ku, rest, x, 1e5, 0.3, 3e-4), mrule=2, brule=2, flags=B.PROJECT_PSD)


@pytest.mark.parametrize("slab", [(0, 40), (40, 41), (41, 90), (90, 128)])
def test_slab_parity(slab):
    _check(W.make_c2(state=1), r0=slab[0], r1=slab[1], flags=B.PROJECT_PSD)


def test_rest_state_zero():
    sh = W.make_sheet(20, 1.0, 0)
    x = np.concatenate([sh.rest_xy, np.zeros((20, 20, 1))], -1)
    s = B.Sheet.from_sheet(sh)
    for path in PATHS:
        E, g, v = _gpu(s, x, path)
        assert abs(E) < 1e-20 and np.abs(g).max() < 1e-12


def test_deterministic_and_partial_outputs():
    sh = W.make_c2(state=2)
    s = B.Sheet.from_sheet(sh)
    xd = torch.from_numpy(sh.x).cuda()
    for path in PATHS:
        E1, g1, v1 = s(xd, B.PROJECT_PSD | path)
        E2, g2, v2 = s(xd, B.PROJECT_PSD | path)
        assert torch.equal(E1, E2) and torch.equal(g1, g2) and torch.equal(v1, v2)
        E3 = torch.zeros(1, dtype=torch.float64, device="cuda")
        s.eval_energy(xd, E3, B.PROJECT_PSD | path)
        g3 = torch.zeros_like(g1)
        s.eval_gradient(xd, g3, B.PROJECT_PSD | path)
        v3 = torch.zeros_like(v1)
        s.assemble_hessian(xd, v3, B.PROJECT_PSD | path)
        # gradient and Hessian: the same bits; the energy-only call sums the same point energies in another order
        # (k_core_energy: one thread per anchor instead of the point warps), so to rounding
        assert torch.equal(g1, g3) and torch.equal(v1, v3)
        assert abs(E1.item() - E3.item()) <= 1e-14 * abs(E1.item())
        assert s.last_launch_count() > 0


def test_energy_only_calls_match_full_calls():
    """Energy-only calls (the line search) through k_core_energy: plain, batched with per-item parameters, and the
    incremental potential; each against the full call's energy (1e-13) and the oracle's (the parity floor)."""
    sh = W.make_c2(state=3)
    s = B.Sheet.from_sheet(sh)
    xd = torch.from_numpy(sh.x).cuda()
    E1, _, _ = s(xd, B.PROJECT_PSD)
    E2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    s.eval_energy(xd, E2, B.PROJECT_PSD)
    torch.cuda.synchronize()
    Er, _, _ = O.Oracle.from_sheet(sh).eval(sh.x, flags=O.FLAG_PROJECT)
    assert abs(E2.item() - E1.item()) <= 1e-13 * abs(E1.item())
    assert abs(E2.item() - Er) <= 1e-11 * abs(Er)
    # batched, per-item parameters (C5 style), energy only vs the full batch
    sheets = W.make_c5(count=3, n=64)
    h = B.Sheet.from_sheet(sheets[0])
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    P = torch.from_numpy(np.stack([B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h))
                                   for q in sheets])).cuda()
    Ef = torch.zeros(3, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((3, h.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    h.eval_all_batch_params(X, P, Ef, G, V, B.PROJECT_PSD)
    Ee = torch.zeros(3, dtype=torch.float64, device="cuda")
    h.eval_all_batch_params(X, P, Ee, None, None, B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert torch.max(torch.abs(Ee - Ef)).item() <= 1e-13 * torch.max(torch.abs(Ef)).item()
    # incremental potential, energy only
    s.set_inertia(0.15, 2e-3, gravity=np.array([0.0, 0.0, -9.81]))
    rng = np.random.default_rng(5)
    xh = torch.from_numpy(sh.x + rng.normal(0, 1e-3, sh.x.shape)).cuda().unsqueeze(0).contiguous()
    X1 = xd.unsqueeze(0).contiguous()
    Ei = torch.zeros(1, dtype=torch.float64, device="cuda")
    Gi = torch.zeros_like(X1)
    Vi = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_ip_batch(X1, xh, Ei, Gi, Vi, B.PROJECT_PSD)
    Eo = torch.zeros(1, dtype=torch.float64, device="cuda")
    s.eval_ip_batch(X1, xh, Eo, None, None, B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert abs(Eo.item() - Ei.item()) <= 1e-13 * abs(Ei.item())
    # a row slab (its core rows only, its own energy share)
    sl = B.Sheet.from_sheet(sh, row_begin=40, row_end=90)
    xs = torch.from_numpy(np.ascontiguousarray(sh.x[sl.x_row_begin:sl.x_row_end])).cuda()
    Es, _, _ = sl(xs, B.PROJECT_PSD)
    Ese = torch.zeros(1, dtype=torch.float64, device="cuda")
    sl.eval_energy(xs, Ese, B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert abs(Ese.item() - Es.item()) <= 1e-13 * abs(Es.item())


def test_c4_full_size():
    """C4 (1024^2, 1.04 M elements) in the bench's launch configuration against ONE full oracle evaluation:
    the energy, every control point's gradient and every one of the 24.07 M Hessian blocks, pattern bit-exact
    (no sampling); then the slab partition property: slab energies sum to the sheet's."""
    sh = W.make_c4()
    s = B.Sheet.from_sheet(sh)
    xd = torch.from_numpy(sh.x).cuda()
    E, g, v = s(xd, B.PROJECT_PSD)
    torch.cuda.synchronize()
    g, v = g.cpu().numpy(), v.cpu().numpy()
    mu = O.material_from_young(sh.E, sh.nu, sh.h)
    o = O.Oracle.from_sheet(sh, mu=mu)
    rp, ci = o.pattern()
    assert np.array_equal(s.pattern()[0], rp) and np.array_equal(s.pattern()[1], ci)
    assert len(ci) == 23 * 1022 ** 2 + 48 * 1022 + 8
    Er, gr, vr = o.eval(sh.x, flags=O.FLAG_PROJECT)
    hd = diag_block_norms(vr, rp, ci, 0, sh.n_u)
    va = o.eval(sh.x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    assert_parity(float(E.item()), g, v, Er, gr, vr, what="C4 full", hdiag=hd, cmax=np.abs(sh.x).max(), vabs=va)
    del v, vr, va
    # energy: sum over a 4-slab partition equals the full-sheet energy
    parts = 0.0
    for r0, r1 in [(0, 256), (256, 512), (512, 768), (768, 1024)]:
        sl = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1)
        parts += _gpu(sl, sh.x, B.PROJECT_PSD)[0]
    assert rel_energy(float(E.item()), parts) <= 1e-12


def test_batch_matches_single_calls():
    """bsf_eval_all_batch over several C2 states equals per-state calls bit for bit (gradient, Hessian; the energy to
    rounding: its per-CTA partial sums follow the launch's row chunking, which depends on the batch size), and the
    oracle."""
    sheets = [W.make_c2(state=k) for k in (0, 7, 42)]
    s = B.Sheet.from_sheet(sheets[0])
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    nb = len(sheets)
    E = torch.zeros(nb, dtype=torch.float64, device="cuda")
    G = torch.zeros((nb,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
    V = torch.zeros((nb, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    for path in PATHS:
        s.eval_all_batch(X, E, G, V, B.PROJECT_PSD | path)
        for k in range(nb):
            E1, g1, v1 = s(X[k].contiguous(), B.PROJECT_PSD | path)
            assert torch.equal(g1, G[k]) and torch.equal(v1, V[k])
            assert rel_energy(float(E1[0]), float(E[k])) <= 1e-13
    o = O.Oracle.from_sheet(sheets[1])
    Er, gr, vr = o.eval(sheets[1].x, flags=O.FLAG_PROJECT)
    rp, ci = o.pattern()
    va = o.eval(sheets[1].x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    assert_parity(float(E[1]), G[1].cpu().numpy(), V[1].cpu().numpy(), Er, gr, vr, what="batch item 1",
                  hdiag=diag_block_norms(vr, rp, ci, 0, sheets[1].n_u), cmax=np.abs(sheets[1].x).max(), vabs=va)


def test_c2_bench_launch_100_states():
    """C2 in exactly the bench's launch (bench.py secondary "C2_batched_100" / --config C2): the 100 seeded states in one
    bsf_eval_all_batch call (one long row chunk per core strip at this batch size).  Three items
    against the oracle; sampled items bit for bit against single-state calls (many short chunks)."""
    sheets = [W.make_c2(state=k) for k in range(100)]
    s = B.Sheet.from_sheet(sheets[0])
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    nb = len(sheets)
    E = torch.zeros(nb, dtype=torch.float64, device="cuda")
    G = torch.zeros((nb,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
    V = torch.zeros((nb, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_all_batch(X, E, G, V, B.PROJECT_PSD)
    torch.cuda.synchronize()
    for k in (0, 37, 99):
        E1, g1, v1 = s(X[k].contiguous(), B.PROJECT_PSD)
        assert torch.equal(g1, G[k]) and torch.equal(v1, V[k])
        assert rel_energy(float(E1.item()), float(E[k])) <= 1e-13
    for k in (0, 51, 99):
        q = sheets[k]
        o = O.Oracle.from_sheet(q)
        Er, gr, vr = o.eval(q.x, flags=O.FLAG_PROJECT)
        rp, ci = o.pattern()
        va = o.eval(q.x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
        assert_parity(float(E[k]), G[k].cpu().numpy(), V[k].cpu().numpy(), Er, gr, vr, what=f"C2 bench item {k}",
                      hdiag=diag_block_norms(vr, rp, ci, 0, q.n_u), cmax=np.abs(q.x).max(), vabs=va)


def test_slab_sheet_nccl_single_rank():
    """The library's NCCL entry points on one rank (unique id, comm init, all-reduce) and the
    SlabSheet driver against the oracle."""
    import os
    import torch.distributed as dist
    from paper_2506_18867_b200 import distributed as D
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        comm = D.NcclComm(0, 1, 0)
        sh = W.make_c2(state=5)
        slab = D.SlabSheet(sh, 0, 1, device=0, comm=comm)
        slab.load_owned(torch.from_numpy(sh.x).cuda())
        E, g, v = slab.assemble(B.PROJECT_PSD)
        buf = torch.tensor([1.5, -2.0], dtype=torch.float64, device="cuda")
        B._check(B.lib().bsf_allreduce_sum(B.C.c_void_p(buf.data_ptr()), 2, comm.comm, B._stream(None)))
        torch.cuda.synchronize()
        assert buf.tolist() == [1.5, -2.0]
        o = O.Oracle.from_sheet(sh)
        Er, gr, vr = o.eval(sh.x, flags=O.FLAG_PROJECT)
        assert rel_energy(float(E.item()), Er) <= TOL
        comm.close()
    finally:
        dist.destroy_process_group()


def _c5_launch(sheets, flags=B.PROJECT_PSD):
    s = B.Sheet.from_sheet(sheets[0])
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    P = torch.from_numpy(np.stack([B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h))
                                   for q in sheets])).cuda()
    nb = len(sheets)
    E = torch.zeros(nb, dtype=torch.float64, device="cuda")
    G = torch.zeros((nb,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
    V = torch.zeros((nb, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_all_batch_params(X, P, E, G, V, flags)
    torch.cuda.synchronize()
    return s, E, G, V


def _c5_item_vs_oracle(q, E, G, V, what):
    o = O.Oracle.from_sheet(q)
    Er, gr, vr = o.eval(q.x, flags=O.FLAG_PROJECT)
    rp, ci = o.pattern()
    va = o.eval(q.x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    assert_parity(float(E), G.cpu().numpy(), V.cpu().numpy(), Er, gr, vr, what=what,
                  hdiag=diag_block_norms(vr, rp, ci, 0, q.n_u), cmax=np.abs(q.x).max(), vabs=va)


def test_c5_bench_launch_8_sheets_256():
    """C5 at full size in the bench's launch (bench.py --config C5: the 8 sheets of rank 0, 256^2 each, per-sheet
    L / E / nu, one bsf_eval_all_batch_params launch), every item against its own oracle."""
    sheets = W.make_c5()[:8]
    assert sheets[0].n_u == 256
    s, E, G, V = _c5_launch(sheets)
    for k, q in enumerate(sheets):
        _c5_item_vs_oracle(q, E[k], G[k], V[k], f"C5 bench item {k}")


def test_c5_all_64_sheets_one_launch():
    """All 64 C5 sheets (256^2) in ONE launch: 8 sampled items against their own oracle, and the items shared
    with the 8-sheet launch bit for bit (the per-row arithmetic does not depend on the launch size)."""
    sheets = W.make_c5()
    assert len(sheets) == 64
    s, E, G, V = _c5_launch(sheets)
    for k in (3, 9, 17, 26, 38, 45, 52, 63):
        _c5_item_vs_oracle(sheets[k], E[k], G[k], V[k], f"C5 64-launch item {k}")
    s8, E8, G8, V8 = _c5_launch(sheets[:8])
    assert torch.equal(G[:8], G8) and torch.equal(V[:8], V8)
    assert float(((E[:8] - E8).abs() / E8.abs()).max()) <= 1e-13


def test_c5_style_batch_of_different_sheets():
    """Config C5 layout: independent sheets of one grid size with per-sheet side length, Young's
    modulus and Poisson ratio in ONE launch (bsf_eval_all_batch_params), each against its own oracle."""
    sheets = W.make_c5(count=4, n=40)
    s = B.Sheet.from_sheet(sheets[0])
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    P = torch.from_numpy(np.stack([B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h))
                                   for q in sheets])).cuda()
    nb = len(sheets)
    E = torch.zeros(nb, dtype=torch.float64, device="cuda")
    G = torch.zeros((nb,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
    V = torch.zeros((nb, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_all_batch_params(X, P, E, G, V, B.PROJECT_PSD)
    torch.cuda.synchronize()
    for k, q in enumerate(sheets):
        o = O.Oracle.from_sheet(q)
        Er, gr, vr = o.eval(q.x, flags=O.FLAG_PROJECT)
        rp, ci = o.pattern()
        va = o.eval(q.x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
        assert_parity(float(E[k]), G[k].cpu().numpy(), V[k].cpu().numpy(), Er, gr, vr, what=f"C5 item {k}",
                      hdiag=diag_block_norms(vr, rp, ci, 0, q.n_u), cmax=np.abs(q.x).max(), vabs=va)


def test_host_buffer_call_matches_device_call():
    """bsf_eval_all_batch_host (chunked upload from pinned host memory, overlapped with the assembly)
    gives the device call's gradient and Hessian bit for bit and its energies to rounding (the energy
    partial sums follow the CTA partition, which depends on the launch size)."""
    sheets = [W.make_c2(state=k) for k in range(7)]
    s = B.Sheet.from_sheet(sheets[0])
    Xh = torch.stack([torch.from_numpy(q.x) for q in sheets]).pin_memory()
    X = Xh.cuda()
    nb = len(sheets)
    out = []
    for host in (False, True):
        E = torch.zeros(nb, dtype=torch.float64, device="cuda")
        G = torch.zeros((nb,) + tuple(X.shape[1:]), dtype=torch.float64, device="cuda")
        V = torch.zeros((nb, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
        Eh = torch.zeros(nb, dtype=torch.float64).pin_memory()
        if host:
            stage = torch.zeros_like(X)
            s.eval_all_batch_host(Xh, stage, E, Eh, G, V, flags=B.PROJECT_PSD, chunk=3)
            torch.cuda.synchronize()
            assert torch.equal(stage, X)
            assert torch.equal(Eh, E.cpu())
        else:
            s.eval_all_batch(X, E, G, V, B.PROJECT_PSD)
            torch.cuda.synchronize()
        out.append((E.cpu().numpy(), G, V))
    assert torch.equal(out[0][1], out[1][1]) and torch.equal(out[0][2], out[1][2])
    assert np.max(np.abs(out[0][0] - out[1][0]) / np.abs(out[0][0])) < 1e-13


@pytest.mark.parametrize("no_band", [False, True])
def test_band_kernel_and_frame_fallback(no_band, monkeypatch):
    """The edge bands (k_band) and, with BSF_NO_BAND, the whole frame in corner-style tiles (k_frame) both
    match the oracle; the band path launches one kernel more (core, band, corners; the energy is reduced by the last
    CTA of the three, no separate launch)."""
    if no_band:
        monkeypatch.setenv("BSF_NO_BAND", "1")
    s, _ = _check(W.make_c2(state=2), flags=B.PROJECT_PSD)
    _gpu(s, W.make_c2(state=2).x, B.PROJECT_PSD)
    assert s.last_launch_count() == (2 if no_band else 3)
    _check(W.make_sheet(40, 1.0, 9, n_modes=4, amp=5e-3, lam=0.2, rigid=True), flags=0)


def test_async_stage_pipelined_host_calls():
    """BSF_ASYNC_STAGE: consecutive host-buffer calls alternating two staging buffers (each upload waits
    only for the last call that read its stage) give the same outputs as plain device calls, per call."""
    sheets = [W.make_c2(state=k) for k in range(6)]
    s = B.Sheet.from_sheet(sheets[0])
    Xh = [torch.stack([torch.from_numpy(q.x) for q in sheets[i:i + 3]]).pin_memory() for i in (0, 3)]
    stages = [torch.zeros_like(Xh[0]).cuda() for _ in range(2)]
    outs = []
    for rep in range(4):   # calls 0..3 alternate inputs and stages; each result copied out in stream order
        i = rep & 1
        E = torch.zeros(3, dtype=torch.float64, device="cuda")
        G = torch.zeros((3,) + tuple(Xh[0].shape[1:]), dtype=torch.float64, device="cuda")
        V = torch.zeros((3, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
        Eh = torch.zeros(3, dtype=torch.float64).pin_memory()
        s.eval_all_batch_host(Xh[i], stages[i], E, Eh, G, V, flags=B.PROJECT_PSD | B.ASYNC_STAGE)
        outs.append((i, E, G.clone(), V.clone(), Eh))
    torch.cuda.synchronize()
    for i, E, G, V, Eh in outs:
        E2 = torch.zeros_like(E); G2 = torch.zeros_like(G); V2 = torch.zeros_like(V)
        s.eval_all_batch(Xh[i].cuda(), E2, G2, V2, B.PROJECT_PSD)
        torch.cuda.synchronize()
        assert torch.equal(G, G2) and torch.equal(V, V2) and torch.equal(E, E2)
        assert torch.equal(Eh, E.cpu())


@pytest.mark.parametrize("case", ["c1", "c2_pinned", "slab", "c3_size"])
def test_incremental_potential_matches_oracle(case):
    """bsf_eval_ip_batch (elastic assembly + lumped-mass inertia, gravity, pinned elimination) against the
    oracle's eval_ip, every path, a batch of 2 items with different predicted positions.  c3_size: a 200^2 sheet,
    whose core, band and corner CTAs overfill the SMs (k_core launched first)."""
    sh = (W.make_c1() if case == "c1" else
          W.make_sheet(200, 1.5, 5, n_modes=4, amp=5e-3, lam=0.2) if case == "c3_size" else W.make_c2(state=4))
    r0, r1 = (40, 90) if case == "slab" else (0, sh.n_v)
    R0, dt, grav = 0.15, 4e-3, np.array([0.0, -9.81, 0.5])
    pinned = None
    if case == "c2_pinned":
        pinned = np.zeros((sh.n_v, sh.n_u), bool)
        pinned[-1, :] = True
        pinned[0, :3] = True
    if case == "slab":   # a pinned row inside the slab and one outside it within the columns' reach
        pinned = np.zeros((sh.n_v, sh.n_u), bool)
        pinned[50, 10:20] = True
        pinned[91, :] = True
    o = O.Oracle.from_sheet(sh, r0=r0, r1=r1)
    m = o.lumped_mass(R0)
    rng = np.random.default_rng(17)
    s = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1)
    s.set_inertia(R0, dt, gravity=grav, pinned=pinned)
    # the library integrates m_a = int R0 N_a directly, the oracle sums the consistent mass rows: the same number
    # up to summation order (1.2e-14 of max m on the 200^2 sheet)
    assert np.max(np.abs(s.lumped_mass() - m)) < 1e-13 * m.max()
    xs = [sh.x, sh.x + rng.normal(0, 1e-3, sh.x.shape)]
    xh = [x[r0:r1] + rng.normal(0, 2e-3, x[r0:r1].shape) for x in xs]
    X = torch.stack([torch.from_numpy(np.ascontiguousarray(x[s.x_row_begin:s.x_row_end])) for x in xs]).cuda()
    XH = torch.from_numpy(np.stack(xh)).cuda()
    for path in PATHS:
        E = torch.zeros(2, dtype=torch.float64, device="cuda")
        G = torch.zeros((2, r1 - r0, sh.n_u, 3), dtype=torch.float64, device="cuda")
        V = torch.zeros((2, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
        s.eval_ip_batch(X, XH, E, G, V, flags=B.PROJECT_PSD | path)
        torch.cuda.synchronize()
        for b in range(2):
            Er, gr, vr = o.eval_ip(xs[b], xh[b], m, dt, grav, pinned, flags=O.FLAG_PROJECT)
            rp, ci = o.pattern()
            hd = diag_block_norms(vr, rp, ci, r0, sh.n_u)
            va = o.eval_ip(xs[b], xh[b], m, dt, grav, pinned, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM,
                           energy=False, gradient=False)[2]
            assert_parity(E[b].item(), G[b].cpu().numpy(), V[b].cpu().numpy(), Er, gr, vr,
                          what=f"ip case={case} path={path} item={b}", hdiag=hd, cmax=np.abs(xs[b]).max(), vabs=va)


def test_cuda_graph_capture_and_replay():
    """A batched call (core + band + corners on the event-forked side stream + energy) captures into a CUDA
    graph after one warm call, and replaying the graph on new positions gives the direct call's outputs."""
    sheets = [W.make_c2(state=k) for k in range(3)]
    s = B.Sheet.from_sheet(sheets[0])
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    E = torch.zeros(3, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((3, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s.eval_all_batch(X, E, G, V, B.PROJECT_PSD, st)   # warm: side stream, events, scratch allocated
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        s.eval_all_batch(X, E, G, V, B.PROJECT_PSD, st)
    X.copy_(torch.stack([torch.from_numpy(W.make_c2(state=k + 5).x) for k in range(3)]))
    g.replay()
    torch.cuda.synchronize()
    E2, G2, V2 = torch.zeros_like(E), torch.zeros_like(G), torch.zeros_like(V)
    s.eval_all_batch(X, E2, G2, V2, B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert torch.equal(G, G2) and torch.equal(V, V2) and torch.equal(E, E2)


def test_set_inertia_repeated_reuses_tables():
    """bsf_set_inertia called again (new dt, gravity, pinned set) updates the tables in place; results follow
    the latest settings."""
    sh = W.make_c1()
    s = B.Sheet.from_sheet(sh)
    o = O.Oracle.from_sheet(sh)
    X = torch.from_numpy(sh.x).cuda().unsqueeze(0)
    XH = X + 1e-3
    for dt, pin_rows in [(1e-2, [15]), (3e-3, []), (5e-3, [0, 15])]:
        pinned = np.zeros((sh.n_v, sh.n_u), bool)
        pinned[pin_rows, :] = True
        s.set_inertia(0.3, dt, gravity=(0, -1.0, 0), pinned=pinned if pin_rows else None)
        E = torch.zeros(1, dtype=torch.float64, device="cuda")
        G = torch.zeros_like(X)
        V = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
        s.eval_ip_batch(X, XH, E, G, V, flags=B.PROJECT_PSD)
        torch.cuda.synchronize()
        m = o.lumped_mass(0.3)
        Er, gr, vr = o.eval_ip(sh.x, XH[0].cpu().numpy(), m, dt, (0, -1.0, 0), pinned if pin_rows else None,
                               flags=O.FLAG_PROJECT)
        rp, ci = o.pattern()
        assert_parity(E.item(), G[0].cpu().numpy(), V[0].cpu().numpy(), Er, gr, vr, what=f"dt={dt}",
                      hdiag=diag_block_norms(vr, rp, ci, 0, sh.n_u), cmax=np.abs(sh.x).max(),
                      vabs=o.eval_ip(sh.x, XH[0].cpu().numpy(), m, dt, (0, -1.0, 0), pinned if pin_rows else None,
                                     flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2])


def test_live_kernel_timing_ring():
    """bsf_set_kernel_timing records k_core / k_band durations of the last calls (oldest first), and
    recording does not change the outputs."""
    sh = W.make_c2(state=7)
    s = B.Sheet.from_sheet(sh)
    x = torch.from_numpy(sh.x).cuda()
    E0, g0, v0 = s(x, B.PROJECT_PSD)
    s.set_kernel_timing(2)
    for _ in range(3):
        E1, g1, v1 = s(x, B.PROJECT_PSD)
    core, band = s.kernel_timing(5)
    assert len(core) == 2 and len(band) == 2 and all(t > 0 for t in core + band), (core, band)
    assert torch.equal(g0, g1) and torch.equal(v0, v1) and torch.equal(E0, E1)
    s.set_kernel_timing(0)
    assert s.kernel_timing(5) == ([], [])


def test_incremental_potential_batch_of_different_sheets():
    """bsf_eval_ip_batch with per-item affine parameters (C5 layout): each item's masses follow its own rest
    map (det J), against each sheet's own oracle incremental potential."""
    sheets = W.make_c5(count=3, n=40)
    s = B.Sheet.from_sheet(sheets[0])
    R0, dt, grav = 0.12, 5e-3, np.array([0.0, 0.0, -9.81])
    s.set_inertia(R0, dt, gravity=grav)
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    rng = np.random.default_rng(21)
    XH = X + torch.from_numpy(rng.normal(0, 1e-3, tuple(X.shape))).cuda()
    P = torch.from_numpy(np.stack([B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h))
                                   for q in sheets])).cuda()
    nb = len(sheets)
    E = torch.zeros(nb, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((nb, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    for path in (0, B.TILE_ONLY):   # fused kernels; epilogue kernel
        s.eval_ip_batch(X, XH, E, G, V, flags=B.PROJECT_PSD | path, params=P)
        torch.cuda.synchronize()
        for k, q in enumerate(sheets):
            o = O.Oracle.from_sheet(q)
            m = o.lumped_mass(R0)
            xh = XH[k].cpu().numpy()
            Er, gr, vr = o.eval_ip(q.x, xh, m, dt, grav, flags=O.FLAG_PROJECT)
            rp, ci = o.pattern()
            va = o.eval_ip(q.x, xh, m, dt, grav, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False,
                           gradient=False)[2]
            assert_parity(float(E[k]), G[k].cpu().numpy(), V[k].cpu().numpy(), Er, gr, vr, what=f"C5 IP item {k}",
                          hdiag=diag_block_norms(vr, rp, ci, 0, q.n_u), cmax=np.abs(q.x).max(), vabs=va)


def test_incremental_potential_curved_rest():
    """Non-affine (curved) rest shape: per-point rest data on the tile path, masses with varying det J, the
    epilogue kernel; against the oracle."""
    base = W.make_sheet(20, 1.0, 12, n_modes=3, amp=3e-3, lam=0.2)
    rest = W.make_curved_rest(20, 20, 5)
    sh = W.Sheet(20, 20, base.knots_u, base.knots_v, rest, base.x, base.E, base.nu, base.h)
    o = O.Oracle.from_sheet(sh)
    R0, dt, grav = 0.3, 2e-3, np.array([0.1, -9.81, 0.0])
    m = o.lumped_mass(R0)
    s = B.Sheet.from_sheet(sh)
    s.set_inertia(R0, dt, gravity=grav)
    assert np.max(np.abs(s.lumped_mass() - m)) < 1e-14 * m.max()
    rng = np.random.default_rng(8)
    xh = sh.x + rng.normal(0, 1e-3, sh.x.shape)
    E = torch.zeros(1, dtype=torch.float64, device="cuda")
    G = torch.zeros((1, 20, 20, 3), dtype=torch.float64, device="cuda")
    V = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_ip_batch(torch.from_numpy(sh.x).cuda().unsqueeze(0), torch.from_numpy(xh).cuda().unsqueeze(0), E, G, V,
                    flags=B.PROJECT_PSD)
    torch.cuda.synchronize()
    Er, gr, vr = o.eval_ip(sh.x, xh, m, dt, grav, flags=O.FLAG_PROJECT)
    rp, ci = o.pattern()
    va = o.eval_ip(sh.x, xh, m, dt, grav, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    assert_parity(E.item(), G[0].cpu().numpy(), V[0].cpu().numpy(), Er, gr, vr, what="IP curved rest",
                  hdiag=diag_block_norms(vr, rp, ci, 0, 20), cmax=np.abs(sh.x).max(), vabs=va)


@pytest.mark.parametrize("seed", list(range(16)) + [100, 101, 102])
def test_random_sizes_slabs_and_batches(seed):
    """Randomised coverage of the launch shapes the chunking and stream logic pick (one-wave slabs, side streams,
    k_core-first ordering, ragged strips, batches): random grid sizes, slab bounds and batch sizes, the full call
    and the energy-only call, against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    lo, hi = (12, 96) if seed < 100 else (200, 420)   # seeds >= 100: grids with many core strips (multi-wave paths)
    n_u, n_v = int(rng.integers(lo, hi)), int(rng.integers(lo, hi))
    ku, kv = W.open_uniform_knots(n_u), W.open_uniform_knots(n_v)
    rest = W.greville_grid(n_u, n_v, float(rng.uniform(0.5, 2.0)), float(rng.uniform(0.5, 2.0)))
    nb = int(rng.integers(1, 4))
    xs = [np.concatenate([rest, np.zeros((n_v, n_u, 1))], -1) + rng.normal(0, 1e-2, (n_v, n_u, 3)) for _ in range(nb)]
    sh = W.Sheet(n_u, n_v, ku, kv, rest, xs[0], 1e5, 0.3, 3e-4)
    r0 = int(rng.integers(0, n_v // 3)) if rng.uniform() < 0.5 else 0
    r1 = int(rng.integers(r0 + 2 + (n_v - r0 - 2) // 2, n_v + 1)) if r0 > 0 else n_v
    o = O.Oracle.from_sheet(sh, r0=r0, r1=r1)
    s = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1)
    X = torch.stack([torch.from_numpy(np.ascontiguousarray(x[s.x_row_begin:s.x_row_end])) for x in xs]).cuda()
    E = torch.zeros(nb, dtype=torch.float64, device="cuda")
    G = torch.zeros((nb, r1 - r0, n_u, 3), dtype=torch.float64, device="cuda")
    V = torch.zeros((nb, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_all_batch(X, E, G, V, B.PROJECT_PSD)
    Ee = torch.zeros(nb, dtype=torch.float64, device="cuda")
    s.eval_all_batch(X, Ee, None, None, B.PROJECT_PSD)
    torch.cuda.synchronize()
    rp, ci = o.pattern()
    for k in range(nb):
        Er, gr, vr = o.eval(xs[k], flags=O.FLAG_PROJECT)
        va = o.eval(xs[k], flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
        assert_parity(E[k].item(), G[k].cpu().numpy(), V[k].cpu().numpy(), Er, gr, vr,
                      what=f"n={n_u}x{n_v} rows [{r0},{r1}) item {k}/{nb}",
                      hdiag=diag_block_norms(vr, rp, ci, r0, n_u), cmax=np.abs(xs[k]).max(), vabs=va)
        assert abs(Ee[k].item() - E[k].item()) <= 1e-13 * max(abs(E[k].item()), 1e-300)
