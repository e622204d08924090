"""GPU parity of the G3-FULL kernel (k_g3, g3.cu) against the CPU oracle under the same rule.

G3-FULL (3x3 Gauss on every span for both energies) is the paper's full-quadrature
comparison rule and BASELINE's C1 rule; SURVEY §8(d) times it as a secondary row for
C2-C4.  Tolerance as tests/parity.py (north star 1e-10); pattern bit-exact.  The generic path
(BSF_GENERIC_PATH) is cross-checked on the same inputs where it exists.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W
from parity import TOL, assert_parity, diag_block_norms, rel_energy

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_18867_b200 as B  # noqa: E402

G3 = B.RULE_G3_FULL


def _oracle(sh, flags, r0=0, r1=None):
    mu = O.material_from_young(sh.E, sh.nu, sh.h)
    o = O.Oracle.from_sheet(sh, G3, G3, r0=r0, r1=r1, mu=mu)
    Er, gr, vr = o.eval(sh.x, flags=flags & 7)
    rp, ci = o.pattern()
    va = o.eval(sh.x, flags=(flags & 7) | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    return o, Er, gr, vr, rp, ci, va


def _gpu(s, x, flags):
    xd = torch.from_numpy(np.ascontiguousarray(x[s.x_row_begin:s.x_row_end])).cuda()
    E, g, v = s(xd, flags)
    torch.cuda.synchronize()
    return float(E.item()), g.cpu().numpy(), v.cpu().numpy()


@pytest.mark.parametrize("case", ["c2", "ragged", "small"])
@pytest.mark.parametrize("flags", [B.PROJECT_PSD, 0])
def test_g3_kernel_matches_oracle(case, flags):
    sh = {"c2": lambda: W.make_c2(state=3), "ragged": lambda: W.make_sheet(37, 1.0, 11, n_modes=4, amp=5e-3),
          "small": lambda: W.make_sheet(7, 1.0, 12, n_modes=2, amp=5e-3)}[case]()
    _, Er, gr, vr, rp, ci, va = _oracle(sh, flags)
    s = B.Sheet.from_sheet(sh, G3, G3)
    assert np.array_equal(s.pattern()[0], rp) and np.array_equal(s.pattern()[1], ci)
    E, g, v = _gpu(s, sh.x, flags)
    assert 1 <= s.last_launch_count() <= 3   # k_g3 (general, interior) + energy: not the generic path
    hd = diag_block_norms(vr, rp, ci, 0, sh.n_u)
    assert_parity(E, g, v, Er, gr, vr, what=f"g3 {case} flags={flags}", hdiag=hd, cmax=np.abs(sh.x).max(), vabs=va)
    if case != "c2":   # the generic gather path on the same handle
        E2, g2, v2 = _gpu(s, sh.x, flags | B.GENERIC_PATH)
        assert_parity(E2, g2, v2, Er, gr, vr, what=f"generic {case}", hdiag=hd, cmax=np.abs(sh.x).max(), vabs=va)


@pytest.mark.parametrize("which", [B.NO_BENDING, B.NO_MEMBRANE])
def test_g3_energy_switches(which):
    sh = W.make_sheet(24, 1.0, 13, n_modes=3, amp=5e-3)
    mu = O.material_from_young(sh.E, sh.nu, sh.h)
    o = O.Oracle.from_sheet(sh, G3, G3, mu=mu)
    Er, gr, vr = o.eval(sh.x, flags=which | O.FLAG_PROJECT)
    rp, ci = o.pattern()
    full = o.eval(sh.x, flags=O.FLAG_PROJECT, energy=False, gradient=False)[2]
    va = o.eval(sh.x, flags=which | O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    s = B.Sheet.from_sheet(sh, G3, G3)
    E, g, v = _gpu(s, sh.x, which | B.PROJECT_PSD)
    assert_parity(E, g, v, Er, gr, vr, what=f"g3 switch {which}", hdiag=diag_block_norms(full, rp, ci, 0, sh.n_u),
                  cmax=np.abs(sh.x).max(), vabs=va)


@pytest.mark.parametrize("slab", [(0, 40), (40, 41), (41, 90), (90, 128)])
def test_g3_slabs(slab):
    sh = W.make_c2(state=8)
    r0, r1 = slab
    _, Er, gr, vr, rp, ci, va = _oracle(sh, B.PROJECT_PSD, r0, r1)
    s = B.Sheet.from_sheet(sh, G3, G3, row_begin=r0, row_end=r1)
    assert np.array_equal(s.pattern()[1], ci)
    E, g, v = _gpu(s, sh.x, B.PROJECT_PSD)
    assert_parity(E, g, v, Er, gr, vr, what=f"g3 slab {slab}", hdiag=diag_block_norms(vr, rp, ci, r0, sh.n_u),
                  cmax=np.abs(sh.x).max(), vabs=va)


def test_g3_batch_and_per_item_params():
    """A batch of C2 states equals per-state calls bit for bit; C5-style sheets with per-sheet L, E, nu in one
    launch (bsf_eval_all_batch_params) each match their own oracle."""
    sheets = [W.make_c2(state=k) for k in (1, 2, 3)]
    s = B.Sheet.from_sheet(sheets[0], G3, G3)
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    E = torch.zeros(3, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((3, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_all_batch(X, E, G, V, B.PROJECT_PSD)
    for k in range(3):
        E1, g1, v1 = s(X[k].contiguous(), B.PROJECT_PSD)
        assert torch.equal(g1, G[k]) and torch.equal(v1, V[k]) and rel_energy(float(E1.item()), float(E[k])) <= 1e-13
    c5 = W.make_c5(count=3, n=40)
    s5 = B.Sheet.from_sheet(c5[0], G3, G3)
    X = torch.stack([torch.from_numpy(q.x) for q in c5]).cuda()
    P = torch.from_numpy(np.stack([B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h)) for q in c5])).cuda()
    E = torch.zeros(3, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((3, s5.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s5.eval_all_batch_params(X, P, E, G, V, B.PROJECT_PSD)
    torch.cuda.synchronize()
    for k, q in enumerate(c5):
        _, Er, gr, vr, rp, ci, va = _oracle(q, B.PROJECT_PSD)
        assert_parity(float(E[k]), G[k].cpu().numpy(), V[k].cpu().numpy(), Er, gr, vr, what=f"g3 C5 item {k}",
                      hdiag=diag_block_norms(vr, rp, ci, 0, q.n_u), cmax=np.abs(q.x).max(), vabs=va)


def test_g3_c4_full_size_sampled_rows():
    """C4 (1024^2) under G3-FULL: 9.4 M points per rule, beyond the generic path's index packing, so only
    k_g3 runs it.  Sampled rows against narrow oracle slabs; energy = sum of GPU slab energies."""
    sh = W.make_c4()
    s = B.Sheet.from_sheet(sh, G3, G3)
    xd = torch.from_numpy(sh.x).cuda()
    E, g, v = s(xd, B.PROJECT_PSD)
    torch.cuda.synchronize()
    rp, ci = s.pattern()
    g, v = g.cpu().numpy(), v.cpu().numpy()
    for r0, r1 in [(0, 2), (600, 602), (1022, 1024)]:
        _, Er, gr, vr, orp, oci, va = _oracle(sh, B.PROJECT_PSD, r0, r1)
        a0, a1 = r0 * sh.n_u, r1 * sh.n_u
        assert np.array_equal(ci[rp[a0]:rp[a1]], oci)
        assert_parity(None, g[r0:r1], v[rp[a0]:rp[a1]], None, gr, vr, what=f"g3 C4 rows {r0}:{r1}",
                      hdiag=diag_block_norms(vr, orp, oci, r0, sh.n_u), cmax=np.abs(sh.x).max(), vabs=va)
    parts = 0.0
    for r0, r1 in [(0, 300), (300, 700), (700, 1024)]:
        parts += _gpu(B.Sheet.from_sheet(sh, G3, G3, row_begin=r0, row_end=r1), sh.x, B.PROJECT_PSD)[0]
    assert rel_energy(float(E.item()), parts) <= 1e-12
    with pytest.raises(B.BsfError):   # no generic fallback at this size
        s(xd, B.PROJECT_PSD | B.GENERIC_PATH)


def test_g3_cuda_graph_capture_and_replay():
    """The G3 launches (frame + interior instances + energy) capture into a CUDA graph after one warm call of
    the same batch size; replaying on new positions gives the direct call's outputs bit for bit."""
    sheets = [W.make_sheet(40, 1.0, 20 + k, n_modes=3, amp=5e-3) for k in range(2)]
    s = B.Sheet.from_sheet(sheets[0], G3, G3)
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    E = torch.zeros(2, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((2, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s.eval_all_batch(X, E, G, V, B.PROJECT_PSD, st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        s.eval_all_batch(X, E, G, V, B.PROJECT_PSD, st)
    X.copy_(torch.stack([torch.from_numpy(W.make_sheet(40, 1.0, 30 + k, n_modes=3, amp=5e-3).x) for k in range(2)]))
    g.replay()
    torch.cuda.synchronize()
    E2, G2, V2 = torch.zeros_like(E), torch.zeros_like(G), torch.zeros_like(V)
    s.eval_all_batch(X, E2, G2, V2, B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert torch.equal(G, G2) and torch.equal(V, V2) and torch.equal(E, E2)


def test_g3_graph_replay_after_other_batch_size():
    """a graph captured at batch size A must replay correctly after a direct call at batch size B
    (the interior row chunking differs between the two; nothing batch-size dependent lives in device memory)."""
    n, A, Bn = 64, 2, 48
    s = B.Sheet.from_sheet(W.make_sheet(n, 1.0, 50, n_modes=3, amp=5e-3), G3, G3)
    mk = lambda seeds: torch.stack([torch.from_numpy(W.make_sheet(n, 1.0, k, n_modes=3, amp=5e-3).x)
                                    for k in seeds]).cuda()
    X = mk(range(60, 60 + A))
    E = torch.zeros(A, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((A, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s.eval_all_batch(X, E, G, V, B.PROJECT_PSD, st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        s.eval_all_batch(X, E, G, V, B.PROJECT_PSD, st)
    XB = mk([70 + (k % 5) for k in range(Bn)])   # direct call at another batch size between capture and replay
    EB = torch.zeros(Bn, dtype=torch.float64, device="cuda")
    VB = torch.zeros((Bn, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_all_batch(XB, EB, None, VB, B.PROJECT_PSD)
    torch.cuda.synchronize()
    X.copy_(mk(range(80, 80 + A)))
    g.replay()
    torch.cuda.synchronize()
    E2, G2, V2 = torch.zeros_like(E), torch.zeros_like(G), torch.zeros_like(V)
    s.eval_all_batch(X, E2, G2, V2, B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert torch.equal(G, G2) and torch.equal(V, V2) and torch.equal(E, E2)
    # and the B-sized call itself is the per-item call
    e1 = torch.zeros(1, dtype=torch.float64, device="cuda")
    v1 = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_all_batch(XB[7:8].contiguous(), e1, None, v1, B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert torch.equal(v1[0], VB[7]) and torch.equal(e1[0], EB[7])


@pytest.mark.parametrize("n,slab", [(5, None), (6, None), (40, (20, 22)), (40, (0, 2)), (40, (38, 40))])
def test_g3_smallest_sheets_and_two_row_slabs(n, slab):
    """Edge cases: the smallest G3 sheets (S = 3, 4: every span is a boundary span, no interior class) and
    2-row slabs at the top, middle and bottom of a sheet."""
    sh = W.make_sheet(n, 1.0, 40 + n, n_modes=2, amp=5e-3)
    r0, r1 = slab if slab else (0, n)
    _, Er, gr, vr, rp, ci, va = _oracle(sh, B.PROJECT_PSD, r0, r1)
    s = B.Sheet.from_sheet(sh, G3, G3, row_begin=r0, row_end=r1)
    E, g, v = _gpu(s, sh.x, B.PROJECT_PSD)
    assert s.last_launch_count() <= 3
    assert_parity(E, g, v, Er, gr, vr, what=f"g3 n={n} slab={slab}", hdiag=diag_block_norms(vr, rp, ci, r0, sh.n_u),
                  cmax=np.abs(sh.x).max(), vabs=va)


def test_g3_incremental_potential():
    """bsf_eval_ip_batch on a G3-FULL handle (k_g3 + the incremental-potential epilogue) against the oracle's
    eval_ip under the same rule, with pinned control points."""
    sh = W.make_sheet(40, 1.0, 77, n_modes=3, amp=5e-3)
    R0, dt, grav = 0.15, 4e-3, np.array([0.0, -9.81, 0.5])
    pinned = np.zeros((sh.n_v, sh.n_u), bool)
    pinned[-1, :] = True
    mu = O.material_from_young(sh.E, sh.nu, sh.h)
    o = O.Oracle.from_sheet(sh, G3, G3, mu=mu)
    m = o.lumped_mass(R0)
    rng = np.random.default_rng(5)
    s = B.Sheet.from_sheet(sh, G3, G3)
    s.set_inertia(R0, dt, gravity=grav, pinned=pinned)
    xh = sh.x + rng.normal(0, 2e-3, sh.x.shape)
    X = torch.from_numpy(sh.x).cuda().unsqueeze(0).contiguous()
    XH = torch.from_numpy(xh).cuda().unsqueeze(0).contiguous()
    E = torch.zeros(1, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_ip_batch(X, XH, E, G, V, flags=B.PROJECT_PSD)
    torch.cuda.synchronize()
    Er, gr, vr = o.eval_ip(sh.x, xh, m, dt, grav, pinned, flags=O.FLAG_PROJECT)
    rp, ci = o.pattern()
    va = o.eval_ip(sh.x, xh, m, dt, grav, pinned, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    assert_parity(E[0].item(), G[0].cpu().numpy(), V[0].cpu().numpy(), Er, gr, vr, what="g3 ip",
                  hdiag=diag_block_norms(vr, rp, ci, 0, sh.n_u), cmax=np.abs(sh.x).max(), vabs=va)


@pytest.mark.parametrize("rules", [(0, 2), (2, 0), (1, 2)])
def test_mixed_rules_fall_back(rules):
    """G3-FULL for one energy only: k_g3 does not apply (both energies must be G3-FULL); the tile / generic
    path computes it, against the oracle under the same rule pair."""
    sh = W.make_sheet(24, 1.0, 61, n_modes=3, amp=5e-3)
    mr, br = rules
    mu = O.material_from_young(sh.E, sh.nu, sh.h)
    o = O.Oracle.from_sheet(sh, mr, br, mu=mu)
    Er, gr, vr = o.eval(sh.x, flags=O.FLAG_PROJECT)
    rp, ci = o.pattern()
    va = o.eval(sh.x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    s = B.Sheet.from_sheet(sh, mr, br)
    assert np.array_equal(s.pattern()[1], ci)
    E, g, v = _gpu(s, sh.x, B.PROJECT_PSD)
    assert_parity(E, g, v, Er, gr, vr, what=f"rules {rules}", hdiag=diag_block_norms(vr, rp, ci, 0, sh.n_u),
                  cmax=np.abs(sh.x).max(), vabs=va)
