"""GPU: contact pullback to the control points (Alg. 1)
against the oracle (oracle_contact_pullback, pinned in test_oracle_contact.py).

  positions      x^alpha = sum N_ij C^ij vs the oracle's weights, 1e-14 relative
  assemble       diagonal blocks (merged into the elastic values) + the off-diagonal contact BSR vs the oracle's
                 dense pulled-back Hessian, 1e-13 relative to its largest entry; the off-diagonal PATTERN exactly
                 (the set of nonzero off-diagonal blocks, rows ascending, columns strictly ascending); gradient
  determinism    two assemblies are bit-identical
  full size      C2 (128^2) with a 16K-vertex mesh and 40K pairs: H_cp y and the gradient vs the chain rule
                 evaluated by numpy with the oracle's weights (an independent route), 1e-12 relative
  Neumann        (D + B) x = b with D = inertia + projected elastic + contact diagonal, B = contact off-diagonal:
                 the residual with the ORACLE's pulled-back matrix <= 1e-10 |b|
  edge cases     no pairs, all-obstacle pairs, a duplicated pair, vertices on knot lines and on the domain
                 boundary, an out-of-range vertex index, a vertex outside the domain, a slab handle
Tolerance: the pullback is a sum of products of nonnegative weights with the pair blocks; the library sums
vertex-pair blocks first and multiplies by the two weights after (Alg. 1's two levels), the oracle multiplies
first, so the two differ by rounding only: a few ulps of the largest block times the number of summed terms.
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


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _assemble(s, cs, vals=None, grad=None, with_g=True):
    s.contact_mesh(cs.uv)
    nnz = s.contact_assemble(_cuda(cs.verts), _cuda(cs.H), _cuda(cs.g) if with_g else None, grad, vals)
    torch.cuda.synchronize()
    return nnz


def _diag_of(s, V):
    """3x3 diagonal blocks of handle-pattern values V [nnzb, 3, 3] -> [n_cp, 3, 3]."""
    rp, ci = s.pattern()
    pos = [rp[a] + int(np.searchsorted(ci[rp[a]:rp[a + 1]], a)) for a in range(len(rp) - 1)]
    return V.cpu().numpy()[pos]


def _gpu_dense(s, V):
    n = s.n_u * s.n_v
    rp, ci, va = (t.cpu().numpy() for t in s.contact_get())
    Bm = sp.bsr_matrix((va, ci, rp), shape=(3 * n, 3 * n)).toarray() if len(ci) else np.zeros((3 * n, 3 * n))
    D = _diag_of(s, V)
    for a in range(n):
        Bm[3 * a:3 * a + 3, 3 * a:3 * a + 3] += D[a]
    return Bm, (rp, ci, va)


CASES = {
    "small": dict(n=9, res=2, pairs=60, obs=0.5),
    "c1": dict(n=16, res=3, pairs=1500, obs=0.3),
    "coarse": dict(n=12, res=1, pairs=400, obs=0.0),
    "one": dict(n=9, res=4, pairs=1, obs=0.0),
    "obstacle_only": dict(n=10, res=2, pairs=300, obs=1.0),
}


@pytest.mark.parametrize("case", list(CASES))
def test_assemble_matches_oracle(case):
    c = CASES[case]
    sh = W.make_sheet(c["n"], 1.0, 7, n_modes=2, amp=5e-3)
    cs = W.make_contact(sh, c["res"], c["pairs"], seed=11, obstacle_frac=c["obs"])
    o = O.Oracle.from_sheet(sh)
    Hcp, gcp = o.contact_pullback(cs.uv, cs.verts, cs.H, cs.g)
    s = B.Sheet.from_sheet(sh)
    V = torch.zeros((s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    G = torch.zeros((sh.n_v, sh.n_u, 3), dtype=torch.float64, device="cuda")
    nnz = _assemble(s, cs, V, G)
    Hg, (rp, ci, va) = _gpu_dense(s, V)
    scale = np.abs(Hcp).max()
    assert np.max(np.abs(Hg - Hcp)) <= 1e-13 * scale, np.max(np.abs(Hg - Hcp)) / scale
    # only the diagonal blocks of the elastic values were touched
    off = V.cpu().numpy().copy()
    rpe, cie = s.pattern()
    for a in range(len(rpe) - 1):
        for k in range(rpe[a], rpe[a + 1]):
            if cie[k] != a:
                assert not off[k].any()
    # the off-diagonal pattern, exactly: the nonzero off-diagonal blocks of the oracle's matrix
    n = sh.n_u * sh.n_v
    blk = np.abs(Hcp.reshape(n, 3, n, 3)).max(axis=(1, 3)) > 0
    np.fill_diagonal(blk, False)
    want = [(i, j) for i, j in zip(*np.nonzero(blk))]
    got = [(a, int(j)) for a in range(n) for j in ci[rp[a]:rp[a + 1]]]
    assert got == want and nnz == len(want) == rp[-1]
    np.testing.assert_allclose(G.cpu().numpy(), gcp, rtol=0, atol=1e-13 * np.abs(gcp).max())


def test_positions_match_oracle_weights():
    sh = W.make_c1()
    cs = W.make_contact(sh, 3, 10, seed=1)
    Wt = O.Oracle.from_sheet(sh).contact_weights(cs.uv)
    s = B.Sheet.from_sheet(sh)
    s.contact_mesh(cs.uv)
    xv = s.contact_positions(_cuda(sh.x)).cpu().numpy()
    ref = Wt @ sh.x.reshape(-1, 3)
    assert np.max(np.abs(xv - ref)) <= 1e-14 * np.abs(ref).max()


def test_deterministic_and_duplicate_pairs():
    sh = W.make_sheet(12, 1.0, 3)
    cs = W.make_contact(sh, 2, 500, seed=5)
    # duplicate a third of the pairs: their blocks must simply add
    k = len(cs.verts) // 3
    dup = W.ContactSet(cs.uv, np.concatenate([cs.verts, cs.verts[:k]]), np.concatenate([cs.H, cs.H[:k]]),
                       np.concatenate([cs.g, cs.g[:k]]))
    s = B.Sheet.from_sheet(sh)
    outs = []
    for _ in range(2):
        V = torch.zeros((s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
        G = torch.zeros((sh.n_v, sh.n_u, 3), dtype=torch.float64, device="cuda")
        _assemble(s, dup, V, G)
        outs.append((V, G) + s.contact_get())
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    Hcp, gcp = O.Oracle.from_sheet(sh).contact_pullback(dup.uv, dup.verts, dup.H, dup.g)
    Hg, _ = _gpu_dense(s, outs[0][0])
    assert np.max(np.abs(Hg - Hcp)) <= 1e-13 * np.abs(Hcp).max()


def test_full_size_c2_against_chain_rule():
    """C2's 128^2 sheet, a 16K-vertex contact mesh, 40K pairs: too large for the oracle's dense matrix, so the
    pulled-back Hessian is checked through its action, y = W^T (H_lin (W x)), with the oracle's weights W."""
    sh = W.make_c2(state=0)
    cs = W.make_contact(sh, 1, 40000, seed=21)
    o = O.Oracle.from_sheet(sh)
    n = sh.n_u * sh.n_v
    rows = []
    for c0 in range(0, len(cs.uv), 2000):
        rows.append(sp.csr_matrix(o.contact_weights(cs.uv[c0:c0 + 2000])))
    Wsp = sp.vstack(rows).tocsr()
    rng = np.random.default_rng(4)
    x = rng.normal(size=(n, 3))
    xv = Wsp @ x
    yv = np.zeros_like(xv)
    gv = np.zeros_like(xv)
    for sa in range(4):
        a = cs.verts[:, sa]
        ma = a >= 0
        np.add.at(gv, a[ma], cs.g[ma, 3 * sa:3 * sa + 3])
        for sb in range(4):
            b = cs.verts[:, sb]
            m = ma & (b >= 0)
            np.add.at(yv, a[m], np.einsum("cij,cj->ci", cs.H[m, 3 * sa:3 * sa + 3, 3 * sb:3 * sb + 3], xv[b[m]]))
    y_ref = Wsp.T @ yv
    g_ref = Wsp.T @ gv
    s = B.Sheet.from_sheet(sh)
    V = torch.zeros((s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    G = torch.zeros((sh.n_v, sh.n_u, 3), dtype=torch.float64, device="cuda")
    _assemble(s, cs, V, G)
    rp, ci, va = (t.cpu().numpy() for t in s.contact_get())
    Bm = sp.bsr_matrix((va, ci, rp), shape=(3 * n, 3 * n))
    y = (Bm @ x.reshape(-1)).reshape(n, 3) + np.einsum("aij,aj->ai", _diag_of(s, V), x)
    assert np.max(np.abs(y - y_ref)) <= 1e-12 * np.abs(y_ref).max()
    assert np.max(np.abs(G.cpu().numpy().reshape(n, 3) - g_ref)) <= 1e-12 * np.abs(g_ref).max()
    # structure: rows ascending, columns strictly ascending, no diagonal blocks
    for a in range(0, n, 97):
        cols = ci[rp[a]:rp[a + 1]]
        assert np.all(np.diff(cols) > 0) and a not in cols


def _ip_values(s, sh, R0=0.15, dt=2e-3):
    rng = np.random.default_rng(3)
    xhat = sh.x + rng.normal(0, 1e-3, sh.x.shape)
    s.set_inertia(R0, dt, gravity=np.array([0.0, 0.0, -9.81]))
    X = _cuda(sh.x).unsqueeze(0).contiguous()
    XH = _cuda(xhat).unsqueeze(0).contiguous()
    E = torch.zeros(1, dtype=torch.float64, device="cuda")
    G = torch.zeros_like(X)
    V = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    s.eval_ip_batch(X, XH, E, G, V, B.PROJECT_PSD)
    torch.cuda.synchronize()
    return G[0].clone(), V[0].clone()


@pytest.mark.parametrize("scale", [0.01, 0.1])
def test_contact_neumann_solve(scale):
    sh = W.make_c1()
    cs = W.make_contact(sh, 2, 400, seed=8, obstacle_frac=0.2, scale=scale)
    s = B.Sheet.from_sheet(sh)
    G, V = _ip_values(s, sh)
    rpe, cie = s.pattern()
    n = sh.n_u * sh.n_v
    A_el = sp.bsr_matrix((V.cpu().numpy(), cie, rpe), shape=(3 * n, 3 * n)).toarray()
    Hcp, gcp = O.Oracle.from_sheet(sh).contact_pullback(cs.uv, cs.verts, cs.H, cs.g)
    _assemble(s, cs, V, G)          # D = inertia + elastic + contact diagonal; gradient += contact gradient
    s.chol_factor(V)
    b = -G
    x, gate, terms = s.contact_neumann_solve(b, max_terms=200, rtol=1e-14)
    torch.cuda.synchronize()
    assert 0.0 < gate < 1.0 and terms >= 2
    A = A_el + Hcp
    bb = b.cpu().numpy().reshape(-1)
    res = np.linalg.norm(bb - A @ x.cpu().numpy().reshape(-1)) / np.linalg.norm(bb)
    assert res <= 1e-10, (res, gate, terms)
    ref = spla.spsolve(sp.csc_matrix(A), bb)
    assert np.linalg.norm(x.cpu().numpy().reshape(-1) - ref) <= 1e-9 * np.linalg.norm(ref)


def test_contact_neumann_gate_refuses_strong_contact():
    sh = W.make_c1()
    cs = W.make_contact(sh, 2, 400, seed=8, obstacle_frac=0.0, scale=1e5)
    s = B.Sheet.from_sheet(sh)
    G, V = _ip_values(s, sh)
    _assemble(s, cs, V, G)
    s.chol_factor(V)
    with pytest.raises(B.BsfError):
        s.contact_neumann_solve(-G)


def test_contact_edge_cases():
    sh = W.make_sheet(9, 1.0, 2)
    s = B.Sheet.from_sheet(sh)
    verts = torch.zeros((1, 4), dtype=torch.int32, device="cuda")
    H = torch.zeros((1, 12, 12), dtype=torch.float64, device="cuda")
    with pytest.raises(B.BsfError):          # no mesh yet
        s.contact_assemble(verts, H)
    S = sh.n_u - 2
    with pytest.raises(B.BsfError):          # a vertex outside the parameter domain
        s.contact_mesh(np.array([[0.5, S + 1e-9]]))
    # vertices on the domain corners / knot lines, no pairs: empty matrix, nothing touched
    s.contact_mesh(np.array([[0.0, 0.0], [S, S], [3.0, 4.0], [S, 0.0]]))
    V = torch.zeros((s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    G = torch.zeros((sh.n_v, sh.n_u, 3), dtype=torch.float64, device="cuda")
    assert s.contact_assemble(verts[:0], H[:0], None, G, V) == 0
    rp, ci, va = s.contact_get()
    assert int(rp.abs().sum()) == 0 and len(ci) == 0 and not V.any() and not G.any()
    with pytest.raises(B.BsfError):          # vertex index >= n_vert
        s.contact_assemble(torch.tensor([[0, 1, 4, -1]], dtype=torch.int32, device="cuda"), H)
    with pytest.raises(ValueError):          # wrong dtype
        s.contact_assemble(verts.long(), H)
    # corner vertices: a single control point each (weight 1), so a pair of the two corners couples the two
    # corner control points: the pattern is structural (the pair's topology), an identity H gives zero blocks
    Hs = torch.eye(12, dtype=torch.float64, device="cuda").unsqueeze(0).contiguous()
    nnz = s.contact_assemble(torch.tensor([[0, 1, -1, -1]], dtype=torch.int32, device="cuda"), Hs, None, None, V)
    n = sh.n_u * sh.n_v
    rp, ci, va = (t.cpu().numpy() for t in s.contact_get())
    assert nnz == 2 and list(ci) == [n - 1, 0] and not va.any()
    D = _diag_of(s, V)
    np.testing.assert_array_equal(D[0], np.eye(3))
    np.testing.assert_array_equal(D[n - 1], np.eye(3))
    assert not np.delete(D, [0, n - 1], axis=0).any()
    slab = B.Sheet.from_sheet(sh, row_begin=2, row_end=5)
    with pytest.raises(B.BsfError):
        slab.contact_mesh(np.array([[0.5, 0.5]]))


_KEYS64 = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle as O, workloads as W, paper_2506_18867_b200 as B
import scipy.sparse as sp
sh = W.make_sheet(12, 1.0, 4, n_modes=2, amp=5e-3)
cs = W.make_contact(sh, 2, 400, seed=2, obstacle_frac=0.2)
Hcp, gcp = O.Oracle.from_sheet(sh).contact_pullback(cs.uv, cs.verts, cs.H, cs.g)
s = B.Sheet.from_sheet(sh)
s.contact_mesh(cs.uv)
V = torch.zeros((s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
G = torch.zeros((sh.n_v, sh.n_u, 3), dtype=torch.float64, device="cuda")
s.contact_assemble(torch.from_numpy(cs.verts).cuda(), torch.from_numpy(cs.H).cuda(), torch.from_numpy(cs.g).cuda(), G, V)
torch.cuda.synchronize()
n = sh.n_u * sh.n_v
rp, ci, va = (t.cpu().numpy() for t in s.contact_get())
Hg = sp.bsr_matrix((va, ci, rp), shape=(3 * n, 3 * n)).toarray()
rpe, cie = s.pattern()
Vn = V.cpu().numpy()
for a in range(n):
    Hg[3 * a:3 * a + 3, 3 * a:3 * a + 3] += Vn[rpe[a] + int(np.searchsorted(cie[rpe[a]:rpe[a + 1]], a))]
print("ERR", np.max(np.abs(Hg - Hcp)) / np.abs(Hcp).max(), np.max(np.abs(G.cpu().numpy() - gcp)) / np.abs(gcp).max())
"""


def test_64bit_sort_keys():
    """The sort keys are 32-bit when their sentinel fits (every test sheet here), else 64-bit (C4-size sheets,
    meshes of > 65535 vertices); BSF_CONTACT_KEYS64=1 forces the 64-bit path (read once per process: run in a
    subprocess) against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, BSF_REBUILD="0", BSF_CONTACT_KEYS64="1")
    r = subprocess.run([sys.executable, "-c", _KEYS64 % root], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    err, gerr = map(float, r.stdout.split("ERR")[1].split())
    assert err <= 1e-13 and gerr <= 1e-13, (err, gerr)
