"""GPU checks of the C-ABI's error reporting: BSF_E_SINGULAR_STRETCH.

A membrane point with |F e_beta| < 1e-12 makes the FBW energy undefined (its 1/|f_beta| terms)
clamps there, this library reports it: the kernel that owns the point's energy stores a code naming the point
into the handle's mapped host word, and the handle's next compute call (or bsf_poll_status after the stream
has synchronised) returns BSF_E_SINGULAR_STRETCH with the point's anchor span and batch item.
"""
import numpy as np
import pytest

import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_18867_b200 as B  # noqa: E402

SINGULAR = -5


@pytest.mark.parametrize("rules,path", [((0, 0), 0), ((0, 0), B.TILE_ONLY), ((0, 0), B.GENERIC_PATH),
                                        ((2, 2), 0), ((1, 1), 0)])
def test_singular_stretch_reported(rules, path):
    sh = W.make_sheet(40, 1.0, 3, n_modes=2, amp=5e-3)
    s = B.Sheet.from_sheet(sh, rules[0], rules[1])
    good = torch.from_numpy(sh.x).cuda()
    E, g, v = s.alloc_outputs()
    s.eval_all(good, E, g, v, B.PROJECT_PSD | path)
    torch.cuda.synchronize()
    s.poll_status()                                 # a regular state reports nothing
    # collapse one control-point row onto its neighbour: F e_2 vanishes on the knot line between them
    bad = sh.x.copy()
    bad[21] = bad[20]
    bad[22] = bad[20]
    s.eval_all(torch.from_numpy(bad).cuda(), E, g, v, B.PROJECT_PSD | path)   # asynchronous: accepted
    torch.cuda.synchronize()
    with pytest.raises(B.BsfError) as e:
        s.eval_all(good, E, g, v, B.PROJECT_PSD | path)                   # surfaced on the next call
    assert e.value.status == SINGULAR and "singular stretch" in str(e.value)
    s.eval_all(good, E, g, v, B.PROJECT_PSD | path)                       # consumed: the next call runs
    torch.cuda.synchronize()
    s.poll_status()
    assert np.isfinite(E.item())
    # poll after synchronising
    s.eval_all(torch.from_numpy(bad).cuda(), E, g, v, B.PROJECT_PSD | path)
    torch.cuda.synchronize()
    with pytest.raises(B.BsfError) as e:
        s.poll_status()
    assert e.value.status == SINGULAR
    s.poll_status()


def test_singular_stretch_names_batch_item():
    sheets = [W.make_sheet(40, 1.0, 10 + k, n_modes=2, amp=5e-3) for k in range(3)]
    s = B.Sheet.from_sheet(sheets[0])
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
    X[2, 30:33] = X[2, 30]
    E = torch.zeros(3, dtype=torch.float64, device="cuda")
    s.eval_all_batch(X, E, None, None, B.PROJECT_PSD)
    torch.cuda.synchronize()
    with pytest.raises(B.BsfError) as e:
        s.poll_status()
    assert "batch item 2" in str(e.value)
    assert np.isfinite(E[:2].cpu().numpy()).all()
