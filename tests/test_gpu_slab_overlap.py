"""GPU: the halo-overlapped slab call (bsf_eval_all_slab).  On one GPU the exchange itself cannot run, so the
split schedule (interior core rows first, then the boundary rows, bands and corners after the `ready`
event) is forced with BSF_SLAB_SPLIT and compared with the plain call and with the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
import oracle as O, workloads as W, paper_2506_18867_b200 as B
from parity import assert_parity, diag_block_norms
sh = W.make_c2(state=6)
for r0, r1 in [(0, 128), (40, 90), (0, 64), (64, 128)]:
    s = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1)
    x = torch.from_numpy(np.ascontiguousarray(sh.x[s.x_row_begin:s.x_row_end])).cuda()
    E1, g1, v1 = s.alloc_outputs(); E2, g2, v2 = s.alloc_outputs()
    s.eval_all(x, E1, g1, v1, B.PROJECT_PSD)
    s.eval_all_slab(x, E2, g2, v2, flags=B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert s.last_launch_count() >= 3, s.last_launch_count()
    assert torch.equal(g1, g2) and torch.equal(v1, v2), (r0, r1)
    assert abs(E1.item() - E2.item()) <= 1e-13 * abs(E1.item())
    # partial outputs on the split schedule: energy only (k_core_energy per row range), gradient only
    E3 = torch.zeros_like(E1); g3 = torch.zeros_like(g1)
    s.eval_all_slab(x, E3, None, None, flags=B.PROJECT_PSD)
    s.eval_all_slab(x, None, g3, None, flags=B.PROJECT_PSD)
    torch.cuda.synchronize()
    assert abs(E3.item() - E1.item()) <= 1e-13 * abs(E1.item()), (r0, r1, E3.item(), E1.item())
    assert torch.equal(g3, g1), (r0, r1)
    o = O.Oracle.from_sheet(sh, r0=r0, r1=r1)
    Er, gr, vr = o.eval(sh.x, flags=O.FLAG_PROJECT)
    rp, ci = o.pattern()
    va = o.eval(sh.x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    assert_parity(E2.item(), g2.cpu().numpy(), v2.cpu().numpy(), Er, gr, vr, what=f"slab {r0}-{r1}",
                  hdiag=diag_block_norms(vr, rp, ci, r0, sh.n_u), cmax=np.abs(sh.x).max(), vabs=va)
print("ok")
'''


def test_split_schedule_matches_plain_call_and_oracle():
    env = dict(os.environ, BSF_SLAB_SPLIT="1", BSF_REBUILD="0")
    r = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + SCRIPT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
