"""Multi-rank row slabs on >= 2 GPUs: torchrun launches one rank per GPU,
each rank runs the library's NCCL halo exchange overlapped with its interior rows (bsf_eval_all_slab) and the
energy all-reduce (bsf_allreduce_sum).  The gathered slabs must equal the one-GPU whole-sheet call bit for bit
(gradient and every Hessian block; the energy to 1e-12) and the oracle within the north star's 1e-10.
Skipped when fewer than 2 GPUs are visible (the driver's GPU runs use one GPU; the exchange plan itself is
covered on CPU by tests/test_distributed.py over gloo)."""
import os
import socket
import subprocess
import sys
import tempfile

import numpy as np
import pytest

import oracle as O
import workloads as W
from parity import assert_parity, diag_block_norms, rel_energy

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2506_18867_b200 as B  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,cfg", [(2, "C2"), (2, "C4")])
def test_nccl_slabs_match_single_gpu_and_oracle(world, cfg):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (found {torch.cuda.device_count()})")
    with tempfile.TemporaryDirectory() as td:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr", "127.0.0.1", "--master-port", str(_port()),
               os.path.join(ROOT, "tests", "_multirank_worker.py"), td, cfg]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        res = [np.load(os.path.join(td, f"r{k}.npz")) for k in range(world)]
        res = [{k: z[k] for k in z.files} for z in res]
    assert all(bool(z["halo_ok"]) for z in res)
    sh = W.make_c4() if cfg == "C4" else W.make_c2(state=6)
    s = B.Sheet.from_sheet(sh)
    E1, g1, v1 = s(torch.from_numpy(sh.x).cuda(), B.PROJECT_PSD)
    torch.cuda.synchronize()
    g1, v1 = g1.cpu().numpy(), v1.cpu().numpy()
    rp, ci = s.pattern()
    g = np.concatenate([z["g"] for z in res])
    v = np.concatenate([z["v"] for z in res])
    assert np.array_equal(g, g1) and np.array_equal(v, v1)
    for z in res:   # every rank holds the all-reduced total
        assert rel_energy(float(z["E"][0]), float(E1.item())) <= 1e-12
    o = O.Oracle.from_sheet(sh)
    Er, gr, vr = o.eval(sh.x, flags=O.FLAG_PROJECT)
    va = o.eval(sh.x, flags=O.FLAG_PROJECT | O.FLAG_ABS_SUM, energy=False, gradient=False)[2]
    assert_parity(float(res[0]["E"][0]), g, v, Er, gr, vr, what=f"{world} ranks {cfg}",
                  hdiag=diag_block_norms(vr, rp, ci, 0, sh.n_u), cmax=np.abs(sh.x).max(), vabs=va)
