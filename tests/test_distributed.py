"""Multi-rank row-slab path on CPU (gloo): partition, halo exchange and slab assembly.

The compute on each rank is the oracle in slab mode (test infrastructure), so the test checks the
distributed host logic: after the 2-row halo exchange every rank holds exactly the rows it needs,
slab energies sum to the sheet energy and the slabs' gradient rows and Hessian block rows
concatenate bit for bit to the unpartitioned result.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

import workloads as W
from paper_2506_18867_b200 import distributed as D


def test_slab_bounds():
    for n_v, world in [(16, 1), (16, 2), (16, 3), (128, 8), (1024, 8), (9, 4), (1024, 5), (11, 3), (1024, 7),
                       (13, 6)]:
        b = D.partition_check(n_v, world)
        sizes = [r1 - r0 for r0, r1 in b]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.slab_bounds(5, 3)


def test_slab_bounds_edge_discount():
    """Edge slabs (which also carry the frame kernels) own fewer rows; the partition stays contiguous, complete
    and >= 2 rows per slab, and reduces to the balanced one for 1-2 ranks or discount 0."""
    for n_v, world in [(1024, 8), (1024, 4), (128, 3), (9, 4), (16, 3)]:
        d = D.edge_rows_discount(n_v, world)
        b = D.slab_bounds(n_v, world, d)
        assert b[0][0] == 0 and b[-1][1] == n_v and all(b[k][1] == b[k + 1][0] for k in range(world - 1))
        sizes = [r1 - r0 for r0, r1 in b]
        if d == 0:   # no discount: the balanced split
            assert b == D.slab_bounds(n_v, world)
            continue
        assert min(sizes) >= 2 and sizes[0] == sizes[-1] <= min(sizes[1:-1])
        mid = sizes[1:-1]
        assert max(mid) - min(mid) <= 1
    assert D.slab_bounds(1024, 8, 24)[0] == (0, 104) and D.slab_bounds(1024, 8, 24)[-1] == (920, 1024)
    assert D.slab_bounds(1024, 2, 24) == D.slab_bounds(1024, 2)
    assert D.slab_bounds(1024, 8, 0) == D.slab_bounds(1024, 8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, cfg):
    import pickle

    import torch
    import torch.distributed as dist

    import oracle as O
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sh = W.make_c1() if cfg == "C1" else W.make_c2(state=4)
        r0, r1 = D.slab_bounds(sh.n_v, world)[rank]
        lo, hi = D.halo_rows(r0, r1, sh.n_v)
        x = torch.from_numpy(D.numpy_slab(sh.x, r0, r1)).clone()
        x[: r0 - lo] = 0.0          # halos unknown before the exchange
        x[r1 - lo:] = 0.0
        x2 = x.clone()
        D.torch_halo_exchange(x, r0, r1, sh.n_v, rank, world)
        halo_ok = bool(np.array_equal(x.numpy(), sh.x[lo:hi]))
        # the library's own exchange plan (host-only handle of this slab; bsf_halo_plan), executed over gloo
        import paper_2506_18867_b200 as B
        hh = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1, device=-1)
        D.plan_halo_exchange(x2, hh.halo_plan(rank, world))
        halo_ok = halo_ok and bool(np.array_equal(x2.numpy(), sh.x[lo:hi]))
        o = O.Oracle.from_sheet(sh, r0=r0, r1=r1)
        E, g, v = o.eval(x.numpy(), flags=O.FLAG_PROJECT, threads=1)
        Et = torch.tensor([E], dtype=torch.float64)
        dist.all_reduce(Et)
        with open(os.path.join(outdir, f"r{rank}.pkl"), "wb") as f:
            pickle.dump(dict(halo_ok=halo_ok, E=E, Etot=float(Et.item()), g=g, v=v, rp=o.pattern()[0],
                             ci=o.pattern()[1]), f)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg", [(2, "C1"), (3, "C1"), (2, "C2")])
def test_gloo_slabs_reproduce_full_sheet(world, cfg):
    import pickle

    import torch.multiprocessing as mp

    import oracle as O
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), td, cfg), nprocs=world, join=True)
        res = [pickle.load(open(os.path.join(td, f"r{k}.pkl"), "rb")) for k in range(world)]
    sh = W.make_c1() if cfg == "C1" else W.make_c2(state=4)
    o = O.Oracle.from_sheet(sh)
    E, g, v = o.eval(sh.x, flags=O.FLAG_PROJECT, threads=1)
    rp, ci = o.pattern()
    assert all(r["halo_ok"] for r in res)
    assert abs(sum(r["E"] for r in res) - E) <= 1e-14 * E
    assert all(abs(r["Etot"] - E) <= 1e-14 * E for r in res)
    assert np.array_equal(np.concatenate([r["g"] for r in res]), g)
    assert np.array_equal(np.concatenate([r["v"] for r in res]), v)
    assert np.array_equal(np.concatenate([r["ci"] for r in res]), ci)
