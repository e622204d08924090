"""Row-slab sharding of one sheet across ranks.

Each rank owns control-point rows [r0, r1) and keeps positions for rows [r0-2, r1+2) (a 2-row halo
from each neighbour, the reach of a 3-row stencil).  Per assembly call:
  1. halo exchange of 2 rows per neighbour (NCCL send/recv through the library, or
     torch.distributed for backends the library does not drive, e.g. gloo in the CPU tests);
  2. the rank's own fused kernels produce its block rows, gradient rows and its partial energy;
  3. one 8-byte sum all-reduce of the energy.
No Hessian or gradient data crosses ranks: the <= 2 rows of quadrature points shared by two slabs
are recomputed on both (their contributions to each slab's rows are disjoint).
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def slab_bounds(n_v: int, world: int, edge_discount: int = 0):
    """Contiguous row slabs; every slab owns >= 2 rows (the halo exchange sends 2 rows).

    edge_discount = 0: balanced.  > 0 (world >= 3): the first and last slab own that many rows fewer than
    the balanced share, the middle slabs share the difference.  The edge slabs also carry the sheet's frame
    (the edge bands and corners, whose kernels take SMs beside the interior kernel), so equal rows are not
    equal time; `edge_rows_discount` gives the value measured for the fused path."""
    if world < 1 or n_v < 2 * world:
        raise ValueError(f"cannot split {n_v} rows into {world} slabs of >= 2 rows")
    if edge_discount < 0:
        raise ValueError("edge_discount must be >= 0")
    base = n_v // world
    d = min(edge_discount, max(0, base - 2)) if world >= 3 else 0
    if d == 0:   # balanced: the plain divmod split (slab sizes differ by at most one row)
        b2, e2 = divmod(n_v, world)
        sizes = [b2 + (1 if k < e2 else 0) for k in range(world)]
    else:
        sizes = [0] * world
        sizes[0] = sizes[-1] = base - d
        mb, mx = divmod(n_v - 2 * (base - d), world - 2)
        for k in range(1, world - 1):
            sizes[k] = mb + (1 if k - 1 < mx else 0)
    out, r = [], 0
    for n in sizes:
        out.append((r, r + n))
        r += n
    assert r == n_v and all(b - a >= 2 for a, b in out)
    return out


def edge_rows_discount(n_v: int, world: int) -> int:
    """Rows taken off each edge slab of the fused path.  Measured (B200, C4, scripts/slab_nch_probe.py with the
    one-wave core chunking and the corner / band kernels on two side streams): at N <= 4 the edge slabs' extra
    corner and band work hides beside their interior kernel (N = 4 balanced: edge 140 us, middle 142 us), so the
    split is balanced; at N = 8 an edge slab takes its interior in 3 chunks (its band kernel needs the SMs) and
    sheds 24 rows (edge 104 rows 86-92 us, middle 136 rows 88-90 us).  At most a quarter of the balanced share."""
    if world <= 4:
        return 0
    return min(24, (n_v // world) // 4)


def halo_rows(r0: int, r1: int, n_v: int):
    """Row range [lo, hi) of a slab's position buffer."""
    return max(0, r0 - 2), min(n_v, r1 + 2)


def torch_halo_exchange(x_local, r0: int, r1: int, n_v: int, rank: int, world: int, group=None):
    """Exchange the 2-row halos of x_local ([hi-lo, n_u, 3], contiguous) with torch.distributed
    point-to-point ops (any backend).  Sends the first / last two owned rows to rank-1 / rank+1."""
    import torch.distributed as dist
    lo, hi = halo_rows(r0, r1, n_v)
    nlo, nhi = r0 - lo, hi - r1
    ops = []
    if rank > 0 and nlo > 0:
        ops.append(dist.P2POp(dist.isend, x_local[r0 - lo:r0 - lo + nlo].contiguous(), rank - 1, group))
        recv_lo = x_local[0:nlo]
        ops.append(dist.P2POp(dist.irecv, recv_lo, rank - 1, group))
    if rank < world - 1 and nhi > 0:
        ops.append(dist.P2POp(dist.isend, x_local[r1 - nhi - lo:r1 - lo].contiguous(), rank + 1, group))
        recv_hi = x_local[r1 - lo:r1 - lo + nhi]
        ops.append(dist.P2POp(dist.irecv, recv_hi, rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return x_local


def plan_halo_exchange(x_local, plan, group=None):
    """Execute the LIBRARY's halo plan (bsf_halo_plan: [(peer, send_off, recv_off, count)] x 2, in doubles of the
    position buffer) with torch.distributed point-to-point ops on any backend (gloo in the CPU tests; the NCCL
    path executes the same plan inside bsf_halo_exchange)."""
    import torch.distributed as dist
    flat = x_local.view(-1)
    ops = []
    for peer, so, ro, n in plan:
        if peer < 0 or n == 0:
            continue
        ops.append(dist.P2POp(dist.isend, flat[so:so + n].contiguous(), int(peer), group))
        ops.append(dist.P2POp(dist.irecv, flat[ro:ro + n], int(peer), group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    return x_local


class NcclComm:
    """NCCL communicator owned by the library (ranks = slabs in row order).  The unique id is
    broadcast over the default torch.distributed group."""

    def __init__(self, rank: int, world: int, device: int):
        import torch
        import torch.distributed as dist

        from . import _check, lib
        L = lib()
        buf = (C.c_char * 128)()
        if rank == 0:
            _check(L.bsf_nccl_get_unique_id(C.cast(buf, C.c_void_p)))
        obj = [bytes(buf) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        idb = (C.c_char * 128).from_buffer_copy(obj[0])
        comm = C.c_void_p()
        _check(L.bsf_nccl_comm_init(world, C.cast(idb, C.c_void_p), rank, device, C.byref(comm)))
        self.comm, self.rank, self.world = comm, rank, world
        torch.cuda.synchronize(device)

    def close(self):
        from . import lib
        if self.comm:
            lib().bsf_nccl_comm_destroy(self.comm)
            self.comm = None


class SlabSheet:
    """One rank's slab of a sheet: handle, position buffer with halos, outputs."""

    def __init__(self, sh, rank: int, world: int, device: int = 0, comm: NcclComm | None = None, material=None,
                 membrane_rule=0, bending_rule=0, edge_discount: int = 0):
        import torch

        from . import Sheet
        self.r0, self.r1 = slab_bounds(sh.n_v, world, edge_discount)[rank]
        self.lo, self.hi = halo_rows(self.r0, self.r1, sh.n_v)
        self.rank, self.world, self.comm = rank, world, comm
        self.n_u, self.n_v = sh.n_u, sh.n_v
        self.h = Sheet.from_sheet(sh, membrane_rule, bending_rule, row_begin=self.r0, row_end=self.r1,
                                  device=device, material=material)
        dev = torch.device("cuda", device)
        self.x = torch.zeros(self.h.x_shape(), dtype=torch.float64, device=dev)
        self.E, self.g, self.v = self.h.alloc_outputs()

    def load_owned(self, x_full_rows):
        """Copy the owned rows (global rows [r0, r1)) into the position buffer (halo untouched)."""
        self.x[self.r0 - self.lo:self.r1 - self.lo].copy_(x_full_rows, non_blocking=True)

    def exchange(self, stream=None):
        from . import _check, _stream, lib
        if self.world == 1:
            return
        if self.comm is None:
            plan_halo_exchange(self.x, self.h.halo_plan(self.rank, self.world))
            return
        _check(lib().bsf_halo_exchange(self.h._h, C.c_void_p(self.x.data_ptr()), self.comm.comm, self.rank,
                                       self.world, _stream(stream)))

    def assemble(self, flags=1, stream=None, reduce_energy=True):
        """Halo exchange, local fused assembly, energy all-reduce.  Returns (E_total[1], g, vals)."""
        from . import _check, _stream, lib
        if self.comm is not None or self.world == 1:
            # library communicator: the exchange overlaps the assembly of the interior rows
            self.h.eval_all_slab(self.x, self.E, self.g, self.v, comm=self.comm.comm if self.comm else None,
                                 rank=self.rank, nranks=self.world, flags=flags, stream=stream)
        else:
            self.exchange(stream)
            self.h.eval_all(self.x, self.E, self.g, self.v, flags, stream)
        if reduce_energy and self.world > 1:
            if self.comm is not None:
                _check(lib().bsf_allreduce_sum(C.c_void_p(self.E.data_ptr()), 1, self.comm.comm, _stream(stream)))
            else:
                import torch.distributed as dist
                dist.all_reduce(self.E)
        return self.E, self.g, self.v


def partition_check(n_v: int, world: int):
    """Host-side invariants of the partition (used by the CPU tests)."""
    b = slab_bounds(n_v, world)
    assert b[0][0] == 0 and b[-1][1] == n_v
    assert all(b[k][1] == b[k + 1][0] for k in range(world - 1))
    assert all(r1 - r0 >= 2 for r0, r1 in b)
    return b


def numpy_slab(x_full: np.ndarray, r0: int, r1: int):
    lo, hi = halo_rows(r0, r1, x_full.shape[0])
    return np.ascontiguousarray(x_full[lo:hi])
