"""Worker of tests/test_gpu_multirank.py (launched by torch.distributed.run, one rank per GPU): the library's
NCCL communicator, bsf_eval_all_slab (halo exchange overlapped with the interior rows) and
bsf_allreduce_sum on one row slab of a sheet; writes the rank's outputs to <outdir>/r<rank>.npz."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(outdir, cfg):
    import torch
    import torch.distributed as dist

    import paper_2506_18867_b200 as B
    import workloads as W
    from paper_2506_18867_b200 import distributed as D
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        sh = W.make_c4() if cfg == "C4" else W.make_c2(state=6)
        comm = D.NcclComm(rank, world, local)
        slab = D.SlabSheet(sh, rank, world, device=local, comm=comm)
        slab.load_owned(torch.from_numpy(np.ascontiguousarray(sh.x[slab.r0:slab.r1])).cuda())
        # halo rows start as garbage: only the exchange can fill them
        slab.x[:slab.r0 - slab.lo].fill_(7.0)
        slab.x[slab.r1 - slab.lo:].fill_(7.0)
        for _ in range(2):
            E, g, v = slab.assemble(B.PROJECT_PSD)
        torch.cuda.synchronize()
        halo = slab.x.cpu().numpy()
        np.savez(os.path.join(outdir, f"r{rank}.npz"), r0=slab.r0, r1=slab.r1, E=E.cpu().numpy(), g=g.cpu().numpy(),
                 v=v.cpu().numpy(), halo_ok=np.array_equal(halo, sh.x[slab.lo:slab.hi]))
        comm.close()
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "C2")
