"""C4 at N = 8 (row slabs with the bench's edge discount): one rank's slab call timed alone for the first (edge)
and a middle rank, under the current core chunking or BSF_CORE_NCH = n (read once per process); SLAB_DISCOUNT overrides the edge
discount, BSF_SIDE_STREAMS = 2 puts the corner and band kernels on two side streams."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402
from paper_2506_18867_b200.distributed import edge_rows_discount, slab_bounds  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
sh = W.make_c4()
disc = int(os.environ["SLAB_DISCOUNT"]) if os.environ.get("SLAB_DISCOUNT") else edge_rows_discount(sh.n_v, N)
bounds = slab_bounds(sh.n_v, N, disc)
out = {"N": N, "nch": os.environ.get("BSF_CORE_NCH"), "side": os.environ.get("BSF_SIDE_STREAMS"), "discount": disc}
for rank in (0, N // 2):
    r0, r1 = bounds[rank]
    s = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1)
    x = torch.from_numpy(np.ascontiguousarray(sh.x[s.x_row_begin:s.x_row_end])).cuda()
    E, g, v = s.alloc_outputs()
    for _ in range(3):
        s.eval_all(x, E, g, v, B.PROJECT_PSD)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.set_kernel_timing(20)
    a.record()
    for _ in range(20):
        s.eval_all(x, E, g, v, B.PROJECT_PSD)
    b.record()
    torch.cuda.synchronize()
    c, bd = s.kernel_timing(20)
    out[f"rank{rank}_rows"] = r1 - r0
    out[f"rank{rank}_call_us"] = a.elapsed_time(b) / 20 * 1e3
    out[f"rank{rank}_core_us"] = float(np.median(c)) * 1e3
    out[f"rank{rank}_band_us"] = float(np.median(bd)) * 1e3
    s.close()
print(json.dumps(out), flush=True)
