"""One-GPU evidence for the C4 strong-scaling row: the compute time of ONE rank's slab of a
1024^2 sheet at N = 1, 2, 4, 8 (slab_bounds(1024, N, d) for the balanced partition and the edge discount d the
bench uses; the slowest of the first, middle and last rank), each rank
timed alone on this GPU with CUDA events (bsf_eval_all on a slab handle, no exchange).  The N-GPU step is
at least max over ranks of this time plus the halo exchange that the library overlaps with the interior
rows; this prints the compute-only efficiency bound T1 / (N * T_N) = T1 / (N * slab time).  No rank waits
on another (nothing here stands in for a multi-GPU run)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import workloads as W
import paper_2506_18867_b200 as B
from paper_2506_18867_b200.distributed import slab_bounds


def time_call(s, x, flags, reps=20):
    E, g, v = s.alloc_outputs()
    for _ in range(3):
        s.eval_all(x, E, g, v, flags)
    torch.cuda.synchronize()
    t = []
    for _ in range(5):   # back-to-back calls (as in a time loop): host launch cost overlaps the device work
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            s.eval_all(x, E, g, v, flags)
        b.record()
        b.synchronize()
        t.append(a.elapsed_time(b) / reps)
    return float(np.median(t))


sh = W.make_c4()
rows = []
t1 = None
from paper_2506_18867_b200.distributed import edge_rows_discount

for N in (1, 2, 4, 8):
  for disc in sorted({0, edge_rows_discount(sh.n_v, N)}):
    bounds = slab_bounds(sh.n_v, N, disc)
    worst = 0.0
    for rank in sorted({0, N // 2, N - 1}):
        r0, r1 = bounds[rank]
        s = B.Sheet.from_sheet(sh, row_begin=r0, row_end=r1)
        x = torch.from_numpy(np.ascontiguousarray(sh.x[s.x_row_begin:s.x_row_end])).cuda()
        ms = time_call(s, x, B.PROJECT_PSD)
        worst = max(worst, ms)
        s.close()
    t1 = worst if N == 1 else t1
    row = {"N": N, "edge_discount": disc, "rows_edge_mid": [bounds[0][1] - bounds[0][0], bounds[N // 2][1] - bounds[N // 2][0]],
           "max_rank_ms": round(worst, 4), "compute_efficiency_bound": round(t1 / (N * worst), 3)}
    rows.append(row)
    print(json.dumps(row), flush=True)
if len(sys.argv) > 1:
    json.dump({"config": "C4 1024^2, PSD, reduced rules; one rank's slab timed alone per N", "rows": rows},
              open(sys.argv[1], "w"), indent=1)
