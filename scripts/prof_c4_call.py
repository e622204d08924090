"""C4 (1024^2) whole-sheet calls for ncu: `ncalls` bsf_eval_all calls (PSD projection) on the bench's inputs.
Each call launches k_frame + k_band (side stream), k_core, k_energy_final."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402

ncalls = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sh = W.make_c4()
h = B.Sheet.from_sheet(sh)
x = torch.from_numpy(sh.x).cuda()
E, g, v = h.alloc_outputs()
for _ in range(ncalls):
    h.eval_all(x, E, g, v, B.PROJECT_PSD)
torch.cuda.synchronize()
print(f"E={E.item():.9e} launches/call={h.last_launch_count()}")
