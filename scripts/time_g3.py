"""Median time of one bsf_eval_all_batch call of 100 C2 states under G3-FULL (BSF_G3_DEBUG phase switches)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import workloads as W
import paper_2506_18867_b200 as B

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
sheets = [W.make_c2(state=k) for k in range(n)]
s = B.Sheet.from_sheet(sheets[0], B.RULE_G3_FULL, B.RULE_G3_FULL)
X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
E = torch.zeros(n, dtype=torch.float64, device="cuda")
G = torch.zeros_like(X)
V = torch.zeros((n, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
t = []
for k in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    s.eval_all_batch(X, E, G, V, B.PROJECT_PSD)
    b.record()
    b.synchronize()
    t.append(a.elapsed_time(b))
print(f"G3 C2 x{n}: {np.median(t[2:]):.3f} ms  (BSF_G3_DEBUG={os.environ.get('BSF_G3_DEBUG', '0')})")
