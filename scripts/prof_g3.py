"""One bsf_eval_all_batch call of 20 C2 states under G3-FULL (for ncu captures of k_g3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import workloads as W
import paper_2506_18867_b200 as B

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
sheets = [W.make_c2(state=k) for k in range(n)]
s = B.Sheet.from_sheet(sheets[0], B.RULE_G3_FULL, B.RULE_G3_FULL)
X = torch.stack([torch.from_numpy(q.x) for q in sheets]).cuda()
E = torch.zeros(n, dtype=torch.float64, device="cuda")
G = torch.zeros_like(X)
V = torch.zeros((n, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
for _ in range(3):
    s.eval_all_batch(X, E, G, V, B.PROJECT_PSD)
torch.cuda.synchronize()
print("ok", float(E[0]))
