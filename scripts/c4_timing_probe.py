import sys, os, statistics
sys.path.insert(0, os.getcwd())
import torch, numpy as np, workloads as W, paper_2506_18867_b200 as B
from paper_2506_18867_b200 import distributed as D
sh = W.make_c4()
slab = D.SlabSheet(sh, 0, 1, device=0, comm=None, edge_discount=0)
owned = torch.from_numpy(np.ascontiguousarray(sh.x)).cuda()
slab.load_owned(owned)
st = torch.cuda.current_stream()
h = B.Sheet.from_sheet(sh)
x = torch.from_numpy(sh.x).cuda()
outs = h.alloc_outputs()
def run(fn, n=20, kt=False, pc=False, obj=None):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    if kt: obj.set_kernel_timing(n)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    t0.record(st)
    for i in range(n):
        if pc: evs[i][0].record(st)
        fn()
        if pc: evs[i][1].record(st)
    t1.record(st); torch.cuda.synchronize()
    if kt: obj.set_kernel_timing(0)
    return t0.elapsed_time(t1) / n * 1e3
for rep in range(2):
    print("eval_all plain %.1f" % run(lambda: h.eval_all(x, *outs, 1, st)))
    print("eval_all kt %.1f" % run(lambda: h.eval_all(x, *outs, 1, st), kt=True, obj=h))
    print("slab plain %.1f" % run(lambda: slab.assemble(1, st)))
    print("slab kt+pc %.1f" % run(lambda: slab.assemble(1, st), kt=True, pc=True, obj=slab.h))
    print("slab pc %.1f" % run(lambda: slab.assemble(1, st), pc=True))
