"""C4 (and C2) per-call time of the partial-output calls a Newton line search uses: bsf_eval_energy (energy only),
bsf_eval_gradient, bsf_assemble_hessian and the full bsf_eval_all (CUDA events, back-to-back calls)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402


def timed(fn, n):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


for tag, sh in (("C2", W.make_c2(0)), ("C4", W.make_c4())):
    h = B.Sheet.from_sheet(sh)
    x = torch.from_numpy(sh.x).cuda()
    E, g, v = h.alloc_outputs()
    n = 50 if tag == "C2" else 20
    f = B.PROJECT_PSD
    out = {"config": tag,
           "energy_us": timed(lambda: h.eval_energy(x, E, f), n),
           "gradient_us": timed(lambda: h.eval_gradient(x, g, f), n),
           "hessian_us": timed(lambda: h.assemble_hessian(x, v, f), n),
           "all_us": timed(lambda: h.eval_all(x, E, g, v, f), n)}
    import statistics
    for name, fn in (("energy", lambda: h.eval_energy(x, E, f)), ("gradient", lambda: h.eval_gradient(x, g, f))):
        h.set_kernel_timing(n)
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
        c, b = h.kernel_timing(n)
        h.set_kernel_timing(0)
        out[name + "_k_core_us"] = statistics.median(c) * 1e3
        out[name + "_k_band_us"] = statistics.median(b) * 1e3
    print(json.dumps(out), flush=True)
