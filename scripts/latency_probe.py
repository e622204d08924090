"""Single-sheet latency probe: C2 (one state) and C3 per-call device time for direct
back-to-back calls and for the same calls replayed from a CUDA graph (host launch overhead removed); run with
different BSF_CORE_MINROWS / BSF_CORE_PROLOGUE settings to compare launch shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402


FLAGS = B.PROJECT_PSD | (B.TILE_ONLY if os.environ.get("PROBE_TILE") else 0)


def probe(sh, n=50, tag=""):
    h = B.Sheet.from_sheet(sh)
    x = torch.from_numpy(sh.x).cuda()
    outs = [h.alloc_outputs() for _ in range(4)]
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for k in range(3):
            h.eval_all(x, *outs[k % 4], FLAGS, st)
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(st)
        for k in range(n):
            h.eval_all(x, *outs[k % 4], FLAGS, st)
        t1.record(st)
        torch.cuda.synchronize()
        direct = t0.elapsed_time(t1) / n
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for k in range(n):
                h.eval_all(x, *outs[k % 4], FLAGS, st)
        g.replay()
        torch.cuda.synchronize()
        t0.record(st)
        g.replay()
        t1.record(st)
        torch.cuda.synchronize()
        graph = t0.elapsed_time(t1) / n
    h.set_kernel_timing(n)
    with torch.cuda.stream(st):
        for k in range(n):
            h.eval_all(x, *outs[k % 4], FLAGS, st)
    torch.cuda.synchronize()
    c, b = h.kernel_timing(n)
    h.set_kernel_timing(0)
    import statistics
    return {"tag": tag, "direct_us": direct * 1e3, "graph_us": graph * 1e3, "launches": h.last_launch_count(),
            "core": h.core_rect(), "k_core_us": statistics.median(c) * 1e3, "k_band_us": statistics.median(b) * 1e3}


env = {k: os.environ.get(k) for k in ("BSF_CORE_MINROWS", "BSF_CORE_PROLOGUE", "PROBE_TILE")}
cases = [("C2", W.make_c2(state=0)), ("C3", W.make_c3())]
if "--c4" in sys.argv:
    cases.append(("C4", W.make_c4()))
for name, sh in cases:
    print(json.dumps({"env": env, **probe(sh, n=20 if name == "C4" else 50, tag=name)}), flush=True)
