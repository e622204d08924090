"""Time the contact pullback (bsf_contact_assemble) on a C2 / C3 sheet with a tessellated contact
mesh and proximity pairs from workloads.make_contact.  The call synchronises (data-dependent pattern size), so it is
timed by wall clock around the call after a device synchronise, median of N.  Prints one JSON line per case."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402


def run(tag, sh, res, pairs, reps=int(os.environ.get("CONTACT_REPS", "20"))):
    cs = W.make_contact(sh, res, pairs, seed=3)
    s = B.Sheet.from_sheet(sh)
    s.contact_mesh(cs.uv)
    verts = torch.from_numpy(cs.verts).cuda()
    H = torch.from_numpy(cs.H).cuda()
    g = torch.from_numpy(cs.g).cuda()
    V = torch.zeros((s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
    G = torch.zeros((sh.n_v, sh.n_u, 3), dtype=torch.float64, device="cuda")
    for _ in range(min(3, reps)):
        nnz = s.contact_assemble(verts, H, g, G, V)
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.contact_assemble(verts, H, g, G, V)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    byt = pairs * (144 + 12) * 8 + pairs * 16
    print(json.dumps({"case": tag, "n_vert": len(cs.uv), "pairs": pairs, "nnzb_offdiag": nnz, "ms": 1e3 * t,
                      "pairs_per_s": pairs / t, "input_GBps": byt / t / 1e9}), flush=True)


if __name__ == "__main__":
    pairs = [int(a) for a in sys.argv[1:]] or [10000, 100000, 400000]
    sh = W.make_c2(state=0)
    for p in pairs:
        run("C2", sh, 2, p)
    if not os.environ.get("CONTACT_C2_ONLY"):
        run("C3", W.make_c3(), 2, 400000)
