"""One small invocation of every assembly kernel for compute-sanitizer (racecheck / synccheck / memcheck /
initcheck; one tool per run): C1 (16^2) and one C2 state (128^2) through k_core + k_band + k_frame (elastic and
fused incremental potential), the tile kernel alone (BSF_TILE_ONLY), the generic path, G3-FULL (k_g3 frame +
interior) and the split slab schedule.  Prints the energies so a run is visibly complete."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2506_18867_b200 as B  # noqa: E402
import workloads as W  # noqa: E402


def run(sh, mrule=0, brule=0, flags=B.PROJECT_PSD, tag=""):
    s = B.Sheet.from_sheet(sh, mrule, brule)
    x = torch.from_numpy(sh.x).cuda()
    E, g, v = s(x, flags)
    torch.cuda.synchronize()
    print(f"{tag}: E={E.item():.6e} launches={s.last_launch_count()}", flush=True)
    return s


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    c1, c2 = W.make_c1(), W.make_c2(state=3)
    for name, sh in (("C1", c1), ("C2", c2)):
        if which in ("all", "core"):
            s = run(sh, tag=f"{name} core+band+frame")
            s.set_inertia(0.15, 4e-3, gravity=np.array([0, -9.81, 0]),
                          pinned=np.pad(np.ones((1, sh.n_u), bool), ((sh.n_v - 1, 0), (0, 0))))
            X = torch.from_numpy(sh.x).cuda().unsqueeze(0).contiguous()
            E = torch.zeros(1, dtype=torch.float64, device="cuda")
            G = torch.zeros_like(X)
            V = torch.zeros((1, s.nnzb, 3, 3), dtype=torch.float64, device="cuda")
            s.eval_ip_batch(X, X, E, G, V, B.PROJECT_PSD)
            torch.cuda.synchronize()
            print(f"{name} incremental potential (fused): E={E.item():.6e}", flush=True)
        if which in ("all", "tile"):
            run(sh, flags=B.PROJECT_PSD | B.TILE_ONLY, tag=f"{name} tile")
        if which in ("all", "generic") and name == "C1":
            run(sh, flags=B.PROJECT_PSD | B.GENERIC_PATH, tag=f"{name} generic")
        if which in ("all", "g3"):
            run(sh if name == "C1" else W.make_sheet(40, 1.0, 8, n_modes=4, amp=5e-3), 2, 2, tag=f"{name} g3")
    if which in ("all", "slab"):
        os.environ["BSF_SLAB_SPLIT"] = "1"
        s = B.Sheet.from_sheet(c2, row_begin=40, row_end=90)
        x = torch.from_numpy(np.ascontiguousarray(c2.x[38:92])).cuda()
        E, g, v = s.alloc_outputs()
        s.eval_all_slab(x, E, g, v, flags=B.PROJECT_PSD)
        torch.cuda.synchronize()
        print(f"C2 slab split: E={E.item():.6e}", flush=True)
    print("SANITIZE_CASE_DONE", flush=True)


if __name__ == "__main__":
    main()
