#!/usr/bin/env python
"""Benchmark of the hot path: FP64 energy + gradient + (PSD-projected) Hessian assembly of the quadratic
B-spline cloth FEM (arXiv 2506.18867) on B200.

Headline workload (BASELINE.json configs[3], "C4", the north star's scaling grid and the largest
single-GPU grid): one 1024x1024-control-point sheet (1,044,484 elements), seeded multi-scale wrinkles,
reduced membrane / bending rules, BSF_PROJECT_PSD.  One step = one assembly of the whole sheet: energy,
gradient and the full BSR Hessian (24.07 M blocks, 1.78 GB written per step, far larger than the 126 MB L2).
N GPUs: row slabs of the same sheet (strong scaling); every step = the library's NCCL halo exchange (2 rows
per neighbour) overlapped with the interior rows, the slab's fused assembly, and a 1-double energy
all-reduce.  At N > 1 the all-reduced energy is checked against a whole-sheet call.

Secondary lines (N = 1, key "secondary"): C2 100 states in one batched call, C2 one state per call (100
back-to-back calls, SURVEY §8(d)'s protocol), C3 one call (the paper's largest scene size), C5 8 sheets of
256^2 with per-sheet parameters in one call.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4|C2|C5]

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run (one rank per
GPU, 127.0.0.1 rendezvous).  --impl reference times the CPU oracle (the paper has no code to install).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "elements/sec for fp64 energy+grad+Hessian assembly; HBM GB/s & FP64 % of peak"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C4", choices=["C4", "C2", "C5"])
    p.add_argument("--states", type=int, default=100)
    p.add_argument("--flags", type=int, default=1, help="1 = BSF_PROJECT_PSD")
    p.add_argument("--generic", action="store_true", help="force the generic gather path")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-secondary", action="store_true")
    return p.parse_args()


def algorithmic_bytes(n_cp, nnzb):
    """positions read once + gradient write + Hessian values write + energy."""
    return 24 * n_cp + 24 * n_cp + 72 * nnzb + 8


def algorithmic_flops(n_membrane, n_bending):
    """SURVEY §8(d) flop model (FMA = 2, symmetric block compute): membrane 24k + 194 + 76 k(k+1)/2 at k = 6
    (the interior stencil), bending 10k + 6 + 4 k(k+1)/2 at k = 8."""
    return n_membrane * (24 * 6 + 194 + 76 * 21) + n_bending * (10 * 8 + 6 + 4 * 36)


def reduced_nnzb(n):
    S = n - 2
    return 23 * S * S + 48 * S + 8


THROTTLE = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}


class Clocks:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, gpu_index):
        self.idx, self.rows, self.proc = gpu_index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _load_json(name):
    try:
        with open(os.path.join(ROOT, name)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def hbm_peak():
    P = _load_json("MEASURED_PEAKS.json")
    if P and "hbm_gbs" in P:
        return float(P["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """DFMA peak measured on the box by scripts/ubench/fp64.cu (profiles/r01_fp64.json), else 148 SMs x 64
    DFMA/clk x 2 flop x 1.965 GHz from the guide's unit counts."""
    P = _load_json(os.path.join("profiles", "r01_fp64.json"))
    for k in ("tflops", "dfma_tflops", "fp64_tflops"):
        if P and k in P:
            return float(P[k]), "measured (profiles/r01_fp64.json, DFMA microbenchmark)"
    return 148 * 64 * 2 * 1.965e9 / 1e12, "derived (148 SMs x 64 DFMA/clk x 1.965 GHz)"


def traffic_info(kernel_prefix):
    """DRAM read+write bytes per algorithmic byte of one call / of its dominant kernel, from the committed
    ncu --set full capture (profiles/r02_traffic.json, else r01)."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        T = _load_json(os.path.join("profiles", name))
        if not T:
            continue
        call = T.get("dram_bytes_per_algorithmic_byte")
        kern = None
        for kname, v in T.get("kernels", {}).items():
            if kname.startswith(kernel_prefix) and "dram_bytes_per_algorithmic_byte" in v:
                kern = float(v["dram_bytes_per_algorithmic_byte"])
        return (float(call) if call is not None else None), kern, T.get("source", ""), name
    return None, None, "", None


def ev_pair(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


# ------------------------------------------------------------------------------- oracle (CPU)
_ORACLE_C4 = {}


def oracle_c4_sample(flags, rows):
    """The CPU oracle as it stands (all host threads) on a row slab of the C4 sheet."""
    import oracle as O
    if rows not in _ORACLE_C4:
        sh = W.make_c4()
        r0 = (sh.n_v - rows) // 2
        _ORACLE_C4[rows] = (sh, r0, O.Oracle.from_sheet(sh, r0=r0, r1=r0 + rows))
    sh, r0, o = _ORACLE_C4[rows]
    th = O.max_threads()
    t0 = time.perf_counter()
    o.eval(sh.x, flags=flags & 7, threads=th)
    t = time.perf_counter() - t0
    el = rows * (sh.n_u - 2)   # elements (knot spans) whose rows the slab owns, ~ its share of the sheet
    return el / t, th, t, f"C4 rows [{r0}, {r0 + rows}) ({rows} of 1024 rows, {el} elements), E+g+H, one pass"


def oracle_states(sheets, flags, budget_s):
    import oracle as O
    th = O.max_threads()
    done_el, t_tot, n = 0, 0.0, 0
    t_start = time.perf_counter()
    for sh in sheets:
        o = O.Oracle.from_sheet(sh)
        t0 = time.perf_counter()
        o.eval(sh.x, flags=flags & 7, threads=th)
        t_tot += time.perf_counter() - t0
        done_el += (sh.n_u - 2) * (sh.n_v - 2)
        n += 1
        if time.perf_counter() - t_start > budget_s:
            break
    return done_el / t_tot, th, n, t_tot


def bench_reference(args, rank, world):
    """The reference arm: the CPU oracle (there is no upstream code), on this arm's config and metric, each step
    a bounded sample of the workload."""
    if rank != 0:
        return
    per_step, th, sample = [], 1, ""
    if args.config == "C4":
        rows = 64
        for _ in range(min(args.warmup, 1)):
            oracle_c4_sample(args.flags, rows)
        els = []
        for _ in range(args.steps):
            v, th, t, sample = oracle_c4_sample(args.flags, rows)
            per_step.append(t)
            els.append(v * t)
        value = sum(els) / sum(per_step)
        sample = f"{args.steps} steps x ({sample})"
    else:
        sheets = [W.make_c2(state=k) for k in range(3)] if args.config == "C2" else W.make_c5(count=2)
        el = (sheets[0].n_u - 2) ** 2
        for step in range(args.steps):
            v, th, n, t = oracle_states(sheets[step % len(sheets):step % len(sheets) + 1], args.flags, 60)
            per_step.append(t)
        value = el * len(per_step) / sum(per_step)
        sample = f"{args.steps} x one {args.config} sheet (E+g+H)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(per_step) / len(per_step),
        "higher_is_better": True, "scaling": "strong" if args.config == "C4" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} (bounded sample per step)", "rules": "reduced membrane + reduced bending",
                   "projection": bool(args.flags & 1)},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": th, "kind": "oracle",
                         "sample": f"{sample}; OpenMP {th} threads"},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- ours (GPU)
def _timed(torch, fn, n, stream, per_call=False):
    """n back-to-back calls of fn on `stream` between CUDA events (synchronised on both sides); returns total ms
    and, with per_call, each call's ms."""
    ev = [ev_pair(torch) for _ in range(n)] if per_call else None
    torch.cuda.synchronize()
    t0, t1 = ev_pair(torch)
    t0.record(stream)
    for i in range(n):
        if per_call:
            ev[i][0].record(stream)
        fn(i)
        if per_call:
            ev[i][1].record(stream)
    t1.record(stream)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1), ([a.elapsed_time(b) for a, b in ev] if per_call else None)


def secondary_lines(args, dev, stream):
    """SURVEY §8(d)'s other configs on one GPU (each: elements/s, ms per call, HBM fraction of the call)."""
    import torch
    import paper_2506_18867_b200 as B
    peak, _ = hbm_peak()
    flags = args.flags
    out = {}

    def line(name, el, alg, ms, calls, note):
        t = ms / calls
        out[name] = {"value": el / (t * 1e-3), "unit": "elements/s", "ms_per_call": t,
                     "roofline_call": {"achieved_gbs": alg / (t * 1e-3) / 1e9, "frac": alg / (t * 1e-3) / 1e9 / peak},
                     "note": note}

    # C2: 100 states, one batched call; and one state per call, 100 back-to-back calls with distinct outputs
    sheets = [W.make_c2(state=k) for k in range(100)]
    h = B.Sheet.from_sheet(sheets[0], device=dev.index)
    X = torch.stack([torch.from_numpy(s.x) for s in sheets]).to(dev)
    E = torch.zeros(100, dtype=torch.float64, device=dev)
    G = torch.zeros_like(X)
    V = torch.zeros((100, h.nnzb, 3, 3), dtype=torch.float64, device=dev)
    alg1 = algorithmic_bytes(128 * 128, h.nnzb)
    for _ in range(3):
        h.eval_all_batch(X, E, G, V, flags, stream)
    ms, _ = _timed(torch, lambda i: h.eval_all_batch(X, E, G, V, flags, stream), 10, stream)
    line("C2_batched_100", 15876 * 100, alg1 * 100, ms, 10,
         "100 independent C2 states in one bsf_eval_all_batch call (2.75 GB of outputs per call)")
    Xs = [X[k] for k in range(100)]
    Es = [E[k:k + 1] for k in range(100)]
    Gs = [G[k] for k in range(100)]
    Vs = [V[k] for k in range(100)]
    for k in range(3):
        h.eval_all(Xs[k], Es[k], Gs[k], Vs[k], flags, stream)
    ms, _ = _timed(torch, lambda i: h.eval_all(Xs[i], Es[i], Gs[i], Vs[i], flags, stream), 100, stream)
    line("C2_single_state", 15876, alg1, ms, 100,
         "one C2 state per bsf_eval_all call, 100 back-to-back calls on the 100 states, distinct output buffers "
         "(SURVEY §8(d) protocol; the paper assembles one sheet per Newton iteration, PAPER.md:620)")
    del X, E, G, V, Xs, Es, Gs, Vs, h
    # C3: 226^2, the paper's largest scene size; 4 rotating output sets (345 MB > L2)
    s3 = W.make_c3()
    h = B.Sheet.from_sheet(s3, device=dev.index)
    x3 = torch.from_numpy(s3.x).to(dev)
    outs = [h.alloc_outputs() for _ in range(4)]
    for k in range(3):
        h.eval_all(x3, *outs[k % 4], flags, stream)
    ms, _ = _timed(torch, lambda i: h.eval_all(x3, *outs[i % 4], flags, stream), 50, stream)
    line("C3_single", 50176, algorithmic_bytes(226 * 226, h.nnzb), ms, 50,
         "one 226^2 sheet per bsf_eval_all call (the paper's largest scene size, PAPER.md:80, 1016-1018); 50 calls "
         "rotating 4 output sets (345 MB > L2)")
    del outs, h
    # C5: 8 sheets of 256^2 with per-sheet L, E, nu in one call
    c5 = W.make_c5()[:8]
    h = B.Sheet.from_sheet(c5[0], device=dev.index)
    X = torch.stack([torch.from_numpy(q.x) for q in c5]).to(dev)
    P = torch.from_numpy(np.stack([B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h))
                                   for q in c5])).to(dev)
    E = torch.zeros(8, dtype=torch.float64, device=dev)
    G = torch.zeros_like(X)
    V = torch.zeros((8, h.nnzb, 3, 3), dtype=torch.float64, device=dev)
    for _ in range(3):
        h.eval_all_batch_params(X, P, E, G, V, flags, stream)
    ms, _ = _timed(torch, lambda i: h.eval_all_batch_params(X, P, E, G, V, flags, stream), 10, stream)
    line("C5_8x256", 254 * 254 * 8, algorithmic_bytes(256 * 256, h.nnzb) * 8, ms, 10,
         "8 C5 sheets (256^2, per-sheet L / E / nu from bsf_affine_params) in one bsf_eval_all_batch_params call")
    return out


def bench_c4(args, rank, world, local_rank):
    import torch
    import paper_2506_18867_b200 as B
    from paper_2506_18867_b200 import distributed as D
    dev = torch.device("cuda", local_rank)
    flags = args.flags | (B.GENERIC_PATH if args.generic else 0)
    sh = W.make_c4()
    el = (sh.n_u - 2) * (sh.n_v - 2)
    # N > 1: the whole-sheet energy on rank 0's GPU, the reference the all-reduced slab energies must match
    E_whole = None
    if world > 1 and rank == 0:
        hw = B.Sheet.from_sheet(sh, device=local_rank)
        Ew, _, _ = hw(torch.from_numpy(sh.x).to(dev), flags)
        torch.cuda.synchronize()
        E_whole = float(Ew.item())
        del hw, Ew
        torch.cuda.empty_cache()
    comm = D.NcclComm(rank, world, local_rank) if world > 1 else None
    # edge slabs also run the frame kernels: they own fewer rows (distributed.edge_rows_discount)
    slab = D.SlabSheet(sh, rank, world, device=local_rank, comm=comm,
                       edge_discount=D.edge_rows_discount(sh.n_v, world))
    owned = torch.from_numpy(np.ascontiguousarray(sh.x[slab.r0:slab.r1])).to(dev)
    owned_host = owned.cpu().pin_memory()
    slab.load_owned(owned)
    stream = torch.cuda.current_stream(dev)
    for _ in range(max(args.warmup, 3)):
        slab.assemble(flags, stream)
    torch.cuda.synchronize()
    launches = slab.h.last_launch_count()
    # N > 1: the step (halo exchange on the library's NCCL communicator, the slab's kernels, the energy
    # all-reduce) is captured once into a CUDA graph and replayed, so the ~10 host launches per step do not pace
    # a ~70 us step; any capture failure falls back to direct calls (reported in config.graph)
    graph = None
    if world > 1:
        try:
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                slab.assemble(flags, stream)
            g.replay()
            torch.cuda.synchronize()
            graph = g
        except Exception as e:   # noqa: BLE001 - fall back to direct calls
            print(f"[bench] rank {rank}: graph capture failed ({e}); direct calls", file=sys.stderr, flush=True)
            torch.cuda.synchronize()
            graph = None
        ok = torch.tensor([1.0 if graph is not None else 0.0], device=dev)
        torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
        if ok.item() < 1.0:
            graph = None
    step = (lambda i: graph.replay()) if graph is not None else (lambda i: slab.assemble(flags, stream))
    core_timed = not (flags & B.GENERIC_PATH) and slab.h.core_rect()[1] > 0 and graph is None
    if core_timed:
        slab.h.set_kernel_timing(args.steps)
    if world > 1:
        torch.distributed.barrier()
    with Clocks(local_rank) as clk:
        ms, _ = _timed(torch, step, args.steps, stream)   # no per-call events: each costs ~2.5 us of the step
    remeasured = False
    if set(clk.summary()["reasons"]) & THROTTLE:   # a throttled run is re-measured once (the contract's rule)
        if core_timed:
            slab.h.set_kernel_timing(args.steps)
        if world > 1:
            torch.distributed.barrier()
        with Clocks(local_rank) as clk:
            ms, _ = _timed(torch, step, args.steps, stream)
        remeasured = True
    core_ms, band_ms = slab.h.kernel_timing(args.steps) if core_timed else ([], [])
    if core_timed:
        slab.h.set_kernel_timing(0)
    E_slabs = float(slab.E.item())
    if world > 1:
        torch.distributed.barrier()
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    value = el * args.steps / (ms * 1e-3)
    # ---- end to end through the public host-buffer API: positions from pinned host memory every step, the
    # energy read back (gradient and Hessian stay on the device for the device-side Newton solve)
    e_host = torch.zeros(1, dtype=torch.float64).pin_memory()
    if world == 1:
        # the public host-buffer call, upload overlapped with the previous step's assembly through two
        # alternating staging buffers (BSF_ASYNC_STAGE)
        X_host = owned_host.unsqueeze(0)
        stages = [slab.x.unsqueeze(0), torch.empty_like(slab.x).unsqueeze(0)]
        G1, V1 = slab.g.unsqueeze(0), slab.v.unsqueeze(0)

        def e2e_step(i):
            slab.h.eval_all_batch_host(X_host, stages[i & 1], slab.E, e_host, G1, V1, flags=flags | B.ASYNC_STAGE,
                                       stream=stream)
    else:
        def e2e_step(i):
            owned.copy_(owned_host, non_blocking=True)
            slab.load_owned(owned)
            slab.assemble(flags, stream)
            e_host.copy_(slab.E, non_blocking=True)
    for i in range(2):
        e2e_step(i)
    if world > 1:
        torch.distributed.barrier()
    e2e_ms, _ = _timed(torch, e2e_step, args.steps, stream)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    if comm is not None:
        comm.close()
    if rank != 0:
        return
    if E_whole is not None:   # strong-scaling correctness inside the run
        rel = abs(E_slabs - E_whole) / abs(E_whole)
        if not rel <= 1e-12:
            raise SystemExit(f"all-reduced slab energy {E_slabs!r} != whole-sheet energy {E_whole!r} (rel {rel:.3e})")
    peak, peak_kind = hbm_peak()
    alg = algorithmic_bytes(sh.n_u * sh.n_v, reduced_nnzb(sh.n_u))
    t_call = ms / args.steps * 1e-3
    achieved = alg / t_call / 1e9 / world
    r4 = slab.h.core_rect()
    n_core = (r4[1] - r4[0]) * (r4[3] - r4[2])
    alg_core = n_core * (48 + 23 * 72)
    call_tr, core_tr, tr_cfg, tr_src = traffic_info("k_core")
    core = None
    if core_ms:
        core_avg = statistics.mean(core_ms) * 1e-3
        core = {"kernel": "k_core", "achieved": alg_core / core_avg / 1e9, "frac": alg_core / core_avg / 1e9 / peak,
                "avg_us": core_avg * 1e6, "units": f"{n_core} core control points x 1704 B (48 + 23 x 72)",
                "share_of_call": core_avg / (ms * 1e-3 / args.steps),
                "traffic": core_tr * alg_core if core_tr else None,
                "k_band_beside_avg_us": statistics.mean(band_ms) * 1e3 if band_ms else None}
    n_mem, n_bend = slab.h.n_membrane, slab.h.n_bending
    flops = algorithmic_flops(n_mem, n_bend)
    f64_peak, f64_kind = fp64_peak()
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, th, t, sample = oracle_c4_sample(args.flags, 512)
        cpu = {"value": v, "unit": "elements/s", "cores": th, "kind": "oracle", "sample": f"{sample}, {t:.1f} s"}
    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C4: one 1024x1024-cp sheet (1,044,484 elements), reduced membrane+bending rules, "
                               f"PSD projection={bool(flags & 1)}; "
                               + ("one GPU, whole sheet" if world == 1 else
                                  f"row slabs over {world} GPUs, 2-row NCCL halos overlapped with the interior rows "
                                  "+ 1-double energy all-reduce"),
                   "elements": el, "nnzb": reduced_nnzb(sh.n_u), "slab_rows": [slab.r0, slab.r1],
                   "path": "generic" if (flags & B.GENERIC_PATH) else "core+band+corners",
                   "graph": graph is not None,
                   "l2": "1.78 GB of outputs per step > 126 MB L2 (no flush needed)",
                   "energy_check": (None if E_whole is None else
                                    {"allreduced": E_slabs, "whole_sheet": E_whole,
                                     "rel": abs(E_slabs - E_whole) / abs(E_whole)})},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": call_tr * alg if call_tr else None, "peak_kind": peak_kind,
                     "per_launch": f"whole assembly call per GPU: {alg} algorithmic bytes (48 B/cp + 72 B/block "
                                   f"+ 8) / {world} GPU(s) / {ms / args.steps * 1e3:.1f} us",
                     "traffic_source": (f"dram read+write per algorithmic byte from profiles/{tr_src} ({tr_cfg}) "
                                        "x this call's algorithmic bytes") if tr_src else None,
                     "kernel": core},
        "fp64": {"achieved_tflops": flops / t_call / 1e12 / world, "peak_tflops": f64_peak,
                 "frac": flops / t_call / 1e12 / world / f64_peak, "peak_kind": f64_kind,
                 "flops_per_call": flops, "model": "SURVEY §8(d) flop model (k = 6 membrane, k = 8 bending stencils)"},
        "cpu_baseline": cpu,
        "e2e": {"value": el * args.steps / (e2e_ms * 1e-3), "unit": "elements/s",
                "h2d_bytes_per_step": int(owned.numel() * 8 * world), "d2h_bytes_per_step": 8,
                "note": "positions uploaded from pinned host memory every step (public host-buffer call at N=1); the "
                        "energy is read back; gradient and Hessian stay on the device (their consumer, the Newton "
                        "solve, runs on the device)"},
        "gpu_launches": launches * args.steps,
        "clocks": dict(clk.summary(), remeasured=remeasured),
    }
    if world == 1 and not args.no_secondary:
        torch.cuda.empty_cache()
        del slab
        line["secondary"] = secondary_lines(args, dev, stream)
    print(json.dumps(line), flush=True)


def bench_batched(args, rank, world, local_rank):
    """--config C2 (100 states per call per GPU) or C5 (8 sheets of 256^2 per GPU): independent units, weak
    scaling, no data-path collective."""
    import torch
    import paper_2506_18867_b200 as B
    dev = torch.device("cuda", local_rank)
    flags = args.flags | (B.GENERIC_PATH if args.generic else 0)
    if args.config == "C2":
        sheets = [W.make_c2(state=(rank * args.states + k) % 100) for k in range(args.states)]
        P = None
    else:
        allsh = W.make_c5()
        sheets = [allsh[(rank * 8 + k) % len(allsh)] for k in range(8)]
    h = B.Sheet.from_sheet(sheets[0], device=local_rank)
    X = torch.stack([torch.from_numpy(s.x) for s in sheets]).to(dev)
    if args.config == "C5":
        P = torch.from_numpy(np.stack([B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h))
                                       for q in sheets])).to(dev)
    X_host = X.cpu().pin_memory()
    nb = len(sheets)
    E = torch.zeros(nb, dtype=torch.float64, device=dev)
    G = torch.zeros_like(X)
    V = torch.zeros((nb, h.nnzb, 3, 3), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(i):
        if P is None:
            h.eval_all_batch(X, E, G, V, flags, stream)
        else:
            h.eval_all_batch_params(X, P, E, G, V, flags, stream)
    for i in range(max(args.warmup, 3)):
        step(i)
    torch.cuda.synchronize()
    launches = h.last_launch_count()
    if world > 1:
        torch.distributed.barrier()
    with Clocks(local_rank) as clk:
        ms, _ = _timed(torch, step, args.steps, stream)
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    t_call = ms * 1e-3 / args.steps
    el = (sheets[0].n_u - 2) ** 2
    value = el * nb * args.steps * world / (ms * 1e-3)
    e_host = torch.zeros(nb, dtype=torch.float64).pin_memory()
    stages = [X, torch.empty_like(X)]
    host_step = lambda i: h.eval_all_batch_host(X_host, stages[i & 1], E, e_host, G, V, params=P,
                                                flags=flags | B.ASYNC_STAGE, stream=stream)
    for i in range(2):
        host_step(i)
    e2e_ms, _ = _timed(torch, host_step, args.steps, stream)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    if rank != 0:
        return
    peak, peak_kind = hbm_peak()
    alg = algorithmic_bytes(sheets[0].n_u ** 2, h.nnzb) * nb
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, th, n, t = oracle_states(sheets, args.flags, 15.0)
        cpu = {"value": v, "unit": "elements/s", "cores": th, "kind": "oracle",
               "sample": f"{n} of the {nb} {args.config} sheets, E+g+H, {t:.1f} s of CPU work, {th} threads"}
    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {nb} sheets/GPU of {sheets[0].n_u}^2 cps in one call",
                   "l2": "%.2f GB of outputs per step > 126 MB L2" % (alg / 1e9)},
        "roofline": {"bound": "hbm", "achieved": alg / t_call / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": alg / t_call / 1e9 / peak, "traffic": None, "peak_kind": peak_kind,
                     "per_launch": "whole batched call"},
        "cpu_baseline": cpu,
        "e2e": {"value": el * nb * args.steps * world / (e2e_ms * 1e-3), "unit": "elements/s",
                "h2d_bytes_per_step": int(X.numel() * 8), "d2h_bytes_per_step": 8 * nb},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def self_launch(args):
    """--gpus N > 1 outside torchrun: re-run this script under torch.distributed.run, one rank per GPU."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        bench_reference(args, rank, world)
        return
    import torch
    torch.cuda.set_device(local_rank)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.config == "C4":
            bench_c4(args, rank, world, local_rank)
        else:
            bench_batched(args, rank, world, local_rank)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
