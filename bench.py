#!/usr/bin/env python
"""Benchmark of the hot path: FP64 energy + gradient + (PSD-projected) Hessian assembly of the
quadratic B-spline cloth FEM (arXiv 2506.18867) on B200.

Workload (BASELINE.json configs[1], "C2"): 128x128-control-point draped sheet, 100 seeded states
(wrinkles + rigid motion), reduced membrane/bending rules, BSF_PROJECT_PSD.  One step = the
assembly of all 100 states (energy, gradient and the full BSR Hessian of each, into 100 separate
output buffers — 2.7 GB of Hessian values per step, far larger than the 126 MB L2, so every step
streams to HBM).  Multi-GPU: the states are independent units, every rank runs its own 100 states
(weak scaling, no data-path collective).

Metric: elements/s (element = one knot span; 126^2 per state).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C2|C4]
"""
from __future__ import annotations

import argparse
import json
import os
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
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2", choices=["C2", "C4", "C5"])
    p.add_argument("--states", type=int, default=100)
    p.add_argument("--flags", type=int, default=1, help="1 = BSF_PROJECT_PSD")
    p.add_argument("--generic", action="store_true", help="force the generic gather path")
    p.add_argument("--no-cpu-baseline", action="store_true")
    return p.parse_args()


def workload(cfg, states, rank=0):
    if cfg == "C2":
        return [W.make_c2(state=(rank * states + k) % 100) for k in range(states)]
    return [W.make_c4()]


def algorithmic_bytes(n_cp, nnzb):
    """positions read once + gradient write + Hessian values write + energy."""
    return 24 * n_cp + 24 * n_cp + 72 * nnzb + 8


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


def traffic_ratio_core():
    """k_core's DRAM bytes per algorithmic byte from the committed ncu capture (None if absent)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            for name, v in json.load(f)["kernels"].items():
                if name.startswith("k_core") and "dram_bytes_per_algorithmic_byte" in v:
                    return float(v["dram_bytes_per_algorithmic_byte"])
    except (OSError, ValueError, KeyError):
        return None
    return None


def traffic_ratio():
    """DRAM bytes per algorithmic byte of one assembly call (k_frame + k_core) from the committed
    ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as f:
            return float(json.load(f)["dram_bytes_per_algorithmic_byte"])
    except (OSError, KeyError, ValueError):
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            P = json.load(f)
        return float(P["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


# ------------------------------------------------------------------------------- oracle (CPU)
def run_oracle_sample(sheets, flags, budget_s=20.0):
    """Time the CPU oracle as it stands (all host cores) on a bounded sample of the workload."""
    import oracle as O
    th = O.max_threads()
    done_el, t_tot, n = 0, 0.0, 0
    t_start = time.perf_counter()
    for sh in sheets:
        o = O.Oracle.from_sheet(sh)
        t0 = time.perf_counter()
        o.eval(sh.x, flags=flags, threads=th)
        t_tot += time.perf_counter() - t0
        done_el += (sh.n_u - 2) * (sh.n_v - 2)
        n += 1
        if time.perf_counter() - t_start > budget_s:
            break
    return done_el / t_tot, th, n, t_tot


def bench_reference(args, rank, world):
    if rank != 0:
        return
    states = workload(args.config, max(1, min(args.states, 3)))
    vals, th, secs = [], 1, 0.0
    for _ in range(args.warmup):
        pass  # the oracle has no warm-up state; each step below is a full independent run
    per_step = []
    for step in range(args.steps):
        v, th, n, t = run_oracle_sample(states[step % len(states):step % len(states) + 1], args.flags, 60)
        per_step.append(t)
        vals.append(v)
    el = (states[0].n_u - 2) * (states[0].n_v - 2)
    value = el * len(per_step) / sum(per_step)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(per_step) / len(per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config} (one state per step: bounded sample of the 100-state step)",
                   "rules": "reduced membrane + reduced bending", "projection": bool(args.flags & 1)},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": th, "kind": "oracle",
                         "sample": f"{args.steps} x one {args.config} state (E+g+H), OpenMP {th} threads"},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------- ours (GPU)
def bench_c4_slabs(args, rank, world, local_rank):
    """C4 (1024^2) row-slab strong scaling: every step = halo exchange (NCCL, 2 rows per neighbour,
    through the library), the rank's fused assembly, energy all-reduce."""
    import torch
    import paper_2506_18867_b200 as B
    from paper_2506_18867_b200 import distributed as D
    dev = torch.device("cuda", local_rank)
    flags = args.flags | (B.GENERIC_PATH if args.generic else 0)
    sh = W.make_c4()
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
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            slab.assemble(flags, stream)
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        torch.distributed.barrier()
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    el = (sh.n_u - 2) * (sh.n_v - 2)
    value = el * args.steps / (ms * 1e-3)
    # e2e: pinned H2D of the owned rows, assembly, D2H of the energy
    e_host = torch.zeros(1, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    if world == 1:
        # one GPU: the public host-buffer call (upload overlapped with the previous step's assembly through
        # two alternating staging buffers, BSF_ASYNC_STAGE)
        h1 = slab.h
        X_host = owned_host.unsqueeze(0)
        stages = [slab.x.unsqueeze(0), torch.empty_like(slab.x).unsqueeze(0)]
        G1, V1 = slab.g.unsqueeze(0), slab.v.unsqueeze(0)
        for i in range(2):
            h1.eval_all_batch_host(X_host, stages[i], slab.E, e_host, G1, V1, flags=flags | B.ASYNC_STAGE, stream=stream)
        torch.cuda.synchronize()
    s0.record(stream)
    for i in range(args.steps):
        if world == 1:
            h1.eval_all_batch_host(X_host, stages[i & 1], slab.E, e_host, G1, V1, flags=flags | B.ASYNC_STAGE,
                                   stream=stream)
            continue
        owned.copy_(owned_host, non_blocking=True)
        slab.load_owned(owned)
        slab.assemble(flags, stream)
        e_host.copy_(slab.E, non_blocking=True)
    s1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = s0.elapsed_time(s1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    if comm is not None:
        comm.close()
    if rank != 0:
        return
    peak, peak_kind = peaks()
    alg = algorithmic_bytes(sh.n_u * sh.n_v, 23 * (sh.n_u - 2) ** 2 + 48 * (sh.n_u - 2) + 8)
    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C4: 1024x1024 cps, row slabs over %d GPUs, 2-row NCCL halos + energy all-reduce" % world,
                   "elements": el, "path": "generic" if (flags & B.GENERIC_PATH) else "tile",
                   "l2": "1.78 GB of outputs per step > 126 MB L2 (no flush needed)"},
        "roofline": {"bound": "hbm", "achieved": alg / (ms / args.steps * 1e-3) / 1e9 / world, "peak": peak,
                     "unit": "GB/s", "frac": alg / (ms / args.steps * 1e-3) / 1e9 / world / peak,
                     "traffic": None, "peak_kind": peak_kind, "per_launch": "per GPU, whole step"},
        "cpu_baseline": None,
        "e2e": {"value": el * args.steps / (e2e_ms * 1e-3), "unit": "elements/s",
                "h2d_bytes_per_step": int(owned.numel() * 8 * world), "d2h_bytes_per_step": 8},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def bench_c5(args, rank, world, local_rank):
    """C5: batch of 256^2 sheets with per-sheet side length / E / nu, 8 sheets per GPU (weak scaling:
    rank r assembles sheets 8r..8r+7 of the 64-sheet set), one bsf_eval_all_batch_params launch."""
    import torch
    import paper_2506_18867_b200 as B
    dev = torch.device("cuda", local_rank)
    per = 8
    allsh = W.make_c5()
    sheets = [allsh[(rank * per + k) % len(allsh)] for k in range(per)]
    h = B.Sheet.from_sheet(sheets[0], device=local_rank)
    X = torch.stack([torch.from_numpy(q.x) for q in sheets]).to(dev)
    X_host = X.cpu().pin_memory()
    P = torch.from_numpy(np.stack([B.affine_params(q.rest_xy, B.material_from_young(q.E, q.nu, q.h))
                                   for q in sheets])).to(dev)
    E = torch.zeros(per, dtype=torch.float64, device=dev)
    G = torch.zeros((per,) + tuple(X.shape[1:]), dtype=torch.float64, device=dev)
    V = torch.zeros((per, h.nnzb, 3, 3), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    step = lambda: h.eval_all_batch_params(X, P, E, G, V, args.flags, stream)
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches = h.last_launch_count()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if world > 1:
        torch.distributed.barrier()
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    el = (sheets[0].n_u - 2) ** 2
    value = el * per * args.steps * world / (ms * 1e-3)
    # e2e through the public host-buffer call (per-item parameters), two alternating staging buffers
    e_host = torch.zeros(per, dtype=torch.float64).pin_memory()
    stages = [X, torch.empty_like(X)]
    host_step = lambda i: h.eval_all_batch_host(X_host, stages[i & 1], E, e_host, G, V, params=P,
                                                flags=args.flags | B.ASYNC_STAGE, stream=stream)
    for i in range(2):
        host_step(i)
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for i in range(args.steps):
        host_step(i)
    s1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = s0.elapsed_time(s1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    if rank != 0:
        return
    peak, peak_kind = peaks()
    alg = algorithmic_bytes(sheets[0].n_u ** 2, h.nnzb) * per
    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C5: %d sheets/GPU of 256x256 cps, per-sheet L/E/nu, one batched launch" % per,
                   "elements_per_sheet": el, "l2": "%.2f GB of outputs per step > 126 MB L2" % (alg / 1e9)},
        "roofline": {"bound": "hbm", "achieved": alg / (ms / args.steps * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": alg / (ms / args.steps * 1e-3) / 1e9 / peak, "traffic": None, "peak_kind": peak_kind},
        "cpu_baseline": None,
        "e2e": {"value": el * per * args.steps * world / (e2e_ms * 1e-3), "unit": "elements/s",
                "h2d_bytes_per_step": int(X.numel() * 8), "d2h_bytes_per_step": 8 * per},
        "gpu_launches": launches * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def bench_ours(args, rank, world, local_rank):
    import torch
    import paper_2506_18867_b200 as B

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    flags = args.flags | (B.GENERIC_PATH if args.generic else 0)
    sheets = workload(args.config, args.states if args.config == "C2" else 1, rank)
    ref = sheets[0]
    h = B.Sheet.from_sheet(ref, device=local_rank)
    n_units = len(sheets)
    X = torch.stack([torch.from_numpy(s.x) for s in sheets]).to(dev)          # [B, n, n, 3]
    X_host = X.cpu().pin_memory()
    Eo = torch.zeros(n_units, dtype=torch.float64, device=dev)
    Go = torch.zeros((n_units,) + tuple(X.shape[1:]), dtype=torch.float64, device=dev)
    Vo = torch.zeros((n_units, h.nnzb, 3, 3), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        h.eval_all_batch(X, Eo, Go, Vo, flags, stream)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    launches_per_step = h.last_launch_count()

    # live per-kernel timing of the timed steps: the library records CUDA events around k_core (on this
    # stream) and k_band (on its side stream) in every call; read after the timed region
    core_timed = not (flags & B.GENERIC_PATH) and h.core_rect()[1] > 0
    if core_timed:
        h.set_kernel_timing(args.steps)
    # ---- timed region (device time, CUDA events on the launching stream) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        t0.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ms = t0.elapsed_time(t1)
    call_ms = [a.elapsed_time(b) for a, b in ev]
    core_ms, band_ms = h.kernel_timing(args.steps) if core_timed else ([], [])
    if core_timed:
        h.set_kernel_timing(0)
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        ms = float(tt.item())
    el_per_unit = (ref.n_u - 2) * (ref.n_v - 2)
    value = el_per_unit * n_units * args.steps * world / (ms * 1e-3)

    # ---- end to end through the public API: bsf_eval_all_batch_host uploads the positions from pinned host
    # memory chunk by chunk (overlapping the assembly of earlier chunks) and reads the energies back; two
    # staging buffers alternate (BSF_ASYNC_STAGE) so that step i+1's upload overlaps step i's assembly ----
    e_host = torch.zeros(n_units, dtype=torch.float64).pin_memory()
    stages = [X, torch.empty_like(X)]
    for i in range(2):   # warm the copy stream and the per-stage events
        h.eval_all_batch_host(X_host, stages[i], Eo, e_host, Go, Vo, flags=flags | B.ASYNC_STAGE, stream=stream)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    s0 = torch.cuda.Event(enable_timing=True)
    s1 = torch.cuda.Event(enable_timing=True)
    s0.record(stream)
    for i in range(args.steps):
        h.eval_all_batch_host(X_host, stages[i & 1], Eo, e_host, Go, Vo, flags=flags | B.ASYNC_STAGE, stream=stream)
    s1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = s0.elapsed_time(s1)
    if world > 1:
        tt = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    e2e_value = el_per_unit * n_units * args.steps * world / (e2e_ms * 1e-3)
    xs = [X]

    if rank != 0:
        return
    peak, peak_kind = peaks()
    n_cp = ref.n_u * ref.n_v
    alg = algorithmic_bytes(n_cp, h.nnzb) * n_units          # one launch covers all states
    call_avg = statistics.mean(call_ms)
    achieved_call = alg / (call_avg * 1e-3) / 1e9
    # roofline of the dominant kernel (k_core): its algorithmic bytes (positions + gradient 48 B per core
    # control point, 23 blocks x 72 B) over its live average duration (events on its stream, band kernel
    # running beside it); the whole-call figure is kept alongside
    r4 = h.core_rect()
    n_core = (r4[1] - r4[0]) * (r4[3] - r4[2])
    alg_core = n_units * n_core * (48 + 23 * 72)
    if core_ms:
        core_avg = statistics.mean(core_ms)
        achieved = alg_core / (core_avg * 1e-3) / 1e9
    else:
        core_avg, achieved = None, achieved_call
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        v, th, n, t = run_oracle_sample(sheets, args.flags, budget_s=15.0)
        cpu = {"value": v, "unit": "elements/s", "cores": th, "kind": "oracle",
               "sample": f"{n} of the {n_units} {args.config} states, E+g+H, {t:.1f} s of CPU work, {th} threads"}
    line = {
        "metric": METRIC, "value": value, "unit": "elements/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {ref.n_u}x{ref.n_v} cps, {n_units} states/step/GPU, "
                               f"reduced membrane+bending rules, PSD projection={bool(flags & 1)}",
                   "elements_per_state": el_per_unit, "nnzb": h.nnzb,
                   "path": "generic" if (flags & B.GENERIC_PATH) else ("core+band+corners" if h.core_rect()[1] else "tile"),
                   "l2": "working set per step = %.2f GB of outputs > 126 MB L2 (no flush needed)" % (alg / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": ((traffic_ratio_core() * alg_core if traffic_ratio_core() else None) if core_ms
                                 else (None if traffic_ratio() is None or (flags & B.GENERIC_PATH)
                                       else traffic_ratio() * alg)),
                     "traffic_source": "k_core's dram read+write per algorithmic byte (ncu --set full of one call, "
                                       "20 C2 states) x its algorithmic bytes per launch; profiles/r01_traffic.json",
                     "peak_kind": peak_kind,
                     "kernel": ("k_core: %d states x %d core control points, %d algorithmic bytes per launch, live avg "
                                "%.1f us (k_band beside it: avg %.1f us)"
                                % (n_units, n_core, alg_core, core_avg * 1e3, statistics.mean(band_ms) * 1e3))
                               if core_ms else "whole call (no core kernel on this path)",
                     "call": {"achieved": achieved_call, "frac": achieved_call / peak,
                              "per_launch": "one bsf_eval_all_batch call (%d states): %d algorithmic bytes, avg %.1f us"
                                            % (n_units, alg, call_avg * 1e3)}},
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "elements/s",
                "h2d_bytes_per_step": int(sum(x.numel() * 8 for x in xs)), "d2h_bytes_per_step": 8 * n_units},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        bench_reference(args, rank, world)
        return
    if world > 1:
        import torch
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        if args.config == "C4":
            bench_c4_slabs(args, rank, world, local_rank)
        elif args.config == "C5":
            bench_c5(args, rank, world, local_rank)
        else:
            bench_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
