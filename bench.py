#!/usr/bin/env python
"""Benchmark of the B200 SBIP-DPPS hot path (BASELINE.json configs[1]).

Workload (one "step"): the full pass search of one world-state frame --
BASELINE configs[1]: SSL Div A 12x9 m, 8v8 (frame F8 = proj/data/bench_16v16.json
truncated to 8 robots per team), SPEC default 128 directions x 64 kick speeds,
flat + chip (16,384 candidate cells, 262,144 pass evaluations point x robot),
value function over every feasible cell and best_pass for all / flat / chip.

  value  pass evaluations/s, device-resident: kernel time per frame from CUDA
         events on the launching stream (the C-ABI context's stream), L2
         flushed (512 MiB write) between timed steps.
  e2e    the same metric through the C-ABI call pp_dpps with host buffers:
         world H2D, kernels, full per-cell result block D2H (pinned), per step.

Multi-GPU (torchrun): a single frame does not shard; every rank
runs an independent replica on its own GPU ("replicas only"), value = all
ranks' evaluations / max-over-ranks time.  --impl reference times the
reference's own CPU implementation (oracle/_ref, compiled from the unmodified
reference sources) on the same frame with every host core.
"""
from __future__ import annotations

import argparse
import ctypes as C
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

from paper_1909_07717_b200 import abi  # noqa: E402

PAIRS_PER_FRAME = 128 * 64 * 2 * 16          # cells x robots (kicker counted), = sbip_calls
FLOP_PER_PAIR = 719.0                        # SURVEY.md 8(d), config 2 (flat+chip) W_pair
METRIC = "candidate pass evaluations/sec (point x robot)"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def load_f8():
    g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
    w = abi.World.from_buffer_copy(g["f8/world"].tobytes())
    p = abi.Params.from_buffer_copy(g["f8/params"].tobytes())
    return w, p, int(g["f8/kicker"][0])


def c2_grid():
    return abi.SearchGrid(128, 64, 1.0, 6.5, 1, 1)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def ncu_traffic():
    """dram bytes per launch of the dominant kernel from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            d = json.load(f)
        return d.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU side: the reference compiled from its own sources (oracle/_ref).

def cpu_reference_time(w, p, grid, kicker, reps, threads):
    from oracle import bindings as B
    lib = B.ref()
    search = (C.c_double * reps)()
    best = (C.c_double * reps)()
    m = B.msgbuf()
    st = lib.ref_time_frame(C.byref(w), C.byref(p), C.byref(grid), kicker, threads, reps, search,
                            best, m, 512)
    if st != 0:
        raise RuntimeError(m.value.decode())
    return [search[i] + best[i] for i in range(reps)], list(search), list(best)


def cpu_baseline(w, p, grid, kicker, seconds):
    from oracle import bindings as B
    if not B.ref_available():
        return None
    cores = os.cpu_count() or 1
    tot, _, _ = cpu_reference_time(w, p, grid, kicker, 1, cores)  # warm-up + sizing
    reps = max(3, min(400, int(seconds * 1000.0 / max(tot[0], 1e-3))))
    tot, search, best = cpu_reference_time(w, p, grid, kicker, reps, cores)
    med = statistics.median(tot)
    return {"value": PAIRS_PER_FRAME / (med / 1e3), "unit": "pair-evals/s", "cores": cores,
            "kind": "reference",
            "sample": f"configs[1] frame F8, run_dpps(workers={cores}) + best_pass, {reps} reps "
                      f"(median {med:.2f} ms/frame: search {statistics.median(search):.2f} ms, "
                      f"best_pass {statistics.median(best):.2f} ms)"}


def run_reference(args, rank, world_size):
    if rank != 0:
        return 0
    w, p, kicker = load_f8()
    grid = c2_grid()
    cores = os.cpu_count() or 1
    from oracle import bindings as B
    if not B.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    cpu_reference_time(w, p, grid, kicker, max(args.warmup, 1), cores)
    t0 = time.perf_counter()
    tot, search, best = cpu_reference_time(w, p, grid, kicker, args.steps, cores)
    wall = time.perf_counter() - t0
    mean_ms = sum(tot) / len(tot)
    value = PAIRS_PER_FRAME / (mean_ms / 1e3)
    sample = (f"configs[1] frame F8 (8v8, 128x64 flat+chip), run_dpps(workers={cores}) + "
              f"best_pass per step, {args.steps} steps")
    out = {"metric": METRIC, "value": value, "unit": "pair-evals/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
           "p50_ms": statistics.median(tot), "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "configs[1]: 8v8 frame F8, 128x64 grid, flat+chip, "
                                  "search + value function + argmax",
                      "cells": 16384, "pairs_per_frame": PAIRS_PER_FRAME},
           "impl": "reference",
           "cpu_baseline": {"value": value, "unit": "pair-evals/s", "cores": cores,
                            "kind": "reference", "sample": sample},
           "e2e": {"value": value, "unit": "pair-evals/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "wall_s": wall,
           "search_ms_p50": statistics.median(search), "best_pass_ms_p50": statistics.median(best)}
    print(json.dumps(out))
    return 0


# ---------------------------------------------------------------------------
# GPU side.

def synthetic_frames(n, seed=0xB200):
    """C5-style frames: 8v8, uniform positions on the pitch, velocity components
    U(-2, 2), ball at rest on the pitch (oracles.hpp:228-258 distribution)."""
    rng = np.random.default_rng(seed)
    frames = (abi.World * n)()
    for i in range(n):
        w = frames[i]
        w.field = abi.Field(12.0, 9.0, 1.8, 1.8, 3.6)
        w.n_ours = w.n_theirs = 8
        xy = rng.uniform([-6.0, -4.5], [6.0, 4.5], size=(17, 2))
        v = rng.uniform(-2.0, 2.0, size=(16, 2))
        for j in range(8):
            w.ours[j].id = j
            w.ours[j].px, w.ours[j].py = xy[j]
            w.ours[j].vx, w.ours[j].vy = v[j]
            w.theirs[j].id = j
            w.theirs[j].px, w.theirs[j].py = xy[8 + j]
            w.theirs[j].vx, w.theirs[j].vy = v[8 + j]
        w.ball_px, w.ball_py = xy[16]
    return frames


def run_ours(args, rank, world_size, local_rank):
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    if world_size > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    lib = abi.load_library()
    ctx = C.c_void_p()
    st = lib.pp_ctx_create(local_rank, C.byref(ctx))
    if st != 0:
        raise RuntimeError(f"pp_ctx_create failed ({st})")
    w, p, kicker = load_f8()
    grid = c2_grid()
    n_cells = 16384
    block_bytes = int(lib.pp_grid_bytes(n_cells))
    hblock = lib.pp_host_alloc(block_bytes)
    st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, abi.PP_COPY_ALL, hblock)
    if st != 0:
        raise RuntimeError(lib.pp_last_error(ctx).decode())
    view = abi.GridBlock(n_cells, buf=(C.c_uint8 * block_bytes).from_address(hblock))
    best = (int(view.summary.best_cell[0]), float(view.summary.best_score[0]))

    stream = torch.cuda.ExternalStream(lib.pp_ctx_stream(ctx), device=local_rank)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=f"cuda:{local_rank}")

    def barrier():
        if world_size > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- value: device-resident kernel time, L2 flushed between steps ----
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            lib.pp_dpps_relaunch(ctx)
    barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clocks:
        barrier()
        t_wall0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()                     # untimed: evict L2 between steps
                starts[i].record(stream)
                lib.pp_dpps_relaunch(ctx)
                ends[i].record(stream)
        barrier()
        t_wall = time.perf_counter() - t_wall0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    dev_total_ms = sum(step_ms)
    if world_size > 1:
        t = torch.tensor([dev_total_ms], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_total_ms = float(t.item())
    ms_per_step = dev_total_ms / args.steps
    value = world_size * PAIRS_PER_FRAME * args.steps / (dev_total_ms / 1e3)

    # ---- e2e: through the C-ABI with host buffers --------------------------
    for _ in range(args.warmup):
        lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, abi.PP_COPY_ALL, hblock)
    barrier()
    e2e_ms = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ts = time.perf_counter()
        st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, abi.PP_COPY_ALL,
                         hblock)
        e2e_ms.append((time.perf_counter() - ts) * 1e3)
        if st != 0:
            raise RuntimeError(lib.pp_last_error(ctx).decode())
    e2e_total = (time.perf_counter() - t0) * 1e3
    barrier()
    if world_size > 1:
        t = torch.tensor([e2e_total], device=f"cuda:{local_rank}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = world_size * PAIRS_PER_FRAME * args.steps / (e2e_total / 1e3)
    if (int(view.summary.best_cell[0]), float(view.summary.best_score[0])) != best:
        raise RuntimeError("result changed between runs")

    # Per-kernel split (CUDA events around each of the two launches) for the
    # roofline of the dominant kernel.
    lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, abi.PP_COPY_SUMMARY, hblock)
    scan_ms, value_ms = C.c_float(), C.c_float()
    lib.pp_dpps_kernel_times(ctx, 50, C.byref(scan_ms), C.byref(value_ms))

    extras = {}
    if rank == 0 and not args.no_extras:
        extras = run_extras(lib, ctx, w, p, kicker)

    if rank == 0:
        peaks = measured_peaks()
        clk = clocks.summary()
        sm_max = clk.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
        # FP32 CUDA-core peak: 148 SMs x 128 lanes x 2 (FMA) x clocks.max.sm.
        # MEASURED_PEAKS.json carries HBM and bf16 tensor figures only.
        peak_tflops = 148 * 128 * 2 * sm_max * 1e6 / 1e12
        # dominant kernel = scan_kernel (the SBIP search the W_pair figure counts)
        achieved = FLOP_PER_PAIR * PAIRS_PER_FRAME / (scan_ms.value / 1e3) / 1e12
        out = {
            "metric": METRIC, "value": value, "unit": "pair-evals/s", "n_gpus": world_size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "p50_ms": statistics.median(step_ms), "p99_ms": float(np.percentile(step_ms, 99)),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "configs[1]: 8v8 frame F8, 128x64 grid, flat+chip, "
                                   "search + value function + argmax (replicas per GPU)",
                       "cells": n_cells, "pairs_per_frame": PAIRS_PER_FRAME,
                       "l2": "flushed (512 MiB write) between timed steps",
                       "parallelism": f"replicas x{world_size}"},
            "e2e": {"value": e2e_value, "unit": "pair-evals/s",
                    "p50_ms": statistics.median(e2e_ms),
                    # the packed frame + robot constants, as kernel parameters
                    "h2d_bytes_per_step": int(lib.pp_dpps_upload_bytes()),
                    "d2h_bytes_per_step": block_bytes},
            "roofline": {"bound": "fp32-core", "achieved": achieved, "peak": peak_tflops,
                         "unit": "TFLOP/s", "frac": achieved / peak_tflops,
                         "traffic": ncu_traffic(),
                         "kernel": "scan_kernel (SBIP search; value_kernel is the second launch)",
                         "kernel_ms": {"scan": scan_ms.value, "value": value_ms.value},
                         "note": "algorithmic FLOP = 719/pair (SURVEY 8(d), C2) x 262,144 pairs "
                                 "per scan launch; peak = nominal FP32 CUDA-core "
                                 "148x128x2xclocks.max.sm (MEASURED_PEAKS has no FP32 figure)"},
            "clocks": clk,
            "gpu_launches": 2 * args.steps,  # scan_kernel + value_kernel per step
            "wall_s": t_wall,
            "best": {"cell": best[0], "score": best[1]},
            "extras": extras,
        }
        if world_size == 1 and not args.no_cpu:
            out["cpu_baseline"] = cpu_baseline(w, p, grid, kicker, args.cpu_seconds)
        print(json.dumps(out))
    lib.pp_host_free(hblock)
    lib.pp_ctx_destroy(ctx)
    if world_size > 1:
        dist.destroy_process_group()
    return 0


def run_extras(lib, ctx, w, p, kicker):
    """Secondary configs (device time, event-timed inside the C-ABI)."""
    ex = {}

    def frame_ms(grid, reps, copy=abi.PP_COPY_SUMMARY):
        n = (grid.flat + grid.chip) * grid.n_directions * grid.n_powers
        blk = abi.GridBlock(n)
        for _ in range(2):
            lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, copy, blk.ptr())
        ms = []
        for _ in range(reps):
            lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, copy, blk.ptr())
            ms.append(blk.summary.device_ms)
        return statistics.median(ms), float(np.percentile(ms, 99)), blk

    c1, c1_99, _ = frame_ms(abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0), 50)
    ex["c1_flat_p50_ms"] = c1
    c3, c3_99, blk = frame_ms(abi.SearchGrid(1200, 900, 1.0, 6.5, 1, 0), 20)
    ex["c3_1200x900_p50_ms"], ex["c3_p99_ms"] = c3, c3_99
    ex["c3_pair_evals_per_s"] = 1200 * 900 * 16 / (c3 / 1e3)
    # C5-style batch: independent frames, one CTA per frame, summaries only.
    n = 16384
    frames = synthetic_frames(n)
    grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)
    if lib.pp_batch_upload(ctx, frames, n, None) == 0:
        ms = C.c_float()
        lib.pp_batch_run(ctx, C.byref(p), C.byref(grid), C.byref(ms))
        runs = []
        for _ in range(3):
            lib.pp_batch_run(ctx, C.byref(p), C.byref(grid), C.byref(ms))
            runs.append(ms.value)
        t = statistics.median(runs)
        ex["batch_frames"] = n
        ex["batch_frames_per_s"] = n / (t / 1e3)
        ex["batch_pair_evals_per_s"] = n * 128 * 64 * 16 / (t / 1e3)
    # C4: running-point map, all zones, 0.1 m and 0.01 m.
    for step in (0.1, 0.01):
        pp = abi.Params.from_buffer_copy(bytes(p))
        pp.thresholds.grid_step = step
        nv = C.c_int64()
        lib.pp_runmap_count(C.byref(w), C.byref(pp), 0xF, C.byref(nv))
        # the caller's result block in pinned memory (as for the DPPS e2e):
        # the kernel writes the map straight into it
        rbytes = abi.runmap_offsets(nv.value)["total"]
        rptr = lib.pp_host_alloc(rbytes)
        req = abi.RunmapRequest(0xF, 0, 4, 0, 0.0, 0.0, 1)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            st = lib.pp_runmap(ctx, C.byref(w), C.byref(pp), C.byref(req), rptr, nv.value)
            ts.append((time.perf_counter() - t0) * 1e3)
            if st != 0:
                raise RuntimeError(lib.pp_last_error(ctx).decode())
        lib.pp_host_free(rptr)
        ex[f"runmap_{step}m_e2e_ms"] = statistics.median(ts[1:])
        ex[f"runmap_{step}m_vertices"] = nv.value
    return ex


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = _env_int("RANK", 0)
    world_size = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world_size)
    return run_ours(args, rank, world_size, local_rank)


if __name__ == "__main__":
    sys.exit(main())
