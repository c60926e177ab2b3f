#!/usr/bin/env python
"""Benchmark of the B200 SBIP-DPPS hot path.

Headline workload (one "step"): the C5 batch of BASELINE.json configs[4] --
65,536 independent world-state frames, frame i =
oracles::random_world(mt19937_64(0xB200 + i), 8, 8) (proj/tests/oracles.hpp:
228-258; regenerated bit for bit by paper_1909_07717_b200/synthetic.py), the
SPEC default 128 directions x 64 kick speeds, flat (C1 grid: 8,192 cells x 16
robots = 131,072 pass evaluations per frame), kicker = the teammate nearest
the ball.  Every frame gets the full search and an exact best_pass for all /
flat / chip (the value function of every feasible cell whose score bound
does not rule it out; results identical to scoring them all).

  value  pass evaluations/s over the whole batch, device-resident: the raw
         frames sit in HBM; one step stages them (id sort, kicker), builds
         the robots' filter constants, and runs scan + value for every frame
         (pp_batch_run).  CUDA events on the launching stream (the C-ABI
         context's), L2 flushed between steps (512 MiB write), max over ranks.
  e2e    the same metric through the public C-ABI call pp_dpps_frames with
         host buffers: frames H2D (pinned), staging, kernels, the 48-byte
         per-frame results D2H, and under torchrun the gather of every
         rank's results on rank 0 -- per step, events, max over ranks.

Multi-GPU (torchrun, one process per GPU): the 65,536 frames shard as
contiguous ranges, no collective inside a frame, one gather of
the results; total work is fixed ("strong" scaling).  The per-frame search
latency of BASELINE's metric is measured on the single frame of configs[1]
(F8, 128 x 64 flat + chip) and reported under "frame".

--impl reference times the reference's own CPU implementation (oracle/_ref,
the unmodified reference sources) on a bounded sample of the same C5 frames
per step: run_dpps_serial + best_pass, frame-parallel on every host core.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1909_07717_b200 import abi, synthetic  # noqa: E402
from paper_1909_07717_b200.sharding import shard_range  # noqa: E402

METRIC = "candidate pass evaluations/sec (point x robot)"
C5_FRAMES = 65536
C5_CELLS = 128 * 64                 # C1 grid, flat
C5_PAIRS_PER_FRAME = C5_CELLS * 16  # cells x robots (kicker counted), = sbip_calls
C2_PAIRS = 128 * 64 * 2 * 16
CONFIG = {
    "workload": "configs[4] C5: 65,536 random 8v8 frames sharded over the GPUs; per frame "
                "run_dpps (128x64 grid, flat: every cell x robot pair searched) + best_pass "
                "all/flat/chip (exact: score_pass of every feasible cell that could be the "
                "best -- cells whose score upper bound is below a scored cell's are skipped, "
                "DESIGN 3.2)",
    "frames": C5_FRAMES,
    "frames_source": "oracles::random_world(mt19937_64(0xB200+i), 8, 8) (proj/tests/oracles.hpp)",
    "grid": "128 directions x 64 powers, flat (C1)",
    "pairs_per_frame": C5_PAIRS_PER_FRAME,
    "kicker": "teammate nearest the ball",
    "l2": "flushed (512 MiB write) between timed steps; device-resident inputs 106 MB",
}


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def c1_grid():
    return abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0)


def default_params(lib):
    p = abi.Params()
    lib.pp_params_default(C.byref(p))
    return p


def load_f8():
    g = np.load(os.path.join(ROOT, "tests", "golden", "grids.npz"))
    w = abi.World.from_buffer_copy(g["f8/world"].tobytes())
    p = abi.Params.from_buffer_copy(g["f8/params"].tobytes())
    return w, p, int(g["f8/kicker"][0])


def cpu_info():
    """Host CPU model, clock and thread count (state the cores)."""
    model, mhz = platform.processor(), None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                elif line.startswith("cpu MHz") and mhz is None:
                    mhz = float(line.split(":", 1)[1])
    except OSError:
        pass
    return {"cpu_model": model, "cpu_mhz": mhz, "nproc": os.cpu_count()}


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


def _load_json(rel):
    try:
        with open(os.path.join(ROOT, rel)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ---------------------------------------------------------------------------
# CPU side: the reference compiled from its own sources (oracle/_ref).

def cpu_batch(frames_np, threads):
    """ref_batch (run_dpps_serial + best_pass per frame, frame-parallel) on
    `frames_np`; returns wall ms."""
    from oracle import bindings as B
    lib = B.ref()
    n = frames_np.shape[0]
    arr, _keep = synthetic.as_ctypes(frames_np)
    p = abi.Params()
    lib.ref_params_default(C.byref(p))
    wall = C.c_double()
    m = B.msgbuf()
    st = lib.ref_batch(arr, n, C.byref(p), C.byref(c1_grid()), None, threads, None, None, None,
                       C.byref(wall), m, 512)
    if st != 0:
        raise RuntimeError(m.value.decode())
    return wall.value


def cpu_baseline_c5(seconds):
    """The reference's best CPU throughput shape on C5 frames, every host
    core, a bounded sample sized to ~`seconds` of CPU time."""
    from oracle import bindings as B
    if not B.ref_available():
        return None
    cores = os.cpu_count() or 1
    probe = max(2 * cores, 32)
    ms = cpu_batch(synthetic.c5_frames(0, probe), cores)
    per_frame_ms = ms / probe
    n = int(min(8192, max(1024, seconds * 1e3 / max(per_frame_ms, 1e-3))))
    ms = cpu_batch(synthetic.c5_frames(0, n), cores)
    value = n * C5_PAIRS_PER_FRAME / (ms / 1e3)
    return {"value": value, "unit": "pair-evals/s", "cores": cores, "kind": "reference",
            "frames_per_s": n / (ms / 1e3),
            "sample": f"C5 frames 0..{n - 1} (of 65,536; frames/s extrapolates linearly: frames "
                      f"are independent), ref_batch = run_dpps_serial + best_pass per frame, "
                      f"frame-parallel on {cores} threads, {ms / 1e3:.1f} s wall",
            **cpu_info()}


def cpu_frame_c2(seconds):
    """configs[1] frame F8 through run_dpps(workers=all cores) + best_pass."""
    from oracle import bindings as B
    if not B.ref_available():
        return None
    w, p, kicker = load_f8()
    grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 1)
    cores = os.cpu_count() or 1
    lib = B.ref()

    def timed(reps):
        search = (C.c_double * reps)()
        best = (C.c_double * reps)()
        m = B.msgbuf()
        st = lib.ref_time_frame(C.byref(w), C.byref(p), C.byref(grid), kicker, cores, reps, search,
                                best, m, 512)
        if st != 0:
            raise RuntimeError(m.value.decode())
        return list(search), list(best)

    s, b = timed(1)
    reps = max(5, min(200, int(seconds * 1e3 / max(s[0] + b[0], 1e-3))))
    s, b = timed(reps)
    tot = [x + y for x, y in zip(s, b)]
    return {"cores": cores, "reps": reps, "frame_ms_p50": statistics.median(tot),
            "search_ms_p50": statistics.median(s), "best_pass_ms_p50": statistics.median(b),
            "search_pair_evals_per_s": C2_PAIRS / (statistics.median(s) / 1e3)}


def run_reference(args, rank, world_size):
    if rank != 0:
        return 0
    from oracle import bindings as B
    if not B.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return 0
    cores = os.cpu_count() or 1
    per_step = max(1, args.ref_frames)
    all_frames = synthetic.c5_frames(0, per_step * min(args.steps + args.warmup, 64))

    def sample(i):
        k = i % (all_frames.shape[0] // per_step)
        return np.ascontiguousarray(all_frames[k * per_step:(k + 1) * per_step])

    for i in range(args.warmup):
        cpu_batch(sample(i), cores)
    t0 = time.perf_counter()
    ms = [cpu_batch(sample(args.warmup + i), cores) for i in range(args.steps)]
    wall = time.perf_counter() - t0
    mean_ms = sum(ms) / len(ms)
    value = per_step * C5_PAIRS_PER_FRAME / (mean_ms / 1e3)
    sample_desc = (f"{per_step} C5 frames per step (rotating through frames 0.."
                   f"{all_frames.shape[0] - 1}), ref_batch = run_dpps_serial + best_pass per "
                   f"frame, frame-parallel on {cores} threads")
    out = {"metric": METRIC, "value": value, "unit": "pair-evals/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_ms,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic", "config": CONFIG, "impl": "reference",
           "frames_per_s": per_step / (mean_ms / 1e3),
           "cpu_baseline": {"value": value, "unit": "pair-evals/s", "cores": cores,
                            "kind": "reference", "sample": sample_desc, **cpu_info()},
           "e2e": {"value": value, "unit": "pair-evals/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0},
           "wall_s": wall}
    print(json.dumps(out))
    return 0


# ---------------------------------------------------------------------------
# GPU side.

def _traffic_per_launch(n_frames, n_launches):
    """ncu DRAM bytes of the dominant kernel per launch of this run: the
    profiled per-frame traffic (profiles/ncu_summary.json, one ncu --set full
    capture) x the frames one scan launch processes here."""
    d = _load_json("profiles/ncu_summary.json")
    per_frame = d.get("dram_bytes_per_frame")
    if per_frame is None or n_launches < 1:
        return d.get("dram_bytes_per_launch")
    return per_frame * n_frames / n_launches


def run_ours(args, rank, world_size, local_rank):
    import torch
    import torch.distributed as dist

    # one process per GPU; (modulo only matters for the functional gloo check,
    # PP_BENCH_DIST_BACKEND=gloo, which may put several ranks on one device)
    gpu = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    backend = os.environ.get("PP_BENCH_DIST_BACKEND", "nccl")
    coll_dev = dev if backend == "nccl" else torch.device("cpu")
    if world_size > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    lib = abi.load_library()
    ctx = C.c_void_p()
    st = lib.pp_ctx_create(gpu, C.byref(ctx))
    if st != 0:
        raise RuntimeError(f"pp_ctx_create failed ({st})")

    def check(st):
        if st != 0:
            raise RuntimeError(lib.pp_last_error(ctx).decode())

    params = default_params(lib)
    grid = c1_grid()
    n_total = args.frames
    lo, hi = shard_range(n_total, rank, world_size)
    n_local = hi - lo
    frames_np = synthetic.c5_frames(lo, hi)
    frames, frames_ptr = synthetic.to_pinned(lib, frames_np)
    out_ptr = lib.pp_host_alloc(max(1, n_local) * C.sizeof(abi.FrameSummary))
    out = (abi.FrameSummary * n_local).from_address(out_ptr)

    stream = torch.cuda.ExternalStream(lib.pp_ctx_stream(ctx), device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world_size > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world_size == 1:
            return x
        t = torch.tensor([x], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- value: device-resident, L2 flushed between steps -------------------
    check(lib.pp_batch_upload(ctx, frames, n_local, None))
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            flush.zero_()
            check(lib.pp_batch_run(ctx, C.byref(params), C.byref(grid), None))
    check(lib.pp_batch_download(ctx, out))
    reference_bytes = bytes(out)
    barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(gpu) as clocks:
        barrier()
        t_wall0 = time.perf_counter()
        with torch.cuda.stream(stream):
            for i in range(args.steps):
                flush.zero_()                     # untimed: evict L2 between steps
                starts[i].record(stream)
                check(lib.pp_batch_run(ctx, C.byref(params), C.byref(grid), None))
                ends[i].record(stream)
        barrier()
        t_wall = time.perf_counter() - t_wall0
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    dev_total_ms = max_over_ranks(sum(step_ms))
    ms_per_step = dev_total_ms / args.steps
    value = n_total * C5_PAIRS_PER_FRAME * args.steps / (dev_total_ms / 1e3)
    check(lib.pp_batch_download(ctx, out))
    if bytes(out) != reference_bytes:
        raise RuntimeError("batch results changed between runs")

    # ---- e2e: pp_dpps_frames with host buffers (+ gather on rank 0) ---------
    gather_buf = None
    if world_size > 1:
        rows = -(-n_total // world_size) + 1
        gather_buf = torch.zeros((rows, C.sizeof(abi.FrameSummary)), dtype=torch.uint8,
                                 device=coll_dev)
        gathered = [torch.zeros_like(gather_buf) for _ in range(world_size)] if rank == 0 \
            else None

    def e2e_step():
        check(lib.pp_dpps_frames(ctx, frames, n_local, C.byref(params), C.byref(grid), None,
                                 out))
        if world_size > 1:
            host = torch.frombuffer(bytearray(bytes(out)), dtype=torch.uint8).view(
                n_local, C.sizeof(abi.FrameSummary))
            gather_buf[:n_local].copy_(host)
            dist.gather(gather_buf, gather_list=gathered, dst=0)

    for _ in range(args.warmup):
        e2e_step()
    e2e_ms = []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        barrier()
        ev0.record(stream)
        e2e_step()
        ev1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        e2e_ms.append(ev0.elapsed_time(ev1))
    e2e_total = max_over_ranks(sum(e2e_ms))
    e2e_value = n_total * C5_PAIRS_PER_FRAME * args.steps / (e2e_total / 1e3)
    if bytes(out) != reference_bytes:
        raise RuntimeError("e2e results differ from the device-resident run")
    # gathered frame-order results on rank 0 (the sharded answer)
    gathered_ok = None
    if world_size > 1 and rank == 0:
        parts = []
        for r in range(world_size):
            a, b = shard_range(n_total, r, world_size)
            parts.append(gathered[r][:b - a].cpu().numpy())
        # every rank's shard is checked on rank 0's own GPU on a sample of its
        # frames (untimed): the gathered rows must be byte-identical
        ok = int(sum(p.shape[0] for p in parts)) == n_total
        for r in range(world_size):
            a, b = shard_range(n_total, r, world_size)
            m = min(64, b - a)
            if m <= 0:
                continue
            chk = (abi.FrameSummary * m)()
            fr, _keep = synthetic.as_ctypes(synthetic.c5_frames(a, a + m))
            check(lib.pp_dpps_frames(ctx, fr, m, C.byref(params), C.byref(grid), None, chk))
            ok = ok and bytes(chk) == parts[r][:m].tobytes()
        gathered_ok = ok

    # ---- kernel split of one step (events between the kernels, no overlap) --
    stage_ms, scan_ms, value_ms = C.c_float(), C.c_float(), C.c_float()
    n_launch = C.c_int32()
    check(lib.pp_batch_upload(ctx, frames, n_local, None))
    check(lib.pp_batch_kernel_times(ctx, C.byref(params), C.byref(grid), 1, C.byref(stage_ms),
                                    C.byref(scan_ms), C.byref(value_ms), C.byref(n_launch)))

    frame = None
    if rank == 0 and not args.no_extras:
        frame = run_frame_c2(lib, ctx, args, torch, stream, flush)
        frame["extras"] = run_extras(lib, ctx)

    if rank == 0:
        peaks = _load_json("MEASURED_PEAKS.json")
        fp = _load_json("profiles/fp_peaks.json")
        work = _load_json("profiles/c5_work.json")
        clk = clocks.summary()
        sm_max = clk.get("sm_max_mhz") or peaks.get("sm_max_mhz") or 1965.0
        if fp.get("fp32_tflops"):
            peak_tflops = fp["fp32_tflops"]
            peak_src = f"measured FP32 FMA throughput ({fp.get('how', 'profiles/fp_peaks.json')})"
        else:
            peak_tflops = 148 * 128 * 2 * sm_max * 1e6 / 1e12
            peak_src = "nominal FP32 148 SMs x 128 lanes x 2 x clocks.max.sm"
        w_pair = work.get("W_pair_flop", 634.2)
        # dominant kernel: scan_kernel (the SBIP search the W_pair figure counts)
        pairs_local = n_local * C5_PAIRS_PER_FRAME
        achieved = w_pair * pairs_local / (scan_ms.value / 1e3) / 1e12
        # stage + consts, then per group of frames: scan, score lower bounds, value
        n_steps_launch = 2 + 3 * int(n_launch.value)
        out_line = {
            "metric": METRIC, "value": value, "unit": "pair-evals/s", "n_gpus": world_size,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": CONFIG,
            "frames_per_s": n_total * args.steps / (dev_total_ms / 1e3),
            "p50_ms": frame["p50_ms"] if frame else None,
            "e2e": {"value": e2e_value, "unit": "pair-evals/s",
                    "frames_per_s": n_total * args.steps / (e2e_total / 1e3),
                    "ms_per_step": e2e_total / args.steps,
                    "h2d_bytes_per_step": n_total * C.sizeof(abi.World),
                    "d2h_bytes_per_step": n_total * C.sizeof(abi.FrameSummary),
                    "path": "pp_dpps_frames (pinned host frames in, 48 B/frame results out)"
                            + (f" + {backend} gather of all {world_size} ranks' results on rank 0"
                               if world_size > 1 else "")},
            "roofline": {"bound": "fp32-core", "achieved": achieved, "peak": peak_tflops,
                         "unit": "TFLOP/s", "frac": achieved / peak_tflops,
                         "traffic": _traffic_per_launch(n_local, int(n_launch.value)),
                         "kernel": "scan_warp_kernel (SBIP search, batch shape: a warp per tile)",
                         "kernel_ms": {"stage+consts": stage_ms.value, "scan": scan_ms.value,
                                       "value (incl. score-bound pre-pass)": value_ms.value,
                                       "scan_launches": int(n_launch.value)},
                         "note": f"algorithmic FLOP = W_pair {w_pair:.1f}/pair (SURVEY 8(d) "
                                 f"formula, counted on C5 frames: profiles/c5_work.json) x "
                                 f"{pairs_local} pairs per step / summed scan time (events); "
                                 f"peak = {peak_src}"},
            "clocks": clk,
            "gpu_launches": n_steps_launch * args.steps,
            "wall_s": t_wall,
            "gathered_ok": gathered_ok,
            "frame": frame,
        }
        if world_size == 1 and not args.no_cpu:
            out_line["cpu_baseline"] = cpu_baseline_c5(args.cpu_seconds)
            if frame is not None:
                cf = cpu_frame_c2(args.cpu_seconds / 4)
                frame["cpu_reference"] = cf
                if cf:
                    frame["search_speedup_vs_cpu"] = frame["search_pair_evals_per_s"] / \
                        cf["search_pair_evals_per_s"]
                    frame["frame_speedup_vs_cpu_e2e"] = cf["frame_ms_p50"] / frame["e2e_p50_ms"]
        print(json.dumps(out_line))
    lib.pp_host_free(frames_ptr)
    lib.pp_host_free(out_ptr)
    lib.pp_ctx_destroy(ctx)
    if world_size > 1:
        dist.destroy_process_group()
    return 0


def run_frame_c2(lib, ctx, args, torch, stream, flush):
    """Per-frame search latency on configs[1] (frame F8, 128 x 64 flat + chip):
    device-resident p50 (L2 flushed), e2e p50 through pp_dpps with host
    buffers, the scan/value kernel split and the search-only evaluation rate."""
    w, p, kicker = load_f8()
    grid = abi.SearchGrid(128, 64, 1.0, 6.5, 1, 1)
    n_cells = 16384
    block_bytes = int(lib.pp_grid_bytes(n_cells))
    hblock = lib.pp_host_alloc(block_bytes)

    def call():
        st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, abi.PP_COPY_ALL,
                         hblock)
        if st != 0:
            raise RuntimeError(lib.pp_last_error(ctx).decode())

    call()
    reps = max(args.steps, 50)
    with torch.cuda.stream(stream):
        for _ in range(5):
            flush.zero_()
            lib.pp_dpps_relaunch(ctx)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    with torch.cuda.stream(stream):
        for i in range(reps):
            flush.zero_()
            starts[i].record(stream)
            lib.pp_dpps_relaunch(ctx)
            ends[i].record(stream)
    torch.cuda.synchronize()
    dev_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    for _ in range(5):
        call()
    e2e = []
    for _ in range(reps):
        t0 = time.perf_counter()
        call()
        e2e.append((time.perf_counter() - t0) * 1e3)
    scan_ms, value_ms = C.c_float(), C.c_float()
    lib.pp_dpps_kernel_times(ctx, 50, C.byref(scan_ms), C.byref(value_ms))
    lib.pp_host_free(hblock)
    cpp_seq = cpp_plan_sequence(max(reps, 200))
    return {"workload": "configs[1]: frame F8 (8v8), 128x64 grid, flat+chip, 16,384 cells, "
                        "262,144 pass evaluations; search + value function + best_pass x3",
            "p50_ms": statistics.median(dev_ms), "p99_ms": float(np.percentile(dev_ms, 99)),
            "pair_evals_per_s": C2_PAIRS / (statistics.median(dev_ms) / 1e3),
            "e2e_p50_ms": statistics.median(e2e), "e2e_p99_ms": float(np.percentile(e2e, 99)),
            "e2e_h2d_bytes": int(lib.pp_dpps_upload_bytes()), "e2e_d2h_bytes": block_bytes,
            "scan_ms": scan_ms.value, "value_ms": value_ms.value,
            "search_pair_evals_per_s": C2_PAIRS / (scan_ms.value / 1e3),
            "reps": reps, "l2": "flushed between device-timed reps",
            "cpp_plan_sequence": cpp_seq}


def cpp_plan_sequence(reps):
    """The reference's plan sequence (run_dpps + best_pass all/flat/chip,
    passplan_main.cpp:87,102-104) through the C++ drop-in on the same frame:
    tests/cpp/build/plan_sequence, host-timed p50."""
    exe = os.path.join(ROOT, "tests", "cpp", "build", "plan_sequence")
    snap = os.path.join(ROOT, "tests", "golden", "data", "bench_16v16.json")
    if not os.path.exists(exe):
        return None
    try:
        r = subprocess.run([exe, snap, str(reps)], capture_output=True, text=True, timeout=300)
        return json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else \
            {"error": r.stderr.strip()[-300:]}
    except (OSError, ValueError, subprocess.TimeoutExpired) as e:
        return {"error": str(e)}


def run_extras(lib, ctx):
    """Secondary configs: C1 frame, C3 1 cm grid (device span and e2e with the
    whole 1.08 M-cell result block copied back), C4 run maps."""
    w, p, kicker = load_f8()
    ex = {}

    def frame_ms(grid, reps, copy):
        n = (grid.flat + grid.chip) * grid.n_directions * grid.n_powers
        nbytes = int(lib.pp_grid_bytes(n))
        ptr = lib.pp_host_alloc(nbytes)
        blk = abi.GridBlock(n, buf=(C.c_uint8 * nbytes).from_address(ptr))
        for _ in range(2):
            lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, copy, ptr)
        dev, e2e = [], []
        for _ in range(reps):
            t0 = time.perf_counter()
            st = lib.pp_dpps(ctx, C.byref(w), C.byref(p), C.byref(grid), kicker, copy, ptr)
            e2e.append((time.perf_counter() - t0) * 1e3)
            if st != 0:
                raise RuntimeError(lib.pp_last_error(ctx).decode())
            dev.append(blk.summary.device_ms)
        lib.pp_host_free(ptr)
        return dev, e2e, nbytes

    dev, _, _ = frame_ms(abi.SearchGrid(128, 64, 1.0, 6.5, 1, 0), 50, abi.PP_COPY_SUMMARY)
    ex["c1_flat_p50_ms"] = statistics.median(dev)
    g3 = abi.SearchGrid(1200, 900, 1.0, 6.5, 1, 0)
    dev, e2e, nbytes = frame_ms(g3, 50, abi.PP_COPY_ALL)
    ex["c3_1200x900_p50_ms"] = statistics.median(dev)
    ex["c3_p99_ms"] = float(np.percentile(dev, 99))
    ex["c3_pair_evals_per_s"] = 1200 * 900 * 16 / (statistics.median(dev) / 1e3)
    ex["c3_e2e_full_map_p50_ms"] = statistics.median(e2e)
    ex["c3_e2e_full_map_p99_ms"] = float(np.percentile(e2e, 99))
    ex["c3_e2e_d2h_bytes"] = nbytes
    for step in (0.1, 0.01):
        pp = abi.Params.from_buffer_copy(bytes(p))
        pp.thresholds.grid_step = step
        nv = C.c_int64()
        lib.pp_runmap_count(C.byref(w), C.byref(pp), 0xF, C.byref(nv))
        rbytes = abi.runmap_offsets(nv.value)["total"]
        rptr = lib.pp_host_alloc(rbytes)
        req = abi.RunmapRequest(0xF, 0, 4, 0, 0.0, 0.0, 1)
        ts = []
        for _ in range(6):
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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--frames", type=int, default=C5_FRAMES,
                    help="C5 frames per step (default: the full 65,536)")
    ap.add_argument("--ref-frames", type=int, default=256,
                    help="reference arm: C5 frames per timed step")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
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
