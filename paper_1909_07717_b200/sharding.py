"""Multi-GPU host logic for batched frames.

Frames are independent, so a batch shards as contiguous frame ranges, one
rank (process) per GPU, with no collective inside a frame.  The only
exchange is the final gather of the per-frame results to rank 0: 48 B per
frame with pp_frame_summary (pp_dpps_frames), 0.5 KB with the full
pp_dpps_summary (pp_dpps_batch).  A single frame never shards ("replicas
only").

`run_sharded` is backend-agnostic: the caller supplies the per-rank runner
(the product's pp_dpps_frames on the rank's GPU; the CPU tests pass the
oracle).
"""
from __future__ import annotations

import ctypes as C
from typing import Callable, Sequence

import numpy as np

from . import abi


def shard_range(n_items: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous range [lo, hi) of rank `rank` out of `world` (balanced)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (rank * n_items) // world, ((rank + 1) * n_items) // world


def summaries_to_array(summaries, row_type=abi.DppsSummary) -> np.ndarray:
    """ctypes array of per-frame results -> raw uint8 rows (one per frame)."""
    n = len(summaries)
    size = C.sizeof(row_type)
    return np.frombuffer(bytes(summaries), dtype=np.uint8).reshape(n, size).copy()


def array_to_summaries(arr: np.ndarray, row_type=abi.DppsSummary):
    n = arr.shape[0]
    out = (row_type * n)()
    C.memmove(out, np.ascontiguousarray(arr).ctypes.data, arr.nbytes)
    return out


def run_sharded(frames: Sequence, runner: Callable, rank: int, world: int, group=None,
                row_type=abi.DppsSummary):
    """Run `runner(frames_slice) -> array of row_type` on this rank's shard
    and gather every frame's result, in frame order, on rank 0 (None
    elsewhere).  Uses torch.distributed (nccl on GPUs, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    lo, hi = shard_range(len(frames), rank, world)
    local = runner(frames[lo:hi]) if hi > lo else (row_type * 0)()
    rows = summaries_to_array(local, row_type) if hi > lo else \
        np.zeros((0, C.sizeof(row_type)), np.uint8)
    if world == 1:
        return array_to_summaries(rows, row_type)
    size = C.sizeof(row_type)
    max_rows = -(-len(frames) // world) + 1
    buf = np.zeros((max_rows, size), np.uint8)
    buf[:rows.shape[0]] = rows
    t = torch.from_numpy(buf)
    backend = dist.get_backend(group)
    if backend == "nccl":
        t = t.cuda()
    gathered = [torch.zeros_like(t) for _ in range(world)] if rank == 0 else None
    dist.gather(t, gather_list=gathered, dst=0, group=group)
    if rank != 0:
        return None
    parts = []
    for r in range(world):
        a, b = shard_range(len(frames), r, world)
        parts.append(gathered[r].cpu().numpy()[:b - a])
    return array_to_summaries(np.concatenate(parts, axis=0), row_type)


def max_over_ranks(value: float, group=None) -> float:
    """Max of a per-rank scalar (timing rule: max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
