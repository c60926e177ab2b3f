"""CPU, world_size 2 over gloo: the multi-GPU host path for batched frames
(contiguous frame shards, no collective inside a frame, final gather on rank
0) reproduces a single-process run bit for bit.  The per-rank runner is the
CPU oracle here; on GPUs it is pp_dpps_frames (tests/test_gpu_batch.py,
test_run_sharded_product_runner_n1)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1909_07717_b200 import abi
from paper_1909_07717_b200.sharding import max_over_ranks, run_sharded, shard_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GRID = abi.SearchGrid(12, 6, 1.0, 6.5, 1, 1)


def _frames(n):
    from paper_1909_07717_b200 import synthetic
    arr, keep = synthetic.as_ctypes(synthetic.c5_frames(0, n))
    return list(arr)


def _oracle_runner(frames):
    from oracle import bindings as B
    orc = B.oracle()
    p = abi.Params()
    orc.or_params_default(C.byref(p))
    n_cells = 2 * 12 * 6
    out = (abi.DppsSummary * len(frames))()
    for i, w in enumerate(frames):
        blk = abi.GridBlock(n_cells)
        k = orc.or_nearest_teammate(C.byref(w))
        assert orc.or_dpps(C.byref(w), C.byref(p), C.byref(GRID), k, blk.ptr(), None, 0) == 0
        out[i] = blk.summary
    return out


def _worker(rank, world, port, n_frames, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        frames = _frames(n_frames)
        got = run_sharded(frames, _oracle_runner, rank, world)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            q.put(("ok", bytes(got), t))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions():
    for n in (0, 1, 7, 65536):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


@pytest.mark.timeout(300)
def test_two_rank_gloo_batch_matches_single_process():
    n_frames = 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, blob, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert status == "ok" and tmax == 2.0
    got = (abi.DppsSummary * n_frames).from_buffer_copy(blob)
    want = _oracle_runner(_frames(n_frames))
    for i in range(n_frames):
        assert bytes(got[i]) == bytes(want[i]), i
    assert any(got[i].best_cell[0] >= 0 for i in range(n_frames))
