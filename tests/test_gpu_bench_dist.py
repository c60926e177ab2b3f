"""GPU: the multi-rank bench path end to end (bench.py --gpus 2 under
torch.distributed.run): each rank uploads its contiguous range of the C5
frames, runs the batch pipeline on its device and the per-frame results are
gathered on rank 0, which re-checks a sample of every rank's rows against its
own GPU (gathered_ok).  Only one B200 is available here, so both ranks share
device 0 and the gather goes over gloo (PP_BENCH_DIST_BACKEND=gloo); the
timings of this run mean nothing, the data path is the N-GPU one."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(600)
def test_bench_two_ranks_shard_and_gather():
    env = dict(os.environ, PP_BENCH_DIST_BACKEND="gloo", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29531", "bench.py", "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--frames", "8192", "--no-cpu", "--no-extras"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=540)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2
    assert line["gathered_ok"] is True
    assert line["frames_per_s"] > 0 and line["e2e"]["frames_per_s"] > 0
