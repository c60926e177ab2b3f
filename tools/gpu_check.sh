#!/bin/bash
# Dev tool (GPU box): GPU test suite, smoke, default bench, launch list.
# usage: tools/gpu_check.sh TAG
tag=${1:-x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/$tag.smi 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/$tag.tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/$tag.tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$tag.smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/$tag.smoke.log
timeout 900 python bench.py > gpurun_out/$tag.bench.json 2> gpurun_out/$tag.bench.err; echo "bench rc=$?" >> gpurun_out/$tag.bench.err
