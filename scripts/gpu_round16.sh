#!/bin/bash
set -u
TAG=${1:-r01v}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ann.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
SVMHSS_TRACE=1 timeout 400 python bench.py --sampling ann --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-predict --max-it 20 > gpurun_out/${TAG}_trace_ann.log 2>&1; echo "trace ann rc=$?"
SVMHSS_TRACE=1 timeout 400 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-predict --max-it 20 --no-variants > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"
