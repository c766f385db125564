#!/bin/bash
set -u
TAG=${1:-r01n}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_errors.py tests/test_gpu_parity.py tests/test_gpu_ann.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
SVMHSS_TRACE=1 timeout 400 python bench.py --sampling ann --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-predict --max-it 20 > gpurun_out/${TAG}_trace_ann.log 2>&1; echo "trace ann rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2>&1; echo "bench rc=$?"
