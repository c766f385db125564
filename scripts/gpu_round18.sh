#!/bin/bash
set -u
TAG=${1:-r01x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-variants --no-predict > gpurun_out/${TAG}_bench.json 2>&1; echo "bench rc=$?"
