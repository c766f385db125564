#!/bin/bash
set -u
TAG=${1:-r01c}
BETA=${2:-1e5}
mkdir -p gpurun_out
./scripts/micro/dfma_rate > gpurun_out/${TAG}_dfma_rate.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_shard.py tests/test_gpu_fused.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
DBG="python bench.py --beta $BETA --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $DBG > gpurun_out/${TAG}_bench_fused.json 2> gpurun_out/${TAG}_bench_fused.err; echo "bench fused rc=$?"
