#!/bin/bash
set -u
TAG=${1:-r01g}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ann.py -m gpu -x -q > gpurun_out/${TAG}_gpu_ann_tests.log 2>&1; echo "ann tests rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 400 python bench.py --sampling ann --beta 1e3 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_ann.json 2>&1; echo "bench ann rc=$?"
timeout 400 python bench.py --beta 1e5 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-predict > gpurun_out/${TAG}_bench.json 2>&1; echo "bench rc=$?"
