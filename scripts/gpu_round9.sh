#!/bin/bash
set -u
TAG=${1:-r01i}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ann.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 400 python bench.py --sampling ann --beta 1e3 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-predict > gpurun_out/${TAG}_bench_ann.json 2>&1; echo "bench ann rc=$?"
timeout 400 python bench.py --beta 1e5 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-predict > gpurun_out/${TAG}_bench.json 2>&1; echo "bench rc=$?"
BIG="python bench.py --sampling ann --beta 1e3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --max-it 5"
timeout 300 $BIG > gpurun_out/${TAG}_big_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv \
    --log-file gpurun_out/${TAG}_ann_launches.csv $BIG > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
