#!/bin/bash
set -u
TAG=${1:-r01f}
BETA=${2:-1e5}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
DBG="python bench.py --beta $BETA --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-predict"
timeout 400 $DBG > gpurun_out/${TAG}_bench.json 2>&1; echo "bench rc=$?"
SMALL="python bench.py --beta $BETA --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --max-it 20"
timeout 300 $SMALL > gpurun_out/${TAG}_small_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'ulv_|admm_|tree_reduce|exch_' -c 120 --csv --log-file gpurun_out/${TAG}_loop_launches.csv $SMALL \
   > gpurun_out/${TAG}_ncu_loop.log 2>&1; echo "ncu loop rc=$?"
