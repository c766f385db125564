#!/bin/bash
set -u
TAG=${1:-r01o}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-predict > gpurun_out/${TAG}_bench.json 2>&1; echo "bench rc=$?"
SVMHSS_TOP_MERGE=0 timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu-baseline --no-predict > gpurun_out/${TAG}_bench_nomerge.json 2>&1; echo "bench nomerge rc=$?"
SMALL="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --max-it 20"
timeout 300 $SMALL > gpurun_out/${TAG}_small_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'ulv_|admm_|tree_reduce|exch_' -c 120 --csv --log-file gpurun_out/${TAG}_loop_launches.csv $SMALL \
   > gpurun_out/${TAG}_ncu_loop.log 2>&1; echo "ncu loop rc=$?"
