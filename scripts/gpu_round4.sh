#!/bin/bash
set -u
TAG=${1:-r01d}
BETA=${2:-1e5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
DBG="python bench.py --beta $BETA --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-predict"
for C in 18 36 72; do
  SVMHSS_FUSE_CLUSTERS=$C timeout 300 $DBG > gpurun_out/${TAG}_bench_c$C.json 2>&1; echo "bench c$C rc=$?"
done
SVMHSS_FUSE_BOTTOM=0 timeout 300 $DBG > gpurun_out/${TAG}_bench_unfused.json 2>&1; echo "bench unfused rc=$?"
SMALL="python bench.py --beta $BETA --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --max-it 20"
timeout 300 $SMALL > gpurun_out/${TAG}_small_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:'ulv_|admm_|tree_reduce|exch_' -c 200 --csv --log-file gpurun_out/${TAG}_loop_launches.csv $SMALL \
   > gpurun_out/${TAG}_ncu_loop.log 2>&1; echo "ncu loop rc=$?"
