#!/bin/bash
set -u
TAG=${1:-r01j}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q -k "kernel_matmul or build_tree or matvec or subtree" > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
SVMHSS_TRACE=1 timeout 400 python bench.py --sampling ann --beta 1e3 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-predict --max-it 50 > gpurun_out/${TAG}_trace_ann.log 2>&1; echo "trace ann rc=$?"
SVMHSS_TRACE=1 timeout 400 python bench.py --beta 1e5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-predict --max-it 50 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"
MID="python bench.py --beta 1e5 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --max-it 5"
timeout 300 $MID > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:kmm_kernel -c 1 --csv \
    --log-file gpurun_out/${TAG}_sketch_counters.csv $MID > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
