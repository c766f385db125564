#!/bin/bash
set -u
TAG=${1:-r01m}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ann.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
SVMHSS_TRACE=1 timeout 400 python bench.py --sampling ann --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-predict --max-it 20 > gpurun_out/${TAG}_trace_ann.log 2>&1; echo "trace ann rc=$?"
BIG="python bench.py --sampling ann --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --max-it 5"
timeout 300 $BIG > gpurun_out/${TAG}_big_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'bgemm_kernel' -s 2 -c 3 \
    -o gpurun_out/${TAG}_bgemm $BIG > gpurun_out/${TAG}_ncu_bgemm.log 2>&1; echo "ncu rc=$?"
