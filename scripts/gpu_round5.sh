#!/bin/bash
set -u
TAG=${1:-r01e}
BETA=${2:-1e5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fused.py -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
DBG="python bench.py --beta $BETA --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-predict"
for C in 16 24 36; do
  SVMHSS_FUSE_CLUSTERS=$C timeout 300 $DBG > gpurun_out/${TAG}_bench_c$C.json 2>&1; echo "bench c$C rc=$?"
done
SVMHSS_FUSE_BOTTOM=0 timeout 300 $DBG > gpurun_out/${TAG}_bench_unfused.json 2>&1; echo "bench unfused rc=$?"
