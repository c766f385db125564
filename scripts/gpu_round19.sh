#!/bin/bash
# cluster CPQR: exactness (forced on every level) + A/B build time
set -u
TAG=${1:-r01y}
mkdir -p gpurun_out
SVMHSS_CPQR_CLUSTER=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ann.py tests/test_gpu_adaptive.py -m gpu -x -q > gpurun_out/${TAG}_tests_forced.log 2>&1; echo "forced tests rc=$?"
for m in 0 2 1; do
  for smp in sketch ann; do
    SVMHSS_TRACE=1 timeout 600 python scripts/cpqr_ab.py $m $smp > gpurun_out/${TAG}_ab_${m}_${smp}.log 2>&1; echo "ab $m $smp rc=$?"
  done
done
grep -h "mode=" gpurun_out/${TAG}_ab_*.log
