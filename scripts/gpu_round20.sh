#!/bin/bash
# DMMA batched GEMM: parity suite + factor A/B against the DFMA kernels
set -u
TAG=${1:-r02b}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_tests.log
for v in 1 0; do
  for smp in sketch ann; do
    SVMHSS_GEMM_DFMA=$v SVMHSS_TRACE=1 timeout 400 python scripts/cpqr_ab.py 2 $smp > gpurun_out/${TAG}_gemm${v}_$smp.log 2>&1; echo "dfma=$v $smp rc=$?"
    grep mode= gpurun_out/${TAG}_gemm${v}_$smp.log
  done
done
