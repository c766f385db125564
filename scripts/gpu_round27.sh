#!/bin/bash
# ncu --set full of the round-2 kernels: factor level-10 launches (QR, Cholesky, TRSM, larft,
# a 512x512x256 GEMM) and the prediction kernel
set -u
TAG=${1:-r02s}
mkdir -p gpurun_out
timeout 300 python scripts/factor_profile.py sketch > gpurun_out/${TAG}_fplain.log 2>&1; echo "factor plain rc=$?"
timeout 300 python scripts/predict_profile.py 16384 > gpurun_out/${TAG}_pplain.log 2>&1; echo "predict plain rc=$?"; cat gpurun_out/${TAG}_pplain.log
for spec in "bgeqrf_tc:1" "bpotrf_tc:1" "btrsm_tc:2" "blarft_blk:1" "bgemm_dmma:12"; do
  k=${spec%%:*}; sk=${spec##*:}
  timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:$k --launch-skip $sk -c 1 \
    -o gpurun_out/${TAG}_$k python scripts/factor_profile.py sketch > gpurun_out/${TAG}_ncu_$k.log 2>&1; echo "ncu $k rc=$?"
done
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:predict_kernel -c 1 \
  -o gpurun_out/${TAG}_predict python scripts/predict_profile.py 16384 > gpurun_out/${TAG}_ncu_predict.log 2>&1; echo "ncu predict rc=$?"
