#!/bin/bash
# ncu evidence of the current kernels: sketch (persistent) at n=65536 and the ULV sweeps +
# epilogue at n=524288, plus the factor GEMM / QR at n=131072.
set -u
TAG=${1:-r01w}
mkdir -p gpurun_out
MID="python bench.py --n 65536 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --no-variants --max-it 5"
timeout 300 $MID > gpurun_out/${TAG}_mid_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kmm_kernel' -c 1 \
    -o gpurun_out/${TAG}_sketch $MID > gpurun_out/${TAG}_ncu_sketch.log 2>&1; echo "ncu sketch rc=$?"
BIG="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --no-variants --max-it 3"
timeout 300 $BIG > gpurun_out/${TAG}_big_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'ulv_fwd_kernel|ulv_bwd_kernel|admm_epilogue' -s 30 -c 5 \
    -o gpurun_out/${TAG}_solve $BIG > gpurun_out/${TAG}_ncu_solve.log 2>&1; echo "ncu solve rc=$?"
FAC="python bench.py --n 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --no-variants --max-it 3"
timeout 300 $FAC > gpurun_out/${TAG}_fac_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'bgemm_big_kernel|bgeqrf|blarft' -c 4 \
    -o gpurun_out/${TAG}_factor $FAC > gpurun_out/${TAG}_ncu_factor.log 2>&1; echo "ncu factor rc=$?"
