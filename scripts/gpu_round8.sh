#!/bin/bash
set -u
TAG=${1:-r01h}
mkdir -p gpurun_out
MID="python bench.py --beta 1e5 --n 131072 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --max-it 5"
timeout 300 $MID > gpurun_out/${TAG}_mid_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'bgemm_kernel|bgeqrf_kernel|btrsm_kernel|bpotrf' -s 40 -c 8 \
    -o gpurun_out/${TAG}_factor $MID > gpurun_out/${TAG}_ncu_factor.log 2>&1; echo "ncu factor rc=$?"
BIG="python bench.py --sampling ann --beta 1e3 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-predict --max-it 5"
timeout 300 $BIG > gpurun_out/${TAG}_big_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv \
    --log-file gpurun_out/${TAG}_ann_launches.csv $BIG > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
