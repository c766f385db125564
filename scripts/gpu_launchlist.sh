#!/bin/bash
# The ncu launch list of the default bench command (B200_PROFILING.md recipe), after the same
# command exited 0 without ncu in the same call.
set -u
TAG=${1:-r01_final}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_bench_plain.json 2> gpurun_out/${TAG}_bench_plain.err && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "rc=$?"
