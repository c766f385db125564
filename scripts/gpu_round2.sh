#!/bin/bash
# GPU call: all -m gpu tests, fused/unfused dev bench lines, targeted ncu counters of the
# sketch at full size, and ncu --set full captures at a reduced size.
set -u
TAG=${1:-r01b}
BETA=${2:-1e5}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
DBG="python bench.py --beta $BETA --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $DBG > gpurun_out/${TAG}_bench_fused.json 2> gpurun_out/${TAG}_bench_fused.err; echo "bench fused rc=$?"
SVMHSS_FUSE_BOTTOM=0 timeout 300 $DBG > gpurun_out/${TAG}_bench_unfused.json 2> gpurun_out/${TAG}_bench_unfused.err; echo "bench unfused rc=$?"
SMALL="python bench.py --beta $BETA --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --max-it 30"
timeout 300 $SMALL > gpurun_out/${TAG}_small_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:kmm_kernel -c 1 --csv --log-file gpurun_out/${TAG}_sketch_counters.csv $SMALL \
    > gpurun_out/${TAG}_ncu_counters.log 2>&1; echo "ncu counters rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${TAG}_launches.csv $SMALL > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
MID="python bench.py --beta $BETA --n 65536 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --max-it 10"
timeout 300 $MID > gpurun_out/${TAG}_mid_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'kmm_kernel|admm_bottom|ulv_(fwd|bwd)_kernel' -c 6 \
    -o gpurun_out/${TAG}_full $MID > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu full rc=$?"
