#!/bin/bash
# One gpurun call: GPU parity tests, the bench line, the launch list and ncu captures of the
# top kernels.  Usage (from the repo root on the box): bash scripts/gpu_round.sh <tag> [beta]
set -u
TAG=${1:-r01}
BETA=${2:-}
BARG=""
[ -n "$BETA" ] && BARG="--beta $BETA"
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${TAG}_smi.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
python bench.py $BARG > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
DBG="python bench.py $BARG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$DBG > gpurun_out/${TAG}_dbg_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/${TAG}_launches.csv $DBG > gpurun_out/${TAG}_ncu_launch.log 2>&1; echo "launch rc=$?"
if [ "${NCU_FULL:-1}" = 1 ]; then
  ncu --set full --clock-control none --import-source on -k regex:'kmm_kernel' -c 1 \
      -o gpurun_out/${TAG}_sketch $DBG > gpurun_out/${TAG}_ncu_sketch.log 2>&1; echo "ncu sketch rc=$?"
  ncu --set full --clock-control none --import-source on -k regex:'ulv_(fwd|bwd)_kernel' -s 40 -c 4 \
      -o gpurun_out/${TAG}_solve $DBG > gpurun_out/${TAG}_ncu_solve.log 2>&1; echo "ncu solve rc=$?"
fi
