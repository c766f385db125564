#!/bin/bash
set -u
TAG=${1:-r02g}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
timeout 300 python scripts/factor_profile.py sketch 2>&1 | tail -1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_factor_launches.csv python scripts/factor_profile.py sketch > gpurun_out/${TAG}_factor_ncu.log 2>&1; echo "ncu rc=$?"
