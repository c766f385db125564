#!/bin/bash
# A/B of an env knob within one box: bash scripts/gpu_ab.sh TAG VAR VALA VALB
set -u
TAG=$1; VAR=$2; A=$3; B=$4
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-variants --no-predict"
for rep in 1 2; do
  env $VAR=$A timeout 600 $CMD > gpurun_out/${TAG}_A$rep.json 2>&1
  env $VAR=$B timeout 600 $CMD > gpurun_out/${TAG}_B$rep.json 2>&1
done
for f in gpurun_out/${TAG}_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value'],1), round(d['hss_build_ulv_s'],3))"; done
