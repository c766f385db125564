#!/bin/bash
# A/B of ADMM-loop launch knobs (env VAR=VALUE pairs per run), config 3, 2 repetitions each
set -u
TAG=$1; shift
mkdir -p gpurun_out
for rep in 1 2; do
  for cfg in "$@"; do
    echo "$cfg rep$rep: $(env $cfg timeout 600 python scripts/admm_profile.py sketch 2>&1 | grep 'loop ms')" >> gpurun_out/${TAG}_admm_ab.log
  done
done
