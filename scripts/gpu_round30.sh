#!/bin/bash
# dataflow top levels: bitwise test + ADMM loop A/B (ms/iteration, 200 iterations)
set -u
timeout 600 python -m pytest tests/test_gpu_topmerge.py -m gpu -x -q 2>&1 | tail -3
for rep in 1 2; do
  for m in 0 2 1; do
    echo -n "top=$m: "; SVMHSS_TOP_MERGE=$m timeout 300 python scripts/admm_profile.py 2>&1 | grep loop
  done
done
