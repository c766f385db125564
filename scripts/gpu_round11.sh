#!/bin/bash
set -u
TAG=${1:-r01l}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/${TAG}_fullsize_tests.log 2>&1; echo "fullsize rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "generators or solve" > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
for C in 0 1 2; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg$C.json 2>&1; echo "bench cfg$C rc=$?"
done
timeout 900 python bench.py --config 4 --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_cfg4.json 2>&1; echo "bench cfg4 rc=$?"
SVMHSS_TRACE=1 timeout 400 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-predict --max-it 20 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"
