#!/bin/bash
# dedicated predict kernel: predict tests + bench timing
set -u
TAG=${1:-r02r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_shard.py -m gpu -x -q -k "predict or fullsize or shard" > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-variants > gpurun_out/${TAG}_bench.json 2>&1; echo "bench rc=$?"
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]);print(d['phases_ms']['predict'], d['roofline_predict'])"
