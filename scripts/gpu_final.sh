#!/bin/bash
# The driver's round-end commands, in order: smoke, -m gpu tests, the reference arm, the bench line.
set -u
TAG=${1:-r01_final}
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err; echo "reference rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --sampling ann > gpurun_out/${TAG}_bench_ann.json 2> gpurun_out/${TAG}_bench_ann.err; echo "bench ann rc=$?"
