#!/bin/bash
# refresh the per-config bench lines (configs 0, 1, 2 and the config-4 grid)
set -u
TAG=${1:-r02zd}
mkdir -p gpurun_out
for c in 0 1 2 4; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/${TAG}_cfg$c.json 2> gpurun_out/${TAG}_cfg$c.err; echo "cfg$c rc=$?"
  tail -1 gpurun_out/${TAG}_cfg$c.json | cut -c1-300
done
