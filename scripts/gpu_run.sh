#!/bin/bash
# One parameterised GPU session (run under gpurun): TAG then any of
#   smoke        __graft_entry__.smoke()
#   tests        pytest -m gpu (TESTK="expr" restricts with -k)
#   reference    bench.py --impl reference (the oracle arm)
#   bench        default bench line, then --sampling ann
#   launchlist   ncu launch list of the default bench command (after it ran clean without ncu)
#   buildprof    ncu launch list of one config-3 build (scripts/build_profile.py sketch)
#   factorprof   ncu launch list of one config-3 factorization
#   admmprof     ncu launch list of 3 ADMM iterations at config 3
#   cpqrab       CPQR mode A/B at config 3
#   ab           bench A/B of one env knob: AB="VAR VALA VALB"
# The driver's round-end order is: smoke tests reference bench.
# usage: bash scripts/gpu_run.sh TAG task [task ...]
set -u
TAG=$1; shift
mkdir -p gpurun_out
NCU="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off"
for t in "$@"; do
  case $t in
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?";;
    tests) if [ -n "${TESTK:-}" ]; then K=(-k "$TESTK"); else K=(); fi
           timeout 2400 python -m pytest tests -m gpu -x -q "${K[@]}" > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?";;
    reference) timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err; echo "reference rc=$?";;
    bench) timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
           timeout 900 python bench.py --sampling ann > gpurun_out/${TAG}_bench_ann.json 2> gpurun_out/${TAG}_bench_ann.err; echo "bench ann rc=$?";;
    launchlist) timeout 900 python bench.py > gpurun_out/${TAG}_bench_plain.json 2> gpurun_out/${TAG}_bench_plain.err && \
                timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
                  --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py > gpurun_out/${TAG}_ncu_bench.log 2>&1; echo "launchlist rc=$?";;
    buildprof) timeout 600 python scripts/build_profile.py sketch > gpurun_out/${TAG}_build_plain.log 2>&1 && \
               timeout 1200 $NCU --log-file gpurun_out/${TAG}_build_launches.csv python scripts/build_profile.py sketch > gpurun_out/${TAG}_build_ncu.log 2>&1; echo "buildprof rc=$?";;
    factorprof) timeout 600 python scripts/factor_profile.py > gpurun_out/${TAG}_factor_plain.log 2>&1 && \
               timeout 1200 $NCU --log-file gpurun_out/${TAG}_factor_launches.csv python scripts/factor_profile.py > gpurun_out/${TAG}_factor_ncu.log 2>&1; echo "factorprof rc=$?";;
    admmprof) timeout 600 python scripts/admm_profile.py sketch > gpurun_out/${TAG}_admm_plain.log 2>&1 && \
              timeout 1200 $NCU --log-file gpurun_out/${TAG}_admm_launches.csv python scripts/admm_profile.py sketch > gpurun_out/${TAG}_admm_ncu.log 2>&1; echo "admmprof rc=$?";;
    cpqrab) for m in 0 1 2; do timeout 600 python scripts/cpqr_ab.py $m sketch >> gpurun_out/${TAG}_cpqr_ab.log 2>&1; done; echo "cpqrab done";;
    ab) set -- ${AB}; VAR=$1; A=$2; B=$3
        CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-variants --no-predict"
        for rep in 1 2; do
          env $VAR=$A timeout 600 $CMD > gpurun_out/${TAG}_A$rep.json 2>&1
          env $VAR=$B timeout 600 $CMD > gpurun_out/${TAG}_B$rep.json 2>&1
        done; echo "ab done";;
    *) echo "unknown task $t";;
  esac
done
