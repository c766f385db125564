#!/bin/bash
# One parameterised GPU session (replaces the per-round lease scripts): TAG then any of
#   tests        pytest -m gpu
#   smoke        __graft_entry__.smoke()
#   bench        default bench line (+ --impl reference)
#   buildprof    ncu launch list of one config-3 build (scripts/build_profile.py sketch)
#   factorprof   ncu launch list of one config-3 factorization
#   admmprof     ncu launch list of 3 ADMM iterations at config 3
# usage: bash scripts/gpu_run.sh TAG task [task ...]
set -u
TAG=$1; shift
mkdir -p gpurun_out
NCU="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --profile-from-start off"
for t in "$@"; do
  case $t in
    tests) timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "tests rc=$?";;
    smoke) timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?";;
    bench) timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
           timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err; echo "reference rc=$?";;
    buildprof) timeout 600 python scripts/build_profile.py sketch > gpurun_out/${TAG}_build_plain.log 2>&1 && \
               timeout 1200 $NCU --log-file gpurun_out/${TAG}_build_launches.csv python scripts/build_profile.py sketch > gpurun_out/${TAG}_build_ncu.log 2>&1; echo "buildprof rc=$?";;
    factorprof) timeout 600 python scripts/factor_profile.py > gpurun_out/${TAG}_factor_plain.log 2>&1 && \
               timeout 1200 $NCU --log-file gpurun_out/${TAG}_factor_launches.csv python scripts/factor_profile.py > gpurun_out/${TAG}_factor_ncu.log 2>&1; echo "factorprof rc=$?";;
    admmprof) timeout 600 python scripts/admm_profile.py sketch > gpurun_out/${TAG}_admm_plain.log 2>&1 && \
              timeout 1200 $NCU --log-file gpurun_out/${TAG}_admm_launches.csv python scripts/admm_profile.py sketch > gpurun_out/${TAG}_admm_ncu.log 2>&1; echo "admmprof rc=$?";;
    cpqrab) for m in 0 1 2; do timeout 600 python scripts/cpqr_ab.py $m sketch >> gpurun_out/${TAG}_cpqr_ab.log 2>&1; done
            SVMHSS_CPQR_NB=4 timeout 600 python scripts/cpqr_ab.py 1 sketch >> gpurun_out/${TAG}_cpqr_ab.log 2>&1; echo "cpqrab done";;
    testsk) timeout 1800 python -m pytest tests -m gpu -q -k "${TESTK:-boundary}" > gpurun_out/${TAG}_gpu_testsk.log 2>&1; echo "testsk rc=$?";;
    *) echo "unknown task $t";;
  esac
done
