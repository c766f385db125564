# scratch GPU session: factor timing trace + the factor/solve parity tests
SVMHSS_TRACE=1 timeout 600 python scripts/factor_profile.py sketch > gpurun_out/q_factor_trace.log 2>&1
tail -1 gpurun_out/q_factor_trace.log
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py tests/test_gpu_fullsize_parity.py tests/test_gpu_admm_variants.py -m gpu -x -q > gpurun_out/q_tests.log 2>&1
tail -3 gpurun_out/q_tests.log
