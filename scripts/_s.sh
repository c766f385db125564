for v in a b c a b c; do cp abso/lib_$v.so paper_2108_04167_b200/libsvmhss.so; echo "V=$v"; timeout 300 python scripts/admm_loop_time.py; done > gpurun_out/leafab.log 2>&1
cat gpurun_out/leafab.log
