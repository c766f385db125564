for v in 64 32 128 64 32 128; do cp abso/lib_rb$v.so paper_2108_04167_b200/libsvmhss.so; echo "KRB=$v"; timeout 300 python scripts/admm_loop_time.py; done > gpurun_out/krb.log 2>&1
cat gpurun_out/krb.log
