for k in 2 4 2 4; do cp abso/lib_k$k.so paper_2108_04167_b200/libsvmhss.so; echo "KCH=$k"; timeout 300 python scripts/kmm_probe.py 131072; done > gpurun_out/kch.log 2>&1
cat gpurun_out/kch.log
