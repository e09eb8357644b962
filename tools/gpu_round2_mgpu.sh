# 2 GPUs at HEAD: multi-GPU tests (mp_check x 4 exchanges incl. the split exchange, LocalCluster)
timeout 3000 python -m pytest tests/test_multi_gpu.py -q > gpurun_out/r2w_multi_gpu.log 2>&1; echo multi rc=$?
tail -n 3 gpurun_out/r2w_multi_gpu.log
tools/k1_variants quick > gpurun_out/r2w_k1_v6.log 2>&1; echo k1v rc=$?
