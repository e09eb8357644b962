tools/k1_variants > gpurun_out/r02_k1_variants_c.log 2>&1; echo k1 rc=$?
ORDER="new nokeep" timeout 900 bash tools/lib_ab.sh 3 > gpurun_out/r02_ab_keep.jsonl 2> gpurun_out/r02_ab_keep.err; echo ab rc=$?
timeout 900 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "audit or multibucket or fused_k12" > gpurun_out/r02_audit.log 2>&1; echo audit rc=$?
