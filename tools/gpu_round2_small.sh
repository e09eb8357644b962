timeout 600 python tools/small_sets.py 50 googlenet layer_1M layer_4M layer_16M > gpurun_out/r02_small_chunks.jsonl 2> gpurun_out/r02_small_chunks.err; echo small rc=$?
timeout 600 python tools/local_latency.py googlenet 2 4 8 > gpurun_out/r02_local_latency.jsonl 2> gpurun_out/r02_local_latency.err; echo lat rc=$?
tools/k1_variants > gpurun_out/r02_k1_variants_b.log 2>&1; echo k1 rc=$?
