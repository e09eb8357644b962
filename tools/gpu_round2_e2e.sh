timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "step_host" > gpurun_out/r2e_tests.log 2>&1; echo tests rc=$?
tail -n 2 gpurun_out/r2e_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --e2e-steps 10 --no-cpu-baseline > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo bench rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --e2e-steps 10 --no-cpu-baseline --workload alexnet > gpurun_out/r2e_bench_alexnet.json 2> gpurun_out/r2e_bench_alexnet.err; echo bench rc=$?
