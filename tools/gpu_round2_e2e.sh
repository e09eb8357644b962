timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "step_host" > gpurun_out/r2e_tests.log 2>&1; echo tests rc=$?
tail -n 2 gpurun_out/r2e_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --e2e-steps 10 --no-cpu-baseline > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo bench rc=$?
timeout 300 python tools/step_timeline.py googlenet > gpurun_out/r2e_tl1_googlenet.json 2> gpurun_out/r2e_tl1_googlenet.err; echo tl rc=$?
timeout 300 python tools/opt_probe.py momentum > gpurun_out/r2e_opt_momentum.log 2>&1; echo opt rc=$?
