# final one-GPU pass at HEAD: smoke, GPU tests, default bench + reference arm, ncu evidence
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2y_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2y_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/r2y_tests.log
timeout 900 python bench.py > gpurun_out/r2y_bench_default.json 2> gpurun_out/r2y_bench_default.err; echo bench rc=$?
timeout 1500 python bench.py --impl reference > gpurun_out/r2y_bench_reference.json 2> gpurun_out/r2y_bench_reference.err; echo ref rc=$?
timeout 1200 bash tools/ncu_round.sh > gpurun_out/r2y_ncu_round.log 2>&1; echo ncu rc=$?
