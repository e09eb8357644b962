# round-2 GPU check on one B200: smoke, the GPU test suite, LocalCluster parity,
# a short bench and the small-set schedule probe (outputs under gpurun_out/)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/r2_tests.log 2>&1; echo tests rc=$?
timeout 300 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo bench rc=$?
timeout 600 python tools/small_sets.py > gpurun_out/r2_small_sets.jsonl 2> gpurun_out/r2_small_sets.err; echo small rc=$?
tail -n 3 gpurun_out/r2_tests.log
