# one-GPU round-2 pass: GPU tests, sanitizers, FixedSize probe, default bench + reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/r2_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/r2_tests.log
timeout 600 python tools/fixed_probe.py > gpurun_out/r2_fixed_probe.json 2> gpurun_out/r2_fixed_probe.err; echo fixed rc=$?
bash tools/sanitize.sh
timeout 900 python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err; echo bench rc=$?
timeout 1500 python bench.py --impl reference > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err; echo ref rc=$?
