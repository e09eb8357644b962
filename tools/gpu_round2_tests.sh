python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo smoke rc=$?
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/r2d_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/r2d_tests.log
