# final: the whole GPU suite on a 4-GPU box at HEAD (incl. mp_check at N = 2 and 4)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2z4_smoke.log 2>&1; echo smoke rc=$?
timeout 4000 python -m pytest tests -q -m gpu > gpurun_out/r2z4_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/r2z4_tests.log
