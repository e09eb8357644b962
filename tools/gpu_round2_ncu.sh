# one GPU: library A/B (K2 L2 demotion on/off) + the ncu round
ORDER="new nodemote" timeout 900 bash tools/lib_ab.sh 3 > gpurun_out/r02_ab_demote.jsonl 2> gpurun_out/r02_ab_demote.err; echo ab rc=$?
timeout 2400 bash tools/ncu_round.sh > gpurun_out/r02_ncu_round.log 2>&1; echo ncu rc=$?
