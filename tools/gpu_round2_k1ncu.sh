# ncu --set full: the bare K1 loop (tools/k1_variants V0) vs the plan's K1, same box
ncu --set full --clock-control none -k regex:"k1_v0" -s 2 -c 1 -o gpurun_out/r2m_k1_v0 -f tools/k1_variants quick > gpurun_out/r2m_ncu_v0.log 2>&1; echo v0 rc=$?
ncu --set full --clock-control none --import-source on -k regex:"k1_stats" -s 2 -c 1 -o gpurun_out/r2m_k1_prod -f python tools/prof_step.py vgg16 3 ungrouped > gpurun_out/r2m_ncu_prod.log 2>&1; echo prod rc=$?
