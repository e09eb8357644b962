#!/bin/bash
# ncu evidence for the current build (one GPU): launch list of bench.py, full captures of
# the attribution kernels (N=1 ungrouped tgb_step: K1 + K2 with fused decode) and of the
# N=4 staged K3. Run each command without ncu first (it must exit 0).
set -x
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench_plain.json || exit 1
python tools/prof_step.py vgg16 3 ungrouped || exit 1
python tools/prof_step.py vgg16 3 k3n4 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01b_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1_stats|k2_ternarize" -s 2 -c 2 \
    -o gpurun_out/r01b_ungrouped -f python tools/prof_step.py vgg16 3 ungrouped > gpurun_out/ncu_u.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k3_decode" -s 1 -c 1 \
    -o gpurun_out/r01b_k3n4 -f python tools/prof_step.py vgg16 2 k3n4 > gpurun_out/ncu_k3.log 2>&1
python tools/ncu_summary.py gpurun_out/r01b_ungrouped.ncu-rep gpurun_out/r01b_k3n4.ncu-rep > gpurun_out/r01b_ncu_summary.txt
ls -la gpurun_out/r01b*
