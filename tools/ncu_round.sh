#!/bin/bash
# ncu evidence for the current build (one GPU). Each command first runs without ncu
# (it must exit 0). Outputs: gpurun_out/r02_*; summaries + traffic.json via tools/ncu_traffic.py.
#  * launch list (gpu__time_duration, --clock-control none) of the default bench command
#  * --set full of the N = 1 attribution kernels (K1, K2 + fused decode) on VGG-16
#  * --set full of the N = 4 staged K3 (one GPU, four unattached plans)
#  * launch list of GoogLeNet N = 1 steps (small-set latency)
set -x
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_bench_plain.json || exit 1
python tools/prof_step.py vgg16 3 ungrouped || exit 1
python tools/prof_step.py vgg16 2 k3n4 || exit 1
python tools/prof_step.py googlenet 20 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02_ncu_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_googlenet_launches.csv \
    python tools/prof_step.py googlenet 20 > gpurun_out/r02_ncu_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k1_stats|k2_ternarize" -s 2 -c 2 \
    -o gpurun_out/r02_ungrouped -f python tools/prof_step.py vgg16 3 ungrouped > gpurun_out/r02_ncu_u.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k3_decode" -s 1 -c 1 \
    -o gpurun_out/r02_k3n4 -f python tools/prof_step.py vgg16 2 k3n4 > gpurun_out/r02_ncu_k3.log 2>&1
python tools/ncu_summary.py gpurun_out/r02_ungrouped.ncu-rep gpurun_out/r02_k3n4.ncu-rep > gpurun_out/r02_ncu_full_summary.txt
python tools/ncu_traffic.py gpurun_out/r02_ungrouped.ncu-rep gpurun_out/r02_k3n4.ncu-rep > gpurun_out/r02_traffic.json
ls -la gpurun_out/r02_*
