#!/bin/bash
# BASELINE configs beyond the headline: single-layer size sweep at N = 1/2/4 and the
# AlexNet / GoogLeNet / VGG-16 gradient sets through bench.py. Output: gpurun_out/cfg_*.
mkdir -p gpurun_out
P=$((29700 + RANDOM % 200))
timeout 600 python tools/size_sweep.py > gpurun_out/cfg_sweep_n1.jsonl 2> gpurun_out/cfg_sweep_n1.err
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((P + n)) tools/size_sweep.py > gpurun_out/cfg_sweep_n$n.jsonl 2> gpurun_out/cfg_sweep_n$n.err
done
for w in googlenet alexnet vgg16; do
  timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/cfg_${w}_n1.json 2> /dev/null
  for n in 2 4; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((P + 10 + n)) bench.py --gpus $n --workload $w > gpurun_out/cfg_${w}_n$n.json 2> /dev/null
  done
done
ls -la gpurun_out/cfg_*
