# round-2 multi-GPU check (run with gpurun --gpus 4): parity on every exchange at
# N = 2 and 4, benches per exchange, plus the single-GPU small-set probe
P=$((29800 + RANDOM % 100))
nvidia-smi topo -m > gpurun_out/r2_topo.txt 2>&1
timeout 600 python tools/small_sets.py > gpurun_out/r2_small_sets.jsonl 2> gpurun_out/r2_small_sets.err; echo small rc=$?
timeout 600 python -m pytest tests/test_parity_gpu.py -q -m gpu -k "fused_k12 or live_kernel" > gpurun_out/r2_k12.log 2>&1; echo k12 rc=$?
for n in 2 4; do
  for ex in auto sharded nccl; do
    TGB_EXCHANGE=$ex timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
      --master-addr 127.0.0.1 --master-port $((P + 10*n)) tools/mp_check.py \
      > gpurun_out/r2_mp_n${n}_$ex.json 2> gpurun_out/r2_mp_n${n}_$ex.err; echo mp n=$n ex=$ex rc=$?
    P=$((P + 1))
  done
done
for n in 2 4; do
  for ex in auto sharded fused; do
    timeout 600 python bench.py --gpus $n --exchange $ex --steps 20 --warmup 5 --no-e2e \
      > gpurun_out/r2_bench_n${n}_$ex.json 2> gpurun_out/r2_bench_n${n}_$ex.err; echo bench n=$n ex=$ex rc=$?
  done
done
