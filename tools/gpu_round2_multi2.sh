# multi-GPU (gpurun --gpus 4): pipelined sharded exchange -- parity, piece sweep, timelines
P=$((29900 + RANDOM % 50))
timeout 900 python tools/local_cluster_check.py 2 3 5 8 > gpurun_out/r2b_lc.json 2> gpurun_out/r2b_lc.err; echo lc rc=$?
TGB_EXCHANGE=sharded timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port $P tools/mp_check.py > gpurun_out/r2b_mp_n4_sharded.json 2> gpurun_out/r2b_mp_n4_sharded.err; echo mp4 rc=$?
TGB_EXCHANGE=sharded timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port $((P+1)) tools/mp_check.py > gpurun_out/r2b_mp_n2_sharded.json 2> gpurun_out/r2b_mp_n2_sharded.err; echo mp2 rc=$?
for n in 4 2; do
  for pc in 1 2 4 6 8; do
    timeout 400 python bench.py --gpus $n --exchange sharded --pieces $pc --steps 20 --warmup 5 --no-e2e \
      > gpurun_out/r2b_bench_n${n}_sh$pc.json 2> gpurun_out/r2b_bench_n${n}_sh$pc.err; echo bench n=$n pieces=$pc rc=$?
  done
  timeout 400 python bench.py --gpus $n --exchange fused --steps 20 --warmup 5 --no-e2e \
    > gpurun_out/r2b_bench_n${n}_fused.json 2> gpurun_out/r2b_bench_n${n}_fused.err; echo bench n=$n fused rc=$?
done
for ex in "sharded 4" "sharded 1" "fused 0"; do
  set -- $ex
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((P+5)) tools/step_timeline.py vgg16 $1 $2 > gpurun_out/r2b_tl4_$1$2.json 2> gpurun_out/r2b_tl4_$1$2.err
  echo tl $1 $2 rc=$?; P=$((P+1))
done
