# 4 GPUs: overlapped exchange -- LocalCluster parity, multi-process parity, benches, timelines
P=$((30100 + RANDOM % 50))
timeout 900 python tools/local_cluster_check.py 2 3 5 8 > gpurun_out/r2c_lc.json 2> gpurun_out/r2c_lc.err; echo lc rc=$?
for ex in auto sharded; do
  TGB_OVERLAP=1 TGB_EXCHANGE=$ex timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port $P tools/mp_check.py > gpurun_out/r2c_mp_n4_${ex}_ov.json 2> gpurun_out/r2c_mp_n4_${ex}_ov.err; echo mp4 $ex rc=$?
  P=$((P+1))
done
for n in 4 2; do
  for cfg in "fused 0 -1" "fused 2 1" "fused 4 1" "fused 8 1" "sharded 0 -1" "sharded 2 1" "sharded 4 1" "sharded 8 1"; do
    set -- $cfg
    timeout 300 python bench.py --gpus $n --exchange $1 --pieces $2 --overlap $3 --steps 20 --warmup 5 --no-e2e \
      > gpurun_out/r2c_bench_n${n}_$1_p$2_o$3.json 2> gpurun_out/r2c_bench_n${n}_$1_p$2_o$3.err; echo bench n=$n $cfg rc=$?
  done
done
for ex in fused sharded; do
  timeout 300 env TGB_TL_OVERLAP=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((P+5)) tools/step_timeline.py vgg16 $ex 4 1 > gpurun_out/r2c_tl4_${ex}_ov.json 2> gpurun_out/r2c_tl4_${ex}_ov.err
  echo tl $ex rc=$?; P=$((P+1))
done
