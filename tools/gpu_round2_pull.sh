# 4 GPUs: split exchange (K3 pulls part of the codes) -- LocalCluster parity, mp parity, benches
P=$((30200 + RANDOM % 50))
timeout 900 python tools/local_cluster_check.py 2 4 8 > gpurun_out/r2e_lc.json 2> gpurun_out/r2e_lc.err; echo lc rc=$?
TGB_PULL=3 TGB_EXCHANGE=fused timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port $P tools/mp_check.py > gpurun_out/r2e_mp_n4_pull3.json 2> gpurun_out/r2e_mp_n4_pull3.err; echo mp4 pull3 rc=$?
for n in 4 2; do
  for pl in 0 1 2 3 4 6 8; do
    timeout 300 python bench.py --gpus $n --exchange fused --pull $pl --steps 20 --warmup 5 --no-e2e \
      > gpurun_out/r2e_bench_n${n}_pull$pl.json 2> gpurun_out/r2e_bench_n${n}_pull$pl.err; echo bench n=$n pull=$pl rc=$?
  done
done
grep -h '"value"' gpurun_out/r2e_bench_*.json | python -c '
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(d["n_gpus"], d["config"].get("pull"), d["ms_per_step"])'
