# 4 GPUs: two-group sharded exchange -- parity (LocalCluster, BASELINE sets, mp), benches
P=$((30300 + RANDOM % 50))
timeout 900 python tools/local_cluster_check.py 2 4 8 > gpurun_out/r2f_lc.json 2> gpurun_out/r2f_lc.err; echo lc rc=$?
timeout 1500 python -m pytest -q -x tests/test_baseline_parity.py -k "alexnet or multiworker" > gpurun_out/r2f_baseline.log 2>&1; echo baseline rc=$?
TGB_EXCHANGE=sharded timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
  --master-addr 127.0.0.1 --master-port $P tools/mp_check.py > gpurun_out/r2f_mp_n4_sharded.json 2> gpurun_out/r2f_mp_n4_sharded.err; echo mp4 sharded rc=$?
for n in 4 2; do
  for cfg in "sharded auto 0" "sharded single 0" "fused auto 0" "fused auto 6"; do
    set -- $cfg
    timeout 300 python bench.py --gpus $n --exchange $1 --schedule $2 --pull $3 --steps 20 --warmup 5 --no-e2e \
      > gpurun_out/r2f_bench_n${n}_$1_$2_$3.json 2> gpurun_out/r2f_bench_n${n}_$1_$2_$3.err; echo bench n=$n $cfg rc=$?
  done
done
for f in gpurun_out/r2f_bench_*.json; do
  python - "$f" <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
if l:
    d = json.loads(l[0]); print(sys.argv[1], d["ms_per_step"], {k: (v["launches_per_step"], round(v["ms_per_launch"], 4)) for k, v in d["kernels_live"].items()})
PY
done
