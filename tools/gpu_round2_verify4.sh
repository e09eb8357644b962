# 4 GPUs at HEAD: K1 probes (same box), parity, multi-GPU parity + benches
tools/k1_variants quick > gpurun_out/r2k_k1_variants.log 2>&1; echo k1v rc=$?
timeout 600 python tools/k1_sets.py > gpurun_out/r2k_k1_sets.jsonl 2> gpurun_out/r2k_k1_sets.err; echo sets rc=$?
timeout 900 python -m pytest -q -x tests/test_parity_gpu.py tests/test_baseline_parity.py > gpurun_out/r2k_parity.log 2>&1; echo parity rc=$?
tail -n 2 gpurun_out/r2k_parity.log
P=$((30400 + RANDOM % 50))
for ex in auto sharded; do
  TGB_EXCHANGE=$ex timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port $P tools/mp_check.py > gpurun_out/r2k_mp_n4_$ex.json 2> gpurun_out/r2k_mp_n4_$ex.err; echo mp4 $ex rc=$?
  P=$((P+1))
done
for n in 1 2 4; do
  timeout 400 python bench.py --gpus $n --no-e2e > gpurun_out/r2k_bench_n$n.json 2> gpurun_out/r2k_bench_n$n.err; echo bench n=$n rc=$?
done
timeout 400 python bench.py --gpus 4 --exchange sharded --no-e2e > gpurun_out/r2k_bench_n4_sharded.json 2> gpurun_out/r2k_bench_n4_sharded.err; echo bench n=4 sharded rc=$?
for f in gpurun_out/r2k_bench_*.json; do
  python - "$f" <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
if l:
    d = json.loads(l[0]); print(sys.argv[1], d["ms_per_step"], d["clocks"]["sm_mhz"], {k: (v["launches_per_step"], round(v["ms_per_launch"], 4)) for k, v in d["kernels_live"].items()})
PY
done
