# GoogLeNet per-kernel live times: N = 1, N = 2 fused, N = 2 nccl (where the N > 1 step time goes)
for cfg in "1 auto" "2 auto" "2 nccl"; do
  set -- $cfg
  timeout 300 python bench.py --gpus $1 --exchange $2 --workload googlenet --steps 200 --warmup 20 --no-e2e --no-cpu-baseline > gpurun_out/r2g2_n$1_$2.json 2> gpurun_out/r2g2_n$1_$2.err
  python - gpurun_out/r2g2_n$1_$2.json $1 $2 <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
if l:
    d = json.loads(l[0]); print("n=" + sys.argv[2], sys.argv[3], round(d["ms_per_step"] * 1e3, 1), {k: (v["launches_per_step"], round(v["ms_per_launch"] * 1e3, 1)) for k, v in d["kernels_live"].items()}, d["clocks"]["sm_mhz"])
PY
done
