# small sets across processes: GoogLeNet and AlexNet at N = 2 / 4 (default exchange)
for n in 2 4; do
  for wl in googlenet alexnet; do
    timeout 300 python bench.py --gpus $n --workload $wl --steps 200 --warmup 20 --no-e2e > gpurun_out/r2r_bench_${wl}_n$n.json 2> gpurun_out/r2r_bench_${wl}_n$n.err; echo $wl n=$n rc=$?
  done
done
for f in gpurun_out/r2r_bench_*.json; do
  python - "$f" <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
if l:
    d = json.loads(l[0]); print(sys.argv[1], round(d["ms_per_step"] * 1e3, 1), "us", d["exchange"][:20], {k: (v["launches_per_step"], round(v["ms_per_launch"] * 1e3, 1)) for k, v in d["kernels_live"].items()})
PY
done
