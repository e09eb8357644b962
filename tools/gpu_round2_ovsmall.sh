# small sets: K2 publishes the barrier record itself (overlap mode, 1 piece) vs the barrier kernel
for r in 1 2; do
  for cfg in "-1 0" "1 1" "1 2"; do
    set -- $cfg
    for n in 2 4; do
      timeout 300 python bench.py --gpus $n --workload googlenet --overlap $1 --pieces $2 --steps 200 --warmup 20 --no-e2e --no-cpu-baseline --no-kernel-timing > gpurun_out/r2ov_${1}_${2}_n${n}_r$r.json 2> gpurun_out/r2ov_${1}_${2}_n${n}_r$r.err
      python - gpurun_out/r2ov_${1}_${2}_n${n}_r$r.json "overlap=$1 pieces=$2 n=$n r$r" <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
print(sys.argv[2], round(json.loads(l[0])["ms_per_step"] * 1e3, 1) if l else "FAIL")
PY
    done
  done
done
