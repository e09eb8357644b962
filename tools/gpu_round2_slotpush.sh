# K2 stores the scaler slots into the peers (K1 no longer does): A/B + the whole GPU suite
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_prod.so
for r in 1 2; do
  for v in base slot; do
    cp build/libtgb_$v.so $LIB
    for cfg in "2 googlenet" "4 googlenet" "2 vgg16" "4 vgg16"; do
      set -- $cfg
      timeout 300 python bench.py --gpus $1 --workload $2 --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r2sp_${v}_$2_n$1_r$r.json 2> gpurun_out/r2sp_${v}_$2_n$1_r$r.err
      python - gpurun_out/r2sp_${v}_$2_n$1_r$r.json $v $2 $1 $r <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
if l:
    d = json.loads(l[0]); print(sys.argv[2], sys.argv[3], "n=" + sys.argv[4], "r" + sys.argv[5], round(d["ms_per_step"] * 1e3, 1), {k: (v["launches_per_step"], round(v["ms_per_launch"] * 1e3, 1)) for k, v in d["kernels_live"].items()}, d["clocks"]["sm_mhz"])
else:
    print(sys.argv[2], sys.argv[3], sys.argv[4], "FAIL")
PY
    done
  done
done
cp build/libtgb_slot.so $LIB
timeout 4000 python -m pytest tests -q -m gpu > gpurun_out/r2sp_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/r2sp_tests.log
cp build/libtgb_prod.so $LIB
