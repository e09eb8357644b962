# K3: decoded-value LUT per item (2N+1 floats) vs per-lane int->float + 2 multiplies; A/B + parity
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_prod.so
for r in 1 2; do
  for v in nolut lut; do
    cp build/libtgb_$v.so $LIB
    for n in 4 2; do
      timeout 300 python bench.py --gpus $n --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2y3_${v}_n${n}_r$r.json 2> gpurun_out/r2y3_${v}_n${n}_r$r.err
      python - gpurun_out/r2y3_${v}_n${n}_r$r.json $v $n $r <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
if l:
    d = json.loads(l[0]); print(sys.argv[2], "n=" + sys.argv[3], "r" + sys.argv[4], round(d["ms_per_step"], 4), {k: (v["launches_per_step"], round(v["ms_per_launch"] * 1e3, 1)) for k, v in d["kernels_live"].items()}, d["clocks"]["sm_mhz"])
else:
    print(sys.argv[2], sys.argv[3], "FAIL")
PY
    done
  done
done
cp build/libtgb_lut.so $LIB
TGB_EXCHANGE=auto timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 30811 tools/mp_check.py > gpurun_out/r2y3_mp_lut.json 2> gpurun_out/r2y3_mp_lut.err; echo mp rc=$?
timeout 900 python tools/local_cluster_check.py 2 3 4 8 > gpurun_out/r2y3_lc_lut.json 2> gpurun_out/r2y3_lc_lut.err; echo lc rc=$?
timeout 1500 python -m pytest -q -x tests/test_parity_gpu.py tests/test_baseline_parity.py > gpurun_out/r2y3_parity.log 2>&1; echo parity rc=$?
tail -n 2 gpurun_out/r2y3_parity.log
cp build/libtgb_prod.so $LIB
