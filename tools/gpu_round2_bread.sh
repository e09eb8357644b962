# K2 CTAs retire after cp.async.bulk.wait_group.read (writes drain after): small + VGG A/B, parity
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_prod.so
for r in 1 2; do
  for v in base bread; do
    cp build/libtgb_$v.so $LIB
    for cfg in "2 googlenet" "4 googlenet" "4 vgg16" "1 googlenet"; do
      set -- $cfg
      timeout 300 python bench.py --gpus $1 --workload $2 --steps 200 --warmup 20 --no-e2e --no-kernel-timing --no-cpu-baseline > gpurun_out/r2x_${v}_$2_n$1_r$r.json 2> gpurun_out/r2x_${v}_$2_n$1_r$r.err
      python - gpurun_out/r2x_${v}_$2_n$1_r$r.json $v $2 $1 $r <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
print(sys.argv[2], sys.argv[3], "n=" + sys.argv[4], "r" + sys.argv[5], round(json.loads(l[0])["ms_per_step"] * 1e3, 1) if l else "FAIL")
PY
    done
  done
done
cp build/libtgb_bread.so $LIB
TGB_EXCHANGE=auto timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 30711 tools/mp_check.py > gpurun_out/r2x_mp_bread.json 2> gpurun_out/r2x_mp_bread.err; echo mp rc=$?
timeout 600 python tools/local_cluster_check.py 2 4 8 > gpurun_out/r2x_lc_bread.json 2> gpurun_out/r2x_lc_bread.err; echo lc rc=$?
cp build/libtgb_prod.so $LIB
