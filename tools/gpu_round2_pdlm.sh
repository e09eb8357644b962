# K2 as K1's programmatic dependent at N > 1 (ungrouped plans): GoogLeNet N = 2 / 4 A/B + parity
LIB=paper_1705_07878_b200/lib/libtgb.so
cp $LIB build/libtgb_prod.so
for r in 1 2; do
  for v in base pdlm; do
    cp build/libtgb_$v.so $LIB
    for n in 2 4; do
      timeout 300 python bench.py --gpus $n --workload googlenet --steps 300 --warmup 20 --no-e2e --no-kernel-timing > gpurun_out/r2s_${v}_n${n}_r$r.json 2> gpurun_out/r2s_${v}_n${n}_r$r.err
      python - gpurun_out/r2s_${v}_n${n}_r$r.json $v $n $r <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
print(sys.argv[2], "n=" + sys.argv[3], "r" + sys.argv[4], round(json.loads(l[0])["ms_per_step"] * 1e3, 1) if l else "FAIL")
PY
    done
  done
done
cp build/libtgb_pdlm.so $LIB
TGB_EXCHANGE=auto timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 \
    --master-addr 127.0.0.1 --master-port 30511 tools/mp_check.py > gpurun_out/r2s_mp_pdlm.json 2> gpurun_out/r2s_mp_pdlm.err; echo mp rc=$?
cp build/libtgb_prod.so $LIB
