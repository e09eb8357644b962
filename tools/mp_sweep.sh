#!/bin/bash
# usage: tools/mp_sweep.sh TAG NPROC [ENV=VAL ...]  -> gpurun_out/mp_TAG.log + one summary line
tag=$1; np=$2; shift 2
env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np \
    --master-addr 127.0.0.1 --master-port $((29500 + RANDOM % 400)) tools/mp_check.py \
    > gpurun_out/mp_$tag.log 2>&1
echo "exit $?" >> gpurun_out/mp_$tag.log
python - "$tag" <<'PY'
import json, sys
tag = sys.argv[1]
l = [x for x in open(f"gpurun_out/mp_{tag}.log") if x.startswith("{")]
if not l:
    print(tag, "FAILED", open(f"gpurun_out/mp_{tag}.log").read()[-800:])
    sys.exit(0)
d = json.loads(l[0])
ok = all(v["ranks_identical"] and v["matches_oracle"] for v in d["checks"].values())
print(tag, d["vgg16_exchange"], round(d["vgg16_ms_per_step_max_over_ranks"], 4),
      {k: round(v, 4) for k, v in d["stage_ms_median_max_over_ranks"].items()},
      "staged", round(d.get("staged_ms_per_step", 0), 4), "parity", ok)
PY
