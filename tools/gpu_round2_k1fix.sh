# K1 descriptor re-fetch (all 8 loads in flight): same-box A/B vs the previous build + parity
timeout 900 python -m pytest -q -x tests/test_parity_gpu.py > gpurun_out/r2g_parity.log 2>&1; echo parity rc=$?
tail -n 2 gpurun_out/r2g_parity.log
ORDER="new old" timeout 900 bash tools/lib_ab.sh 3 > gpurun_out/r2g_lib_ab.jsonl 2> gpurun_out/r2g_lib_ab.err; echo ab rc=$?
python - <<'PY'
import json
for l in open("gpurun_out/r2g_lib_ab.jsonl"):
    d = json.loads(l); x = d["line"]
    print(d["build"], d["round"], round(x["ms_per_step"], 4), {k: round(v["ms_per_launch"], 4) for k, v in x["kernels_live"].items()}, x.get("k1_l2_state", {}) and round(x["k1_l2_state"]["clean_l2_ms"], 4), x["clocks"]["sm_mhz"])
PY
timeout 600 python tools/fixed_probe.py > gpurun_out/r2g_fixed_probe.json 2> gpurun_out/r2g_fixed_probe.err; echo fixed rc=$?
