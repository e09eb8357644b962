"""Where the plan's K1 loses time against tools/k1_variants' bare loop (84 us on a clean L2):
K1 (plan.stats(), CUDA events, a 256 MB read before each launch) over several tensor
layouts of the same 138,357,544 elements, N = 1 (L2-policy loads, finalize) and N = 2
(unattached: plain .cs loads).

    python tools/k1_sets.py > gpurun_out/k1_sets.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402
from paper_1705_07878_b200 import layersets  # noqa: E402

dev = torch.device("cuda", 0)
TOTAL = 138357544
vgg = layersets.get("vgg16")
sets = {
    "vgg16": ([n for n, _ in vgg], [int(torch.Size(s).numel()) for _, s in vgg]),
    "one_tensor": (["g"], [TOTAL]),
    "32_equal": ([f"t{i}" for i in range(32)], [TOTAL // 32] * 31 + [TOTAL - 31 * (TOTAL // 32)]),
    "fc6_only": (["fc6"], [102760448]),
}
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
K = 30
for name, (names, ns) in sets.items():
    for nw in (1, 2):
        p = tg.Plan(names, ns, tg.CodecConfig(seed=42), worker=0, n_workers=nw, device=dev)
        p.set_schedule("single")
        gf, gv = tg.aligned_flat(ns, dev)
        of, ov = tg.aligned_flat(ns, dev)
        gf.normal_(0.0, 1e-3, generator=torch.Generator(device=dev).manual_seed(1))
        p.bind(gv, ov)
        for _ in range(3):
            p.stats()
        res = {}
        for cond in ("clean", "hot"):
            es = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                  for _ in range(K)]
            for k in range(K):
                if cond == "clean":
                    flush.sum()
                es[k][0].record()
                p.stats()
                es[k][1].record()
            torch.cuda.synchronize()
            ts = sorted(a.elapsed_time(b) * 1e3 for a, b in es)
            res[cond] = {"mean_us": sum(ts) / K, "min_us": ts[0], "median_us": ts[K // 2]}
        el = sum(ns)
        print(json.dumps({"set": name, "n_workers": nw, "tensors": len(ns), "elements": el,
                          "k1": res, "frac_clean_mean": 4 * el / (res["clean"]["mean_us"] * 1e-6) / 6549.1e9}),
              flush=True)
        p.close()
        del gf, gv, of, ov
        torch.cuda.empty_cache()
