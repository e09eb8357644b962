"""PCIe probe: pinned H2D / D2H / both at once for a VGG-16-sized buffer (553 MB),
one big copy vs 32 per-tensor copies. Prints one JSON line."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1705_07878_b200 import layersets  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    ns = [int(torch.Size(s).numel()) for _, s in layersets.get("vgg16")]
    n = sum(ns)
    hin = torch.empty(n, dtype=torch.float32, pin_memory=True)
    hout = torch.empty(n, dtype=torch.float32, pin_memory=True)
    din = torch.empty(n, dtype=torch.float32, device=dev)
    dout = torch.empty(n, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {"bytes": 4 * n}

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def h2d():
        with torch.cuda.stream(s1):
            din.copy_(hin, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            hout.copy_(dout, non_blocking=True)

    def both():
        h2d()
        d2h()

    offs = [0]
    for k in ns:
        offs.append(offs[-1] + k)

    def h2d_split():
        with torch.cuda.stream(s1):
            for a, b in zip(offs[:-1], offs[1:]):
                din[a:b].copy_(hin[a:b], non_blocking=True)

    def d2h_split():
        with torch.cuda.stream(s2):
            for a, b in zip(offs[:-1], offs[1:]):
                hout[a:b].copy_(dout[a:b], non_blocking=True)

    def both_split():
        h2d_split()
        d2h_split()

    for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both), ("h2d_split", h2d_split),
                     ("d2h_split", d2h_split), ("both_split", both_split)]:
        ms = timed(fn)
        res[name] = {"ms": ms, "GB/s_per_direction": 4 * n / (ms * 1e-3) / 1e9}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
