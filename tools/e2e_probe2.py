"""e2e probe 2: which part of the host-buffer step costs what (pinned, VGG-16 size)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_07878_b200 as tg  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    layers = tg.layersets.get("vgg16")
    sw = tg.SyncWorker([n for n, _ in layers], [s for _, s in layers], tg.CodecConfig(seed=42),
                       device=dev)
    hin, hv, hout, ov = sw.host_buffers()
    hin.normal_(0, 1e-3)
    n = hin.numel()
    st = torch.cuda.current_stream(dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    res = {}

    def timeit(name, fn, K=6):
        for t in range(2):
            fn(t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0 = time.perf_counter()
        e0.record(st)
        for t in range(K):
            fn(100 + t)
        h1 = time.perf_counter()
        for s in (s1, s2):
            st.wait_stream(s)
        e1.record(st)
        torch.cuda.synchronize()
        res[name] = {"ms": e0.elapsed_time(e1) / K, "host_enqueue_ms": (h1 - h0) * 1e3 / K}

    def h2d(t):
        with torch.cuda.stream(s1):
            sw.grad_flat[:n].copy_(hin, non_blocking=True)

    def d2h(t):
        with torch.cuda.stream(s2):
            hout.copy_(sw.out_flat[:n], non_blocking=True)

    timeit("h2d_only", h2d)
    timeit("d2h_only", d2h)
    timeit("h2d_d2h_free", lambda t: (h2d(t), d2h(t)))

    def lock(t):  # both copies, joined every step
        h2d(t)
        d2h(t)
        st.wait_stream(s1)
        st.wait_stream(s2)
        s1.wait_stream(st)
        s2.wait_stream(st)

    timeit("h2d_d2h_lockstep", lock)

    def lock_step(t):
        lock(t)
        sw.step(t)
        s1.wait_stream(st)
        s2.wait_stream(st)

    timeit("lockstep_plus_step", lock_step)
    timeit("step_host", lambda t: sw.step_host(t, hv, ov))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
