"""e2e probe: tgb_step_host vs a torch emulation of the same copy/compute pattern."""
import json
import os
import sys

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
    st = torch.cuda.current_stream(dev)
    res = {}

    def timeit(fn, K=6):
        for t in range(2):
            fn(t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for t in range(K):
            fn(100 + t)
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    res["step_host"] = timeit(lambda t: sw.step_host(t, hv, ov))
    res["step_only"] = timeit(lambda t: sw.step(t))
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev = {}
    n = hin.numel()

    def emu(t, flat=True):
        comp = ev.get("comp")
        if comp is not None:
            s1.wait_event(comp)
        with torch.cuda.stream(s1):
            sw.grad_flat[:n].copy_(hin, non_blocking=True)
        e_h = torch.cuda.Event()
        e_h.record(s1)
        st.wait_event(e_h)
        if "d2h" in ev:
            st.wait_event(ev["d2h"])
        sw.step(t)
        c = torch.cuda.Event()
        c.record(st)
        ev["comp"] = c
        s2.wait_event(c)
        with torch.cuda.stream(s2):
            hout.copy_(sw.out_flat[:n], non_blocking=True)
        d = torch.cuda.Event()
        d.record(s2)
        ev["d2h"] = d
        st.wait_event(d)

    res["torch_emulation"] = timeit(emu)
    ev.clear()

    def emu_nowait(t):  # D2H of step t does not gate step t+1's compute (output double-buffer)
        comp = ev.get("comp")
        if comp is not None:
            s1.wait_event(comp)
        with torch.cuda.stream(s1):
            sw.grad_flat[:n].copy_(hin, non_blocking=True)
        e_h = torch.cuda.Event()
        e_h.record(s1)
        st.wait_event(e_h)
        sw.step(t)
        c = torch.cuda.Event()
        c.record(st)
        ev["comp"] = c
        s2.wait_event(c)
        with torch.cuda.stream(s2):
            hout.copy_(sw.out_flat[:n], non_blocking=True)
        d = torch.cuda.Event()
        d.record(s2)
        st.wait_event(d)

    res["torch_emulation_tail_wait"] = timeit(emu_nowait)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
