"""Plan / communicator / worker-sync wrappers over the C-ABI.

``SyncWorker`` is the device replacement for the reference worker's sync
segment (cluster.hpp:283-297): encode_step -> push -> ParameterServer::step
-> pull -> decode_pull becomes K1 -> K2 -> NCCL allgather -> K3 on every rank.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import torch

from . import _lib
from ._lib import check, load
from .codec import CodecConfig, CodecError, ProtocolError, ShareMode, fnv1a64, _dev


class _CudaBuf:
    """Zero-copy torch view of plan-owned device memory."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False), "version": 3,
        }


def _view(ptr: int, nbytes: int, device: torch.device) -> torch.Tensor:
    if nbytes == 0 or ptr == 0:
        return torch.empty(0, dtype=torch.uint8, device=device)
    return torch.as_tensor(_CudaBuf(ptr, nbytes), device=device)


def aligned_flat(ns: Sequence[int], device, align_elems: int = 4, dtype=torch.float32,
                 pin_memory: bool = False):
    """One flat buffer holding every tensor at a 16-byte aligned offset.

    Returns (flat, views). This is the gradient-bucket layout the kernels
    stream with 128-bit accesses (pin_memory: page-locked host buffer)."""
    offs, pos = [], 0
    for n in ns:
        offs.append(pos)
        pos += (int(n) + align_elems - 1) // align_elems * align_elems
    flat = torch.zeros(max(pos, 1), dtype=dtype, device=device, pin_memory=pin_memory)
    views = [flat[o:o + int(n)] for o, n in zip(offs, ns)]
    return flat, views


class Comm:
    """NCCL communicator created through the C-ABI (tgb_comm_init)."""

    def __init__(self, rank: int, world_size: int, unique_id: Optional[bytes] = None,
                 group=None):
        L = load()
        self.rank, self.world_size = rank, world_size
        if unique_id is None:
            import torch.distributed as dist

            buf = [None]
            if rank == 0:
                raw = C.create_string_buffer(_lib.UNIQUE_ID_BYTES)
                check(L.tgb_comm_unique_id(raw), "tgb_comm_unique_id")
                buf[0] = bytes(raw.raw)
            dist.broadcast_object_list(buf, src=0, group=group)
            unique_id = buf[0]
        h = C.c_void_p()
        check(L.tgb_comm_init(unique_id, world_size, rank, C.byref(h)), "tgb_comm_init")
        self.h = h

    @staticmethod
    def unique_id() -> bytes:
        raw = C.create_string_buffer(_lib.UNIQUE_ID_BYTES)
        check(load().tgb_comm_unique_id(raw), "tgb_comm_unique_id")
        return bytes(raw.raw)

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            load().tgb_comm_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Plan:
    """tgb_plan: one worker's layer table, push/gather buffers and workspace."""

    def __init__(self, names: Sequence[str], ns: Sequence[int], cfg: CodecConfig, worker: int = 0,
                 n_workers: int = 1, device=None, passthrough: Optional[Sequence[bool]] = None):
        cfg.validate()
        self.device = _dev(device)
        self.names = list(names)
        self.ns = [int(n) for n in ns]
        self.cfg = cfg
        self.worker, self.n_workers = int(worker), int(n_workers)
        L = load()
        nl = len(self.names)
        if passthrough is None:  # CodecConfig::passthrough / float_mode (cluster.hpp:274-275)
            passthrough = [cfg.float_mode or name in cfg.passthrough for name in self.names]
        self.passthrough = [bool(x) for x in passthrough]
        descs = (_lib.LayerDesc * max(nl, 1))()
        for l, (name, n) in enumerate(zip(self.names, self.ns)):
            flags = _lib.TGB_LAYER_PASSTHROUGH if self.passthrough[l] else 0
            descs[l] = _lib.LayerDesc(n, fnv1a64(name), flags, 0)
        params = cfg.params()
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            check(L.tgb_plan_create(descs, nl, C.byref(params), self.worker, self.n_workers,
                                    C.byref(h)), "tgb_plan_create")
        self.h = h
        # the reference wire format carries tensor names (serialize_push / decode_pull)
        cn = (C.c_char_p * max(nl, 1))(*[x.encode() for x in self.names])
        check(L.tgb_plan_set_names(h, cn), "tgb_plan_set_names")
        info = _lib.PlanInfo()
        check(L.tgb_plan_get_info(h, C.byref(info)), "tgb_plan_get_info")
        self.info = info
        self.code_offsets, self.slots = [], []
        for l in range(nl):
            off, slot = C.c_uint64(), C.c_int32()
            check(L.tgb_plan_layer_layout(h, l, C.byref(off), C.byref(slot)), "layout")
            self.code_offsets.append(off.value)
            self.slots.append(slot.value)
        # blocks of the encoded gradient (EncodedGradient::blocks, codec.hpp:70-76)
        self.blocks: List[_lib.BlockInfo] = []
        for b in range(info.n_blocks):
            bi = _lib.BlockInfo()
            check(L.tgb_plan_block_info(h, b, C.byref(bi)), "tgb_plan_block_info")
            self.blocks.append(bi)
        push, gathered, bounds = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(L.tgb_plan_buffers(h, C.byref(push), C.byref(gathered), C.byref(bounds)), "buffers")
        self.push = _view(push.value or 0, info.push_bytes, self.device)
        self.gathered = _view(gathered.value or 0, info.push_bytes * self.n_workers
                              if self.n_workers > 1 else 0, self.device)
        nb = len(self.blocks)  # clip bound per block (its tensor's bound)
        self.bounds = _view(bounds.value or 0, 4 * nb, self.device).view(torch.float32) \
            if nb else torch.empty(0, device=self.device)
        self._grads = self._outs = None
        self.attached = False
        self.grouped = info.n_groups == 2  # tgb_step overlaps the dominant layer with the rest
        self.last_t = None  # iteration of the last step issued (iteration-skew messages)

    # -- options -------------------------------------------------------------
    def set_option(self, option: int, value: int):
        """tgb_plan_set_option (schedule / exchange / fused optimizer); rebuilds the
        work tables, so bind() afterwards if gradients were bound before."""
        with torch.cuda.device(self.device):
            check(load().tgb_plan_set_option(self.h, int(option), int(value)),
                  "tgb_plan_set_option")
        self._refresh()

    SCHEDULES = {"auto": _lib.TGB_SCHEDULE_AUTO, "single": _lib.TGB_SCHEDULE_SINGLE,
                 "groups": _lib.TGB_SCHEDULE_GROUPS, "unfused": _lib.TGB_SCHEDULE_UNFUSED,
                 "fused12": _lib.TGB_SCHEDULE_FUSED12}

    def set_schedule(self, schedule: str):
        """"auto" | "single" (one stream, each kernel covers the whole set) | "groups" |
        "unfused" (K1 and K2 always separate launches) | "fused12" (always one launch)"""
        self.set_option(_lib.TGB_PLAN_OPT_SCHEDULE, self.SCHEDULES[schedule])

    def set_exchange(self, exchange: str):
        """"auto" (fused N <= 4, sharded from 5) | "fused" | "sharded"; before attaching"""
        self.set_option(_lib.TGB_PLAN_OPT_EXCHANGE, {"auto": _lib.TGB_EXCHANGE_AUTO,
                                                     "fused": _lib.TGB_EXCHANGE_FUSED,
                                                     "sharded": _lib.TGB_EXCHANGE_SHARDED}[exchange])

    def set_overlap(self, on: bool):
        """overlapped exchange (N > 1): K2 publishes finished pieces, their decode
        overlaps the later pieces' K2; before attaching"""
        self.set_option(_lib.TGB_PLAN_OPT_OVERLAP, 1 if on else 0)

    def set_pull(self, eighths: int):
        """fused exchange: eighths (0..8) of the code items the decode pulls from the
        peers' memory instead of K2 storing them into every peer; before attaching"""
        self.set_option(_lib.TGB_PLAN_OPT_PULL, int(eighths))

    def set_pieces(self, pieces: int):
        """sharded exchange: pieces of the K2 work list (0 = auto); before attaching"""
        self.set_option(_lib.TGB_PLAN_OPT_PIECES, int(pieces))

    def _refresh(self):
        L = load()
        info = _lib.PlanInfo()
        check(L.tgb_plan_get_info(self.h, C.byref(info)), "tgb_plan_get_info")
        self.info = info
        self.grouped = info.n_groups == 2
        push, gathered, bounds = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(L.tgb_plan_buffers(self.h, C.byref(push), C.byref(gathered), C.byref(bounds)),
              "buffers")
        self.gathered = _view(gathered.value or 0, info.push_bytes * self.n_workers
                              if self.n_workers > 1 else 0, self.device)
        if self._grads is not None:
            self.bind(self._grads, self._outs)

    @property
    def exchange(self) -> str:
        return _lib.EXCHANGE_NAMES[self.info.exchange]

    def audit(self):
        """tgb_plan_audit: raise if any kernel region lies outside its allocation"""
        st = load().tgb_plan_audit(self.h)
        if st == _lib.TGB_ERR_PROTOCOL:
            raise AssertionError(load().tgb_last_error_message().decode())
        check(st, "tgb_plan_audit")

    def traffic(self) -> "TrafficStats":
        """one step of this worker's TrafficStats terms (tgb_plan_traffic)"""
        t = _lib.Traffic()
        check(load().tgb_plan_traffic(self.h, C.byref(t)), "tgb_plan_traffic")
        return TrafficStats.of(t)

    # -- binding -------------------------------------------------------------
    def bind(self, grads: Sequence[torch.Tensor], outs: Optional[Sequence[torch.Tensor]]):
        """Bind per-layer device gradients (input) and averaged outputs."""
        if outs is None:
            outs = [torch.empty(0, device=self.device)] * len(grads)
        for g, n in zip(grads, self.ns):
            if g.numel() != n or g.dtype != torch.float32 or not g.is_contiguous():
                raise ValueError("bind: gradient must be contiguous float32 of the planned size")
            if n and g.device != self.device:
                raise ValueError("bind: gradient on the wrong device")
        nl = len(self.ns)
        gp = (C.c_void_p * max(nl, 1))(*[g.data_ptr() if g.numel() else 0 for g in grads])
        op = (C.c_void_p * max(nl, 1))(*[o.data_ptr() if o.numel() else 0 for o in outs])
        # decode outputs are optional for encode-only use: point at the gradient
        for l in range(nl):
            if not op[l]:
                op[l] = gp[l]
        check(load().tgb_plan_bind(self.h, gp, op), "tgb_plan_bind")
        self._grads, self._outs = list(grads), list(outs)

    def _st(self, stream=None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        return C.c_void_p(s.cuda_stream)

    # -- pipeline stages -----------------------------------------------------
    def stats(self, stream=None):
        check(load().tgb_stats(self.h, self._st(stream)), "tgb_stats")

    def ternarize_pack(self, t: int, stream=None):
        check(load().tgb_ternarize_pack(self.h, int(t), self._st(stream)), "tgb_ternarize_pack")
        self.last_t = int(t)

    def encode(self, t: int, stream=None):
        check(load().tgb_encode(self.h, int(t), self._st(stream)), "tgb_encode")
        self.last_t = int(t)

    def share_scalers(self, comm: Comm, stream=None):
        check(load().tgb_share_scalers(self.h, comm.h, self._st(stream)), "tgb_share_scalers")

    def sync(self, comm: Optional[Comm], stream=None):
        """NCCL allgather of push buffers, or (peers attached) the step barrier."""
        check(load().tgb_sync(self.h, comm.h if comm is not None else None, self._st(stream)),
              "tgb_sync")

    def decode_average(self, src: Optional[torch.Tensor], n_workers: int, stream=None):
        """K3 over `src` (N push buffers back to back); None = this step's gather buffer."""
        ptr = C.c_void_p(src.data_ptr()) if src is not None else None
        check(load().tgb_decode_average(self.h, ptr, int(n_workers), self._st(stream)),
              "tgb_decode_average")

    def attach_peers(self, comm: Comm):
        """Peer exchange over NVLink (CUDA IPC): fused or sharded (set_exchange);
        collective over all ranks. Raises ProtocolError when the ranks' plans differ
        (the reference server's "block structure mismatch", cluster.hpp:169-172)."""
        with torch.cuda.device(self.device):
            st = load().tgb_plan_attach_peers(self.h, comm.h)
        if st == _lib.TGB_ERR_PROTOCOL:
            raise ProtocolError(load().tgb_last_error_message().decode())
        check(st, "tgb_plan_attach_peers")
        self.attached = True
        self._refresh()

    @staticmethod
    def attach_local(plans: Sequence["Plan"]):
        """Exchange between the N plans of this process (workers 0..N-1;
        tgb_plan_attach_local); step them together with Plan.local_step."""
        arr = (C.c_void_p * len(plans))(*[p.h.value for p in plans])
        st = load().tgb_plan_attach_local(arr, len(plans))
        if st == _lib.TGB_ERR_PROTOCOL:
            raise ProtocolError(load().tgb_last_error_message().decode())
        check(st, "tgb_plan_attach_local")
        for p in plans:
            p.attached = True
            p._refresh()

    @staticmethod
    def local_step(plans: Sequence["Plan"], ts: Sequence[int], streams):
        """tgb_local_step: plan w steps iteration ts[w] on streams[w]"""
        n = len(plans)
        arr = (C.c_void_p * n)(*[p.h.value for p in plans])
        tv = (C.c_uint64 * n)(*[int(t) for t in ts])
        sv = (C.c_void_p * n)(*[s.cuda_stream for s in streams])
        check(load().tgb_local_step(arr, n, tv, sv), "tgb_local_step")
        for p, t in zip(plans, ts):
            p.last_t = int(t)

    def last_buffers(self):
        """(own push area, gather buffer) of the last step, as uint8 views."""
        push, gathered = C.c_void_p(), C.c_void_p()
        check(load().tgb_plan_last_buffers(self.h, C.byref(push), C.byref(gathered)),
              "tgb_plan_last_buffers")
        P = self.info.push_bytes
        return (_view(push.value or 0, P, self.device),
                _view(gathered.value or 0, P * self.n_workers, self.device))

    def step(self, t: int, comm: Optional[Comm] = None, stream=None):
        check(load().tgb_step(self.h, comm.h if comm is not None else None, int(t),
                              self._st(stream)), "tgb_step")
        self.last_t = int(t)

    def step_host(self, t: int, host_grads: Sequence[torch.Tensor],
                  host_outs: Sequence[torch.Tensor], comm: Optional[Comm] = None, stream=None):
        """tgb_step_host: per-layer host (pinned) gradients in, averaged gradients out;
        completes in `stream` order, the next call's H2D overlaps this call's D2H."""
        nl = len(self.ns)
        for h, n in zip(list(host_grads) + list(host_outs), self.ns + self.ns):
            if h.device.type != "cpu" or h.numel() != n or h.dtype != torch.float32 or \
                    not h.is_contiguous():
                raise ValueError("step_host: host tensors must be contiguous float32 of the "
                                 "planned sizes")
        gp = (C.c_void_p * max(nl, 1))(*[h.data_ptr() if h.numel() else 0 for h in host_grads])
        op = (C.c_void_p * max(nl, 1))(*[h.data_ptr() if h.numel() else 0 for h in host_outs])
        check(load().tgb_step_host(self.h, comm.h if comm is not None else None, int(t), gp, op,
                                   self._st(stream)), "tgb_step_host")
        self.last_t = int(t)

    def error(self) -> _lib.Error:
        e = _lib.Error()
        st = load().tgb_check(self.h, C.byref(e))
        if st not in (_lib.TGB_OK, _lib.TGB_ERR_CODEC):
            check(st, "tgb_check")
        return e

    # -- reference wire format ----------------------------------------------
    def serialize_push(self, t: int, stream=None) -> bytes:
        """frame(Message{Push, t, worker, serialize_encoded(last encode)}) (wire.hpp:41-53)"""
        n = C.c_uint64()
        check(load().tgb_plan_push_frame_size(self.h, C.byref(n)), "tgb_plan_push_frame_size")
        buf = (C.c_uint8 * n.value)()
        check(load().tgb_plan_serialize_push(self.h, int(t), buf, self._st(stream)),
              "tgb_plan_serialize_push")
        return bytes(buf)

    def decode_pull(self, frame: bytes, stream=None) -> int:
        """decode_pull(deserialize_pull(unframe(frame).payload)) into the bound outputs;
        returns the frame's iteration (wire.hpp:57-75, 147-228)"""
        buf = (C.c_uint8 * len(frame)).from_buffer_copy(frame) if frame else (C.c_uint8 * 1)()
        it = C.c_uint64()
        st = load().tgb_plan_decode_pull(self.h, buf, len(frame), C.byref(it), self._st(stream))
        if st == _lib.TGB_ERR_PROTOCOL:
            raise ProtocolError(load().tgb_last_error_message().decode())
        check(st, "tgb_plan_decode_pull")
        return it.value

    def enable_timing(self, capacity: int):
        """Bracket the next `capacity` kernel launches of this plan with CUDA events on
        their own streams (0 = off); resets the records (tgb_plan_enable_timing)."""
        check(load().tgb_plan_enable_timing(self.h, int(capacity)), "tgb_plan_enable_timing")
        self._t_cap = int(capacity)

    def read_timing(self) -> List[dict]:
        """One record per timed launch: kernel, group, ms, elements, algorithmic HBM and
        NVLink bytes (waits for the recorded events)."""
        cap = getattr(self, "_t_cap", 0)
        arr = (_lib.KernelTime * max(cap, 1))()
        n = C.c_int32()
        check(load().tgb_plan_read_timing(self.h, arr, cap, C.byref(n)), "tgb_plan_read_timing")
        return [{"kernel": _lib.KERNEL_NAMES.get(r.kind, str(r.kind)), "group": r.group,
                 "ms": r.ms, "start_ms": r.start_ms, "elements": r.elements, "hbm_bytes": r.hbm_bytes,
                 "nvlink_bytes": r.nvlink_bytes} for r in arr[:min(n.value, cap)]]

    def enable_code_stats(self, on: bool = True):
        """count nonzero codes inside K2 from the next step on (telemetry, off by default)"""
        check(load().tgb_plan_enable_code_stats(self.h, int(on)), "tgb_plan_enable_code_stats")

    def code_stats(self):
        """(nonzero codes, ternary elements) of the last encode, counted inside K2"""
        nz, tot = C.c_uint64(), C.c_uint64()
        check(load().tgb_plan_code_stats(self.h, C.byref(nz), C.byref(tot)), "tgb_plan_code_stats")
        return nz.value, tot.value

    def zero_fraction(self) -> float:
        """Worker::zero_fraction of the last encode (cluster.hpp:336-346)"""
        nz, tot = self.code_stats()
        return (tot - nz) / tot if tot else 0.0

    def block_of(self, layer: int, index: int) -> int:
        """block holding element `index` of `layer` (first block if none)."""
        first = None
        for b, bi in enumerate(self.blocks):
            if bi.layer == layer:
                first = b if first is None else first
                if bi.offset <= index < bi.offset + bi.n:
                    return b
        return first if first is not None else -1

    def raise_errors(self):
        """Rethrow the device error word with the reference's CodecError /
        ProtocolError text."""
        e = self.error()
        if e.flags & _lib.TGB_E_SKEW:  # cluster.hpp:141-143
            raise ProtocolError(f"server: iteration skew, expected {self.last_t} got {e.aux}")
        if e.flags:
            name = self.names[e.layer] if 0 <= e.layer < len(self.names) else "?"
            b = self.block_of(e.layer, e.index) if 0 <= e.layer < len(self.names) else -1
            k = e.index - self.blocks[b].offset if b >= 0 else e.index
            if e.flags & _lib.TGB_E_NONFINITE:
                raise CodecError("encode_step: non-finite gradient " + name)
            if e.flags & _lib.TGB_E_CORRUPT_CODE:
                raise CodecError(f"corrupt ternary code 11 in block {name} at element {k}")
            if e.flags & _lib.TGB_E_PEER_TIMEOUT:
                raise CodecError(f"fused exchange: peer {e.index} never reached the step barrier")
            raise CodecError(f"codec error flags {e.flags:#x} in {name}")

    def scalers(self) -> torch.Tensor:
        """this worker's scaler slots (one per ternary block, canonical order)"""
        push, _ = self.last_buffers()
        return push[:4 * self.info.n_slots].view(torch.float32)

    def block_region(self, b: int, worker: Optional[int] = None) -> torch.Tensor:
        """block b's packed codes (uint8) or raw values (float32) in the last
        step's own push area, or in worker `worker`'s area of the gather buffer"""
        bi = self.blocks[b]
        raw = bool(bi.flags & _lib.TGB_LAYER_PASSTHROUGH)
        nbytes = 4 * bi.n if raw else (bi.n + 3) // 4
        push, gathered = self.last_buffers()
        if worker is None:
            r = push[bi.region_offset:bi.region_offset + nbytes]
        else:
            base = worker * self.info.push_bytes + bi.region_offset
            r = gathered[base:base + nbytes]
        return r.view(torch.float32) if raw else r

    def layer_codes(self, l: int, worker: Optional[int] = None) -> torch.Tensor:
        """codes of layer l's first block (the whole layer unless FixedSize)"""
        return self.block_region(next(b for b, bi in enumerate(self.blocks) if bi.layer == l),
                                 worker)

    def close(self):
        if getattr(self, "h", None) and self.h.value:
            load().tgb_plan_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class SyncWorker:
    """One data-parallel worker's gradient synchronisation on one B200.

    Mirrors Worker::run's sync segment (cluster.hpp:283-297): ``step(t)``
    encodes this rank's gradients, exchanges scalers+codes with every rank
    and decodes the identical averaged gradient into ``out``.
    """

    def __init__(self, names: Sequence[str], shapes: Sequence[Sequence[int]], cfg: CodecConfig,
                 rank: int = 0, world_size: int = 1, comm: Optional[Comm] = None, device=None,
                 exchange: str = "auto", schedule: str = "auto", pieces: int = 0,
                 overlap: Optional[bool] = None, pull: int = 0):
        """exchange: "auto" | "fused" | "sharded" (NVLink peer stores, attached at
        construction) | "nccl" (ncclAllGather of push areas); schedule: see
        Plan.set_schedule."""
        self.device = _dev(device)
        self.names = list(names)
        self.shapes = [list(s) for s in shapes]
        self.ns = [int(torch.Size(s).numel()) if len(s) else 0 for s in self.shapes]
        self.rank, self.world_size = rank, world_size
        if world_size > 1 and comm is None:
            raise ValueError("SyncWorker: world_size > 1 needs a Comm")
        if exchange not in ("auto", "fused", "sharded", "nccl"):
            raise ValueError(f"SyncWorker: unknown exchange {exchange!r}")
        self.comm = comm
        self.plan = Plan(self.names, self.ns, cfg, worker=rank, n_workers=world_size,
                         device=self.device)
        if schedule != "auto":
            self.plan.set_schedule(schedule)
        if world_size > 1 and exchange in ("fused", "sharded"):
            self.plan.set_exchange(exchange)
        if overlap is not None and world_size > 1:
            self.plan.set_overlap(overlap)
        if pieces:
            self.plan.set_pieces(pieces)
        if pull and world_size > 1:
            self.plan.set_pull(pull)
        self.grad_flat, self.grads = aligned_flat(self.ns, self.device)
        self.out_flat, self.outs = aligned_flat(self.ns, self.device)
        self.plan.bind(self.grads, self.outs)
        if world_size > 1 and exchange != "nccl":  # K2 stores codes into the peers (NVLink)
            self.plan.attach_peers(comm)
        self.traffic = TrafficStats()
        self._step_traffic = None

    def step(self, t: int, stream=None, check: bool = False) -> List[torch.Tensor]:
        """Worker::run sync segment: encode -> exchange -> decode into ``outs``.
        check=True synchronises and rethrows a codec / protocol error of this step
        (otherwise errors stay in the device error word until ``check()``)."""
        self.plan.step(t, self.comm, stream)
        self._count_traffic()
        if check:
            self.check()
        return self.outs

    def _count_traffic(self):
        if self._step_traffic is None:
            self._step_traffic = self.plan.traffic()
        self.traffic += self._step_traffic

    def host_buffers(self, pinned: bool = True):
        """pinned host buffers for step_host: (in_flat, in_views, out_flat, out_views)"""
        gi, gv = aligned_flat(self.ns, torch.device("cpu"), pin_memory=pinned)
        go, ov = aligned_flat(self.ns, torch.device("cpu"), pin_memory=pinned)
        return gi, gv, go, ov

    def step_host(self, t: int, host_grads: Sequence[torch.Tensor],
                  host_outs: Sequence[torch.Tensor], stream=None):
        """Worker::run sync segment with host buffers: gradients in, averaged out."""
        self.plan.step_host(t, host_grads, host_outs, self.comm, stream)
        self._count_traffic()

    def bind_optimizer(self, cfg, params: Sequence[torch.Tensor]):
        """Parameters (device, one per layer) updated by step_apply with
        OptimizerState::apply semantics (optimizer.hpp:80-125); state zero-initialised."""
        n = cfg.n_state()
        self.params = list(params)
        self.opt_state1 = [torch.zeros_like(p) for p in self.params] if n >= 1 else None
        self.opt_state2 = [torch.zeros_like(p) for p in self.params] if n >= 2 else None
        nl = len(self.ns)
        P = C.c_void_p * max(nl, 1)
        opt = cfg.c()
        check(load().tgb_plan_bind_optimizer(
            self.plan.h, C.byref(opt), P(*[p.data_ptr() for p in self.params]),
            P(*[b.data_ptr() for b in self.opt_state1]) if self.opt_state1 else None,
            P(*[b.data_ptr() for b in self.opt_state2]) if self.opt_state2 else None),
            "tgb_plan_bind_optimizer")

    def step_apply(self, t: int, rate: float, stream=None):
        """Worker::run sync segment + opt.apply (cluster.hpp:283-299) in one call"""
        check(load().tgb_step_apply(self.plan.h, self.comm.h if self.comm is not None else None,
                                    int(t), float(rate), self.plan._st(stream)), "tgb_step_apply")

    def check(self):
        self.plan.raise_errors()


class LocalCluster:
    """N data-parallel workers in ONE process (the reference's run_cluster over
    InProcessHub, cluster.hpp:378-397): one plan per worker, attached to each
    other with tgb_plan_attach_local and stepped together with tgb_local_step,
    each worker on its own stream. The exchange kernels are the ones the
    multi-process path runs (K2 peer stores, K3 or the sharded reduce/expand);
    the streams are ordered by CUDA events instead of spinning flag barriers, so
    N = 8 workers can run on one GPU with no launch-environment settings.
    ``devices``: one device for all, or one per worker."""

    def __init__(self, names: Sequence[str], shapes: Sequence[Sequence[int]], cfg: CodecConfig,
                 n_workers: int, devices=None, exchange: str = "auto", schedule: str = "auto",
                 pieces: int = 0, overlap: Optional[bool] = None, pull: int = 0):
        if not isinstance(devices, (list, tuple)):
            devices = [devices] * n_workers
        self.devices = [_dev(d) for d in devices]
        self.names = list(names)
        self.ns = [int(torch.Size(s).numel()) if len(s) else 0 for s in shapes]
        self.n_workers = int(n_workers)
        self.plans, self.grad_flat, self.grads, self.out_flat, self.outs = [], [], [], [], []
        for w in range(self.n_workers):
            dev = self.devices[w]
            p = Plan(self.names, self.ns, cfg, worker=w, n_workers=self.n_workers, device=dev)
            if schedule != "auto":
                p.set_schedule(schedule)
            if self.n_workers > 1 and exchange != "auto":
                p.set_exchange(exchange)
            if overlap is not None and self.n_workers > 1:
                p.set_overlap(overlap)
            if pieces:
                p.set_pieces(pieces)
            if pull and self.n_workers > 1:
                p.set_pull(pull)
            gf, gv = aligned_flat(self.ns, dev)
            of, ov = aligned_flat(self.ns, dev)
            p.bind(gv, ov)
            self.plans.append(p)
            self.grad_flat.append(gf)
            self.grads.append(gv)
            self.out_flat.append(of)
            self.outs.append(ov)
        if self.n_workers > 1:
            Plan.attach_local(self.plans)
        self.streams = [torch.cuda.Stream(d) for d in self.devices]
        self.traffic = TrafficStats()  # ParameterServer::traffic(): all workers (cluster.hpp:147-160)
        self._step_traffic = None

    @property
    def exchange(self) -> str:
        return self.plans[0].exchange

    def step(self, t, check: bool = False) -> List[List[torch.Tensor]]:
        """Every worker's step for iteration t (an int, or one per worker), each on
        its own stream (ordered after work already queued on each device's current
        stream, e.g. the gradients' producers)."""
        ts = list(t) if isinstance(t, (list, tuple)) else [int(t)] * self.n_workers
        for s, d in zip(self.streams, self.devices):
            s.wait_stream(torch.cuda.current_stream(d))
        Plan.local_step(self.plans, ts, self.streams)
        if self._step_traffic is None:
            self._step_traffic = TrafficStats()
            for p in self.plans:
                self._step_traffic += p.traffic()
        self.traffic += self._step_traffic
        if check:
            self.check()
        return self.outs

    def synchronize(self):
        for s in self.streams:
            s.synchronize()

    def check(self):
        for p in self.plans:
            p.raise_errors()

    def close(self):
        self.synchronize()
        for p in self.plans:
            p.close()


class TrafficStats:
    """The reference's TrafficStats (cluster.hpp:62-74): framed bytes up/down in
    the reference's wire format and the same tensors at raw fp32, plus what this
    build's device exchange moved over NVLink."""

    def __init__(self, bytes_up=0, bytes_down=0, float_bytes_up=0, float_bytes_down=0,
                 device_bytes_out=0, device_bytes_in=0):
        self.bytes_up, self.bytes_down = int(bytes_up), int(bytes_down)
        self.float_bytes_up, self.float_bytes_down = int(float_bytes_up), int(float_bytes_down)
        self.device_bytes_out, self.device_bytes_in = int(device_bytes_out), int(device_bytes_in)

    @classmethod
    def of(cls, t: "_lib.Traffic") -> "TrafficStats":
        return cls(t.bytes_up, t.bytes_down, t.float_bytes_up, t.float_bytes_down,
                   t.device_bytes_out, t.device_bytes_in)

    @classmethod
    def for_layers(cls, names: Sequence[str], ns: Sequence[int], cfg: CodecConfig,
                   n_workers: int, passthrough: Optional[Sequence[bool]] = None) -> "TrafficStats":
        """one worker-step's terms from a layer table alone (no device;
        tgb_traffic_for_layers)"""
        nl = len(names)
        if passthrough is None:
            passthrough = [cfg.float_mode or n in cfg.passthrough for n in names]
        descs = (_lib.LayerDesc * max(nl, 1))()
        for l, (name, n) in enumerate(zip(names, ns)):
            descs[l] = _lib.LayerDesc(int(n), fnv1a64(name),
                                      _lib.TGB_LAYER_PASSTHROUGH if passthrough[l] else 0, 0)
        cn = (C.c_char_p * max(nl, 1))(*[x.encode() for x in names])
        params = cfg.params()
        t = _lib.Traffic()
        check(load().tgb_traffic_for_layers(descs, cn, nl, C.byref(params), int(n_workers),
                                            C.byref(t)), "tgb_traffic_for_layers")
        return cls.of(t)

    def __iadd__(self, o: "TrafficStats") -> "TrafficStats":
        self.bytes_up += o.bytes_up
        self.bytes_down += o.bytes_down
        self.float_bytes_up += o.float_bytes_up
        self.float_bytes_down += o.float_bytes_down
        self.device_bytes_out += o.device_bytes_out
        self.device_bytes_in += o.device_bytes_in
        return self

    def up_reduction(self) -> float:
        return self.float_bytes_up / self.bytes_up if self.bytes_up else 1.0

    def down_reduction(self) -> float:
        return self.float_bytes_down / self.bytes_down if self.bytes_down else 1.0

    def __repr__(self):
        return (f"TrafficStats(up={self.bytes_up}, down={self.bytes_down}, "
                f"float_up={self.float_bytes_up}, float_down={self.float_bytes_down}, "
                f"device_out={self.device_bytes_out}, device_in={self.device_bytes_in})")
