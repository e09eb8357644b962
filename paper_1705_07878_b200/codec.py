"""Reference-shaped codec API (namespace ``terngrad`` of the CPU reference) on the
B200 kernels.

Same names, argument meaning and error behaviour as
``/root/reference/proj/include/terngrad/{rng,tensor,codec}.hpp``; tensors live
in HBM (``torch.Tensor`` on a CUDA device) instead of ``std::vector<float>``.
Everything computes through libtgb.so's C-ABI; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum
from typing import Iterable, List, Optional, Sequence, Set, Union

import torch

from . import _lib
from ._lib import check, load


class ProtocolError(RuntimeError):
    """wire.hpp:14-16"""


class CodecError(RuntimeError):
    """terngrad::CodecError (codec.hpp:25-27)."""


def fnv1a64(name: str) -> int:
    """rng.hpp:37-44 (host side)."""
    b = name.encode()
    return load().tgb_fnv1a64(b, len(b))


def _stream(device: torch.device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None and t.numel() > 0 else 0)


def _dev(device=None) -> torch.device:
    _lib.require_device()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError("terngrad_b200 tensors live on CUDA devices")
    return d


def _fmt_float(x: float) -> str:
    """std::to_string(float) formatting ("%f")."""
    return "%f" % x


def _raise_layer_error(e: _lib.Error, name: str) -> None:
    f = e.flags
    if f & _lib.TGB_E_NONFINITE:
        raise CodecError("encode_step: non-finite gradient " + name)
    if f & _lib.TGB_E_S0_NONZERO:
        raise CodecError("ternarize: s=0 but gradient has nonzero element")
    if f & _lib.TGB_E_CORRUPT_CODE:
        raise CodecError(f"corrupt ternary code 11 in block {name} at element {e.index}")
    raise CodecError(f"codec error flags {f:#x} in {name}")


def _layer_check(device: torch.device, name: str, scaler: Optional[float] = None) -> None:
    e = _lib.Error()
    st = load().tgb_layer_check(_stream(device), C.byref(e))
    if st == _lib.TGB_ERR_CODEC:
        if e.flags & _lib.TGB_E_SCALER_BELOW_MAX:
            raise CodecError(f"ternarize: scaler {_fmt_float(scaler or 0.0)} below max |g| in {name}")
        _raise_layer_error(e, name)
    check(st, "tgb_layer_check")


# ------------------------------------------------------------------ rng.hpp
class RngStream:
    """rng.hpp:48-84. Host derives the key; bits/uniform are computed on the device."""

    def __init__(self, seed: int, iteration: int, tensor_name: str, worker: int = 0):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
        self.iteration = int(iteration) & 0xFFFFFFFFFFFFFFFF
        self.name = tensor_name
        self.worker = int(worker) & 0xFFFFFFFFFFFFFFFF
        self.name_hash = fnv1a64(tensor_name)

    def bits_range(self, k0: int, n: int, device=None) -> torch.Tensor:
        dev = _dev(device)
        out = torch.empty(n, dtype=torch.int32, device=dev)
        check(load().tgb_rng_bits(self.seed, self.iteration, self.name_hash, self.worker, k0, n,
                                  _ptr(out), _stream(dev)), "tgb_rng_bits")
        return out

    def bits(self, index: int) -> int:
        return int(self.bits_range(index, 1).cpu().item()) & 0xFFFFFFFF

    def uniform(self, index: int) -> float:
        # float(bits) * 2^-32, round-to-nearest (rng.hpp:69-71)
        b = torch.tensor([self.bits(index)], dtype=torch.float64)
        return float(b.to(torch.float32).item()) * 2.0 ** -32


# --------------------------------------------------------------- tensor.hpp
class GradTensor:
    """tensor.hpp:14-43 with device-resident values."""

    def __init__(self, name: str, shape: Sequence[int], values: Optional[torch.Tensor] = None,
                 device=None):
        self.name = name
        self.shape = list(shape)
        n = self.element_count(self.shape)
        if values is None:
            values = torch.zeros(n, dtype=torch.float32, device=_dev(device))
        values = values.reshape(-1)
        if values.numel() != n:
            raise ValueError(f"GradTensor {name}: values/shape mismatch")
        if values.dtype != torch.float32:
            raise TypeError("GradTensor values must be float32")
        self.values = values.contiguous()

    @staticmethod
    def element_count(shape: Sequence[int]) -> int:
        if len(shape) == 0:
            return 0
        n = 1
        for d in shape:
            n *= int(d)
        return n

    def size(self) -> int:
        return self.values.numel()

    def all_finite(self) -> bool:
        return bool(torch.isfinite(self.values).all().item())


# ---------------------------------------------------------------- codec.hpp
class Bucketing(IntEnum):
    PerTensor = _lib.TGB_BUCKET_PER_TENSOR
    Global = _lib.TGB_BUCKET_GLOBAL
    FixedSize = _lib.TGB_BUCKET_FIXED


class ShareMode(IntEnum):
    REF = _lib.TGB_SHARE_REF               # post-hoc max, bit-exact with the reference
    PRESHARED = _lib.TGB_SHARE_PRESHARED   # paper Eq. 4: shared max before ternarize


@dataclass
class CodecConfig:
    """codec.hpp:80-96."""

    clip_factor: float = 2.5
    clipping_enabled: bool = True
    bucketing: Bucketing = Bucketing.PerTensor
    bucket_size: int = 0
    scaler_sharing: bool = True
    float_mode: bool = False
    passthrough: Set[str] = field(default_factory=set)
    seed: int = 0
    share_mode: ShareMode = ShareMode.REF

    def validate(self) -> None:
        if not (self.clip_factor > 0.0):
            raise ValueError("codec: clip factor must be positive")
        if self.bucketing == Bucketing.FixedSize and self.bucket_size < 1:
            raise ValueError("codec: fixed-size bucket needs k >= 1")

    def params(self) -> _lib.CodecParams:
        return _lib.CodecParams(float(self.clip_factor), int(self.clipping_enabled),
                                int(self.bucketing), int(self.scaler_sharing),
                                int(self.bucket_size), int(self.seed) & 0xFFFFFFFFFFFFFFFF,
                                int(self.share_mode), 0)


@dataclass
class TernaryBlock:
    """codec.hpp:30-61; codes are ceil(n/4) bytes in HBM."""

    name: str
    n: int
    s: float
    codes: torch.Tensor

    def code_at(self, k: int) -> int:
        c = (int(self.codes[k // 4].item()) >> (2 * (k % 4))) & 3
        if c == 0:
            return 0
        if c == 1:
            return 1
        if c == 2:
            return -1
        raise CodecError(f"corrupt ternary code 11 in block {self.name} at element {k}")

    def zero_fraction(self) -> float:
        if self.n == 0:
            return 0.0
        c = self.codes.to(torch.int32)
        nz = sum(int((((c >> (2 * e)) & 3) != 0).sum().item()) for e in range(4))
        return (self.n - nz) / self.n


@dataclass
class PassthroughBlock:
    name: str
    values: torch.Tensor


GradBlock = Union[TernaryBlock, PassthroughBlock]


@dataclass
class EncodedGradient:
    iteration: int = 0
    worker: int = 0
    blocks: List[GradBlock] = field(default_factory=list)


@dataclass
class EncodeResult:
    encoded: EncodedGradient
    local_scalers: List[float]


def scaler(values: Union[torch.Tensor, GradTensor]) -> float:
    """codec.hpp:128-134."""
    v = values.values if isinstance(values, GradTensor) else values.reshape(-1).contiguous()
    dev = v.device
    out = torch.empty(1, dtype=torch.float32, device=_dev(dev))
    check(load().tgb_layer_scaler(_ptr(v), v.numel(), _ptr(out), _stream(dev)), "tgb_layer_scaler")
    _layer_check(dev, "scaler")
    return float(out.item())


def share_scalers(locals_: Sequence[float]) -> float:
    """codec.hpp:136-141 (host: it is the max-allreduce's local semantics)."""
    if len(locals_) == 0:
        raise CodecError("share_scalers: empty scaler list")
    m = 0.0
    for s in locals_:
        m = max(m, float(s))
    return m


def clip(g: GradTensor, c: float) -> GradTensor:
    """codec.hpp:117-124; returns a new tensor."""
    if g.size() < 2:
        return GradTensor(g.name, g.shape, g.values.clone())
    out = torch.empty_like(g.values)
    bound = torch.empty(1, dtype=torch.float32, device=g.values.device)
    check(load().tgb_layer_clip(_ptr(g.values), g.size(), float(c), _ptr(out), _ptr(bound),
                                _stream(g.values.device)), "tgb_layer_clip")
    _layer_check(g.values.device, g.name)
    return GradTensor(g.name, g.shape, out)


def clip_bound(g: GradTensor, c: float) -> float:
    """float(c * stddev(g)) (codec.hpp:119), +inf for n < 2."""
    if g.size() < 2:
        return float("inf")
    out = torch.empty_like(g.values)
    bound = torch.empty(1, dtype=torch.float32, device=g.values.device)
    check(load().tgb_layer_clip(_ptr(g.values), g.size(), float(c), _ptr(out), _ptr(bound),
                                _stream(g.values.device)), "tgb_layer_clip")
    _layer_check(g.values.device, g.name)
    return float(bound.item())


def ternarize(name: Union[str, GradTensor], g=None, s: float = None, rng: RngStream = None,
              rng_base: int = 0) -> TernaryBlock:
    """codec.hpp:148-175 (and the GradTensor overload :173-175)."""
    if isinstance(name, GradTensor):  # ternarize(g, s, rng)
        gt, s, rng = name, g, s
        name, values = gt.name, gt.values
    else:
        values = g.values if isinstance(g, GradTensor) else g.reshape(-1).contiguous()
    n = values.numel()
    dev = values.device
    codes = torch.zeros((n + 3) // 4, dtype=torch.uint8, device=_dev(dev))
    check(load().tgb_layer_ternarize(_ptr(values), n, float(s), rng.seed, rng.iteration,
                                     rng.name_hash, rng.worker, int(rng_base), _ptr(codes),
                                     _stream(dev)), "tgb_layer_ternarize")
    _layer_check(dev, name, float(s))
    return TernaryBlock(name, n, float(s), codes)


def decode(blk: TernaryBlock) -> GradTensor:
    """codec.hpp:177-182."""
    dev = blk.codes.device if blk.codes.numel() else _dev()
    out = torch.empty(blk.n, dtype=torch.float32, device=dev)
    check(load().tgb_layer_decode(_ptr(blk.codes), blk.n, float(blk.s), _ptr(out), _stream(dev)),
          "tgb_layer_decode")
    _layer_check(dev, blk.name)
    return GradTensor(blk.name, [blk.n], out)


# ------------------------------------------------------------- telemetry
@dataclass
class HistogramBin:
    """codec.hpp:485-488"""
    edge: float  # left edge
    count: int


def histogram(values: Union[torch.Tensor, GradTensor], bins: int) -> List[HistogramBin]:
    """codec.hpp:491-517 on the device (equal-width bins over [min, max])."""
    if bins < 1:
        raise ValueError("histogram: bins must be >= 1")
    v = values.values if isinstance(values, GradTensor) else values.reshape(-1).contiguous()
    dev = v.device if v.numel() else _dev()
    counts = torch.zeros(bins, dtype=torch.int64, device=dev)
    edges = torch.zeros(bins, dtype=torch.float64, device=dev)
    check(load().tgb_layer_histogram(_ptr(v), v.numel(), int(bins), _ptr(counts), _ptr(edges),
                                     _stream(dev)), "tgb_layer_histogram")
    return [HistogramBin(float(e), int(c)) for e, c in zip(edges.cpu().tolist(),
                                                           counts.cpu().tolist())]


# ------------------------------------------------------------- encode_step
class _PlanCache:
    def __init__(self):
        self.plans = {}

    def get(self, key, make):
        p = self.plans.get(key)
        if p is None:
            p = make()
            self.plans[key] = p
        return p


_plans = _PlanCache()


def encode_step(grads: Sequence[GradTensor], cfg: CodecConfig, t: int, worker: int) -> EncodeResult:
    """codec.hpp:194-239 through one B200 plan (K1 stats + K2 ternarize/copy).

    Blocks come back in canonical order: one TernaryBlock per bucket (FixedSize)
    or tensor, one PassthroughBlock per tensor named in cfg.passthrough; the
    codes/values are views of one copy of the plan's push area."""
    from .plan import Plan  # local import: plan.py builds on this module

    cfg.validate()
    dev = grads[0].values.device if grads else _dev()
    names = [g.name for g in grads]
    ns = [g.size() for g in grads]
    passthrough = tuple(name in cfg.passthrough for name in names)
    key = ("enc", tuple(names), tuple(ns), passthrough, cfg.clip_factor, cfg.clipping_enabled,
           int(cfg.bucketing), cfg.bucket_size, cfg.scaler_sharing, cfg.seed,
           int(cfg.share_mode), worker, str(dev))
    plan = _plans.get(key, lambda: Plan(names, ns, cfg, worker=worker, n_workers=1, device=dev,
                                        passthrough=list(passthrough)))
    plan.bind([g.values for g in grads], None)
    plan.encode(t)
    plan.raise_errors()
    push = plan.push.clone()
    scal = push[:4 * plan.info.n_slots].view(torch.float32).cpu().tolist()
    blocks: List[GradBlock] = []
    for bi in plan.blocks:
        name = names[bi.layer]
        o = bi.region_offset
        if bi.flags & _lib.TGB_LAYER_PASSTHROUGH:
            blocks.append(PassthroughBlock(name, push[o:o + 4 * bi.n].view(torch.float32)))
        else:
            blocks.append(TernaryBlock(name, bi.n, scal[bi.slot], push[o:o + (bi.n + 3) // 4]))
    return EncodeResult(EncodedGradient(t, worker, blocks), scal)


def average(encoded: Sequence[EncodedGradient], N: int, scaler_sharing: bool) -> List[GradTensor]:
    """codec.hpp:245-311 (K3 per block)."""
    if len(encoded) != N or N == 0:
        raise CodecError(f"average: expected {N} messages, got {len(encoded)}")
    nblocks = len(encoded[0].blocks)
    for e in encoded:
        if e.iteration != encoded[0].iteration:
            raise CodecError("average: mismatched iterations")
        if len(e.blocks) != nblocks:
            raise CodecError("average: mismatched block structure")
    out: List[GradTensor] = []
    lib = load()
    for b in range(nblocks):
        first = encoded[0].blocks[b]
        if isinstance(first, PassthroughBlock):  # codec.hpp:269-279
            dev = first.values.device if first.values.numel() else _dev()
            avg = torch.empty(first.values.numel(), dtype=torch.float32, device=dev)
            for e in encoded:
                blk = e.blocks[b]
                if not isinstance(blk, PassthroughBlock) or blk.name != first.name or \
                        blk.values.numel() != first.values.numel():
                    raise CodecError("average: block structure mismatch at " + first.name)
            if avg.numel():
                vals = [e.blocks[b].values.contiguous() for e in encoded]
                ptrs = (C.c_void_p * N)(*[v.data_ptr() for v in vals])
                check(lib.tgb_layer_average_raw(N, ptrs, avg.numel(), _ptr(avg), _stream(dev)),
                      "tgb_layer_average_raw")
                _layer_check(dev, first.name)
            _append(out, first.name, avg)
            continue
        for e in encoded:
            blk = e.blocks[b]
            if not isinstance(blk, TernaryBlock) or blk.name != first.name or blk.n != first.n:
                raise CodecError("average: block structure mismatch at " + first.name)
        dev = first.codes.device if first.codes.numel() else _dev()
        avg = torch.empty(first.n, dtype=torch.float32, device=dev)
        if first.n:
            ptrs = (C.c_void_p * N)(*[e.blocks[b].codes.data_ptr() for e in encoded])
            s = torch.tensor([e.blocks[b].s for e in encoded], dtype=torch.float32, device=dev)
            check(lib.tgb_layer_average(N, ptrs, _ptr(s), first.n, int(scaler_sharing), _ptr(avg),
                                        _stream(dev)), "tgb_layer_average")
            _layer_check(dev, first.name)
        _append(out, first.name, avg)
    return out


def _append(out: List[GradTensor], name: str, avg: torch.Tensor) -> None:
    """merge bucket runs by name (codec.hpp:259-265)"""
    if out and out[-1].name == name:
        merged = torch.cat([out[-1].values, avg])
        out[-1] = GradTensor(name, [merged.numel()], merged)
    else:
        out.append(GradTensor(name, [avg.numel()], avg))
