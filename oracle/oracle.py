"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the parity checkers.

* ``Restated``  -> oracle/_build/libtgoracle.so (plain-C restatement, tg_oracle.c)
* ``Reference`` -> oracle/_ref/libtgref.so (the reference headers compiled
  unmodified from /root/reference by oracle/Makefile)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference
arm may import this module. The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(HERE, "_build", "libtgoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libtgref.so")

_u8p = C.POINTER(C.c_uint8)
_f32p = C.POINTER(C.c_float)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int32)

PER_TENSOR, GLOBAL, FIXED_SIZE = 0, 1, 2


def build() -> None:
    """Compile the checkers (restatement always; reference when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


@dataclass
class Config:
    """Mirror of terngrad::CodecConfig (codec.hpp:80-96)."""

    clip_factor: float = 2.5
    clipping_enabled: bool = True
    bucketing: int = PER_TENSOR
    bucket_size: int = 0
    scaler_sharing: bool = True
    seed: int = 0


class _TgoConfig(C.Structure):
    _fields_ = [
        ("clip_factor", C.c_float),
        ("clipping_enabled", C.c_int),
        ("bucketing", C.c_int),
        ("bucket_size", C.c_uint64),
        ("scaler_sharing", C.c_int),
        ("seed", C.c_uint64),
    ]


class _TgoRng(C.Structure):
    _fields_ = [("key", C.c_uint32 * 2), ("hi", C.c_uint32 * 2)]


def block_layout(ns: Sequence[int], cfg: Config, passthrough=None):
    """Per-block (tensor, offset, len) list in canonical order (codec.hpp:218-237)."""
    out = []
    for l, n in enumerate(ns):
        if passthrough is not None and passthrough[l]:
            continue
        if n == 0:
            out.append((l, 0, 0))
            continue
        bucket = cfg.bucket_size if cfg.bucketing == FIXED_SIZE else n
        off = 0
        while off < n:
            ln = min(bucket, n - off)
            out.append((l, off, ln))
            off += bucket
    return out


class Restated:
    """The plain-C restatement (tg_oracle.c)."""

    def __init__(self, path: str = RESTATED_SO):
        if not os.path.exists(path):
            build()
        L = self.L = C.CDLL(path)
        L.tgo_fnv1a64.restype = C.c_uint64
        L.tgo_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
        L.tgo_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
        L.tgo_rng_init.argtypes = [C.POINTER(_TgoRng), C.c_uint64, C.c_uint64, C.c_char_p,
                                   C.c_size_t, C.c_uint64]
        L.tgo_rng_bits.restype = C.c_uint32
        L.tgo_rng_bits.argtypes = [C.POINTER(_TgoRng), C.c_uint64]
        L.tgo_rng_uniform.restype = C.c_float
        L.tgo_rng_uniform.argtypes = [C.POINTER(_TgoRng), C.c_uint64]
        L.tgo_rng_normal_fill.argtypes = [C.POINTER(_TgoRng), C.c_uint64, C.c_size_t, C.c_float,
                                          _f32p]
        L.tgo_stddev.restype = C.c_double
        L.tgo_stddev.argtypes = [_f32p, C.c_size_t]
        L.tgo_clip.restype = C.c_float
        L.tgo_clip.argtypes = [_f32p, C.c_size_t, C.c_float, _f32p]
        L.tgo_scaler.restype = C.c_float
        L.tgo_scaler.argtypes = [_f32p, C.c_size_t]
        L.tgo_ternarize.restype = C.c_int
        L.tgo_ternarize.argtypes = [_f32p, C.c_size_t, C.c_float, C.POINTER(_TgoRng), C.c_uint64,
                                    _u8p]
        L.tgo_decode.restype = C.c_int
        L.tgo_decode.argtypes = [_u8p, C.c_size_t, C.c_float, _f32p]
        L.tgo_encode_step.restype = C.c_int
        L.tgo_encode_step.argtypes = [C.c_int, C.POINTER(C.c_char_p), _u64p,
                                      C.POINTER(_f32p), C.POINTER(C.c_int),
                                      C.POINTER(_TgoConfig), C.c_uint64, C.c_uint16, _u8p, _f32p,
                                      _f32p, C.POINTER(C.c_int)]
        L.tgo_average_block.restype = C.c_int
        L.tgo_average_block.argtypes = [C.c_int, _f32p, C.POINTER(_u8p), C.c_size_t, C.c_int,
                                        _f32p]
        L.tgo_average_passthrough.argtypes = [C.c_int, C.POINTER(_f32p), C.c_size_t, _f32p]

    # --- rng.hpp ---
    def philox(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        self.L.tgo_philox4x32_10(c, k, o)
        return list(o)

    def fnv1a64(self, name: str) -> int:
        b = name.encode()
        return self.L.tgo_fnv1a64(b, len(b))

    def rng(self, seed, t, name, worker=0):
        r = _TgoRng()
        b = name.encode()
        self.L.tgo_rng_init(C.byref(r), seed, t, b, len(b), worker)
        return r

    def bits(self, seed, t, name, worker, idx: Sequence[int]):
        r = self.rng(seed, t, name, worker)
        return [self.L.tgo_rng_bits(C.byref(r), i) for i in idx]

    def uniform(self, seed, t, name, worker, idx: Sequence[int]):
        r = self.rng(seed, t, name, worker)
        return np.array([self.L.tgo_rng_uniform(C.byref(r), i) for i in idx], dtype=np.float32)

    def normal(self, seed, t, name, n, scale=1.0, worker=0, k0=0):
        r = self.rng(seed, t, name, worker)
        out = np.empty(n, dtype=np.float32)
        self.L.tgo_rng_normal_fill(C.byref(r), k0, n, scale, _ptr(out, _f32p))
        return out

    # --- codec.hpp ---
    def stddev(self, v):
        v = _f32(v)
        return self.L.tgo_stddev(_ptr(v, _f32p), v.size)

    def clip(self, v, c=2.5):
        v = _f32(v)
        out = np.empty_like(v)
        b = self.L.tgo_clip(_ptr(v, _f32p), v.size, c, _ptr(out, _f32p))
        return out, b

    def scaler(self, v):
        v = _f32(v)
        return self.L.tgo_scaler(_ptr(v, _f32p), v.size)

    def ternarize(self, g, s, seed, t, name, worker=0, rng_base=0):
        g = _f32(g)
        codes = np.zeros((g.size + 3) // 4, dtype=np.uint8)
        r = self.rng(seed, t, name, worker)
        st = self.L.tgo_ternarize(_ptr(g, _f32p), g.size, s, C.byref(r), rng_base,
                                  _ptr(codes, _u8p))
        return st, codes

    def decode(self, codes, n, s):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        out = np.empty(n, dtype=np.float32)
        st = self.L.tgo_decode(_ptr(codes, _u8p), n, s, _ptr(out, _f32p))
        return st, out

    def encode_step(self, names, grads, cfg: Config, t, worker, passthrough=None):
        """Returns (status, codes-per-block list, scalers array, bounds array, bad_tensor)."""
        n_t = len(names)
        grads = [_f32(g) for g in grads]
        ns = np.array([g.size for g in grads], dtype=np.uint64)
        pt = np.array(passthrough if passthrough is not None else [0] * n_t, dtype=np.int32)
        layout = block_layout([int(x) for x in ns], cfg, pt)
        total = sum((ln + 3) // 4 for (_, _, ln) in layout)
        codes = np.zeros(max(total, 1), dtype=np.uint8)
        scal = np.zeros(max(len(layout), 1), dtype=np.float32)
        bounds = np.zeros(max(n_t, 1), dtype=np.float32)
        bad = C.c_int(-1)
        cn = (C.c_char_p * n_t)(*[x.encode() for x in names])
        gp = (_f32p * n_t)(*[_ptr(g, _f32p) for g in grads])
        tc = _TgoConfig(cfg.clip_factor, int(cfg.clipping_enabled), cfg.bucketing,
                        cfg.bucket_size, int(cfg.scaler_sharing), cfg.seed)
        st = self.L.tgo_encode_step(n_t, cn, _ptr(ns, _u64p), gp,
                                    pt.ctypes.data_as(C.POINTER(C.c_int)), C.byref(tc), t, worker,
                                    _ptr(codes, _u8p), _ptr(scal, _f32p), _ptr(bounds, _f32p),
                                    C.byref(bad))
        blocks, pos = [], 0
        for (_, _, ln) in layout:
            nb = (ln + 3) // 4
            blocks.append(codes[pos:pos + nb].copy())
            pos += nb
        return st, blocks, scal[:len(layout)], bounds[:n_t], bad.value

    def average_block(self, s, codes_per_worker, n, sharing=True):
        N = len(codes_per_worker)
        s = _f32(s)
        cs = [np.ascontiguousarray(c, dtype=np.uint8) for c in codes_per_worker]
        cp = (_u8p * N)(*[_ptr(c, _u8p) for c in cs])
        out = np.empty(n, dtype=np.float32)
        st = self.L.tgo_average_block(N, _ptr(s, _f32p), cp, n, int(sharing), _ptr(out, _f32p))
        return st, out

    def histogram(self, v, bins):
        """codec.hpp:491-517 restated: lo/hi by the reference's sequential std::min/max
        chain from v[0], width = (hi - lo) / bins in double, b = size_t((x - lo) / width)
        clamped to bins - 1 (NaN -> last bin, like the x86-64 conversion)."""
        v = _f32(v)
        if bins < 1:
            raise ValueError("histogram: bins must be >= 1")
        if v.size == 0:
            return np.zeros(bins, np.float64), np.zeros(bins, np.uint64)
        lo = hi = float(v[0])
        for x in v.astype(np.float64):  # small cases only (pure-Python loop)
            lo = x if x < lo else lo
            hi = x if hi < x else hi
        width = (hi - lo) / float(bins)
        edges = np.array([lo + width * float(b) for b in range(bins)], np.float64)
        counts = np.zeros(bins, np.uint64)
        for x in v.astype(np.float64):
            if width > 0.0:
                q = (x - lo) / width
                b = int(q) if q == q and q < 2.0 ** 64 else bins - 1
            else:
                b = 0
            counts[min(b, bins - 1)] += 1
        return edges, counts

    @staticmethod
    def optimizer_run(rule, w, grads, rates, momentum=0.9, beta1=0.9, beta2=0.999,
                      epsilon=1e-8, weight_decay=0.0):
        """optimizer.hpp:80-125 restated in numpy (one op per IEEE rounding, no FMA):
        len(rates) applies of one OptimizerState to one tensor."""
        f32, f64 = np.float32, np.float64
        w = _f32(w).copy()
        s1 = np.zeros_like(w)
        s2 = np.zeros_like(w)
        for step, (g, rate) in enumerate(zip(grads, rates), start=1):
            g = _f32(g)
            if rule == 2:  # Adam, double precision (optimizer.hpp:108-121)
                bc1 = 1.0 - f64(beta1) ** f64(step)
                bc2 = 1.0 - f64(beta2) ** f64(step)
                eff = g.astype(f64) + f64(weight_decay) * w.astype(f64)
                s1 = (f64(beta1) * s1.astype(f64) + (1.0 - f64(beta1)) * eff).astype(f32)
                s2 = (f64(beta2) * s2.astype(f64) + (1.0 - f64(beta2)) * eff * eff).astype(f32)
                mhat = s1.astype(f64) / bc1
                vhat = s2.astype(f64) / bc2
                w = (w - (f64(rate) * mhat / (np.sqrt(vhat) + f64(epsilon))).astype(f32)).astype(f32)
                continue
            eff = (g + f32(weight_decay) * w).astype(f32)
            if rule == 1:  # Momentum (optimizer.hpp:98-105)
                s1 = (f32(momentum) * s1 + eff).astype(f32)
                w = (w - f32(rate) * s1).astype(f32)
            else:  # Vanilla (optimizer.hpp:91-96)
                w = (w - f32(rate) * eff).astype(f32)
        return w

    def average_passthrough(self, vals):
        N = len(vals)
        vs = [_f32(v) for v in vals]
        vp = (_f32p * N)(*[_ptr(v, _f32p) for v in vs])
        out = np.empty(vs[0].size, dtype=np.float32)
        self.L.tgo_average_passthrough(N, vp, vs[0].size, _ptr(out, _f32p))
        return out


class Reference:
    """The unmodified reference headers behind oracle/ref_shim.cpp."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where "
                                    "/root/reference is present")
        L = self.L = C.CDLL(path)
        L.tgref_last_error.restype = C.c_char_p
        L.tgref_fnv1a64.restype = C.c_uint64
        L.tgref_fnv1a64.argtypes = [C.c_char_p, C.c_size_t]
        L.tgref_philox.argtypes = [_u32p, _u32p, _u32p]
        L.tgref_rng_bits.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64, C.c_uint64,
                                     C.c_size_t, _u32p]
        L.tgref_rng_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64,
                                        C.c_uint64, C.c_size_t, _f32p]
        L.tgref_normal_fill.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64,
                                        C.c_uint64, C.c_size_t, C.c_float, _f32p]
        L.tgref_stddev.restype = C.c_double
        L.tgref_stddev.argtypes = [_f32p, C.c_size_t]
        L.tgref_clip.argtypes = [_f32p, C.c_size_t, C.c_float, _f32p, _f32p]
        L.tgref_optimizer_run.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double,
                                          C.c_double, C.c_double, C.c_int, C.c_size_t, _f32p,
                                          _f32p, C.POINTER(C.c_double)]
        L.tgref_histogram.argtypes = [_f32p, C.c_size_t, C.c_size_t, C.POINTER(C.c_double),
                                      C.POINTER(C.c_uint64)]
        L.tgref_scaler.restype = C.c_float
        L.tgref_scaler.argtypes = [_f32p, C.c_size_t]
        L.tgref_ternarize.restype = C.c_int
        L.tgref_ternarize.argtypes = [C.c_char_p, _f32p, C.c_size_t, C.c_float, C.c_uint64,
                                      C.c_uint64, C.c_uint64, C.c_uint64, _u8p]
        L.tgref_decode.restype = C.c_int
        L.tgref_decode.argtypes = [_u8p, C.c_size_t, C.c_float, _f32p]
        L.tgref_encode_step.restype = C.c_int
        L.tgref_encode_step.argtypes = [C.c_int, C.POINTER(C.c_char_p), _u64p, C.POINTER(_f32p),
                                        C.POINTER(C.c_int), C.c_float, C.c_int, C.c_int,
                                        C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, C.c_uint16,
                                        _u8p, _f32p, _u64p]
        L.tgref_average_encoded.restype = C.c_int
        L.tgref_average_encoded.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_char_p), _u64p,
                                            C.POINTER(_f32p), C.POINTER(C.c_int), C.c_float,
                                            C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64,
                                            C.c_uint64, _f32p]
        L.tgref_cluster_create.restype = C.c_void_p
        L.tgref_cluster_create.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_char_p), _u64p,
                                           C.POINTER(_f32p), C.POINTER(C.c_int), C.c_float,
                                           C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_uint64]
        L.tgref_cluster_step.restype = C.c_double
        L.tgref_cluster_step.argtypes = [C.c_void_p, C.c_uint64]
        L.tgref_cluster_output.argtypes = [C.c_void_p, C.c_int, _f32p]
        L.tgref_cluster_destroy.argtypes = [C.c_void_p]

    def err(self) -> str:
        return self.L.tgref_last_error().decode()

    def philox(self, ctr, key):
        c = (C.c_uint32 * 4)(*ctr)
        k = (C.c_uint32 * 2)(*key)
        o = (C.c_uint32 * 4)()
        self.L.tgref_philox(c, k, o)
        return list(o)

    def fnv1a64(self, name: str) -> int:
        b = name.encode()
        return self.L.tgref_fnv1a64(b, len(b))

    def bits(self, seed, t, name, worker, k0, n):
        out = np.empty(n, dtype=np.uint32)
        self.L.tgref_rng_bits(seed, t, name.encode(), worker, k0, n, _ptr(out, _u32p))
        return out

    def uniform(self, seed, t, name, worker, k0, n):
        out = np.empty(n, dtype=np.float32)
        self.L.tgref_rng_uniform(seed, t, name.encode(), worker, k0, n, _ptr(out, _f32p))
        return out

    def normal(self, seed, t, name, n, scale=1.0, worker=0, k0=0):
        out = np.empty(n, dtype=np.float32)
        self.L.tgref_normal_fill(seed, t, name.encode(), worker, k0, n, scale, _ptr(out, _f32p))
        return out

    def stddev(self, v):
        v = _f32(v)
        return self.L.tgref_stddev(_ptr(v, _f32p), v.size)

    def clip(self, v, c=2.5):
        v = _f32(v)
        out = np.empty_like(v)
        b = C.c_float()
        self.L.tgref_clip(_ptr(v, _f32p), v.size, c, _ptr(out, _f32p), C.byref(b))
        return out, b.value

    def scaler(self, v):
        v = _f32(v)
        return self.L.tgref_scaler(_ptr(v, _f32p), v.size)

    def optimizer_run(self, rule, w, grads, rates, momentum=0.9, beta1=0.9, beta2=0.999,
                      epsilon=1e-8, weight_decay=0.0):
        """OptimizerState(cfg).apply() len(rates) times on one tensor (optimizer.hpp:80-125)"""
        w = _f32(w).copy()
        g = np.ascontiguousarray(np.stack([_f32(x) for x in grads]), dtype=np.float32)
        r = np.ascontiguousarray(rates, dtype=np.float64)
        st = self.L.tgref_optimizer_run(int(rule), momentum, beta1, beta2, epsilon, weight_decay,
                                        len(rates), w.size, _ptr(w, _f32p), _ptr(g, _f32p),
                                        r.ctypes.data_as(C.POINTER(C.c_double)))
        return (st, self.err() if st else ""), w

    def histogram(self, v, bins):
        """codec.hpp:491-517 -> ((status, msg), edges float64[bins], counts uint64[bins])"""
        v = _f32(v)
        edges = np.zeros(bins, np.float64)
        counts = np.zeros(bins, np.uint64)
        st = self.L.tgref_histogram(_ptr(v, _f32p), v.size, bins,
                                    edges.ctypes.data_as(C.POINTER(C.c_double)),
                                    counts.ctypes.data_as(C.POINTER(C.c_uint64)))
        return (st, self.err() if st else ""), edges, counts

    def ternarize(self, g, s, seed, t, name, worker=0, rng_base=0):
        g = _f32(g)
        codes = np.zeros((g.size + 3) // 4, dtype=np.uint8)
        st = self.L.tgref_ternarize(name.encode(), _ptr(g, _f32p), g.size, s, seed, t, worker,
                                    rng_base, _ptr(codes, _u8p))
        return (st, self.err() if st else ""), codes

    def decode(self, codes, n, s):
        codes = np.ascontiguousarray(codes, dtype=np.uint8)
        out = np.empty(n, dtype=np.float32)
        st = self.L.tgref_decode(_ptr(codes, _u8p), n, s, _ptr(out, _f32p))
        return (st, self.err() if st else ""), out

    def encode_step(self, names, grads, cfg: Config, t, worker, passthrough=None):
        n_t = len(names)
        grads = [_f32(g) for g in grads]
        ns = np.array([g.size for g in grads], dtype=np.uint64)
        pt = np.array(passthrough if passthrough is not None else [0] * n_t, dtype=np.int32)
        layout = block_layout([int(x) for x in ns], cfg, pt)
        total = sum((ln + 3) // 4 for (_, _, ln) in layout)
        codes = np.zeros(max(total, 1), dtype=np.uint8)
        scal = np.zeros(max(len(layout), 1), dtype=np.float32)
        nb = C.c_uint64()
        cn = (C.c_char_p * n_t)(*[x.encode() for x in names])
        gp = (_f32p * n_t)(*[_ptr(g, _f32p) for g in grads])
        st = self.L.tgref_encode_step(n_t, cn, _ptr(ns, _u64p), gp,
                                      pt.ctypes.data_as(C.POINTER(C.c_int)), cfg.clip_factor,
                                      int(cfg.clipping_enabled), cfg.bucketing, cfg.bucket_size,
                                      int(cfg.scaler_sharing), cfg.seed, t, worker,
                                      _ptr(codes, _u8p), _ptr(scal, _f32p), C.byref(nb))
        blocks, pos = [], 0
        for (_, _, ln) in layout:
            n_b = (ln + 3) // 4
            blocks.append(codes[pos:pos + n_b].copy())
            pos += n_b
        return (st, self.err() if st else ""), blocks, scal[:len(layout)]

    def average_encoded(self, names, grads_per_worker, cfg: Config, t, passthrough=None):
        """grads_per_worker[w][l]; returns (status, flat averaged output)."""
        N = len(grads_per_worker)
        n_t = len(names)
        gs = [[_f32(g) for g in gw] for gw in grads_per_worker]
        ns = np.array([g.size for g in gs[0]], dtype=np.uint64)
        pt = np.array(passthrough if passthrough is not None else [0] * n_t, dtype=np.int32)
        flat = [_ptr(g, _f32p) for gw in gs for g in gw]
        gp = (_f32p * len(flat))(*flat)
        cn = (C.c_char_p * n_t)(*[x.encode() for x in names])
        out = np.empty(int(ns.sum()), dtype=np.float32)
        st = self.L.tgref_average_encoded(N, n_t, cn, _ptr(ns, _u64p), gp,
                                          pt.ctypes.data_as(C.POINTER(C.c_int)),
                                          cfg.clip_factor, int(cfg.clipping_enabled),
                                          cfg.bucketing, cfg.bucket_size,
                                          int(cfg.scaler_sharing), cfg.seed, t,
                                          _ptr(out, _f32p))
        return (st, self.err() if st else ""), out


class RefCluster:
    """ParameterServer + N workers over InProcessHub (the reference as shipped)."""

    def __init__(self, ref: Reference, names, grads_per_worker, cfg: Config, passthrough=None):
        self.ref = ref
        N = self.N = len(grads_per_worker)
        n_t = len(names)
        self._gs = [[_f32(g) for g in gw] for gw in grads_per_worker]
        ns = np.array([g.size for g in self._gs[0]], dtype=np.uint64)
        self.total = int(ns.sum())
        pt = np.array(passthrough if passthrough is not None else [0] * n_t, dtype=np.int32)
        flat = [_ptr(g, _f32p) for gw in self._gs for g in gw]
        gp = (_f32p * len(flat))(*flat)
        cn = (C.c_char_p * n_t)(*[x.encode() for x in names])
        self.h = ref.L.tgref_cluster_create(N, n_t, cn, _ptr(ns, _u64p), gp,
                                            pt.ctypes.data_as(C.POINTER(C.c_int)),
                                            cfg.clip_factor, int(cfg.clipping_enabled),
                                            cfg.bucketing, cfg.bucket_size,
                                            int(cfg.scaler_sharing), cfg.seed)
        if not self.h:
            raise RuntimeError(ref.err())
        # the C++ side copied the gradients; drop ours
        self._gs = None

    def frame(self, worker: int, which: int) -> bytes:
        """last step's push (which=0) or received pull (which=1) frame of `worker`"""
        L = self.ref.L
        L.tgref_cluster_frame.restype = C.c_size_t
        L.tgref_cluster_frame.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_size_t]
        n = L.tgref_cluster_frame(self.h, worker, which, None, 0)
        buf = (C.c_uint8 * max(n, 1))()
        L.tgref_cluster_frame(self.h, worker, which, buf, n)
        return bytes(buf)[:n]

    def step(self, t: int) -> float:
        dt = self.ref.L.tgref_cluster_step(self.h, t)
        if dt < 0:
            raise RuntimeError(self.ref.err())
        return dt

    def output(self, worker=0) -> np.ndarray:
        out = np.empty(self.total, dtype=np.float32)
        self.ref.L.tgref_cluster_output(self.h, worker, _ptr(out, _f32p))
        return out

    def close(self):
        if self.h:
            self.ref.L.tgref_cluster_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()
