"""ctypes binding of libtgb.so (the C-ABI in include/tgb/terngrad_b200.h).

There is deliberately no fallback: if the shared library is missing or no
CUDA device is visible, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

_lock = threading.Lock()
_lib = None

TGB_OK = 0
TGB_ERR_INVALID_ARGUMENT = 1
TGB_ERR_CODEC = 2
TGB_ERR_CUDA = 3
TGB_ERR_NCCL = 4
TGB_ERR_UNSUPPORTED = 5
TGB_ERR_PROTOCOL = 6

TGB_E_NONFINITE = 0x1
TGB_E_SCALER_BELOW_MAX = 0x2
TGB_E_S0_NONZERO = 0x4
TGB_E_CORRUPT_CODE = 0x8
TGB_E_PEER_TIMEOUT = 0x10
TGB_E_SKEW = 0x20

TGB_LAYER_PASSTHROUGH = 0x1
TGB_BUCKET_PER_TENSOR, TGB_BUCKET_GLOBAL, TGB_BUCKET_FIXED = 0, 1, 2
TGB_SHARE_REF, TGB_SHARE_PRESHARED = 0, 1
UNIQUE_ID_BYTES = 128
TGB_EXCHANGE_AUTO = -1
TGB_EXCHANGE_NONE, TGB_EXCHANGE_NCCL, TGB_EXCHANGE_FUSED, TGB_EXCHANGE_SHARDED = 0, 1, 2, 3
EXCHANGE_NAMES = ["none", "nccl", "fused", "sharded"]
TGB_PLAN_OPT_SCHEDULE, TGB_PLAN_OPT_EXCHANGE, TGB_PLAN_OPT_FUSED_OPTIMIZER = 0, 1, 2
TGB_PLAN_OPT_PIECES = 3
TGB_PLAN_OPT_CHUNK = 4
TGB_PLAN_OPT_OVERLAP = 5
TGB_PLAN_OPT_PULL = 6
TGB_SCHEDULE_AUTO, TGB_SCHEDULE_SINGLE, TGB_SCHEDULE_GROUPS = 0, 1, 2
TGB_SCHEDULE_UNFUSED, TGB_SCHEDULE_FUSED12 = 3, 4

# every symbol the header declares (checked by tests/test_capi.py)
EXPORTS = [
    "tgb_version", "tgb_status_string", "tgb_fnv1a64", "tgb_device_count",
    "tgb_plan_create", "tgb_plan_destroy", "tgb_plan_get_info", "tgb_plan_layer_layout",
    "tgb_plan_block_info", "tgb_plan_set_option",
    "tgb_plan_bind", "tgb_plan_buffers", "tgb_stats", "tgb_ternarize_pack", "tgb_encode",
    "tgb_share_scalers", "tgb_sync", "tgb_decode_average", "tgb_step", "tgb_step_host", "tgb_check",
    "tgb_plan_code_stats", "tgb_plan_enable_code_stats", "tgb_plan_enable_timing",
    "tgb_plan_read_timing",
    "tgb_plan_attach_peers", "tgb_plan_attach_local", "tgb_local_step", "tgb_plan_last_buffers",
    "tgb_traffic_for_layers", "tgb_plan_traffic", "tgb_plan_audit",
    "tgb_optimizer_apply", "tgb_plan_bind_optimizer", "tgb_step_apply",
    "tgb_last_error_message", "tgb_plan_set_names", "tgb_plan_push_frame_size",
    "tgb_plan_serialize_push", "tgb_plan_decode_pull",
    "tgb_comm_unique_id", "tgb_comm_init", "tgb_comm_destroy",
    "tgb_layer_scaler", "tgb_layer_clip", "tgb_layer_ternarize", "tgb_layer_decode",
    "tgb_layer_average", "tgb_layer_average_raw", "tgb_layer_histogram", "tgb_rng_bits",
    "tgb_layer_check",
]


class LayerDesc(C.Structure):
    _fields_ = [("n", C.c_uint64), ("name_hash", C.c_uint64), ("flags", C.c_uint32),
                ("reserved", C.c_uint32)]


class CodecParams(C.Structure):
    _fields_ = [("clip_factor", C.c_float), ("clipping_enabled", C.c_int32),
                ("bucketing", C.c_int32), ("scaler_sharing", C.c_int32),
                ("bucket_size", C.c_uint64), ("seed", C.c_uint64),
                ("share_mode", C.c_int32), ("reserved", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("total_elements", C.c_uint64), ("push_bytes", C.c_uint64),
                ("code_bytes", C.c_uint64), ("scaler_offset", C.c_uint64),
                ("codes_offset", C.c_uint64), ("n_layers", C.c_int32), ("n_slots", C.c_int32),
                ("n_chunks", C.c_int32), ("n_workers", C.c_int32), ("chunk_elems", C.c_uint32),
                ("n_groups", C.c_uint32), ("n_blocks", C.c_int32), ("exchange", C.c_int32)]


class KernelTime(C.Structure):
    _fields_ = [("kind", C.c_int32), ("group", C.c_int32), ("ms", C.c_float),
                ("start_ms", C.c_float), ("elements", C.c_uint64), ("hbm_bytes", C.c_uint64),
                ("nvlink_bytes", C.c_uint64)]


KERNEL_NAMES = {0: "K1_stats", 1: "K2_ternarize_pack", 2: "peer_barrier", 3: "K3_decode",
                4: "K3a_shard_reduce", 5: "K3b_shard_expand", 6: "K12_fused", 7: "nccl"}


class Traffic(C.Structure):
    """tgb_traffic: one worker's per-step TrafficStats terms (cluster.hpp:62-74)"""
    _fields_ = [("bytes_up", C.c_uint64), ("bytes_down", C.c_uint64),
                ("float_bytes_up", C.c_uint64), ("float_bytes_down", C.c_uint64),
                ("device_bytes_out", C.c_uint64), ("device_bytes_in", C.c_uint64)]


class BlockInfo(C.Structure):
    _fields_ = [("layer", C.c_int32), ("slot", C.c_int32), ("offset", C.c_uint64),
                ("n", C.c_uint64), ("region_offset", C.c_uint64), ("flags", C.c_uint32),
                ("reserved", C.c_uint32)]


class Optimizer(C.Structure):
    _fields_ = [("rule", C.c_int32), ("reserved", C.c_int32), ("momentum", C.c_double),
                ("beta1", C.c_double), ("beta2", C.c_double), ("epsilon", C.c_double),
                ("weight_decay", C.c_double)]


class Error(C.Structure):
    _fields_ = [("flags", C.c_uint32), ("layer", C.c_int32), ("index", C.c_uint64),
                ("aux", C.c_uint64)]


_vp = C.c_void_p
_u64 = C.c_uint64
_i32 = C.c_int32


def _declare(L):
    S = C.c_int  # tgb_status
    sig = {
        "tgb_version": (C.c_char_p, []),
        "tgb_status_string": (C.c_char_p, [S]),
        "tgb_fnv1a64": (_u64, [C.c_char_p, C.c_size_t]),
        "tgb_device_count": (_i32, []),
        "tgb_plan_create": (S, [C.POINTER(LayerDesc), _i32, C.POINTER(CodecParams), C.c_uint16,
                                _i32, C.POINTER(_vp)]),
        "tgb_plan_destroy": (None, [_vp]),
        "tgb_plan_get_info": (S, [_vp, C.POINTER(PlanInfo)]),
        "tgb_plan_layer_layout": (S, [_vp, _i32, C.POINTER(_u64), C.POINTER(_i32)]),
        "tgb_plan_block_info": (S, [_vp, _i32, C.POINTER(BlockInfo)]),
        "tgb_plan_set_option": (S, [_vp, _i32, C.c_int64]),
        "tgb_plan_bind": (S, [_vp, C.POINTER(_vp), C.POINTER(_vp)]),
        "tgb_plan_buffers": (S, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
        "tgb_stats": (S, [_vp, _vp]),
        "tgb_ternarize_pack": (S, [_vp, _u64, _vp]),
        "tgb_encode": (S, [_vp, _u64, _vp]),
        "tgb_share_scalers": (S, [_vp, _vp, _vp]),
        "tgb_sync": (S, [_vp, _vp, _vp]),
        "tgb_decode_average": (S, [_vp, _vp, _i32, _vp]),
        "tgb_step": (S, [_vp, _vp, _u64, _vp]),
        "tgb_step_host": (S, [_vp, _vp, _u64, C.POINTER(_vp), C.POINTER(_vp), _vp]),
        "tgb_check": (S, [_vp, C.POINTER(Error)]),
        "tgb_plan_code_stats": (S, [_vp, C.POINTER(_u64), C.POINTER(_u64)]),
        "tgb_plan_enable_code_stats": (S, [_vp, _i32]),
        "tgb_plan_enable_timing": (S, [_vp, _i32]),
        "tgb_plan_read_timing": (S, [_vp, C.POINTER(KernelTime), _i32, C.POINTER(_i32)]),
        "tgb_plan_attach_peers": (S, [_vp, _vp]),
        "tgb_plan_attach_local": (S, [C.POINTER(_vp), _i32]),
        "tgb_local_step": (S, [C.POINTER(_vp), _i32, C.POINTER(_u64), C.POINTER(_vp)]),
        "tgb_traffic_for_layers": (S, [C.POINTER(LayerDesc), C.POINTER(C.c_char_p), _i32,
                                       C.POINTER(CodecParams), _i32, C.POINTER(Traffic)]),
        "tgb_plan_traffic": (S, [_vp, C.POINTER(Traffic)]),
        "tgb_plan_audit": (S, [_vp]),
        "tgb_plan_last_buffers": (S, [_vp, C.POINTER(_vp), C.POINTER(_vp)]),
        "tgb_optimizer_apply": (S, [C.POINTER(Optimizer), _u64, C.c_double, _i32,
                                    C.POINTER(_u64), C.POINTER(_vp), C.POINTER(_vp),
                                    C.POINTER(_vp), C.POINTER(_vp), _vp]),
        "tgb_plan_bind_optimizer": (S, [_vp, C.POINTER(Optimizer), C.POINTER(_vp),
                                        C.POINTER(_vp), C.POINTER(_vp)]),
        "tgb_step_apply": (S, [_vp, _vp, _u64, C.c_double, _vp]),
        "tgb_last_error_message": (C.c_char_p, []),
        "tgb_plan_set_names": (S, [_vp, C.POINTER(C.c_char_p)]),
        "tgb_plan_push_frame_size": (S, [_vp, C.POINTER(_u64)]),
        "tgb_plan_serialize_push": (S, [_vp, _u64, _vp, _vp]),
        "tgb_plan_decode_pull": (S, [_vp, _vp, _u64, C.POINTER(_u64), _vp]),
        "tgb_comm_unique_id": (S, [C.c_char_p]),
        "tgb_comm_init": (S, [C.c_char_p, _i32, _i32, C.POINTER(_vp)]),
        "tgb_comm_destroy": (None, [_vp]),
        "tgb_layer_scaler": (S, [_vp, _u64, _vp, _vp]),
        "tgb_layer_clip": (S, [_vp, _u64, C.c_float, _vp, _vp, _vp]),
        "tgb_layer_ternarize": (S, [_vp, _u64, C.c_float, _u64, _u64, _u64, _u64, _u64, _vp,
                                    _vp]),
        "tgb_layer_decode": (S, [_vp, _u64, C.c_float, _vp, _vp]),
        "tgb_layer_average": (S, [_i32, C.POINTER(_vp), _vp, _u64, _i32, _vp, _vp]),
        "tgb_layer_average_raw": (S, [_i32, C.POINTER(_vp), _u64, _vp, _vp]),
        "tgb_layer_histogram": (S, [_vp, _u64, C.c_uint32, _vp, _vp, _vp]),
        "tgb_rng_bits": (S, [_u64, _u64, _u64, _u64, _u64, _u64, _vp, _vp]),
        "tgb_layer_check": (S, [_vp, C.POINTER(Error)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libtgb.so (building it first when the CUDA toolchain is present)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if build_if_missing and (not os.path.exists(path) or _build.needs_build()):
            if os.path.exists(_build.NVCC):
                _build.build()
        if not os.path.exists(path):
            raise RuntimeError(f"libtgb.so not built ({path}); run __graft_entry__.build()")
        L = C.CDLL(path)
        _declare(L)
        _lib = L
        return L


class TgbError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {load().tgb_status_string(status).decode()} ({status})")


def check(status: int, what: str) -> None:
    if status != TGB_OK:
        raise TgbError(status, what)


def require_device() -> None:
    if load().tgb_device_count() < 1:
        raise RuntimeError("terngrad_b200 needs a CUDA (sm_100a) device; there is no CPU path")
