"""B200-native TernGrad gradient synchronisation (arXiv 1705.07878).

Public surface mirrors the reference's namespace ``terngrad``
(codec.hpp / rng.hpp / tensor.hpp) plus the worker sync entry point.
All compute runs in libtgb.so (sm_100a); there is no CPU fallback.
"""
from .codec import (Bucketing, CodecConfig, CodecError, EncodedGradient, EncodeResult,
                    GradTensor, HistogramBin, PassthroughBlock, RngStream, ShareMode,
                    ProtocolError, TernaryBlock, average, clip, clip_bound, decode, encode_step,
                    fnv1a64, histogram, scaler, share_scalers, ternarize)
from .optimizer import OptimizerConfig, OptimizerRule, OptimizerState
from .plan import Comm, LocalCluster, Plan, SyncWorker, TrafficStats, aligned_flat
from . import layersets

__all__ = [
    "Bucketing", "CodecConfig", "CodecError", "EncodedGradient", "EncodeResult", "GradTensor",
    "HistogramBin", "histogram", "PassthroughBlock", "ProtocolError", "RngStream", "ShareMode", "TernaryBlock", "average", "clip",
    "clip_bound", "decode", "encode_step", "fnv1a64", "scaler", "share_scalers", "ternarize",
    "Comm", "LocalCluster", "Plan", "SyncWorker", "TrafficStats", "aligned_flat", "layersets",
    "OptimizerConfig", "OptimizerRule", "OptimizerState",
]
