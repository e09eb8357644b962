"""Optimizer mirror (optimizer.hpp:60-125): OptimizerState::apply on the device
(tgb_optimizer_apply, and fused into the decode by tgb_step_apply), bit-identical to
the reference's float/double operation order. (Learning-rate schedules,
optimizer.hpp:15-55, are outside the hot path: callers pass the step's rate.)"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import IntEnum
from typing import List, Optional, Sequence, Union

import torch

from . import _lib
from ._lib import check, load
from .codec import GradTensor, _dev, _stream


class OptimizerRule(IntEnum):
    Vanilla = 0
    Momentum = 1
    Adam = 2


@dataclass
class OptimizerConfig:
    """optimizer.hpp:60-67"""

    rule: OptimizerRule = OptimizerRule.Vanilla
    momentum: float = 0.9
    beta1: float = 0.9
    beta2: float = 0.999
    epsilon: float = 1e-8
    weight_decay: float = 0.0

    def c(self) -> _lib.Optimizer:
        return _lib.Optimizer(int(self.rule), 0, self.momentum, self.beta1, self.beta2,
                              self.epsilon, self.weight_decay)

    def n_state(self) -> int:
        return {OptimizerRule.Vanilla: 0, OptimizerRule.Momentum: 1, OptimizerRule.Adam: 2}[
            self.rule]


def _vals(x: Union[GradTensor, torch.Tensor]) -> torch.Tensor:
    return x.values if isinstance(x, GradTensor) else x


class OptimizerState:
    """optimizer.hpp:70-125: per-worker state, applied identically at every worker."""

    def __init__(self, cfg: OptimizerConfig):
        self.cfg = cfg
        self._step = 0
        self.buffers: List[torch.Tensor] = []
        self.buffers2: List[torch.Tensor] = []

    def step_count(self) -> int:
        return self._step

    def apply(self, params: Sequence[Union[GradTensor, torch.Tensor]],
              avg_grad: Sequence[Union[GradTensor, torch.Tensor]], rate: float) -> None:
        if len(params) != len(avg_grad):
            raise ValueError("optimizer: param/grad count mismatch")
        ws = [_vals(p) for p in params]
        gs = [_vals(g).reshape(-1).contiguous() for g in avg_grad]
        for p, w, g in zip(params, ws, gs):
            if w.numel() != g.numel():
                name = p.name if isinstance(p, GradTensor) else "?"
                raise ValueError("optimizer: shape mismatch on " + name)
        if not self.buffers:
            n = self.cfg.n_state()
            self.buffers = [torch.zeros_like(w) for w in ws] if n >= 1 else []
            self.buffers2 = [torch.zeros_like(w) for w in ws] if n >= 2 else []
        self._step += 1
        nl = len(ws)
        dev = ws[0].device if nl else _dev()
        P = C.c_void_p * max(nl, 1)
        ns = (C.c_uint64 * max(nl, 1))(*[w.numel() for w in ws])
        s1 = P(*[b.data_ptr() for b in self.buffers]) if self.buffers else None
        s2 = P(*[b.data_ptr() for b in self.buffers2]) if self.buffers2 else None
        opt = self.cfg.c()
        check(load().tgb_optimizer_apply(C.byref(opt), self._step, float(rate), nl, ns,
                                         P(*[w.data_ptr() for w in ws]),
                                         P(*[g.data_ptr() for g in gs]), s1, s2, _stream(dev)),
              "tgb_optimizer_apply")
