"""Optimizer mirror (optimizer.hpp): learning-rate schedules (host arithmetic, as
in the reference) and OptimizerState::apply on the device (tgb_optimizer_apply),
bit-identical to the reference's float/double operation order."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from enum import IntEnum
from typing import List, Optional, Sequence, Union

import torch

from . import _lib
from ._lib import check, load
from .codec import GradTensor, _dev, _stream


class ScheduleKind(IntEnum):
    Constant = 0
    Polynomial = 1
    Staircase = 2


@dataclass
class LrSchedule:
    """optimizer.hpp:15-55"""

    kind: ScheduleKind = ScheduleKind.Constant
    base: float = 0.1
    power: float = 0.5
    max_iter: int = 1
    factor: float = 0.1
    step: int = 1

    @staticmethod
    def constant(base: float) -> "LrSchedule":
        return LrSchedule(ScheduleKind.Constant, base)

    @staticmethod
    def polynomial(base: float, power: float, max_iter: int) -> "LrSchedule":
        return LrSchedule(ScheduleKind.Polynomial, base, power=power, max_iter=max_iter)

    @staticmethod
    def staircase(base: float, factor: float, step: int) -> "LrSchedule":
        return LrSchedule(ScheduleKind.Staircase, base, factor=factor, step=step)

    def lr(self, t: int) -> float:
        if self.kind == ScheduleKind.Polynomial:
            tc = min(t, self.max_iter)
            return self.base * math.pow(1.0 - tc / self.max_iter, self.power)
        if self.kind == ScheduleKind.Staircase:
            return self.base * math.pow(self.factor, float(t // self.step))
        return self.base


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
