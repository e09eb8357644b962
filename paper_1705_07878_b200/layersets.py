"""Synthetic gradient sets of the BASELINE configs.

Names and shapes are pinned in layersets.json (generated once by
tools/gen_layersets.py from torchvision); names key the Philox streams.
"""
from __future__ import annotations

import json
import os
from typing import List, Tuple

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "layersets.json")
_cache = None


def _load():
    global _cache
    if _cache is None:
        with open(_PATH) as f:
            _cache = json.load(f)["sets"]
    return _cache


def names() -> List[str]:
    return sorted(_load().keys())


def get(name: str) -> List[Tuple[str, List[int]]]:
    """[(tensor name, shape)] in canonical parameter order."""
    return [(n, list(s)) for n, s in _load()[name]]


def numel(shape) -> int:
    if len(shape) == 0:
        return 0
    p = 1
    for d in shape:
        p *= int(d)
    return p


def total(name: str) -> int:
    return sum(numel(s) for _, s in get(name))
