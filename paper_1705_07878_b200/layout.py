"""Push-buffer layout of one worker (mirrors tgb_plan_create in csrc/capi.cu).

    [scaler slot per layer, f32][pad to 256 B][layer l codes at a 16-B aligned
    offset, ceil(n_l/4) bytes each][pad to 256 B]

Every rank's push buffer has the same layout, so the allgathered buffer is N
push buffers back to back and worker w's codes of layer l sit at
w*push_bytes + code_offset[l]. Pure host logic (no device), used by the
CPU/gloo tests and by tools that parse a gathered buffer.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence

ALIGN_CODES = 16
ALIGN_PUSH = 256
CHUNK = 16384  # elements per device work item (tgb_device.cuh kChunk)


def _up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


@dataclass
class PushLayout:
    ns: List[int]
    codes_offset: int
    code_offsets: List[int]
    push_bytes: int
    code_bytes: int

    @property
    def n_layers(self) -> int:
        return len(self.ns)

    def n_chunks(self) -> int:
        return sum((n + CHUNK - 1) // CHUNK for n in self.ns)


def push_layout(ns: Sequence[int]) -> PushLayout:
    ns = [int(n) for n in ns]
    codes_offset = _up(4 * len(ns), ALIGN_PUSH)
    off, offs, code_bytes = codes_offset, [], 0
    for n in ns:
        offs.append(off)
        nb = (n + 3) // 4
        code_bytes += nb
        off += _up(nb, ALIGN_CODES)
    return PushLayout(ns, codes_offset, offs, _up(off, ALIGN_PUSH), code_bytes)


def pack_push(layout: PushLayout, scalers: Sequence[float], codes: Sequence[bytes]) -> bytearray:
    """Assemble one push buffer from per-layer scalers and packed codes."""
    import struct

    buf = bytearray(layout.push_bytes)
    for l, s in enumerate(scalers):
        buf[4 * l:4 * l + 4] = struct.pack("<f", s)
    for l, c in enumerate(codes):
        o = layout.code_offsets[l]
        buf[o:o + len(c)] = bytes(c)
    return buf


def unpack_gathered(layout: PushLayout, gathered: bytes, n_workers: int):
    """-> (scalers[w][l], codes[w][l]) from N push buffers back to back."""
    import struct

    P = layout.push_bytes
    sc, cs = [], []
    for w in range(n_workers):
        base = w * P
        sc.append([struct.unpack_from("<f", gathered, base + 4 * l)[0]
                   for l in range(layout.n_layers)])
        cs.append([bytes(gathered[base + layout.code_offsets[l]:
                                  base + layout.code_offsets[l] + (n + 3) // 4])
                   for l, n in enumerate(layout.ns)])
    return sc, cs
