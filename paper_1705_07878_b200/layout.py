"""Push-buffer layout of one worker (mirrors tgb_plan_create in csrc/capi.cu).

Blocks follow EncodedGradient::blocks (codec.hpp:70-76, built by encode_step
:218-236): a ternary tensor is one block (PerTensor / Global) or ceil(n/k)
buckets (FixedSize; an empty tensor is still one empty block); a passthrough
tensor is one raw-fp32 block.

    [scaler slot per ternary block, f32][pad to 256 B]
    [block regions in order, each at a 16-B aligned offset:
       ternary: ceil(n/4) packed code bytes, passthrough: 4n raw bytes][pad to 256 B]

Every rank's push buffer has the same layout, so the allgathered buffer is N
push buffers back to back and worker w's region of block b sits at
w*push_bytes + region_offset[b]. Pure host logic (no device), used by the
CPU/gloo tests and by tools that parse a gathered buffer.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

ALIGN_CODES = 16
ALIGN_PUSH = 256
PER_TENSOR, GLOBAL, FIXED_SIZE = 0, 1, 2


def _up(x: int, a: int) -> int:
    return (x + a - 1) // a * a


@dataclass
class Block:
    layer: int
    offset: int          # first element inside the layer (ternarize rng_base)
    n: int
    slot: int            # scaler slot, -1 for passthrough
    region_offset: int
    passthrough: bool

    @property
    def nbytes(self) -> int:
        return 4 * self.n if self.passthrough else (self.n + 3) // 4


@dataclass
class PushLayout:
    ns: List[int]
    blocks: List[Block]
    n_slots: int
    codes_offset: int
    push_bytes: int
    code_bytes: int

    @property
    def n_layers(self) -> int:
        return len(self.ns)

    @property
    def code_offsets(self) -> List[int]:
        """region offset of each layer's first block"""
        first = {}
        for b in self.blocks:
            first.setdefault(b.layer, b.region_offset)
        return [first[l] for l in range(len(self.ns))]


def push_layout(ns: Sequence[int], passthrough: Optional[Sequence[bool]] = None,
                bucketing: int = PER_TENSOR, bucket_size: int = 0) -> PushLayout:
    ns = [int(n) for n in ns]
    pt = [bool(x) for x in passthrough] if passthrough is not None else [False] * len(ns)
    spans = []  # (layer, offset, n, passthrough)
    for l, n in enumerate(ns):
        if pt[l] or bucketing != FIXED_SIZE or n == 0:
            spans.append((l, 0, n, pt[l]))
        else:
            spans.extend((l, off, min(bucket_size, n - off), False)
                         for off in range(0, n, bucket_size))
    n_slots = sum(1 for s in spans if not s[3])
    codes_offset = _up(4 * n_slots, ALIGN_PUSH)
    off, slot, code_bytes, blocks = codes_offset, 0, 0, []
    for l, o, n, p in spans:
        b = Block(l, o, n, -1 if p else slot, off, p)
        slot += 0 if p else 1
        code_bytes += 0 if p else (n + 3) // 4
        off += _up(b.nbytes, ALIGN_CODES)
        blocks.append(b)
    return PushLayout(ns, blocks, n_slots, codes_offset, _up(off, ALIGN_PUSH), code_bytes)


def pack_push(layout: PushLayout, scalers: Sequence[float], regions: Sequence[bytes]) -> bytearray:
    """Assemble one push buffer from the ternary-block scalers and every
    block's region bytes (codes, or raw float32 bytes for passthrough)."""
    import struct

    buf = bytearray(layout.push_bytes)
    for i, s in enumerate(scalers):
        buf[4 * i:4 * i + 4] = struct.pack("<f", s)
    for b, r in zip(layout.blocks, regions):
        buf[b.region_offset:b.region_offset + len(r)] = bytes(r)
    return buf


def unpack_gathered(layout: PushLayout, gathered: bytes, n_workers: int):
    """-> (scalers[w][slot], regions[w][block]) from N push buffers back to back."""
    import struct

    P = layout.push_bytes
    sc, rs = [], []
    for w in range(n_workers):
        base = w * P
        sc.append([struct.unpack_from("<f", gathered, base + 4 * i)[0]
                   for i in range(layout.n_slots)])
        rs.append([bytes(gathered[base + b.region_offset:base + b.region_offset + b.nbytes])
                   for b in layout.blocks])
    return sc, rs
