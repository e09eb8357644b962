"""C-ABI boundary checks that need no GPU (-m "not gpu").

* libtgb.so loads and exports every symbol include/tgb/terngrad_b200.h declares;
* host-only helpers (fnv1a64) agree with the oracle;
* every compute entry point refuses to run without a device (no CPU fallback);
* the Python plan layout restatement agrees with the header's documented layout.
"""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_1705_07878_b200 import _lib
from paper_1705_07878_b200.layout import push_layout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tgb", "terngrad_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\w[\w\s\*]*?\b(tgb_\w+)\s*\(", src, re.M)))


def test_header_declares_expected_symbols():
    assert header_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_header_symbol():
    L = _lib.load()
    for s in header_symbols():
        assert hasattr(L, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.lib_path()], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (tgb_\w+)", out))
    assert set(header_symbols()) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.lib_path()], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_fnv_host_matches_oracle(restated):
    L = _lib.load()
    for name in ["", "fc.weight", "classifier.0.weight", "features.28.bias"]:
        b = name.encode()
        assert L.tgb_fnv1a64(b, len(b)) == restated.fnv1a64(name)


def test_version_and_status_strings():
    L = _lib.load()
    assert b"sm_100a" in L.tgb_version()
    assert L.tgb_status_string(_lib.TGB_ERR_CODEC) == b"codec error"


def test_no_cpu_fallback_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("host has a GPU")
    L = _lib.load()
    assert L.tgb_device_count() == 0
    d = (_lib.LayerDesc * 1)(_lib.LayerDesc(16, 1, 0, 0))
    p = _lib.CodecParams(2.5, 1, 0, 1, 0, 42, 0, 0)
    h = C.c_void_p()
    st = L.tgb_plan_create(d, 1, C.byref(p), 0, 1, C.byref(h))
    assert st == _lib.TGB_ERR_CUDA and not h.value
    out = (C.c_uint32 * 4)()
    assert L.tgb_rng_bits(1, 2, 3, 4, 0, 4, C.cast(out, C.c_void_p), None) == _lib.TGB_ERR_CUDA
    from paper_1705_07878_b200 import codec

    with pytest.raises(RuntimeError, match="no CPU path"):
        codec._dev()


def test_plan_argument_validation():
    L = _lib.load()
    d = (_lib.LayerDesc * 1)(_lib.LayerDesc(16, 1, 0, 0))
    h = C.c_void_p()
    bad = _lib.CodecParams(0.0, 1, 0, 1, 0, 42, 0, 0)   # clip factor must be positive
    assert L.tgb_plan_create(d, 1, C.byref(bad), 0, 1, C.byref(h)) == _lib.TGB_ERR_INVALID_ARGUMENT
    fixed = _lib.CodecParams(2.5, 1, 2, 1, 0, 42, 0, 0)  # FixedSize with k = 0
    assert L.tgb_plan_create(d, 1, C.byref(fixed), 0, 1, C.byref(h)) == \
        _lib.TGB_ERR_INVALID_ARGUMENT
    ok = _lib.CodecParams(2.5, 1, 0, 1, 0, 42, 0, 0)
    assert L.tgb_plan_create(d, 1, C.byref(ok), 0, 0, C.byref(h)) == _lib.TGB_ERR_INVALID_ARGUMENT
    assert L.tgb_plan_create(d, 1, C.byref(ok), 0, 65, C.byref(h)) == _lib.TGB_ERR_INVALID_ARGUMENT


def test_push_layout():
    lay = push_layout([5, 0, 16, 1000003])
    assert lay.codes_offset == 256
    assert lay.code_offsets == [256, 272, 272, 288]
    assert lay.code_bytes == 2 + 0 + 4 + 250001
    assert lay.push_bytes % 256 == 0 and lay.push_bytes >= 288 + 250001
    assert all(o % 16 == 0 for o in lay.code_offsets)


def test_push_layout_blocks():
    # FixedSize k = 6 over [13, 0, 3] with layer 2 passthrough:
    # blocks (0,0,6) (0,6,6) (0,12,1) (1,0,0) | raw (2,0,3)
    lay = push_layout([13, 0, 3], [False, False, True], bucketing=2, bucket_size=6)
    assert [(b.layer, b.offset, b.n, b.slot) for b in lay.blocks] == \
        [(0, 0, 6, 0), (0, 6, 6, 1), (0, 12, 1, 2), (1, 0, 0, 3), (2, 0, 3, -1)]
    assert lay.n_slots == 4 and lay.codes_offset == 256
    assert [b.region_offset for b in lay.blocks] == [256, 272, 288, 304, 304]
    assert lay.blocks[-1].nbytes == 12 and lay.code_bytes == 2 + 2 + 1 + 0
    assert lay.push_bytes == 512


def test_attach_local_and_timing_argument_validation():
    """tgb_plan_attach_local / tgb_plan_enable_timing / tgb_plan_read_timing reject bad
    arguments before touching a device (no plan exists without a GPU)."""
    L = _lib.load()
    assert L.tgb_plan_attach_local(None, 2) == _lib.TGB_ERR_INVALID_ARGUMENT
    arr = (C.c_void_p * 2)(None, None)
    assert L.tgb_plan_attach_local(arr, 2) == _lib.TGB_ERR_INVALID_ARGUMENT
    assert L.tgb_plan_attach_local(arr, 0) == _lib.TGB_ERR_INVALID_ARGUMENT
    assert L.tgb_plan_attach_local(arr, 9) == _lib.TGB_ERR_INVALID_ARGUMENT
    assert L.tgb_plan_enable_timing(None, 4) == _lib.TGB_ERR_INVALID_ARGUMENT
    n = C.c_int32()
    assert L.tgb_plan_read_timing(None, None, 0, C.byref(n)) == _lib.TGB_ERR_INVALID_ARGUMENT
    assert C.sizeof(_lib.KernelTime) == 40
