"""The drop-in boundary: both product libraries load and export every C symbol
declared in include/*.h (no compute calls here — this runs without a GPU)."""
import ctypes
import os
import re

import pytest

from paper_2605_09735_b200 import kvrail as kv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DECL = re.compile(r"^(?:const\s+)?\w+\s*\*?\s*(kvr_\w+)\s*\(", re.M)


def declared(header: str) -> list[str]:
    with open(os.path.join(ROOT, "include", header)) as f:
        text = f.read()
    return sorted(set(DECL.findall(text)))


@pytest.mark.parametrize("header,lib", [("kvrail_c.h", "libkvrail.so"), ("kvr_cuda.h", "libkvr_cuda.so")])
def test_every_declared_symbol_is_exported(header, lib):
    names = declared(header)
    assert len(names) > 10
    so = ctypes.CDLL(os.path.join(kv.LIB_DIR, lib))
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, f"{lib} lacks {missing}"


def test_errc_names_match_reference_taxonomy():
    lib = kv.native_lib()
    lib.kvr_errc_name.restype = ctypes.c_char_p
    for i, name in enumerate(kv.ERRC_NAMES):
        assert lib.kvr_errc_name(i + 1).decode() == name
    assert lib.kvr_errc_name(kv.KVR_E_CUDA).decode() == "CudaError"


def test_errors_carry_reference_messages():
    p = kv.Pager(kv.PagerConfig(512, 8, 1, 8, 2))
    with pytest.raises(kv.KvrailError) as e:
        p.reserve(99, 1)
    assert e.value.code == "UnknownSession" and str(e.value) == "UnknownSession: session 99"


def test_struct_layouts_match_headers():
    """The ctypes mirrors have exactly the C compiler's struct sizes."""
    lib = kv.native_lib()
    out = (ctypes.c_uint64 * 64)()
    n = ctypes.c_uint64()
    assert lib.kvr_abi_struct_sizes(out, 64, ctypes.byref(n)) == 0
    sizes = list(out)[:n.value]
    mirrors = {0: kv.PagerConfig, 1: kv.TokenRange, 2: kv.ViewEntry, 3: kv.ViewInfo,
               4: kv.ReservedBlock, 5: kv.ArenaStats, 6: kv.WorkCounters, 7: kv.FreeRun,
               8: kv.FrameDelta, 9: kv.StagedSpan, 10: kv.StageNeed, 11: kv.Descriptor,
               12: kv.TransportConfig, 13: kv.Train, 14: kv.StepRecord, 15: kv.Geometry,
               27: kv.MassRun}
    for i, cls in mirrors.items():
        assert ctypes.sizeof(cls) == sizes[i], cls.__name__


def test_no_device_without_gpu_is_a_loud_error():
    if kv.device_count() > 0:
        pytest.skip("a GPU is present")
    g = kv.Geometry()
    g.device = 0
    with pytest.raises(kv.KvrailError):
        kv.Device(g)
