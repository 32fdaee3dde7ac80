"""The C-ABI library (the product) loads on a CPU-only host, exports every entry point
include/tsb.h declares, and refuses to run without an sm_100 GPU (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from paper_2505_05356_b200 import _abi

HAS_GPU = os.path.exists("/dev/nvidia0")


def declared_functions():
    text = _abi.HEADER_PATH.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tsb_\w+)\s*\(", text)))


def test_header_symbols_exported_and_bound():
    L = _abi.lib()
    names = declared_functions()
    assert len(names) >= 40
    for n in names:
        assert hasattr(L, n), f"{n} declared in tsb.h but not exported by libtsb.so"
        assert n in _abi.SIGNATURES, f"{n} has no ctypes signature"
    assert L.tsb_abi_version() == 3


def test_library_is_sm100a_code():
    data = _abi.LIB_PATH.read_bytes()
    assert b"sm_100a" in data or b"sm_100" in data


@pytest.mark.skipif(HAS_GPU, reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    import paper_2505_05356_b200 as tsb
    with pytest.raises(tsb.TsbError) as e:
        tsb.Context(0)
    assert e.value.code == _abi.TSB_ERR_CUDA


def test_invalid_arguments_are_errors():
    L = _abi.lib()
    out = C.c_void_p()
    assert L.tsb_ctx_create(0, None) == _abi.TSB_ERR_INVALID
    assert L.tsb_scene_create(None, None, C.byref(out)) == _abi.TSB_ERR_INVALID
    assert b"null" in L.tsb_last_error()
    assert L.tsb_pass_prepare(None, None, None, None, None) == _abi.TSB_ERR_INVALID
