"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
public headers declare, and refuses to compute without a GPU (there is no CPU
fallback)."""
import ctypes
import os
import re

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2305_09781_b200", "libspectree_b200.so")


def declared_symbols():
    syms = set()
    for name in os.listdir(os.path.join(ROOT, "include")):
        if name.endswith(".h"):
            src = open(os.path.join(ROOT, "include", name)).read()
            syms |= set(re.findall(r"\b(st_[a-z0-9_]+)\s*\(", src))
    return syms


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        pytest.skip("library not built (run __graft_entry__.build())")
    return ctypes.CDLL(LIB)


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 10
    missing = [s for s in sorted(syms) if not hasattr(lib, s)]
    assert not missing, f"declared but not exported: {missing}"


def test_python_binding_covers_exports(lib):
    from paper_2305_09781_b200 import _capi
    assert declared_symbols() <= set(_capi.SIGNATURES), \
        sorted(declared_symbols() - set(_capi.SIGNATURES))


def test_abi_version(lib):
    assert lib.st_abi_version() == 5


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the CPU-only host behaviour")
def test_no_cpu_fallback(lib):
    from paper_2305_09781_b200 import _capi
    L = _capi.lib()
    assert L.st_device_count() == 0
    st = L.st_build_masks(None, None, 1, 1, 1, None, None)
    assert st == 100  # ST_ERR_NO_DEVICE
    assert b"no CPU fallback" in L.st_last_error_message()
