"""CPU checks of the drop-in boundary: libphx.so loads without a GPU, exports
every symbol include/phx.h declares, and fails loudly (no CPU fallback) when
no device is present."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2509_26475_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    with open(os.path.join(ROOT, "include", "phx.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"\b(phx_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    lib = C.CDLL(P.lib_path())
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(P.ABI_SYMBOLS)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    rp = np.array([0, 1], dtype=np.int64)
    with pytest.raises(P.CudaError):
        P.CsrOperator(1, rp, np.array([0], dtype=np.int32), np.array([1.0]))


def test_invalid_csr_rejected_before_device():
    rp = np.array([0, 2, 1], dtype=np.int64)  # not monotone
    with pytest.raises(ValueError, match="row_ptr not monotone"):
        P.CsrOperator(2, rp, np.array([0, 1], dtype=np.int32), np.array([1.0, 2.0]))
    rp = np.array([0, 1], dtype=np.int64)
    with pytest.raises(ValueError, match="column index out of range"):
        P.CsrOperator(1, rp, np.array([3], dtype=np.int32), np.array([1.0]))
    with pytest.raises(ValueError, match="non-finite"):
        P.CsrOperator(1, rp, np.array([0], dtype=np.int32), np.array([np.nan]))
