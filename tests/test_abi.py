"""CPU tests of the drop-in boundary: the C-ABI library loads, exports every
symbol include/quik_b200.h declares, and fails loudly (no CPU fallback) when no
sm_100 device is present. No compute calls are made here."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_functions():
    text = (ROOT / "include" / "quik_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(quik_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for required in ("quik_quantize_activations_fused", "quik_quantize_activations", "quik_int_matmul",
                     "quik_dequantize_epilogue", "quik_linear_forward", "quik_layer_create",
                     "quik_rtn_quantize_weights"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2310_09259_b200 import _lib

    lib = C.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.EXPORTED_SYMBOLS) <= set(declared_functions())


def test_abi_version_and_status_strings():
    from paper_2310_09259_b200 import _lib

    lib = _lib.load()
    assert lib.quik_abi_version() == 3
    assert lib.quik_status_string(3) == b"numerical error"
    assert lib.quik_linear_forward_launches(2) == 2


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2310_09259_b200 import _lib

    lib = _lib.load()
    h = C.c_void_p()
    st = lib.quik_ctx_create(0, C.byref(h))
    assert st == _lib.QUIK_ERR_CUDA
    assert b"no CUDA device" in lib.quik_last_error() or b"sm_100" in lib.quik_last_error()
    import paper_2310_09259_b200 as q

    with pytest.raises(_lib.QuikCudaError):
        q.quantize_activations(np.zeros((1, 4), np.float32), 4)


def test_argument_errors_map_to_reference_exceptions():
    """Argument checks happen before any device work, like the reference's throws."""
    from paper_2310_09259_b200 import _lib

    lib = _lib.load()
    # int_matmul bit-width mismatch -> std::invalid_argument (packed.cpp:94-97)
    st = lib.quik_int_matmul(C.c_void_p(1), None, 2, 3, 4, None, 2, 3, 8, None, None)
    assert st == _lib.QUIK_ERR_INVALID_ARGUMENT
    st = lib.quik_set_gemm_tile(3, 7)
    assert st == _lib.QUIK_ERR_INVALID_ARGUMENT
    with pytest.raises(ValueError):
        _lib.check(_lib.QUIK_ERR_INVALID_ARGUMENT)
    with pytest.raises(IndexError):
        _lib.check(_lib.QUIK_ERR_OUT_OF_RANGE)
    with pytest.raises(_lib.NumericalError):
        _lib.check(_lib.QUIK_ERR_NUMERICAL)


def test_sass_contains_tcgen05_and_tma():
    """The shipped kernels are native sm_100a tcgen05/TMA code (UTC*MMA, UTMALDG)."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    from paper_2310_09259_b200 import _lib

    out = subprocess.run([cuobjdump, "-sass", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert re.search(r"UTC\w*MMA", out), "no tcgen05 MMA in SASS"
    assert "UTMALDG" in out and "UTMASTG" in out, "no TMA in SASS"
    assert "LDTM" in out and "STTM" in out
    assert "HMMA" not in out.replace("UTCHMMA", ""), "legacy mma.sync path present"
