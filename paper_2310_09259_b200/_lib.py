"""ctypes binding of the C ABI in include/quik_b200.h (libquik_b200.so).

The library is built in-tree by paper_2310_09259_b200/build.py. There is no
fallback: if the library is missing or no sm_100 GPU is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libquik_b200.so"

QUIK_OK = 0
QUIK_ERR_INVALID_ARGUMENT = 1
QUIK_ERR_OUT_OF_RANGE = 2
QUIK_ERR_NUMERICAL = 3
QUIK_ERR_CUDA = 4
QUIK_ERR_NCCL = 5
QUIK_ERR_UNSUPPORTED = 6
QUIK_ERR_FORMAT = 7

QUIK_F16 = 0
QUIK_F32 = 1

QUIK_WEIGHTS_SPEED = 0
QUIK_WEIGHTS_INT4 = 1

EXPORTED_SYMBOLS = (
    "quik_last_error", "quik_status_string", "quik_abi_version", "quik_ctx_create", "quik_ctx_destroy",
    "quik_ctx_sync", "quik_layer_create", "quik_layer_destroy", "quik_layer_info",
    "quik_quantize_activations_fused", "quik_quantize_activations", "quik_int_matmul",
    "quik_dequantize_epilogue", "quik_linear_forward", "quik_linear_forward_strided",
    "quik_linear_forward_launches", "quik_linear_forward_ex", "quik_rtn_quantize_weights",
    "quik_set_gemm_tile", "quik_set_probe_mode", "quik_linear_forward_host",
    "quik_quantize_activations_gemm", "quik_layer_is_sparse", "quik_set_gemm_multicast",
    "quik_bundle_open", "quik_bundle_weights",
    "quik_bundle_tensor", "quik_bundle_close", "quik_layer_load_bundle", "quik_layer_create_gated",
    "quik_linear_forward_weight_only", "quik_linear_forward_sharded", "quik_set_int4_decode",
    "quik_gptq_quantize", "quik_hessian_accumulate", "quik_ctx_clear_error", "quik_ctx_reserve", "quik_layer_layout",
    "quik_linear_forward_timed", "quik_split_activations", "quik_unpack_values", "quik_compute_wreduced",
    "quik_dequantize_weights", "quik_elementwise", "quik_ipc_handle_get", "quik_ipc_handle_open",
    "quik_ipc_handle_close", "quik_layer_device_bytes", "quik_gated_mlp_forward",
)


class NumericalError(RuntimeError):
    """reference: quik::NumericalError (matrix.hpp:18-21) — non-finite activations."""


class FormatError(RuntimeError):
    """reference: quik::FormatError (matrix.hpp:12-15) — malformed layer bundle / container."""


class QuikCudaError(RuntimeError):
    """CUDA failure inside the native library (no CPU fallback exists)."""


class IpcHandle(C.Structure):
    """quik_ipc_handle: a cudaIpcMemHandle_t + the pointer's offset in its allocation."""
    _fields_ = [("bytes", C.c_ubyte * 64), ("offset", C.c_int64)]


class WeightsDesc(C.Structure):
    _fields_ = [
        ("in_features", C.c_int64),
        ("out_features", C.c_int64),
        ("bits", C.c_int),
        ("act_bits", C.c_int),
        ("base", C.c_void_p),
        ("scales", C.c_void_p),
        ("wreduced", C.c_void_p),
        ("outlier_weights", C.c_void_p),
        ("outlier_indices", C.c_void_p),
        ("n_outlier", C.c_int64),
        ("bias", C.c_void_p),
        ("row_begin", C.c_int64),
        ("row_end", C.c_int64),
        ("sparsity", C.c_int),
        ("weight_mode", C.c_int),
    ]


_lib = None
_lock = threading.Lock()


def load() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: the QUIK B200 kernels are not built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
        lib = C.CDLL(str(LIB_PATH))
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int
        sig = {
            "quik_last_error": (C.c_char_p, []),
            "quik_status_string": (C.c_char_p, [i32]),
            "quik_abi_version": (i32, []),
            "quik_ctx_create": (i32, [i32, C.POINTER(vp)]),
            "quik_ctx_destroy": (i32, [vp]),
            "quik_ctx_sync": (i32, [vp, vp]),
            "quik_layer_create": (i32, [vp, C.POINTER(WeightsDesc), C.POINTER(vp)]),
            "quik_layer_destroy": (i32, [vp]),
            "quik_layer_info": (i32, [vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i32)]),
            "quik_quantize_activations_fused": (i32, [vp, vp, vp, i32, i64, vp, vp, vp, vp, vp]),
            "quik_quantize_activations": (i32, [vp, vp, i32, i64, i64, i32, vp, vp, vp, vp]),
            "quik_int_matmul": (i32, [vp, vp, i64, i64, i32, vp, i64, i64, i32, vp, vp]),
            "quik_dequantize_epilogue": (i32, [vp, vp, i64, i64, vp, vp, i32, vp, vp, vp, vp]),
            "quik_linear_forward": (i32, [vp, vp, vp, i32, i64, vp, i32, i32, vp]),
            "quik_linear_forward_strided": (i32, [vp, vp, vp, i32, i64, vp, i32, i64, i32, vp]),
            "quik_linear_forward_launches": (i32, [i32]),
            "quik_linear_forward_ex": (i32, [vp, vp, vp, i32, i64, vp, i32, i64, i32, vp, vp]),
            "quik_gated_mlp_forward": (i32, [vp, vp, vp, vp, i32, i64, vp, i64, vp, i32, i64, vp]),
            "quik_rtn_quantize_weights": (i32, [vp, vp, i64, i64, vp, i64, i32, i32, vp, vp, vp, vp, vp]),
            "quik_ctx_clear_error": (i32, [vp, vp]),
            "quik_ctx_reserve": (i32, [vp, vp, i64]),
            "quik_layer_layout": (i32, [vp, C.POINTER(i64), C.POINTER(i64)]),
            "quik_linear_forward_timed": (i32, [vp, vp, vp, i32, i64, vp, i32, i64, i32, vp, vp, vp]),
            "quik_split_activations": (i32, [vp, vp, vp, i32, i64, vp, vp, vp]),
            "quik_unpack_values": (i32, [vp, vp, i64, i64, i32, vp, vp]),
            "quik_compute_wreduced": (i32, [vp, vp, i64, i64, i32, vp, vp, vp]),
            "quik_dequantize_weights": (i32, [vp, vp, i64, i64, i32, vp, vp, vp, i64, vp, vp]),
            "quik_elementwise": (i32, [vp, i32, vp, vp, vp, i64, vp]),
            "quik_ipc_handle_get": (i32, [vp, vp, C.POINTER(IpcHandle)]),
            "quik_ipc_handle_open": (i32, [vp, C.POINTER(IpcHandle), C.POINTER(vp)]),
            "quik_ipc_handle_close": (i32, [vp, vp, C.POINTER(IpcHandle)]),
            "quik_layer_device_bytes": (i64, [vp]),
            "quik_set_gemm_tile": (i32, [i32, i32]),
            "quik_set_probe_mode": (i32, [i32]),
            "quik_linear_forward_host": (i32, [vp, vp, vp, i32, i64, vp, i32, i64, vp]),
            "quik_quantize_activations_gemm": (i32, [vp, vp, vp, i32, i64, vp, vp, vp, vp, vp]),
            "quik_layer_is_sparse": (i32, [vp]),
            "quik_set_gemm_multicast": (i32, [i32]),
            "quik_bundle_open": (i32, [C.c_char_p, C.POINTER(vp)]),
            "quik_bundle_weights": (i32, [vp, C.POINTER(WeightsDesc)]),
            "quik_bundle_tensor": (i32, [vp, C.c_char_p, C.POINTER(vp), C.POINTER(i32), C.POINTER(i64),
                                         C.POINTER(i32)]),
            "quik_bundle_close": (i32, [vp]),
            "quik_layer_load_bundle": (i32, [vp, C.c_char_p, i64, i64, C.POINTER(vp)]),
            "quik_layer_create_gated": (i32, [vp, C.POINTER(WeightsDesc), C.POINTER(WeightsDesc), C.POINTER(vp)]),
            "quik_linear_forward_weight_only": (i32, [vp, vp, vp, i32, i64, vp, i32, i64, vp]),
            "quik_linear_forward_sharded": (i32, [vp, vp, vp, i32, i64, C.POINTER(vp), i32, i64, i64, vp]),
            "quik_set_int4_decode": (i32, [i32]),
            "quik_gptq_quantize": (i32, [vp, vp, i64, i64, vp, C.c_double, vp, i64, i32, i32, i32, vp, vp, vp, vp, vp]),
            "quik_hessian_accumulate": (i32, [vp, vp, i64, i64, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
        return lib


def check(status: int) -> None:
    """Maps a quik_status to the reference's exception types (runtime.cpp / packed.cpp)."""
    if status == QUIK_OK:
        return
    msg = (load().quik_last_error() or b"").decode(errors="replace")
    if status == QUIK_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # std::invalid_argument
    if status == QUIK_ERR_OUT_OF_RANGE:
        raise IndexError(msg)  # std::out_of_range
    if status == QUIK_ERR_NUMERICAL:
        raise NumericalError(msg)
    if status == QUIK_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == QUIK_ERR_FORMAT:
        raise FormatError(msg)
    raise QuikCudaError(msg)
