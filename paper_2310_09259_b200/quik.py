"""Host-side mirror of the reference's C++ layer API (namespace quik), running on
the B200 kernels through the C ABI (include/quik_b200.h).

Reference-facing functions keep the reference's names, argument meaning and
error behaviour (runtime.hpp, packed.hpp, quantizer.hpp, calibration.hpp):
host arrays in, host arrays out, ValueError for std::invalid_argument,
IndexError for std::out_of_range, NumericalError for quik::NumericalError.

`QuikLinear` is the device-resident hot path: weights repacked once, torch CUDA
tensors in and out, asynchronous on the current stream.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import FormatError, NumericalError  # noqa: F401  (re-export)


# --------------------------------------------------------------------------- types


class PipelineVariant(enum.IntEnum):
    """reference: runtime.hpp:31. All three are bit-identical."""
    V1Unfused = 0
    V2FusedQuant = 1
    V3FusedEpilogue = 2


def row_bytes(cols: int, bits: int) -> int:
    return (cols + 1) // 2 if bits == 4 else cols


@dataclass
class PackedIntMatrix:
    """reference: packed.hpp:17-36 (i4p: low nibble = even column, stored = v+8)."""
    rows: int
    cols: int
    bits: int
    data: np.ndarray  # uint8 [rows * row_bytes]

    def row_bytes(self) -> int:
        return row_bytes(self.cols, self.bits)

    def get(self, r: int, c: int) -> int:
        if self.bits == 8:
            return int(self.data[r * self.cols + c].astype(np.int8))
        b = int(self.data[r * self.row_bytes() + c // 2])
        return ((b & 0xF) if c % 2 == 0 else (b >> 4)) - 8


def pack_values(values: np.ndarray, rows: int, cols: int, bits: int) -> PackedIntMatrix:
    """reference: pack_values / pack_int4 / pack_int8 (packed.cpp:30-66), same errors."""
    if bits not in (4, 8):
        raise ValueError("pack_values: bits must be 4 or 8")
    v = np.asarray(values, dtype=np.int64).reshape(-1)
    if v.size != rows * cols:
        raise ValueError(f"pack: expected {rows * cols} values, got {v.size}")
    lo, hi = (-8, 7) if bits == 4 else (-128, 127)
    bad = np.nonzero((v < lo) | (v > hi))[0]
    if bad.size:
        i = int(bad[0])
        raise IndexError(f"pack: value {int(v[i])} at row {i // cols}, col {i % cols} outside [{lo}, {hi}]")
    v = v.reshape(rows, cols)
    if bits == 8:
        return PackedIntMatrix(rows, cols, 8, v.astype(np.int8).view(np.uint8).reshape(-1).copy())
    rb = row_bytes(cols, 4)
    biased = (v + 8).astype(np.uint8)
    out = np.zeros((rows, rb), dtype=np.uint8)
    out[:, : (cols + 1) // 2] |= biased[:, 0::2]
    out[:, : cols // 2] |= (biased[:, 1::2] << 4).astype(np.uint8)
    return PackedIntMatrix(rows, cols, 4, out.reshape(-1))


def unpack_values(m: PackedIntMatrix) -> np.ndarray:
    """reference: unpack_values (packed.cpp:86-91) -> int8 [rows][cols]."""
    if m.bits == 8:
        return m.data.view(np.int8).reshape(m.rows, m.cols).copy()
    b = m.data.reshape(m.rows, m.row_bytes())
    out = np.empty((m.rows, m.cols), dtype=np.int8)
    out[:, 0::2] = (b[:, : (m.cols + 1) // 2] & 0xF).astype(np.int8) - 8
    out[:, 1::2] = (b[:, : m.cols // 2] >> 4).astype(np.int8) - 8
    return out


@dataclass
class OutlierSet:
    """reference: calibration.hpp:37-48; from_indices calibration.cpp:69-91."""
    feature_count: int
    indices: np.ndarray      # int64, sorted ascending
    permutation: np.ndarray  # int64 [feature_count]: non-outliers ascending, then outliers

    @staticmethod
    def from_indices(feature_count: int, indices) -> "OutlierSet":
        idx = np.sort(np.asarray(indices, dtype=np.int64).reshape(-1))
        if idx.size and (idx[0] < 0 or idx[-1] >= feature_count):
            bad = int(idx[0] if idx[0] < 0 else idx[-1])
            raise ValueError(f"OutlierSet: index {bad} outside feature range")
        if idx.size > 1 and np.any(idx[1:] == idx[:-1]):
            raise ValueError(f"OutlierSet: duplicate index {int(idx[1:][idx[1:] == idx[:-1]][0])}")
        mask = np.ones(feature_count, dtype=bool)
        mask[idx] = False
        perm = np.concatenate([np.nonzero(mask)[0].astype(np.int64), idx])
        return OutlierSet(feature_count, idx, perm)

    @staticmethod
    def none(feature_count: int) -> "OutlierSet":
        return OutlierSet.from_indices(feature_count, [])

    def outlier_count(self) -> int:
        return int(self.indices.size)

    def base_count(self) -> int:
        return self.feature_count - self.outlier_count()


@dataclass
class QuantizedWeights:
    """reference: quantizer.hpp:48-58 (permuted column order, outliers at the tail)."""
    base: PackedIntMatrix
    scales: np.ndarray           # f32 [out]
    outlier_weights: np.ndarray  # f32 [out][n_outlier]
    wreduced: np.ndarray         # f32 [out]
    mask: Optional[np.ndarray] = None

    def bits(self) -> int:
        return self.base.bits

    def out_features(self) -> int:
        return self.base.rows

    def base_features(self) -> int:
        return self.base.cols


@dataclass
class QuikLinearLayer:
    """reference: runtime.hpp:33-44 (Quik mode)."""
    weights: QuantizedWeights
    outliers: OutlierSet
    bias: Optional[np.ndarray] = None
    act_bits: int = 4

    def in_features(self) -> int:
        return self.outliers.feature_count

    def out_features(self) -> int:
        return self.weights.out_features()

    def validate(self) -> None:
        """reference: QuikLinearLayer::validate (runtime.cpp:150-167)."""
        ow = np.asarray(self.weights.outlier_weights)
        if self.outliers.outlier_count() != (ow.shape[1] if ow.ndim == 2 else 0):
            raise ValueError(f"layer: outlier index count {self.outliers.outlier_count()} != outlier weight columns")
        if self.outliers.base_count() != self.weights.base_features():
            raise ValueError("layer: base column count mismatch")
        if self.bias is not None and len(self.bias) != self.out_features():
            raise ValueError("layer: bias length != out_features")
        if self.act_bits != self.weights.bits():
            raise ValueError("layer: activation bits must match weight bits in quik mode")
        if self.act_bits not in (4, 8):
            raise ValueError("activation bits must be 4 or 8")


@dataclass
class ActQuantResult:
    """reference: runtime.hpp:18-23."""
    packed: PackedIntMatrix
    scale: np.ndarray
    zero: np.ndarray
    half_range: int = 8


@dataclass
class StageTimes:
    """reference: runtime.hpp:72-80 (milliseconds, CUDA events on the device)."""
    split_ms: float = 0.0
    quantize_ms: float = 0.0
    int_matmul_ms: float = 0.0
    fp_matmul_ms: float = 0.0
    dequantize_ms: float = 0.0
    add_ms: float = 0.0
    quantize_fused: bool = False
    dequantize_fused: bool = False

    def total_ms(self) -> float:
        return self.split_ms + self.quantize_ms + self.int_matmul_ms + self.fp_matmul_ms + self.dequantize_ms + self.add_ms


# --------------------------------------------------------------------------- device plumbing


def _torch():
    import torch  # plumbing only: device memory, streams

    if not torch.cuda.is_available():
        raise _lib.QuikCudaError("no CUDA device visible: the QUIK B200 path has no CPU fallback")
    return torch


class Context:
    """Owns a quik_ctx_t (scratch + error flag) for one device."""

    def __init__(self, device: int = 0):
        self._lib = _lib.load()
        self.device = device
        h = C.c_void_p()
        _lib.check(self._lib.quik_ctx_create(device, C.byref(h)))
        self.handle = h

    def sync(self, stream) -> None:
        _lib.check(self._lib.quik_ctx_sync(self.handle, C.c_void_p(stream)))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.quik_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_ctx_lock = threading.Lock()
_ctxs: dict = {}


def context(device: Optional[int] = None) -> Context:
    torch = _torch()
    dev = torch.cuda.current_device() if device is None else device
    key = (threading.get_ident(), dev)
    with _ctx_lock:
        c = _ctxs.get(key)
        if c is None:
            c = _ctxs[key] = Context(dev)
        return c


def _stream_ptr(torch, device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t) -> C.c_void_p:
    return C.c_void_p(t.data_ptr() if t is not None and t.numel() else None)


def _dev(torch, a: np.ndarray, device: int):
    return torch.from_numpy(np.ascontiguousarray(a)).to(f"cuda:{device}")


WEIGHT_MODES = {"speed": _lib.QUIK_WEIGHTS_SPEED, "int4": _lib.QUIK_WEIGHTS_INT4}


def _host_desc(layer: QuikLinearLayer, sparse: Optional[bool] = None, row_begin: int = 0, row_end: int = 0,
               weights: str = "speed"):
    """-> (WeightsDesc over host copies, the copies to keep alive)."""
    w = layer.weights
    n_out = layer.outliers.outlier_count()
    keep = dict(
        base=np.ascontiguousarray(w.base.data, dtype=np.uint8),
        scales=np.ascontiguousarray(w.scales, dtype=np.float32),
        wreduced=np.ascontiguousarray(w.wreduced, dtype=np.float32),
        ow=np.ascontiguousarray(np.asarray(w.outlier_weights, dtype=np.float32).reshape(-1)
                                if n_out and w.out_features() else np.zeros(1, np.float32)),
        idx=np.ascontiguousarray(layer.outliers.indices, dtype=np.int64),
        bias=None if layer.bias is None else np.ascontiguousarray(layer.bias, dtype=np.float32),
    )
    d = _lib.WeightsDesc(
        in_features=layer.in_features(), out_features=w.out_features(), bits=w.bits(), act_bits=layer.act_bits,
        base=keep["base"].ctypes.data if keep["base"].size else None,
        scales=keep["scales"].ctypes.data, wreduced=keep["wreduced"].ctypes.data,
        outlier_weights=keep["ow"].ctypes.data, outlier_indices=keep["idx"].ctypes.data if keep["idx"].size else None,
        n_outlier=n_out, bias=None if keep["bias"] is None else keep["bias"].ctypes.data,
        row_begin=row_begin, row_end=row_end,
        sparsity=int(bool(w.mask is not None if sparse is None else sparse)), weight_mode=WEIGHT_MODES[weights])
    return d, keep


class QuikLinear:
    """Device-resident QUIK linear layer (the hot path).

    Construction uploads the reference-format weights once (quik_layer_create:
    i4p/i8 -> device GEMM layout, outliers -> f16). forward() runs K1 + the fused
    tcgen05 kernel on the current CUDA stream. `row_begin/row_end` select an
    output-row shard (multi-GPU column sharding)."""

    def __init__(self, layer: QuikLinearLayer, device: Optional[int] = None, row_begin: int = 0, row_end: int = 0,
                 sparse: Optional[bool] = None, weights: str = "speed"):
        """sparse: request the 2:4 sparse GEMM (default: when the weights carry a
        SparsityMask, i.e. come from sparsegpt_joint, quantizer.cpp:299-337).
        weights: device copy of 4-bit dense weights, "speed" (INT8 for the prefill GEMM +
        INT4 for decode) or "int4" (the INT4 copy only: QUIK's memory footprint)."""
        if weights not in WEIGHT_MODES:
            raise ValueError(f"weights must be one of {sorted(WEIGHT_MODES)}")
        torch = _torch()
        layer.validate()
        self._lib = _lib.load()
        self.ctx = context(device)
        self.device = self.ctx.device
        w = layer.weights
        self.in_features = layer.in_features()
        self.n_outlier = layer.outliers.outlier_count()
        self.bits = w.bits()
        self._keep = dict(
            base=np.ascontiguousarray(w.base.data, dtype=np.uint8),
            scales=np.ascontiguousarray(w.scales, dtype=np.float32),
            wreduced=np.ascontiguousarray(w.wreduced, dtype=np.float32),
            ow=np.ascontiguousarray(np.asarray(w.outlier_weights, dtype=np.float32).reshape(-1)
                                    if self.n_outlier and w.out_features() else np.zeros(1, np.float32)),
            idx=np.ascontiguousarray(layer.outliers.indices, dtype=np.int64),
            bias=None if layer.bias is None else np.ascontiguousarray(layer.bias, dtype=np.float32),
        )
        k = self._keep
        d = _lib.WeightsDesc(
            in_features=self.in_features, out_features=w.out_features(), bits=self.bits, act_bits=layer.act_bits,
            base=k["base"].ctypes.data if k["base"].size else None,
            scales=k["scales"].ctypes.data, wreduced=k["wreduced"].ctypes.data,
            outlier_weights=k["ow"].ctypes.data, outlier_indices=k["idx"].ctypes.data if k["idx"].size else None,
            n_outlier=self.n_outlier, bias=None if k["bias"] is None else k["bias"].ctypes.data,
            row_begin=row_begin, row_end=row_end,
            sparsity=int(bool(w.mask is not None if sparse is None else sparse)), weight_mode=WEIGHT_MODES[weights])
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._lib.quik_layer_create(self.ctx.handle, C.byref(d), C.byref(h)))
        self.handle = h
        self._keep = None  # host copies no longer needed
        of = C.c_int64()
        self._lib.quik_layer_info(h, None, C.byref(of), None, None)
        self.out_features = of.value

    @classmethod
    def from_device(cls, outliers: OutlierSet, base, scales, wreduced, outlier_weights, bits: int, bias=None,
                    row_begin: int = 0, row_end: int = 0, sparse: bool = False, weights: str = "speed") -> "QuikLinear":
        """Builds the layer straight from device tensors in the reference formats
        (e.g. the output of rtn_quantize_weights_device) without a host round trip."""
        torch = _torch()
        self = cls.__new__(cls)
        self._lib = _lib.load()
        self.ctx = context(base.device.index)
        self.device = self.ctx.device
        self.in_features = outliers.feature_count
        self.n_outlier = outliers.outlier_count()
        self.bits = bits
        idx = np.ascontiguousarray(outliers.indices, dtype=np.int64)
        ow = outlier_weights.contiguous() if self.n_outlier else None
        d = _lib.WeightsDesc(
            in_features=self.in_features, out_features=scales.numel(), bits=bits, act_bits=bits,
            base=base.data_ptr(), scales=scales.data_ptr(), wreduced=wreduced.data_ptr(),
            outlier_weights=None if ow is None else ow.data_ptr(),
            outlier_indices=idx.ctypes.data if idx.size else None, n_outlier=self.n_outlier,
            bias=None if bias is None else bias.data_ptr(), row_begin=row_begin, row_end=row_end,
            sparsity=int(sparse), weight_mode=WEIGHT_MODES[weights])
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            torch.cuda.current_stream().synchronize()
            _lib.check(self._lib.quik_layer_create(self.ctx.handle, C.byref(d), C.byref(h)))
        self.handle = h
        of = C.c_int64()
        self._lib.quik_layer_info(h, None, C.byref(of), None, None)
        self.out_features = of.value
        return self

    @classmethod
    def gated(cls, up: QuikLinearLayer, gate: QuikLinearLayer, device: Optional[int] = None, row_begin: int = 0,
              row_end: int = 0, weights: str = "speed") -> "QuikLinear":
        """Gated MLP projection h = silu(gate(x)) * up(x) (reference forward_model with
        gated_mlp_ops, runtime.cpp:320-392) as ONE layer: shared quantizer, one GEMM
        whose epilogue forms silu(gate) * up (C ABI quik_layer_create_gated)."""
        torch = _torch()
        up.validate()
        gate.validate()
        self = cls.__new__(cls)
        self._lib = _lib.load()
        self.ctx = context(device)
        self.device = self.ctx.device
        du, ku = _host_desc(up, row_begin=row_begin, row_end=row_end, weights=weights)
        dg, kg = _host_desc(gate, row_begin=row_begin, row_end=row_end, weights=weights)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._lib.quik_layer_create_gated(self.ctx.handle, C.byref(du), C.byref(dg), C.byref(h)))
        self.handle = h
        inf, of, no, bits = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        self._lib.quik_layer_info(h, C.byref(inf), C.byref(of), C.byref(no), C.byref(bits))
        self.in_features, self.out_features, self.n_outlier, self.bits = inf.value, of.value, no.value, bits.value
        return self

    @classmethod
    def from_bundle(cls, path, device: Optional[int] = None, row_begin: int = 0, row_end: int = 0) -> "QuikLinear":
        """Bundle -> device GEMM layout in one call (C ABI quik_layer_load_bundle, SURVEY.md
        §8f.1); `row_begin/row_end` load only an output-row shard. A bundle with a
        sparsity mask (sparsegpt_joint) gets the 2:4 sparse GEMM."""
        torch = _torch()
        self = cls.__new__(cls)
        self._lib = _lib.load()
        self.ctx = context(device)
        self.device = self.ctx.device
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(self._lib.quik_layer_load_bundle(self.ctx.handle, str(path).encode(), row_begin, row_end,
                                                        C.byref(h)))
        self.handle = h
        inf, of, no, bits = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        self._lib.quik_layer_info(h, C.byref(inf), C.byref(of), C.byref(no), C.byref(bits))
        self.in_features, self.out_features, self.n_outlier, self.bits = inf.value, of.value, no.value, bits.value
        return self

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.quik_layer_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def device_bytes(self) -> int:
        """Device memory this layer holds (C ABI quik_layer_device_bytes)."""
        return int(self._lib.quik_layer_device_bytes(self.handle))

    @property
    def is_sparse(self) -> bool:
        """True when the layer runs the 2:4 sparse tcgen05 GEMM."""
        return bool(self._lib.quik_layer_is_sparse(self.handle))

    @staticmethod
    def launches(variant: PipelineVariant = PipelineVariant.V3FusedEpilogue) -> int:
        return int(_lib.load().quik_linear_forward_launches(int(variant)))

    def forward(self, x, out=None, out_dtype=None, variant: PipelineVariant = PipelineVariant.V3FusedEpilogue,
                mid_event=None):
        """x: CUDA tensor [M][in_features] f16/f32 -> [M][out_features] (f16 default).
        mid_event: optional torch.cuda.Event recorded between the quantizer and the
        GEMM kernel (per-kernel timing)."""
        torch = _torch()
        if x.dim() != 2 or x.shape[1] != self.in_features:
            raise ValueError(f"quik_matmul: input has {x.shape[-1]} features, layer expects {self.in_features}")
        if x.dtype not in (torch.float16, torch.float32):
            raise ValueError("quik_matmul: input must be float16 or float32")
        x = x.contiguous()
        M = x.shape[0]
        out = self._check_out(torch, x, out, out_dtype, "quik_matmul")
        ydt = _lib.QUIK_F16 if out.dtype == torch.float16 else _lib.QUIK_F32
        xdt = _lib.QUIK_F16 if x.dtype == torch.float16 else _lib.QUIK_F32
        _lib.check(self._lib.quik_linear_forward_ex(
            self._ctx_handle(), self.handle, _ptr(x), xdt, M, _ptr(out), ydt, out.stride(0), int(variant),
            C.c_void_p(_stream_ptr(torch, x.device)), C.c_void_p(mid_event.cuda_event if mid_event else None)))
        return out

    def _ctx_handle(self):
        """The calling thread's context on this layer's device (scratch is per context)."""
        return context(self.device).handle

    def _check_out(self, torch, x, out, out_dtype, what):
        """Allocates or validates the output: f16 / f32, row-major, >= M rows and
        out_features columns, on the layer's device (as x)."""
        M = x.shape[0]
        if x.device.type != "cuda" or x.device.index != self.device:
            raise ValueError(f"{what}: input must live on cuda:{self.device}")
        if out is None:
            dt = out_dtype or torch.float16
            if dt not in (torch.float16, torch.float32):
                raise ValueError(f"{what}: output dtype must be float16 or float32")
            return torch.empty((M, self.out_features), dtype=dt, device=x.device)
        if out.dtype not in (torch.float16, torch.float32):
            raise ValueError(f"{what}: output dtype must be float16 or float32, got {out.dtype}")
        if out.device != x.device:
            raise ValueError(f"{what}: output on {out.device}, input on {x.device}")
        if out.dim() != 2 or out.shape[0] < M or out.shape[1] < self.out_features:
            raise ValueError(f"{what}: output must be at least [{M}][{self.out_features}], got {tuple(out.shape)}")
        if out.stride(1) != 1 or out.stride(0) < self.out_features:
            raise ValueError(f"{what}: output must be row-major with pitch >= out_features")
        return out

    def reserve(self, max_tokens: int) -> None:
        """Sizes this thread's context scratch for forwards of up to max_tokens (C ABI
        quik_ctx_reserve) so that forwards can be captured into a CUDA graph."""
        _lib.check(self._lib.quik_ctx_reserve(self._ctx_handle(), self.handle, int(max_tokens)))

    def check_numerics(self) -> None:
        """Waits for the current stream and raises NumericalError if a forward since the
        last check saw a non-finite activation (reference runtime.cpp:52)."""
        torch = _torch()
        _lib.check(self._lib.quik_ctx_sync(self._ctx_handle(), C.c_void_p(_stream_ptr(torch, self.device))))

    __call__ = forward

    def forward_sharded(self, x, outs, col_offset: int):
        """Shard forward with the all-gather fused into the epilogue (C ABI
        quik_linear_forward_sharded): this layer's f16 output columns land at
        `col_offset` of every tensor in `outs` ([M][N_total] f16; outs[0] local, the
        others e.g. peer-GPU tensors with peer access enabled)."""
        torch = _torch()
        x = x.contiguous()
        M = x.shape[0]
        ldy = outs[0].stride(0)
        for o in outs:
            if o.dtype != torch.float16 or o.stride(1) != 1 or o.stride(0) != ldy or o.shape[0] != M:
                raise ValueError("sharded outputs must be row-major f16 [M][N] with one pitch")
        arr = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
        xdt = _lib.QUIK_F16 if x.dtype == torch.float16 else _lib.QUIK_F32
        _lib.check(self._lib.quik_linear_forward_sharded(
            self._ctx_handle(), self.handle, _ptr(x), xdt, M, arr, len(outs), ldy, col_offset,
            C.c_void_p(_stream_ptr(torch, x.device))))
        return outs

    def forward_sharded_ptrs(self, x, dests, ldy: int, col_offset: int):
        """forward_sharded with raw device pointers as destinations (e.g. peer outputs
        opened through CUDA IPC, sharded.FusedAllGatherOutput); row pitch ldy elements."""
        torch = _torch()
        x = x.contiguous()
        arr = (C.c_void_p * len(dests))(*dests)
        xdt = _lib.QUIK_F16 if x.dtype == torch.float16 else _lib.QUIK_F32
        _lib.check(self._lib.quik_linear_forward_sharded(
            self._ctx_handle(), self.handle, _ptr(x), xdt, x.shape[0], arr, len(dests), ldy, col_offset,
            C.c_void_p(_stream_ptr(torch, x.device))))

    def weight_only(self, x, out=None, out_dtype=None):
        """LayerMode::WeightOnly (reference weight_only_forward, runtime.cpp:115-136):
        activations stay floating point, y = (bias + x_o W_o^T) + x_b (q * scale)^T.
        x: CUDA tensor [M][in_features] f16/f32 -> [M][out_features] (f16 default).
        Asynchronous on the current stream (C ABI quik_linear_forward_weight_only)."""
        torch = _torch()
        if x.dim() != 2 or x.shape[1] != self.in_features:
            raise ValueError(f"weight_only_forward: input has {x.shape[-1]} features, layer expects {self.in_features}")
        if x.dtype not in (torch.float16, torch.float32):
            raise ValueError("weight_only_forward: input must be float16 or float32")
        x = x.contiguous()
        M = x.shape[0]
        out = self._check_out(torch, x, out, out_dtype, "weight_only_forward")
        ydt = _lib.QUIK_F16 if out.dtype == torch.float16 else _lib.QUIK_F32
        xdt = _lib.QUIK_F16 if x.dtype == torch.float16 else _lib.QUIK_F32
        _lib.check(self._lib.quik_linear_forward_weight_only(
            self._ctx_handle(), self.handle, _ptr(x), xdt, M, _ptr(out), ydt, out.stride(0),
            C.c_void_p(_stream_ptr(torch, x.device))))
        return out

    def quantize_gemm_layout(self, x):
        """Diagnostics: K1 as the hot path runs it (C ABI quik_quantize_activations_gemm).
        Returns (codes int8 [M][kpad], scale [M], zero [M], x_outlier f16 [M][opad])."""
        torch = _torch()
        M = x.shape[0]
        kp, op = C.c_int64(), C.c_int64()
        _lib.check(self._lib.quik_layer_layout(self.handle, C.byref(kp), C.byref(op)))
        kpad, opad = kp.value, op.value
        dev = x.device
        codes = torch.empty((M, kpad), dtype=torch.int8, device=dev)
        scale = torch.empty(M, dtype=torch.float32, device=dev)
        zero = torch.empty(M, dtype=torch.float32, device=dev)
        xo = torch.empty((M, opad), dtype=torch.float16, device=dev)
        xdt = _lib.QUIK_F16 if x.dtype == torch.float16 else _lib.QUIK_F32
        _lib.check(self._lib.quik_quantize_activations_gemm(
            self._ctx_handle(), self.handle, _ptr(x.contiguous()), xdt, M, _ptr(codes), _ptr(scale), _ptr(zero), _ptr(xo),
            C.c_void_p(_stream_ptr(torch, dev))))
        _lib.check(self._lib.quik_ctx_sync(self._ctx_handle(), C.c_void_p(_stream_ptr(torch, dev))))
        return codes, scale, zero, xo

    def forward_host(self, x, out, chunk_tokens: int = 0):
        """Host (CPU, ideally pinned) x [M][in_features] -> host out [M][out_features],
        chunked so the H2D copy, the kernels and the D2H copy overlap
        (C ABI quik_linear_forward_host). Asynchronous on the current stream."""
        torch = _torch()
        if x.dim() != 2 or x.shape[1] != self.in_features:
            raise ValueError(f"quik_matmul: input has {x.shape[-1]} features, layer expects {self.in_features}")
        if x.device.type != "cpu" or out.device.type != "cpu":
            raise ValueError("forward_host: x and out must be host tensors")
        if x.dtype not in (torch.float16, torch.float32) or out.dtype not in (torch.float16, torch.float32):
            raise ValueError("forward_host: float16 or float32 tensors expected")
        if not (x.is_contiguous() and out.is_contiguous()) or tuple(out.shape) != (x.shape[0], self.out_features):
            raise ValueError("forward_host: contiguous x [M][in] and out [M][out] expected")
        xdt = _lib.QUIK_F16 if x.dtype == torch.float16 else _lib.QUIK_F32
        ydt = _lib.QUIK_F16 if out.dtype == torch.float16 else _lib.QUIK_F32
        dev = torch.device("cuda", self.device)
        _lib.check(self._lib.quik_linear_forward_host(
            self._ctx_handle(), self.handle, C.c_void_p(x.data_ptr()), xdt, x.shape[0], C.c_void_p(out.data_ptr()), ydt,
            int(chunk_tokens), C.c_void_p(_stream_ptr(torch, dev))))
        return out


# --------------------------------------------------------------------------- reference-facing API


def _outlier_handle(torch, outliers: OutlierSet, bits: int, device: int) -> QuikLinear:
    """A weight-less layer carrying only the outlier permutation tables."""
    K = outliers.feature_count
    kb = outliers.base_count()
    w = QuantizedWeights(PackedIntMatrix(0, kb, bits, np.zeros(0, np.uint8)), np.zeros(0, np.float32),
                         np.zeros((0, outliers.outlier_count()), np.float32), np.zeros(0, np.float32))
    return QuikLinear(QuikLinearLayer(w, outliers, None, bits), device)


def quantize_activations_fused(x: np.ndarray, outliers: OutlierSet, bits: int):
    """reference: quantize_activations_fused (runtime.hpp:55-56) -> (ActQuantResult, x_outlier)."""
    if bits not in (4, 8):
        raise ValueError("activation bits must be 4 or 8")
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2 or x.shape[1] != outliers.feature_count:
        raise ValueError("fused quantization: input features do not match outlier set")
    torch = _torch()
    ctx = context()
    M = x.shape[0]
    kb = outliers.base_count()
    L = _outlier_handle(torch, outliers, bits, ctx.device)
    dx = _dev(torch, x, ctx.device)
    packed = torch.empty(max(M * row_bytes(kb, bits), 1), dtype=torch.uint8, device=dx.device)
    scale = torch.empty(max(M, 1), dtype=torch.float32, device=dx.device)
    zero = torch.empty(max(M, 1), dtype=torch.float32, device=dx.device)
    xo = torch.empty(max(M * outliers.outlier_count(), 1), dtype=torch.float32, device=dx.device)
    s = _stream_ptr(torch, dx.device)
    _lib.check(L._lib.quik_ctx_clear_error(ctx.handle, C.c_void_p(s)))  # report this call's errors only
    _lib.check(L._lib.quik_quantize_activations_fused(ctx.handle, L.handle, _ptr(dx), _lib.QUIK_F32, M,
                                                      _ptr(packed), _ptr(scale), _ptr(zero), _ptr(xo), C.c_void_p(s)))
    ctx.sync(s)
    pk = packed.cpu().numpy()[: M * row_bytes(kb, bits)]
    res = ActQuantResult(PackedIntMatrix(M, kb, bits, pk), scale.cpu().numpy()[:M], zero.cpu().numpy()[:M],
                         1 << (bits - 1))
    return res, xo.cpu().numpy()[: M * outliers.outlier_count()].reshape(M, outliers.outlier_count())


def quantize_activations(x_base: np.ndarray, bits: int) -> ActQuantResult:
    """reference: quantize_activations (runtime.hpp:51, runtime.cpp:188-197)."""
    if bits not in (4, 8):
        raise ValueError("activation bits must be 4 or 8")
    x = np.ascontiguousarray(x_base, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError("quantize_activations: expected a 2-D matrix")
    torch = _torch()
    ctx = context()
    M, K = x.shape
    dx = _dev(torch, x, ctx.device)
    packed = torch.empty(max(M * row_bytes(K, bits), 1), dtype=torch.uint8, device=dx.device)
    scale = torch.empty(max(M, 1), dtype=torch.float32, device=dx.device)
    zero = torch.empty(max(M, 1), dtype=torch.float32, device=dx.device)
    s = _stream_ptr(torch, dx.device)
    _lib.check(_lib.load().quik_ctx_clear_error(ctx.handle, C.c_void_p(s)))
    _lib.check(_lib.load().quik_quantize_activations(ctx.handle, _ptr(dx), _lib.QUIK_F32, M, K, bits, _ptr(packed),
                                                     _ptr(scale), _ptr(zero), C.c_void_p(s)))
    ctx.sync(s)
    return ActQuantResult(PackedIntMatrix(M, K, bits, packed.cpu().numpy()[: M * row_bytes(K, bits)]),
                          scale.cpu().numpy()[:M], zero.cpu().numpy()[:M], 1 << (bits - 1))


def int_matmul(x: PackedIntMatrix, w: PackedIntMatrix) -> np.ndarray:
    """reference: int_matmul (packed.hpp:58, packed.cpp:93-132) -> int32 [x.rows][w.rows]."""
    torch = _torch()
    ctx = context()
    dxp = _dev(torch, x.data if x.data.size else np.zeros(1, np.uint8), ctx.device)
    dwp = _dev(torch, w.data if w.data.size else np.zeros(1, np.uint8), ctx.device)
    out = torch.empty(max(x.rows * w.rows, 1), dtype=torch.int32, device=dxp.device)
    s = _stream_ptr(torch, dxp.device)
    _lib.check(_lib.load().quik_int_matmul(ctx.handle, _ptr(dxp), x.rows, x.cols, x.bits, _ptr(dwp), w.rows, w.cols,
                                           w.bits, _ptr(out), C.c_void_p(s)))
    ctx.sync(s)
    return out.cpu().numpy()[: x.rows * w.rows].reshape(x.rows, w.rows)


def dequantize_epilogue(acc: np.ndarray, a: ActQuantResult, weight_scales, wreduced) -> np.ndarray:
    """reference: dequantize_epilogue (runtime.hpp:66-68, runtime.cpp:222-244)."""
    acc = np.ascontiguousarray(acc, dtype=np.int32)
    M, N = acc.shape
    if M != len(a.scale):
        raise ValueError("dequantize_epilogue: token count mismatch")
    if len(weight_scales) != N or len(wreduced) != N:
        raise ValueError("dequantize_epilogue: per-row vector length mismatch")
    torch = _torch()
    ctx = context()
    d = lambda v: _dev(torch, np.ascontiguousarray(v, dtype=np.float32), ctx.device)  # noqa: E731
    dacc = _dev(torch, acc, ctx.device)
    sa, za, sw, wr = d(a.scale), d(a.zero), d(weight_scales), d(wreduced)
    out = torch.empty((M, N), dtype=torch.float32, device=dacc.device)
    s = _stream_ptr(torch, dacc.device)
    _lib.check(_lib.load().quik_dequantize_epilogue(ctx.handle, _ptr(dacc), M, N, _ptr(sa), _ptr(za), a.half_range,
                                                    _ptr(sw), _ptr(wr), _ptr(out), C.c_void_p(s)))
    ctx.sync(s)
    return out.cpu().numpy()


def _bundle_tensor(lib, h, name):
    """-> numpy copy of one bundle tensor (f32 -> float32, i8 / i4p -> raw uint8 bytes), or None."""
    data, dt, nd = C.c_void_p(), C.c_int(), C.c_int()
    shape = (C.c_int64 * 4)()
    if lib.quik_bundle_tensor(h, name.encode(), C.byref(data), C.byref(dt), shape, C.byref(nd)) != _lib.QUIK_OK:
        return None, None, None
    shp = tuple(int(shape[i]) for i in range(nd.value))
    if not data.value or (shp and int(np.prod(shp)) == 0):
        return (np.zeros(shp, np.float32) if dt.value == 0 else np.zeros(0, np.uint8)), dt.value, shp
    if dt.value == 0:
        n = int(np.prod(shp)) if shp else 0
        arr = np.ctypeslib.as_array((C.c_float * max(n, 1)).from_address(data.value))[:n].copy().reshape(shp)
    else:
        rows = shp[0] if len(shp) == 2 else 1
        nbytes = rows * ((shp[-1] + 1) // 2 if dt.value == 2 else shp[-1]) if shp else 0
        arr = np.ctypeslib.as_array((C.c_uint8 * max(nbytes, 1)).from_address(data.value))[:nbytes].copy()
    return arr, dt.value, shp


class QuikGatedMLP:
    """The reference's gated MLP block (gated_mlp_ops, runtime.cpp:380-388:
    down(silu(gate(x)) * up(x))) on the device: the fused gated projection (one K1 +
    one GEMM) followed by the down projection (its own K1 + GEMM)."""

    def __init__(self, up: QuikLinearLayer, gate: QuikLinearLayer, down: QuikLinearLayer,
                 device: Optional[int] = None, weights: str = "speed"):
        """weights: "speed" or "int4" for both projections (QuikLinear)."""
        self.proj = QuikLinear.gated(up, gate, device, weights=weights)
        self.down = QuikLinear(down, device, weights=weights)
        if self.down.in_features != self.proj.out_features:
            raise ValueError("gated MLP: down projection input != up/gate output features")

    def forward(self, x, out=None, out_dtype=None, hidden_dtype=None, fused: bool = True):
        """hidden_dtype: dtype of h between the projections (default: x's dtype).
        With an f16 hidden state the block runs through quik_gated_mlp_forward: the
        gated GEMM's epilogue also reduces the down projection's per-token min / max, so
        the down quantizer skips its reduction pass (bit-identical to the two forwards;
        fused=False runs them separately)."""
        return self.forward_with_hidden(x, out, out_dtype, hidden_dtype, fused)[0]

    def forward_with_hidden(self, x, out=None, out_dtype=None, hidden_dtype=None, fused: bool = True,
                            hidden=None):
        """forward() that also returns the hidden state h: (y, h). hidden: optional f16
        [M][>= F] row-major buffer for h (any row pitch >= F; the fused path)."""
        torch = _torch()
        hd = hidden_dtype or x.dtype
        if hd != torch.float16 or not fused:
            h = self.proj(x, out_dtype=hd)
            return self.down(h, out=out, out_dtype=out_dtype), h
        if x.dim() != 2 or x.shape[1] != self.proj.in_features:
            raise ValueError(f"quik_matmul: input has {x.shape[-1]} features, layer expects {self.proj.in_features}")
        if x.dtype not in (torch.float16, torch.float32):
            raise ValueError("quik_matmul: input must be float16 or float32")
        x = x.contiguous()
        M = x.shape[0]
        h = self.proj._check_out(torch, x, hidden, torch.float16, "gated MLP")
        if h.dtype != torch.float16:
            raise ValueError("gated MLP: the hidden state must be float16")
        out = self.down._check_out(torch, x, out, out_dtype, "gated MLP")
        ydt = _lib.QUIK_F16 if out.dtype == torch.float16 else _lib.QUIK_F32
        xdt = _lib.QUIK_F16 if x.dtype == torch.float16 else _lib.QUIK_F32
        _lib.check(self.proj._lib.quik_gated_mlp_forward(
            self.proj._ctx_handle(), self.proj.handle, self.down.handle, _ptr(x), xdt, M, _ptr(h), h.stride(0),
            _ptr(out), ydt, out.stride(0), C.c_void_p(_stream_ptr(torch, x.device))))
        return out, h

    __call__ = forward


def load_layer(path) -> QuikLinearLayer:
    """reference: load_layer (layer_io.hpp, layer_io.cpp:32-74): a layer bundle
    (manifest.json + blobs) -> QuikLinearLayer, host arrays. Malformed bundles raise
    FormatError (C ABI quik_bundle_open, which repeats every reference check)."""
    lib = _lib.load()
    h = C.c_void_p()
    _lib.check(lib.quik_bundle_open(str(path).encode(), C.byref(h)))
    try:
        d = _lib.WeightsDesc()
        _lib.check(lib.quik_bundle_weights(h, C.byref(d)))
        base, bdt, bshape = _bundle_tensor(lib, h, "weight_base")
        scales, _, _ = _bundle_tensor(lib, h, "weight_scales")
        wred, _, _ = _bundle_tensor(lib, h, "wreduced")
        ow, _, _ = _bundle_tensor(lib, h, "outlier_weights")
        bias, _, _ = _bundle_tensor(lib, h, "bias")
        mask, mdt, mshape = _bundle_tensor(lib, h, "sparsity_mask")
        idx = np.ctypeslib.as_array((C.c_int64 * max(d.n_outlier, 1)).from_address(d.outlier_indices or 0)) \
            if d.n_outlier else np.zeros(0, np.int64)
        idx = np.array(idx[: d.n_outlier], dtype=np.int64)
        bits = 4 if bdt == 2 else 8
        weights = QuantizedWeights(PackedIntMatrix(bshape[0], bshape[1], bits, base), scales.reshape(-1),
                                   ow.reshape(bshape[0], -1), wred.reshape(-1),
                                   None if mask is None else mask.reshape(mshape))
        return QuikLinearLayer(weights, OutlierSet.from_indices(int(d.in_features), idx),
                               None if bias is None else bias.reshape(-1), int(d.act_bits))
    finally:
        lib.quik_bundle_close(h)


def rtn_quantize_weights_device(w, outliers: OutlierSet, bits: int, use_clipping: bool = False):
    """reference: rtn_quantize_weights (quantizer.cpp:339-371; use_clipping -> per-row
    clip_search, :266-290), on the device.

    w: CUDA f32 tensor [out][in]. Returns device tensors (base_packed u8
    [out*row_bytes], scales, wreduced, outlier_weights [out][n_outlier])."""
    torch = _torch()
    if bits not in (4, 8):
        raise ValueError("weight bits must be 4 or 8")
    if w.dim() != 2 or w.shape[1] != outliers.feature_count:
        raise ValueError(f"outlier set covers {outliers.feature_count} features, weights have {w.shape[-1]}")
    w = w.contiguous().float()
    ctx = context(w.device.index)
    N, K = w.shape
    kb = outliers.base_count()
    O = outliers.outlier_count()
    base = torch.empty(max(N * row_bytes(kb, bits), 1), dtype=torch.uint8, device=w.device)
    scales = torch.empty(max(N, 1), dtype=torch.float32, device=w.device)
    wred = torch.empty(max(N, 1), dtype=torch.float32, device=w.device)
    ow = torch.empty(max(N * O, 1), dtype=torch.float32, device=w.device)
    idx = np.ascontiguousarray(outliers.indices, dtype=np.int64)
    s = _stream_ptr(torch, w.device)
    _lib.check(_lib.load().quik_rtn_quantize_weights(
        ctx.handle, _ptr(w), N, K, C.c_void_p(idx.ctypes.data if idx.size else None), O, bits, int(use_clipping),
        _ptr(base),
        _ptr(scales), _ptr(wred), _ptr(ow), C.c_void_p(s)))
    return base[: N * row_bytes(kb, bits)], scales[:N], wred[:N], ow[: N * O].view(N, O)


def hessian_device(batches, device: Optional[int] = None):
    """reference: build_hessian / Hessian::accumulate (quantizer.cpp:193-240) on the device:
    the FP64 sum of x x^T over the calibration batches (host or CUDA f32 [T][K]).
    Returns a CUDA float64 tensor [K][K] (before damping)."""
    torch = _torch()
    h = None
    for x in batches:
        xt = torch.as_tensor(x)
        if xt.dtype != torch.float32:
            xt = xt.float()
        xt = xt.contiguous()
        T, K = xt.shape
        ctx = context(device if xt.device.type != "cuda" else xt.device.index)
        if h is None:
            h = torch.zeros((K, K), dtype=torch.float64, device=f"cuda:{ctx.device}")
        if h.shape[0] != K:
            raise ValueError(f"Hessian: batch has {K} features, expected {h.shape[0]}")
        _lib.check(_lib.load().quik_hessian_accumulate(ctx.handle, C.c_void_p(xt.data_ptr()), T, K, _ptr(h)))
    if h is None:
        raise ValueError("build_hessian: no calibration tokens")
    return h


def gptq_quantize_device(w, outliers: OutlierSet, bits: int, hessian_sum, damping_frac: float = 0.01,
                         use_clipping: bool = False, sparse: bool = False,
                         device: Optional[int] = None) -> QuantizedWeights:
    """reference: gptq_quantize (quantizer.cpp:292-297) or, sparse=True,
    sparsegpt_joint (:299-337), computed on the device in FP64. w: f32 [out][in] (numpy
    or torch); hessian_sum: [in][in] f64 sum of x x^T (numpy or torch, e.g.
    hessian_device). Returns host QuantizedWeights (mask set when sparse)."""
    torch = _torch()
    if bits not in (4, 8):
        raise ValueError("weight bits must be 4 or 8")
    wt = torch.as_tensor(w).float().contiguous()
    N, K = wt.shape
    if K != outliers.feature_count:
        raise ValueError(f"outlier set covers {outliers.feature_count} features, weights have {K}")
    ht = torch.as_tensor(hessian_sum, dtype=torch.float64).contiguous()
    if tuple(ht.shape) != (K, K):
        raise ValueError(f"Hessian dim {ht.shape[0]} does not match weight columns {K}")
    ctx = context(device)
    kb = outliers.base_count()
    O = outliers.outlier_count()
    base = np.zeros(max(N * row_bytes(kb, bits), 1), np.uint8)
    scales = np.zeros(max(N, 1), np.float32)
    wred = np.zeros(max(N, 1), np.float32)
    ow = np.zeros(max(N * O, 1), np.float32)
    mask = np.zeros(max(N * kb, 1), np.uint8) if sparse else None
    idx = np.ascontiguousarray(outliers.indices, dtype=np.int64)
    if wt.device.type == "cpu":
        wt = wt.numpy()
        wptr = C.c_void_p(wt.ctypes.data)
    else:
        wptr = C.c_void_p(wt.data_ptr())
    if ht.device.type == "cpu":
        ht = ht.numpy()
        hptr = C.c_void_p(ht.ctypes.data)
    else:
        hptr = C.c_void_p(ht.data_ptr())
    _lib.check(_lib.load().quik_gptq_quantize(
        ctx.handle, wptr, N, K, hptr, C.c_double(damping_frac), C.c_void_p(idx.ctypes.data if idx.size else None), O,
        bits, int(use_clipping), int(sparse), C.c_void_p(base.ctypes.data), C.c_void_p(scales.ctypes.data),
        C.c_void_p(wred.ctypes.data), C.c_void_p(ow.ctypes.data), C.c_void_p(mask.ctypes.data) if sparse else None))
    qw = QuantizedWeights(PackedIntMatrix(N, kb, bits, base[: N * row_bytes(kb, bits)]), scales[:N],
                          ow[: N * O].reshape(N, O), wred[:N])
    if sparse:
        qw.mask = mask[: N * kb].reshape(N, kb)
    return qw


def rtn_quantize_weights(w: np.ndarray, outliers: OutlierSet, bits: int, use_clipping: bool = False) -> QuantizedWeights:
    """reference: rtn_quantize_weights (quantizer.hpp:89-90), bit-exact incl. use_clipping.
    Host f32 [out][in] in, QuantizedWeights (host arrays) out; computed on the GPU."""
    torch = _torch()
    w = np.ascontiguousarray(w, dtype=np.float32)
    if w.ndim != 2 or w.shape[1] != outliers.feature_count:
        raise ValueError(f"outlier set covers {outliers.feature_count} features, weights have {w.shape[-1]}")
    ctx = context()
    dw = _dev(torch, w, ctx.device)
    base, sc, wr, ow = rtn_quantize_weights_device(dw, outliers, bits, use_clipping)
    ctx.sync(_stream_ptr(torch, dw.device))
    N = w.shape[0]
    return QuantizedWeights(PackedIntMatrix(N, outliers.base_count(), bits, base.cpu().numpy()), sc.cpu().numpy(),
                            ow.cpu().numpy(), wr.cpu().numpy())


def quik_matmul(layer: QuikLinearLayer, x: np.ndarray,
                variant: PipelineVariant = PipelineVariant.V3FusedEpilogue,
                times: Optional[StageTimes] = None, out_dtype: str = "float32") -> np.ndarray:
    """reference: quik_matmul (runtime.hpp:85-87): host FP32 in, host FP32 out.

    Uploads the layer on every call like the reference re-reads its weights; keep a
    QuikLinear for repeated calls."""
    layer.validate()
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2 or x.shape[1] != layer.in_features():
        raise ValueError(f"quik_matmul: input has {x.shape[-1]} features, layer expects {layer.in_features()}")
    torch = _torch()
    dev = QuikLinear(layer)
    dx = _dev(torch, x, dev.device)
    dt = torch.float32 if out_dtype == "float32" else torch.float16
    y = torch.empty((x.shape[0], dev.out_features), dtype=dt, device=dx.device)
    s = C.c_void_p(_stream_ptr(torch, dx.device))
    h = dev._ctx_handle()
    _lib.check(dev._lib.quik_ctx_clear_error(h, s))  # report this call's errors only
    ydt = _lib.QUIK_F16 if dt == torch.float16 else _lib.QUIK_F32
    if times is not None:
        # per-stage CUDA-event times, the reference's fused-stage convention (C ABI
        # quik_linear_forward_timed; runtime.cpp:265-315)
        ms = (C.c_double * 6)()
        fl = (C.c_int * 2)()
        _lib.check(dev._lib.quik_linear_forward_timed(h, dev.handle, _ptr(dx), _lib.QUIK_F32, x.shape[0], _ptr(y), ydt,
                                                      dev.out_features, int(variant), s, ms, fl))
        (times.split_ms, times.quantize_ms, times.int_matmul_ms, times.fp_matmul_ms, times.dequantize_ms,
         times.add_ms) = list(ms)
        times.quantize_fused, times.dequantize_fused = bool(fl[0]), bool(fl[1])
    else:
        dev.forward(dx, out=y, variant=variant)
    _lib.check(dev._lib.quik_ctx_sync(h, s))
    return y.float().cpu().numpy()


def split_activations(x: np.ndarray, outliers: OutlierSet):
    """reference: split_activations (runtime.hpp:48, runtime.cpp:169-186) on the device:
    x [M][K] -> (base [M][K_b] in permuted order, outlier columns [M][n_outlier]), f32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2 or x.shape[1] != outliers.feature_count:
        raise ValueError(f"split_activations: input has {x.shape[-1]} features, outlier set covers "
                         f"{outliers.feature_count}")
    torch = _torch()
    ctx = context()
    M = x.shape[0]
    kb, O = outliers.base_count(), outliers.outlier_count()
    L = _outlier_handle(torch, outliers, 4, ctx.device)
    dx = _dev(torch, x, ctx.device)
    base = torch.empty(max(M * kb, 1), dtype=torch.float32, device=dx.device)
    outl = torch.empty(max(M * O, 1), dtype=torch.float32, device=dx.device)
    s = _stream_ptr(torch, dx.device)
    _lib.check(L._lib.quik_split_activations(ctx.handle, L.handle, _ptr(dx), _lib.QUIK_F32, M, _ptr(base), _ptr(outl),
                                             C.c_void_p(s)))
    ctx.sync(s)
    return base.cpu().numpy()[: M * kb].reshape(M, kb), outl.cpu().numpy()[: M * O].reshape(M, O)


def _unpack_device(m: PackedIntMatrix) -> np.ndarray:
    torch = _torch()
    ctx = context()
    n = m.rows * m.cols
    if n == 0:
        return np.zeros((m.rows, m.cols), np.int8)
    dp = _dev(torch, m.data, ctx.device)
    out = torch.empty(n, dtype=torch.int8, device=dp.device)
    s = _stream_ptr(torch, dp.device)
    _lib.check(_lib.load().quik_unpack_values(ctx.handle, _ptr(dp), m.rows, m.cols, m.bits, _ptr(out), C.c_void_p(s)))
    ctx.sync(s)
    return out.cpu().numpy().reshape(m.rows, m.cols)


def unpack_int4(m: PackedIntMatrix) -> np.ndarray:
    """reference: unpack_int4 (packed.hpp:48, packed.cpp:68-84) on the device; ValueError
    (std::invalid_argument) unless m.bits == 4."""
    if m.bits != 4:
        raise ValueError("unpack_int4: matrix is not 4-bit")
    return _unpack_device(m)


def compute_wreduced(q: QuantizedWeights) -> np.ndarray:
    """reference: compute_wreduced (quantizer.hpp:94, quantizer.cpp:373-382) on the device."""
    torch = _torch()
    ctx = context()
    N = q.base.rows
    if N == 0:
        return np.zeros(0, np.float32)
    db = _dev(torch, q.base.data if q.base.data.size else np.zeros(1, np.uint8), ctx.device)
    ds = _dev(torch, np.ascontiguousarray(q.scales, np.float32), ctx.device)
    out = torch.empty(N, dtype=torch.float32, device=db.device)
    s = _stream_ptr(torch, db.device)
    _lib.check(_lib.load().quik_compute_wreduced(ctx.handle, _ptr(db), N, q.base.cols, q.base.bits, _ptr(ds),
                                                 _ptr(out), C.c_void_p(s)))
    ctx.sync(s)
    return out.cpu().numpy()


def dequantize_weights(q: QuantizedWeights, outliers: OutlierSet) -> np.ndarray:
    """reference: dequantize_weights (quantizer.hpp:98, quantizer.cpp:384-403) on the
    device: the de-permuted f32 [out][in] reconstruction."""
    ow = np.asarray(q.outlier_weights, np.float32).reshape(q.base.rows, -1) if q.base.rows else \
        np.zeros((0, outliers.outlier_count()), np.float32)
    if outliers.base_count() != q.base.cols or outliers.outlier_count() != ow.shape[1]:
        raise ValueError("dequantize_weights: outlier set does not match weights")
    torch = _torch()
    ctx = context()
    N, K = q.base.rows, outliers.feature_count
    if N * K == 0:
        return np.zeros((N, K), np.float32)
    db = _dev(torch, q.base.data if q.base.data.size else np.zeros(1, np.uint8), ctx.device)
    ds = _dev(torch, np.ascontiguousarray(q.scales, np.float32), ctx.device)
    dow = _dev(torch, ow if ow.size else np.zeros(1, np.float32), ctx.device)
    out = torch.empty((N, K), dtype=torch.float32, device=db.device)
    idx = np.ascontiguousarray(outliers.indices, np.int64)
    s = _stream_ptr(torch, db.device)
    rb = q.base.row_bytes()
    O = outliers.outlier_count()
    for r0 in range(0, N, 65535):
        nr = min(65535, N - r0)
        _lib.check(_lib.load().quik_dequantize_weights(
            ctx.handle, C.c_void_p(db.data_ptr() + r0 * rb), nr, K, q.base.bits, C.c_void_p(ds.data_ptr() + 4 * r0),
            C.c_void_p(dow.data_ptr() + 4 * r0 * O), C.c_void_p(idx.ctypes.data if idx.size else None), O,
            C.c_void_p(out.data_ptr() + 4 * r0 * K), C.c_void_p(s)))
    ctx.sync(s)
    return out.cpu().numpy()


@dataclass
class BlockOp:
    """reference: BlockOp (runtime.hpp:91-101): value 0 is the model input, op i produces
    value i + 1."""

    class Kind(enum.IntEnum):
        Linear = 0
        Silu = 1
        Multiply = 2
        Add = 3

    kind: "BlockOp.Kind" = 0
    a: int = 0
    b: int = -1
    layer: int = -1


def gated_mlp_ops():
    """reference: gated_mlp_ops (runtime.cpp:373-382), layers {0: up, 1: gate, 2: down}."""
    K = BlockOp.Kind
    return [BlockOp(K.Linear, 0, -1, 0), BlockOp(K.Linear, 0, -1, 1), BlockOp(K.Silu, 2, -1, -1),
            BlockOp(K.Multiply, 3, 1, -1), BlockOp(K.Linear, 4, -1, 2)]


def forward_model_trace(layers, ops, x: np.ndarray):
    """reference: forward_model_trace (runtime.hpp:105-107, runtime.cpp:325-371) with every
    value on the device: Linear -> the QUIK forward of the layer (f32 in/out), Silu /
    Multiply / Add -> quik_elementwise. Returns all values (host f32)."""
    torch = _torch()
    ctx = context()
    x = np.ascontiguousarray(x, np.float32)
    dev_layers = {}
    vals = [_dev(torch, x, ctx.device)]
    s = _stream_ptr(torch, vals[0].device)
    lib = _lib.load()

    def value(i):
        if i < 0 or i >= len(vals):
            raise ValueError(f"forward_model: op references undefined value {i}")
        return vals[i]

    for op in ops:
        k = BlockOp.Kind(op.kind)
        if k == BlockOp.Kind.Linear:
            if op.layer < 0 or op.layer >= len(layers):
                raise ValueError(f"forward_model: op references undefined layer {op.layer}")
            if op.layer not in dev_layers:
                dev_layers[op.layer] = QuikLinear(layers[op.layer], ctx.device)
            vals.append(dev_layers[op.layer](value(op.a), out_dtype=torch.float32))
        elif k == BlockOp.Kind.Silu:
            a = value(op.a)
            out = torch.empty_like(a)
            _lib.check(lib.quik_elementwise(ctx.handle, 0, _ptr(a), None, _ptr(out), a.numel(), C.c_void_p(s)))
            vals.append(out)
        else:
            a, b = value(op.a), value(op.b)
            if a.shape != b.shape:
                raise ValueError(f"forward_model elementwise op: shape mismatch ({a.shape[0]}x{a.shape[1]} vs "
                                 f"{b.shape[0]}x{b.shape[1]})")
            out = torch.empty_like(a)
            _lib.check(lib.quik_elementwise(ctx.handle, 1 if k == BlockOp.Kind.Multiply else 2, _ptr(a), _ptr(b),
                                            _ptr(out), a.numel(), C.c_void_p(s)))
            vals.append(out)
    if len(vals) == 1:
        raise ValueError("forward_model: empty op list")
    ctx.sync(s)
    return [x] + [v.cpu().numpy() for v in vals[1:]]


def forward_model(layers, ops, x: np.ndarray) -> np.ndarray:
    """reference: forward_model (runtime.hpp:103-104)."""
    return forward_model_trace(layers, ops, x)[-1]
