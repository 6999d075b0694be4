"""ctypes access to the two CPU checkers (TEST INFRASTRUCTURE ONLY):

  Oracle  oracle/build/libquik_oracle.so  — plain-C restatement (oracle/quik_oracle.c)
  Ref     oracle/_ref/libquik_ref.so      — the reference's own sources + C shim

Both expose the same methods so tests can parametrize over them.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "build" / "libquik_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libquik_ref.so"


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def row_bytes(cols, bits):
    return (cols + 1) // 2 if bits == 4 else cols


class _Base:
    prefix = ""

    def __init__(self, path: Path):
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (run __graft_entry__.build())")
        self.lib = C.CDLL(str(path))

    def f(self, name):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = C.c_int
        return fn

    # ------------------------------------------------------------- packing
    def pack(self, vals, rows, cols, bits):
        v = np.ascontiguousarray(vals, dtype=np.int8).reshape(-1)
        out = np.zeros(max(rows * row_bytes(cols, bits), 1), np.uint8)
        st = self._pack(v, rows, cols, bits, out)
        return st, out[: rows * row_bytes(cols, bits)]

    def unpack(self, packed, rows, cols, bits):
        out = np.zeros(max(rows * cols, 1), np.int8)
        self._unpack(np.ascontiguousarray(packed, np.uint8), rows, cols, bits, out)
        return out[: rows * cols].reshape(rows, cols)

    def int_matmul(self, xp, t, k, xbits, wp, n, wk=None, wbits=None):
        wk = k if wk is None else wk
        wbits = xbits if wbits is None else wbits
        out = np.zeros(max(t * n, 1), np.int32)
        st = self.f("int_matmul")(_p(np.ascontiguousarray(xp, np.uint8)), C.c_int64(t), C.c_int64(k), xbits,
                                  _p(np.ascontiguousarray(wp, np.uint8)), C.c_int64(n), C.c_int64(wk), wbits, _p(out))
        return st, out[: t * n].reshape(t, n)

    # ------------------------------------------------------------- calibration
    def select_outliers(self, x, k):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros(max(k, 1), np.int64)
        st = self.f("select_outliers")(_p(x), C.c_int64(x.shape[0]), C.c_int64(x.shape[1]), C.c_int64(k), _p(out))
        assert st == 0, st
        return out[:k]

    def permutation(self, features, idx):
        idx = np.ascontiguousarray(idx, np.int64)
        out = np.zeros(max(features, 1), np.int64)
        st = self.f("outlier_permutation")(C.c_int64(features), _p(idx), C.c_int64(idx.size), _p(out))
        return st, out[:features]

    # ------------------------------------------------------------- runtime
    def quantize(self, x_base, bits):
        x = np.ascontiguousarray(x_base, np.float32)
        M, K = x.shape
        packed = np.zeros(max(M * row_bytes(K, bits), 1), np.uint8)
        scale = np.zeros(max(M, 1), np.float32)
        zero = np.zeros(max(M, 1), np.float32)
        st = self.f("quantize_activations")(_p(x), C.c_int64(M), C.c_int64(K), bits, _p(packed), _p(scale), _p(zero))
        return st, packed[: M * row_bytes(K, bits)], scale[:M], zero[:M]

    def dequantize_epilogue(self, acc, sa, za, hr, sw, wr):
        acc = np.ascontiguousarray(acc, np.int32)
        M, N = acc.shape
        out = np.zeros((M, N), np.float32)
        a = [np.ascontiguousarray(v, np.float32) for v in (sa, za, sw, wr)]
        self.f("dequantize_epilogue")(_p(acc), C.c_int64(M), C.c_int64(N), _p(a[0]), _p(a[1]), hr, _p(a[2]),
                                      _p(a[3]), _p(out))
        return out

    def rtn_quantize_weights(self, w, idx, bits, use_clipping=False):
        w = np.ascontiguousarray(w, np.float32)
        N, K = w.shape
        idx = np.ascontiguousarray(idx, np.int64)
        kb = K - idx.size
        base = np.zeros(max(N * row_bytes(kb, bits), 1), np.uint8)
        scales = np.zeros(max(N, 1), np.float32)
        wred = np.zeros(max(N, 1), np.float32)
        ow = np.zeros(max(N * idx.size, 1), np.float32)
        st = self.f("rtn_quantize_weights_clip")(_p(w), C.c_int64(N), C.c_int64(K), _p(idx), C.c_int64(idx.size), bits,
                                                 int(use_clipping), _p(base), _p(scales), _p(wred), _p(ow))
        assert st == 0, st
        return dict(base=base[: N * row_bytes(kb, bits)], scales=scales[:N], wreduced=wred[:N],
                    outlier_weights=ow[: N * idx.size].reshape(N, idx.size))


    def compute_wreduced(self, base, N, kb, bits, scales):
        out = np.zeros(max(N, 1), np.float32)
        self.f("compute_wreduced")(_p(np.ascontiguousarray(base, np.uint8)), C.c_int64(N), C.c_int64(kb), bits,
                                   _p(np.ascontiguousarray(scales, np.float32)), _p(out))
        return out[:N]

    def dequantize_weights(self, base, N, K, idx, bits, scales, ow):
        idx = np.ascontiguousarray(idx, np.int64)
        out = np.zeros(max(N * K, 1), np.float32)
        st = self.f("dequantize_weights")(_p(np.ascontiguousarray(base, np.uint8)), C.c_int64(N), C.c_int64(K), _p(idx),
                                          C.c_int64(idx.size), bits, _p(np.ascontiguousarray(scales, np.float32)),
                                          _p(np.ascontiguousarray(ow, np.float32).reshape(-1)
                                             if np.asarray(ow).size else np.zeros(1, np.float32)), _p(out))
        assert st == 0, st
        return out[: N * K].reshape(N, K)


class Oracle(_Base):
    prefix = "qo_"

    def _pack(self, v, rows, cols, bits, out):
        return self.f("pack")(_p(v), C.c_int64(rows), C.c_int64(cols), bits, _p(out), None, None)

    def _unpack(self, p, rows, cols, bits, out):
        fn = self.lib.qo_unpack
        fn.restype = None
        fn(_p(p), C.c_int64(rows), C.c_int64(cols), bits, _p(out))

    def quantize_fused(self, x, idx, bits):
        x = np.ascontiguousarray(x, np.float32)
        M, K = x.shape
        idx = np.ascontiguousarray(idx, np.int64)
        st, perm = self.permutation(K, idx)
        kb = K - idx.size
        packed = np.zeros(max(M * row_bytes(kb, bits), 1), np.uint8)
        scale = np.zeros(max(M, 1), np.float32)
        zero = np.zeros(max(M, 1), np.float32)
        xo = np.zeros(max(M * idx.size, 1), np.float32)
        st = self.f("quantize_activations_fused")(_p(x), C.c_int64(M), C.c_int64(K), _p(perm), C.c_int64(kb),
                                                  _p(idx), C.c_int64(idx.size), bits, _p(packed), _p(scale),
                                                  _p(zero), _p(xo))
        return st, packed[: M * row_bytes(kb, bits)], scale[:M], zero[:M], xo[: M * idx.size].reshape(M, idx.size)

    def quik_matmul(self, L, x, variant=2):
        """L: dict(in_features, out_features, bits, base, scales, wreduced, outlier_weights, idx, bias)."""
        class QoLayer(C.Structure):
            _fields_ = [("in_features", C.c_int64), ("out_features", C.c_int64), ("n_outlier", C.c_int64),
                        ("bits", C.c_int), ("act_bits", C.c_int), ("base", C.c_void_p), ("scales", C.c_void_p),
                        ("wreduced", C.c_void_p), ("outlier_weights", C.c_void_p), ("outlier_idx", C.c_void_p),
                        ("bias", C.c_void_p)]
        keep = {k: np.ascontiguousarray(L[k]) for k in ("base", "scales", "wreduced", "outlier_weights", "idx")}
        bias = None if L.get("bias") is None else np.ascontiguousarray(L["bias"], np.float32)
        lay = QoLayer(L["in_features"], L["out_features"], keep["idx"].size, L["bits"], L.get("act_bits", L["bits"]),
                      keep["base"].ctypes.data, keep["scales"].ctypes.data, keep["wreduced"].ctypes.data,
                      keep["outlier_weights"].ctypes.data, keep["idx"].ctypes.data,
                      None if bias is None else bias.ctypes.data)
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((x.shape[0], L["out_features"]), np.float32)
        fn = self.lib.qo_weight_only_forward if variant == "weight_only" else None
        if fn is not None:
            st = fn(C.byref(lay), _p(x), C.c_int64(x.shape[0]), _p(out))
        else:
            st = self.lib.qo_quik_matmul(C.byref(lay), _p(x), C.c_int64(x.shape[0]), variant, _p(out))
        return st, out

    def weight_only(self, L, x):
        """runtime.cpp:115-136 (LayerMode::WeightOnly) restated in C."""
        return self.quik_matmul(L, x, variant="weight_only")


class Ref(_Base):
    prefix = "qr_"

    def _pack(self, v, rows, cols, bits, out):
        return self.f("pack")(_p(v), C.c_int64(rows), C.c_int64(cols), bits, _p(out))

    def _unpack(self, p, rows, cols, bits, out):
        self.f("unpack")(_p(p), C.c_int64(rows), C.c_int64(cols), bits, _p(out))

    def quantize_fused(self, x, idx, bits):
        x = np.ascontiguousarray(x, np.float32)
        M, K = x.shape
        idx = np.ascontiguousarray(idx, np.int64)
        kb = K - idx.size
        packed = np.zeros(max(M * row_bytes(kb, bits), 1), np.uint8)
        scale = np.zeros(max(M, 1), np.float32)
        zero = np.zeros(max(M, 1), np.float32)
        xo = np.zeros(max(M * idx.size, 1), np.float32)
        st = self.f("quantize_activations_fused")(_p(x), C.c_int64(M), C.c_int64(K), _p(idx), C.c_int64(idx.size),
                                                  bits, _p(packed), _p(scale), _p(zero), _p(xo))
        return st, packed[: M * row_bytes(kb, bits)], scale[:M], zero[:M], xo[: M * idx.size].reshape(M, idx.size)

    def _layer_args(self, L):
        keep = {k: np.ascontiguousarray(L[k]) for k in ("base", "scales", "wreduced", "outlier_weights", "idx")}
        for k in ("scales", "wreduced", "outlier_weights"):
            keep[k] = keep[k].astype(np.float32)
        keep["base"] = keep["base"].astype(np.uint8)
        keep["idx"] = keep["idx"].astype(np.int64)
        if keep["base"].size == 0:
            keep["base"] = np.zeros(1, np.uint8)
        if keep["outlier_weights"].size == 0:
            keep["outlier_weights"] = np.zeros(1, np.float32)
        bias = None if L.get("bias") is None else np.ascontiguousarray(L["bias"], np.float32)
        keep["bias"] = bias
        args = [C.c_int64(L["in_features"]), C.c_int64(L["out_features"]), L["bits"], L.get("act_bits", L["bits"]),
                _p(keep["base"]), _p(keep["scales"]), _p(keep["wreduced"]), _p(keep["outlier_weights"]),
                _p(keep["idx"]), C.c_int64(np.asarray(L["idx"]).size), _p(bias)]
        return keep, args

    def quik_matmul(self, L, x, variant=2, times=None):
        keep, args = self._layer_args(L)
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((x.shape[0], L["out_features"]), np.float32)
        t = np.zeros(6, np.float64)
        st = self.f("quik_matmul")(*args, _p(x), C.c_int64(x.shape[0]), variant, _p(out), _p(t))
        if times is not None:
            times[:] = t
        return st, out

    def weight_only(self, L, x):
        """The reference's quik_matmul with layer.mode = LayerMode::WeightOnly."""
        keep, args = self._layer_args(L)
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((x.shape[0], L["out_features"]), np.float32)
        st = self.f("weight_only")(*args, _p(x), C.c_int64(x.shape[0]), _p(out))
        return st, out

    def layer_create(self, L):
        keep, args = self._layer_args(L)
        fn = self.lib.qr_layer_create
        fn.restype = C.c_void_p
        h = fn(*args)
        assert h, "qr_layer_create failed"
        return h, keep

    def layer_forward(self, h, x, n_out, variant=2, times=None):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((x.shape[0], n_out), np.float32)
        t = np.zeros(6, np.float64)
        st = self.f("layer_forward")(C.c_void_p(h), _p(x), C.c_int64(x.shape[0]), variant, _p(out), _p(t))
        if times is not None:
            times[:] = t
        return st, out

    def layer_destroy(self, h):
        self.lib.qr_layer_destroy.restype = None
        self.lib.qr_layer_destroy(C.c_void_p(h))

    def sparsegpt_joint(self, w, idx, bits, hsum=None, tokens=0):
        """The reference's sparsegpt_joint (quantizer.cpp:299-337): 2:4 pruning +
        quantization. hsum: K x K FP64 Hessian sum or None (identity)."""
        w = np.ascontiguousarray(w, np.float32)
        N, K = w.shape
        idx = np.ascontiguousarray(idx, np.int64)
        kb = K - idx.size
        base = np.zeros(max(N * row_bytes(kb, bits), 1), np.uint8)
        sc = np.zeros(max(N, 1), np.float32)
        wr = np.zeros(max(N, 1), np.float32)
        ow = np.zeros(max(N * idx.size, 1), np.float32)
        mask = np.zeros(max(N * kb, 1), np.uint8)
        h = None if hsum is None else np.ascontiguousarray(hsum, np.float64)
        st = self.f("sparsegpt_joint")(_p(w), C.c_int64(N), C.c_int64(K), _p(idx), C.c_int64(idx.size), bits,
                                       _p(h) if h is not None else None, C.c_int64(tokens), _p(base), _p(sc), _p(wr),
                                       _p(ow), _p(mask))
        return st, dict(base=base[: N * row_bytes(kb, bits)], scales=sc[:N], wreduced=wr[:N],
                        outlier_weights=ow[: N * idx.size].reshape(N, idx.size), mask=mask[: N * kb].reshape(N, kb))

    def gptq(self, w, idx, bits, hsum=None, tokens=1, damping=0.01, use_clipping=False, sparse=False):
        """The reference's gptq_quantize / sparsegpt_joint with an explicit Hessian sum."""
        w = np.ascontiguousarray(w, np.float32)
        N, K = w.shape
        idx = np.ascontiguousarray(idx, np.int64)
        kb = K - idx.size
        base = np.zeros(max(N * row_bytes(kb, bits), 1), np.uint8)
        sc = np.zeros(max(N, 1), np.float32)
        wr = np.zeros(max(N, 1), np.float32)
        ow = np.zeros(max(N * idx.size, 1), np.float32)
        mask = np.zeros(max(N * kb, 1), np.uint8)
        h = None if hsum is None else np.ascontiguousarray(hsum, np.float64)
        fn = self.f("gptq")
        fn.argtypes = None
        st = fn(_p(w), C.c_int64(N), C.c_int64(K), _p(idx), C.c_int64(idx.size), C.c_int(bits),
                _p(h) if h is not None else None, C.c_int64(tokens), C.c_double(damping), C.c_int(int(use_clipping)),
                C.c_int(int(sparse)), _p(base), _p(sc), _p(wr), _p(ow), _p(mask))
        return st, dict(base=base[: N * row_bytes(kb, bits)], scales=sc[:N], wreduced=wr[:N],
                        outlier_weights=ow[: N * idx.size].reshape(N, idx.size),
                        mask=mask[: N * kb].reshape(N, kb) if sparse else None)

    def build_hessian(self, x):
        x = np.ascontiguousarray(x, np.float32)
        T, K = x.shape
        h = np.zeros((K, K), np.float64)
        st = self.f("build_hessian")(_p(x), C.c_int64(T), C.c_int64(K), _p(h))
        assert st == 0, st
        return h

    def gated_mlp(self, up, gate, down, x):
        """The reference's forward_model(gated_mlp_ops): -> (st, out, h = silu(gate) * up)."""
        hs = [self.layer_create(L) for L in (up, gate, down)]
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((x.shape[0], down["out_features"]), np.float32)
        h = np.zeros((x.shape[0], up["out_features"]), np.float32)
        st = self.f("gated_mlp")(C.c_void_p(hs[0][0]), C.c_void_p(hs[1][0]), C.c_void_p(hs[2][0]), _p(x),
                                 C.c_int64(x.shape[0]), _p(out), _p(h))
        for hh, _ in hs:
            self.layer_destroy(hh)
        return st, out, h

    def save_layer(self, path, L, mask=None, wfp32=None):
        """The reference's save_layer (layer_io.cpp:7-30) -> bundle directory."""
        keep, args = self._layer_args(L)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        w = None if wfp32 is None else np.ascontiguousarray(wfp32, np.float32)
        return self.f("save_layer")(str(path).encode(), C.c_int64(L["in_features"]), C.c_int64(L["out_features"]),
                                    L["bits"], L.get("act_bits", L["bits"]), _p(keep["base"]), _p(keep["scales"]),
                                    _p(keep["wreduced"]), _p(keep["outlier_weights"]), _p(keep["idx"]),
                                    C.c_int64(np.asarray(L["idx"]).size), _p(keep["bias"]), _p(m), _p(w))

    def random_matrix(self, seed, rows, cols, stddev=1.0):
        out = np.zeros(max(rows * cols, 1), np.float32)
        fn = self.lib.qr_random_matrix
        fn.restype = None
        fn(C.c_uint32(seed), C.c_int64(rows), C.c_int64(cols), C.c_float(stddev), _p(out))
        return out[: rows * cols].reshape(rows, cols)


_oracle = None
_ref = None


def oracle() -> Oracle:
    global _oracle
    if _oracle is None:
        _oracle = Oracle(ORACLE_SO)
    return _oracle


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref(REF_SO)
    return _ref


def make_layer(rng: np.random.Generator, tokens, in_f, out_f, bits, n_outliers, heavy_cols=0, with_bias=True,
               fp16_inputs=True, checker=None):
    """Seeded layer in the style of test_runtime.cpp:27-45 (W ~ N(0,.5), x ~ N(0,1),
    heavy columns x100, outliers selected from x, RTN weights, bias ~ N(0,.1)).
    With fp16_inputs, x and the outlier weights are rounded to f16-representable
    values so the f16 device path and the f32 CPU checker see identical numbers."""
    chk = checker or oracle()
    w = rng.normal(0.0, 0.5, size=(out_f, in_f)).astype(np.float32)
    x = rng.normal(0.0, 1.0, size=(tokens, in_f)).astype(np.float32)
    for _ in range(heavy_cols):
        c = int(rng.integers(0, in_f))
        x[:, c] *= 100.0
    if fp16_inputs:
        x = x.astype(np.float16).astype(np.float32)
    idx = chk.select_outliers(x, n_outliers)
    q = chk.rtn_quantize_weights(w, idx, bits)
    ow = q["outlier_weights"]
    if fp16_inputs:
        ow = ow.astype(np.float16).astype(np.float32)
    bias = rng.normal(0.0, 0.1, size=out_f).astype(np.float32) if with_bias else None
    L = dict(in_features=in_f, out_features=out_f, bits=bits, act_bits=bits, base=q["base"], scales=q["scales"],
             wreduced=q["wreduced"], outlier_weights=ow, idx=idx, bias=bias)
    return L, x, w


def weight_only_f64(L, x, checker=None):
    """The reference test's FP64 oracle for LayerMode::WeightOnly (test_runtime.cpp:
    284-300): x times the de-permuted dequantized weights (q * scale in the base
    columns, the outlier weights in theirs) plus bias, in float64."""
    chk = checker or oracle()
    K, N = L["in_features"], L["out_features"]
    idx = np.asarray(L["idx"], np.int64)
    kb = K - idx.size
    st, perm = chk.permutation(K, idx)
    assert st == 0, st
    q = chk.unpack(L["base"], N, kb, L["bits"]).astype(np.float64)
    w = np.zeros((N, K), np.float64)
    w[:, perm[:kb]] = q * np.asarray(L["scales"], np.float64)[:, None]
    if idx.size:
        w[:, idx] = np.asarray(L["outlier_weights"], np.float64)
    y = np.asarray(x, np.float64) @ w.T
    if L.get("bias") is not None:
        y += np.asarray(L["bias"], np.float64)[None, :]
    return y


def rel_frobenius(ref_, out):
    ref_ = np.asarray(ref_, np.float64)
    return float(np.linalg.norm(np.asarray(out, np.float64) - ref_) / max(np.linalg.norm(ref_), 1e-300))


def f16_output_bound(L, x, want, y_is_f16=True):
    """Per-element bound on |y_device - want| for the Quik-mode forward.

    want = the reference's f32 output on the same f16-representable x and outlier weights,
    computed as r = fl(fl(bias + sum_seq x_o*w_o) + D) (runtime.cpp:96-113, :288-301);
    the device computes v = TC-accumulate(fl(bias + D); x_o*w_o) in f32 and rounds it to
    f16 (D, the dequant term, is bit-identical on both sides; every x_o*w_o product of
    two f16 values is exact in f32). With u = 2^-24 and
    T = |bias| + |D| + sum|x_o*w_o|  (<= |want| + 2|bias| + 2 sum|x_o*w_o|):
      |r - exact| <= (O + 1) u T          sequential f32 sum of bias + O products, + D
      |v - exact| <= (O/8 + 2) u T        init rounding + <= 2u of the running magnitude
                                          per 16-deep tcgen05 kind::f16 MMA step
      |f16(v) - v| <= 2^-11 |v| + 2^-25   round to nearest (normal / subnormal f16)
    so |y - r| <= 2^-11 |r| + 2^-25 + (1 + 2^-11) (1.125 O + 3) u T."""
    idx = np.asarray(L["idx"])
    O = idx.size
    xo = np.asarray(x, np.float64)[:, idx]
    ow = np.asarray(L["outlier_weights"], np.float64).reshape(-1, O) if O else None
    P = np.abs(xo) @ np.abs(ow).T if O else 0.0
    B = np.abs(np.asarray(L["bias"], np.float64))[None, :] if L.get("bias") is not None else 0.0
    r = np.abs(np.asarray(want, np.float64))
    T = r + 2.0 * B + 2.0 * P
    delta = (1.0 + 2.0 ** -11) * (1.125 * O + 3.0) * 2.0 ** -24 * T
    if not y_is_f16:
        return delta
    return 2.0 ** -11 * r + 2.0 ** -25 + delta
