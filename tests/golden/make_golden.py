"""Generates tests/golden/quik_golden.npz from the REFERENCE implementation itself
(oracle/_ref/libquik_ref.so = /root/reference/proj/src/{packed,calibration,
quantizer,runtime}.cpp compiled unchanged + oracle/ref_shim.cpp).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Cases:
  ref_test_layer_127   the reference unit test fixture "random 64x128 layer with 16
                       outliers" (test_runtime.cpp:241-246): make_layer(mt19937(127),
                       64, 128, 48, bits=4, outliers=16, heavy=4, bias) reproduced by
                       the reference's own generator (qr_make_test_layer)
  ref_test_layer_8bit  same generator, 8-bit, 24 x 200 -> 72, 8 outliers
  f16_*                numpy-seeded layers with f16-representable x and outlier
                       weights (device f16 path), weights from the reference RTN
  bundle_<case>/       the f16_w4_o64 and sp24_w4_o16 layers as reference layer bundles
  sp24_*               2:4 sparse layers from the reference's sparsegpt_joint (identity
                       or random-PSD Hessian), mask stored; *_tail2 / *_tail3 have a
                       trailing dense remainder group of 2 / 3 base columns
For every case the npz stores the layer, x, and the reference outputs:
quantize_activations_fused (packed / scale / zero / x_out), int_matmul of the
packed activations with the packed weights, and quik_matmul V1 / V2 / V3.
"""
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
from oracle_lib import make_layer, ref, row_bytes  # noqa: E402


def ref_layer(r, seed, tokens, in_f, out_f, bits, O, heavy):
    import ctypes as C

    x = np.zeros((tokens, in_f), np.float32)
    w = np.zeros((out_f, in_f), np.float32)
    idx = np.zeros(max(O, 1), np.int64)
    kb = in_f - O
    base = np.zeros(out_f * row_bytes(kb, bits), np.uint8)
    sc = np.zeros(out_f, np.float32)
    wr = np.zeros(out_f, np.float32)
    ow = np.zeros(max(out_f * O, 1), np.float32)
    bias = np.zeros(out_f, np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    st = r.lib.qr_make_test_layer(C.c_uint32(seed), C.c_int64(tokens), C.c_int64(in_f), C.c_int64(out_f), bits,
                                  C.c_int64(O), C.c_int64(heavy), 1, p(x), p(w), p(idx), p(base), p(sc), p(wr),
                                  p(ow), p(bias))
    assert st == 0, st
    L = dict(in_features=in_f, out_features=out_f, bits=bits, act_bits=bits, base=base, scales=sc, wreduced=wr,
             outlier_weights=ow[: out_f * O].reshape(out_f, O), idx=idx[:O], bias=bias)
    return L, x


def sparse_layer(r, rng, M, K, N, O, bits, psd):
    x = rng.normal(0.0, 1.0, size=(M, K)).astype(np.float32)
    for c in rng.choice(K, size=3, replace=False):
        x[:, c] *= 100.0
    x = x.astype(np.float16).astype(np.float32)
    idx = r.select_outliers(x, O)
    w = rng.normal(0.0, 0.5, size=(N, K)).astype(np.float32)
    hsum = None
    if psd:
        xc = rng.normal(0.0, 1.0, size=(4 * K, K))
        hsum = xc.T @ xc
    st, q = r.sparsegpt_joint(w, idx, bits, hsum=hsum, tokens=4 * K if psd else 0)
    assert st == 0, st
    bias = rng.normal(0.0, 0.1, size=N).astype(np.float32)
    L = dict(in_features=K, out_features=N, bits=bits, act_bits=bits, base=q["base"], scales=q["scales"],
             wreduced=q["wreduced"], outlier_weights=q["outlier_weights"].astype(np.float16).astype(np.float32),
             idx=idx, bias=bias, mask=q["mask"])
    return L, x


def outputs(r, L, x):
    bits = L["bits"]
    st, pk, sc, ze, xo = r.quantize_fused(x, L["idx"], bits)
    assert st == 0
    kb = L["in_features"] - len(L["idx"])
    st, acc = r.int_matmul(pk, x.shape[0], kb, bits, L["base"], L["out_features"])
    assert st == 0
    outs = {}
    for v in (0, 1, 2):
        st, o = r.quik_matmul(L, x, v)
        assert st == 0
        outs[f"out_v{v + 1}"] = o
    return dict(packed=pk, scale=sc, zero=ze, x_out=xo, acc=acc, **outs)


def main():
    r = ref()
    cases = {}
    cases["ref_test_layer_127"] = ref_layer(r, 127, 64, 128, 48, 4, 16, 4)
    cases["ref_test_layer_8bit"] = ref_layer(r, 2024, 24, 200, 72, 8, 8, 3)
    rng = np.random.default_rng(20231017)
    for name, (M, K, N, O, bits, heavy) in {
        "f16_w4_o64": (16, 512, 256, 64, 4, 8),
        "f16_w8_o8": (9, 96, 40, 8, 8, 2),
        "f16_w4_o0": (33, 300, 77, 0, 4, 3),
        "f16_w4_o32_ragged": (48, 641, 129, 32, 4, 5),
    }.items():
        L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=heavy, checker=r)
        cases[name] = (L, x)
    # 2:4 sparse layers (cfg5 path) from the reference's sparsegpt_joint, f16-representable
    # x and outlier weights; the mask is stored so the device builds the sparse GEMM
    srng = np.random.default_rng(240)
    for name, (M, K, N, O, bits, psd) in {
        "sp24_w4_o16": (40, 256, 160, 16, 4, False),
        "sp24_w4_o64_psd": (24, 512, 200, 64, 4, True),
        "sp24_w8_o32_psd": (17, 384, 136, 32, 8, True),
        "sp24_w4_o0": (64, 640, 256, 0, 4, True),
        "sp24_w4_o0_tail2": (12, 262, 96, 0, 4, False),
        "sp24_w4_o0_tail3": (12, 259, 96, 0, 4, False),
    }.items():
        cases[name] = sparse_layer(r, srng, M, K, N, O, bits, psd)
    blob, manifest = {}, {}
    for name, (L, x) in cases.items():
        out = outputs(r, L, x)
        manifest[name] = dict(M=int(x.shape[0]), K=int(L["in_features"]), N=int(L["out_features"]),
                              outliers=int(len(L["idx"])), bits=int(L["bits"]))
        blob[f"{name}.x"] = x
        for k in ("base", "scales", "wreduced", "outlier_weights", "idx", "bias", "mask"):
            if k in L:
                blob[f"{name}.{k}"] = np.asarray(L[k])
        for k, v in out.items():
            blob[f"{name}.{k}"] = v
    # layer bundles written by the reference's own save_layer (layer_io.cpp:7-30) for the
    # bundle-loader GPU tests
    import shutil
    for name in ("f16_w4_o64", "sp24_w4_o16"):
        L, _ = cases[name]
        d = HERE / f"bundle_{name}"
        shutil.rmtree(d, ignore_errors=True)
        assert r.save_layer(d, L, mask=L.get("mask")) == 0
    np.savez_compressed(HERE / "quik_golden.npz", **blob)
    (HERE / "quik_golden.json").write_text(json.dumps(
        dict(generator="tests/golden/make_golden.py", source="oracle/_ref/libquik_ref.so (reference proj/src compiled "
             "unchanged with -O3 -fopenmp -ffp-contract=off)", cases=manifest), indent=1))
    print("wrote", HERE / "quik_golden.npz", sum(v.nbytes for v in blob.values()), "bytes raw")


if __name__ == "__main__":
    main()
