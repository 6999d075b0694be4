"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Bit-exact: packed activation codes, per-token scale/zero, outlier gather, INT32
base accumulators, the dequantisation epilogue, and the whole layer when it has
no outliers (f32 output). Tolerance: f16 outlier products (tensor-core
summation order) and the f16 output rounding, SURVEY.md Appendix A.3:
  |y - ref| <= 2^-11 |ref| + 2^-20 * S   (S = sum of term magnitudes), and
  rel_frobenius(y, ref) <= 5e-4 (f16 out) / 1e-5 (f32 out).
Cases follow the reference tests (test_packed.cpp, test_runtime.cpp,
acceptance.cpp criteria 4/5) plus BASELINE.json shapes.
"""
import numpy as np
import pytest

from oracle_lib import f16_output_bound, make_layer, oracle, ref, row_bytes

pytestmark = pytest.mark.gpu

F16_REL = 2.0 ** -11


def q():
    import paper_2310_09259_b200 as m

    return m


def to_layer(L):
    m = q()
    kb = L["in_features"] - np.asarray(L["idx"]).size
    w = m.QuantizedWeights(m.PackedIntMatrix(L["out_features"], kb, L["bits"], np.asarray(L["base"], np.uint8)),
                           np.asarray(L["scales"], np.float32), np.asarray(L["outlier_weights"], np.float32),
                           np.asarray(L["wreduced"], np.float32))
    return m.QuikLinearLayer(w, m.OutlierSet.from_indices(L["in_features"], L["idx"]), L.get("bias"), L["bits"])


def rel_frob(ref_, got):
    ref_ = ref_.astype(np.float64)
    got = got.astype(np.float64)
    d = np.sqrt(((got - ref_) ** 2).sum())
    n = np.sqrt((ref_ ** 2).sum())
    return d if n == 0 else d / n


# --------------------------------------------------------------------------- K1 quantizer


def test_quantize_kat_direct_formula():
    # test_runtime.cpp:80-87: [0, .5, 1, 1.5] -> scale 0.1, zero 0, codes [-8,-3,2,7]
    m = q()
    r = m.quantize_activations(np.array([[0.0, 0.5, 1.0, 1.5]], np.float32), 4)
    assert abs(r.scale[0] - 0.1) < 1e-7 and r.zero[0] == 0.0
    assert list(m.unpack_values(r.packed)[0]) == [-8, -3, 2, 7]


def test_quantize_kat_constant_row():
    # test_runtime.cpp:89-97
    m = q()
    r = m.quantize_activations(np.array([[5.0, 5.0, 5.0]], np.float32), 4)
    assert r.scale[0] == 1.0 and r.zero[0] == 5.0
    assert list(m.unpack_values(r.packed)[0]) == [-8, -8, -8]


def test_quantize_rejects_non_finite():
    # test_runtime.cpp:110-116
    m = q()
    for bad in (np.nan, np.inf):
        with pytest.raises(m.NumericalError):
            m.quantize_activations(np.array([[1.0, bad]], np.float32), 4)


@pytest.mark.parametrize("bits", [4, 8])
def test_fused_quantizer_bit_exact_random(bits):
    # fused == reference on seeded random shapes (test_runtime.cpp:134-156 style)
    m = q()
    o = oracle()
    for seed in range(40):
        rng = np.random.default_rng(1000 + seed)
        K = int(rng.integers(8, 400))
        M = int(rng.integers(1, 20))
        x = rng.normal(0, 1.5, size=(M, K)).astype(np.float32)
        k = int(rng.integers(0, K))
        idx = o.select_outliers(x, k)
        st, pk, sc, ze, xo = o.quantize_fused(x, idx, bits)
        assert st == 0
        r, gxo = m.quantize_activations_fused(x, m.OutlierSet.from_indices(K, idx), bits)
        np.testing.assert_array_equal(r.packed.data, pk)
        np.testing.assert_array_equal(r.scale.view(np.uint32), sc.view(np.uint32))
        np.testing.assert_array_equal(r.zero.view(np.uint32), ze.view(np.uint32))
        np.testing.assert_array_equal(gxo, xo)


def test_fused_quantizer_ties_and_signed_zero():
    # exact .5 ties (lround ties-away) and the first-seen sign of a zero minimum
    m = q()
    o = oracle()
    x = np.array([[0.0, 1.0, 0.5, 15.0, 7.5, 2.5, 1.5],
                  [-0.0, 0.0, 3.0, 1.0, 2.0, 0.0, 0.6],
                  [0.0, -0.0, 3.0, 1.0, 2.0, -0.0, 0.6]], np.float32)
    for bits in (4, 8):
        st, pk, sc, ze, _ = o.quantize_fused(x, np.zeros(0, np.int64), bits)
        r, _ = m.quantize_activations_fused(x, m.OutlierSet.none(x.shape[1]), bits)
        np.testing.assert_array_equal(r.packed.data, pk)
        np.testing.assert_array_equal(r.zero.view(np.uint32), ze.view(np.uint32))
        np.testing.assert_array_equal(r.scale.view(np.uint32), sc.view(np.uint32))


def test_fused_quantizer_boundaries():
    # test_runtime.cpp:158-170: empty outlier set, all-outlier set
    m = q()
    x = np.array([[1.0, 2.0, 3.0]], np.float32)
    a, xo = m.quantize_activations_fused(x, m.OutlierSet.none(3), 4)
    plain = m.quantize_activations(x, 4)
    np.testing.assert_array_equal(a.packed.data, plain.packed.data)
    assert xo.shape == (1, 0)
    b, allx = m.quantize_activations_fused(x, m.OutlierSet.from_indices(3, [0, 1, 2]), 4)
    assert b.packed.cols == 0
    np.testing.assert_array_equal(allx, x)


# --------------------------------------------------------------------------- INT GEMM


def test_int_matmul_kat():
    # test_packed.cpp:78-92
    m = q()
    x = m.pack_values([1, -2, 3, 4], 2, 2, 8)
    w = m.pack_values([5, 6, -7, 8], 2, 2, 8)
    np.testing.assert_array_equal(m.int_matmul(x, w), [[-7, -23], [39, 11]])
    x4 = m.pack_values([1, -2, 3, 4], 2, 2, 4)
    w4 = m.pack_values([5, 6, -7, 7], 2, 2, 4)
    out4 = m.int_matmul(x4, w4)
    assert out4[0, 0] == 1 * 5 + -2 * 6 and out4[1, 1] == 3 * -7 + 4 * 7


def test_int_matmul_rejects_mismatch():
    # test_packed.cpp:153-157
    m = q()
    a = m.pack_values([1] * 6, 2, 3, 4)
    b = m.pack_values([1] * 8, 2, 4, 4)
    c = m.pack_values([1] * 6, 2, 3, 8)
    with pytest.raises(ValueError):
        m.int_matmul(a, b)
    with pytest.raises(ValueError):
        m.int_matmul(a, c)


def test_int_matmul_random_shapes_vs_naive():
    # test_packed.cpp:104-128: 100 random shapes with dims 1..40, bits alternating
    m = q()
    o = oracle()
    rng = np.random.default_rng(7)
    for trial in range(100):
        bits = 4 if trial % 2 == 0 else 8
        lim = 7 if bits == 4 else 127
        t, k, n = (int(v) for v in rng.integers(1, 41, size=3))
        xv = rng.integers(-lim - 1, lim + 1, size=(t, k))
        wv = rng.integers(-lim - 1, lim + 1, size=(n, k))
        x = m.pack_values(xv, t, k, bits)
        w = m.pack_values(wv, n, k, bits)
        got = m.int_matmul(x, w)
        st, want = o.int_matmul(x.data, t, k, bits, w.data, n)
        assert st == 0
        np.testing.assert_array_equal(got, want)
        np.testing.assert_array_equal(got, xv @ wv.T)


@pytest.mark.parametrize("bits,t,k,n", [(4, 300, 1000, 500), (8, 257, 4100, 129), (4, 16, 3968, 4096),
                                        (8, 1, 10320, 300), (4, 2048, 256, 384)])
def test_int_matmul_large_exact(bits, t, k, n):
    m = q()
    rng = np.random.default_rng(t * 7 + k)
    lim = 7 if bits == 4 else 127
    xv = rng.integers(-lim - 1, lim + 1, size=(t, k))
    wv = rng.integers(-lim - 1, lim + 1, size=(n, k))
    got = m.int_matmul(m.pack_values(xv, t, k, bits), m.pack_values(wv, n, k, bits))
    np.testing.assert_array_equal(got, (xv @ wv.T).astype(np.int64))


def test_int_matmul_linearity():
    # test_packed.cpp:131-151
    m = q()
    rng = np.random.default_rng(11)
    t, k, n = 33, 300, 70
    xv = rng.integers(-8, 8, size=(t, k))
    w1 = rng.integers(-4, 4, size=(n, k))
    w2 = rng.integers(-4, 4, size=(n, k))
    x = m.pack_values(xv, t, k, 4)
    s = m.int_matmul(x, m.pack_values(w1 + w2, n, k, 4))
    a = m.int_matmul(x, m.pack_values(w1, n, k, 4))
    b = m.int_matmul(x, m.pack_values(w2, n, k, 4))
    np.testing.assert_array_equal(s, a + b)


# --------------------------------------------------------------------------- epilogue


def test_dequantize_epilogue_bit_exact():
    m = q()
    o = oracle()
    rng = np.random.default_rng(3)
    M, N = 37, 211
    acc = rng.integers(-400000, 400000, size=(M, N)).astype(np.int32)
    sa = rng.uniform(0.01, 2, M).astype(np.float32)
    za = rng.normal(0, 3, M).astype(np.float32)
    sw = rng.uniform(0.001, 0.1, N).astype(np.float32)
    wr = rng.normal(0, 5, N).astype(np.float32)
    want = o.dequantize_epilogue(acc, sa, za, 8, sw, wr)
    a = m.ActQuantResult(m.PackedIntMatrix(M, 0, 4, np.zeros(0, np.uint8)), sa, za, 8)
    got = m.dequantize_epilogue(acc, a, sw, wr)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_dequantize_epilogue_hand_example():
    # test_runtime.cpp:172-186: acc = -23, out = -0.5
    m = q()
    aq = m.quantize_activations(np.array([[1.0, 3.0]], np.float32), 4)
    assert list(m.unpack_values(aq.packed)[0]) == [-8, 7]
    acc = m.int_matmul(aq.packed, m.pack_values([2, -1], 1, 2, 4))
    assert acc[0, 0] == -23
    out = m.dequantize_epilogue(acc, aq, np.array([0.5], np.float32), np.array([0.5], np.float32))
    assert abs(out[0, 0] + 0.5) < 1e-6


# --------------------------------------------------------------------------- full layer


@pytest.mark.parametrize("bits", [4, 8])
@pytest.mark.parametrize("with_bias", [False, True])
def test_layer_no_outliers_f32_bit_exact(bits, with_bias):
    """With O = 0 every op of the layer is defined op-by-op: the f32 output must be
    bit-identical to the reference quik_matmul (runtime.cpp:246-318)."""
    m = q()
    o = oracle()
    rng = np.random.default_rng(17 + bits)
    for (M, K, N) in [(9, 96, 40), (64, 128, 48), (33, 1000, 257), (130, 512, 300)]:
        L, x, _ = make_layer(rng, M, K, N, bits, 0, heavy_cols=2, with_bias=with_bias)
        st, want = o.quik_matmul(L, x, 2)
        assert st == 0
        got = m.quik_matmul(to_layer(L), x)
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("bits", [4, 8])
def test_layer_with_outliers_f32(bits):
    m = q()
    o = oracle()
    rng = np.random.default_rng(23 + bits)
    for (M, K, N, O) in [(9, 96, 40, 8), (64, 128, 48, 16), (48, 2048, 512, 256), (5, 300, 77, 64)]:
        L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=4)
        st, want = o.quik_matmul(L, x, 2)
        assert st == 0
        got = m.quik_matmul(to_layer(L), x)
        assert rel_frob(want, got) < 1e-5, (M, K, N, O, rel_frob(want, got))


def elementwise_bound(L, x, want):
    """Per-element f16 tolerance, SURVEY.md Appendix A.3."""
    idx = np.asarray(L["idx"])
    xo = x[:, idx].astype(np.float64)
    ow = np.asarray(L["outlier_weights"], np.float64)
    S = np.abs(xo) @ np.abs(ow).T + np.abs(want).astype(np.float64)
    if L.get("bias") is not None:
        S += np.abs(L["bias"])[None, :]
    return F16_REL * np.abs(want) + 2.0 ** -20 * S + 1e-30


@pytest.mark.parametrize("bits", [4, 8])
def test_layer_f16_output_tolerance(bits):
    m = q()
    o = oracle()
    import torch

    rng = np.random.default_rng(29 + bits)
    for (M, K, N, O) in [(16, 512, 384, 128), (200, 1024, 640, 64), (3, 640, 128, 0)]:
        L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=4)
        st, want = o.quik_matmul(L, x, 2)
        dev = m.QuikLinear(to_layer(L))
        y = dev(torch.from_numpy(x).half().cuda()).float().cpu().numpy()
        err = np.abs(y - want)
        bound = f16_output_bound(L, x, want)
        assert np.all(err <= bound), float((err / bound).max())
        assert rel_frob(want, y) <= 5e-4


def test_variants_bit_identical():
    # test_runtime.cpp:270-281 / acceptance criterion 5
    m = q()
    import torch

    rng = np.random.default_rng(31)
    for trial in range(6):
        bits = 4 if trial % 2 == 0 else 8
        L, x, _ = make_layer(rng, 5 + 13 * trial, 48 + 40 * trial, 24 + 50 * trial, bits, 8 * (trial % 3), 1)
        dev = m.QuikLinear(to_layer(L))
        xt = torch.from_numpy(x).cuda()
        outs = [dev(xt, out_dtype=torch.float32, variant=v).cpu().numpy() for v in m.PipelineVariant]
        np.testing.assert_array_equal(outs[0].view(np.uint32), outs[1].view(np.uint32))
        np.testing.assert_array_equal(outs[0].view(np.uint32), outs[2].view(np.uint32))


def test_layer_matches_compiled_reference():
    """Same seeded layer through the reference sources themselves (oracle/_ref)."""
    m = q()
    r = ref()
    rng = np.random.default_rng(37)
    L, x, _ = make_layer(rng, 24, 640, 200, 4, 0, heavy_cols=3, checker=r)
    st, want = r.quik_matmul(L, x, 2)
    assert st == 0
    got = m.quik_matmul(to_layer(L), x)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


def test_cfg1_oracle_shape():
    """BASELINE configs[0]: 16 tokens x 4096 -> 4096, 128 outliers, W4A4."""
    m = q()
    o = oracle()
    import torch

    rng = np.random.default_rng(41)
    L, x, _ = make_layer(rng, 16, 4096, 4096, 4, 128, heavy_cols=128)
    st, want = o.quik_matmul(L, x, 2)
    dev = m.QuikLinear(to_layer(L))
    y32 = dev(torch.from_numpy(x).cuda(), out_dtype=torch.float32).cpu().numpy()
    assert rel_frob(want, y32) < 1e-5
    y16 = dev(torch.from_numpy(x).half().cuda()).float().cpu().numpy()
    assert rel_frob(want, y16) < 5e-4


@pytest.mark.parametrize("M,K,N,bits,O", [(1024, 8192, 4096, 4, 0), (4096, 1024, 8192, 4, 0), (3000, 2048, 6000, 8, 0),
                                         (4096, 1024, 8192, 4, 128), (2500, 2048, 5000, 8, 256)])
def test_large_layer_token_subset_exact(M, K, N, bits, O):
    """Full-size property: tokens and output rows are independent, so the oracle on a
    subset of tokens and rows checks the full-size device run (O = 0: exactly, f32).
    The 4096 x 8192 / 3000 x 6000 outputs are several tiles per persistent CTA (pair):
    TMEM accumulator double buffering and the tile scheduler's phases across tiles."""
    m = q()
    o = oracle()
    import torch

    rng = np.random.default_rng(43 + M + O)
    L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=min(O, 4))
    dev = m.QuikLinear(to_layer(L))
    y = dev(torch.from_numpy(x).cuda(), out_dtype=torch.float32).cpu().numpy()
    toks = np.unique(np.concatenate([rng.choice(M, 6, replace=False), [0, M - 1]]))
    rows = np.unique(np.concatenate([rng.choice(N, 300, replace=False), [0, N - 1]]))
    rb = row_bytes(K - O, bits)
    sub = dict(L)
    sub["out_features"] = rows.size
    sub["base"] = np.asarray(L["base"]).reshape(N, rb)[rows].reshape(-1)
    sub["scales"] = L["scales"][rows]
    sub["wreduced"] = L["wreduced"][rows]
    sub["outlier_weights"] = np.asarray(L["outlier_weights"]).reshape(N, O)[rows]
    sub["bias"] = L["bias"][rows]
    st, want = o.quik_matmul(sub, x[toks], 2)
    assert st == 0
    got = y[np.ix_(toks, rows)]
    if O == 0:
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    else:
        assert rel_frob(want, got) < 1e-5


def test_non_finite_input_flags_numerical_error():
    m = q()
    import torch

    rng = np.random.default_rng(47)
    L, x, _ = make_layer(rng, 4, 64, 32, 4, 4)
    lay = to_layer(L)
    dev = m.QuikLinear(lay)
    base_col = int(lay.outliers.permutation[0])
    x[2, base_col] = np.nan
    dev(torch.from_numpy(x).cuda())
    with pytest.raises(m.NumericalError):
        dev.ctx.sync(torch.cuda.current_stream().cuda_stream)
    with pytest.raises(m.NumericalError):
        m.quik_matmul(lay, x)


# --------------------------------------------------------------------------- every tile configuration


@pytest.fixture(params=[0, 1], ids=["default", "alt"])
def tile(request):
    """Forces a GEMM tile. "alt": CTA-pair tiles of 8-bit dense layers run as 4-CTA
    TMA-multicast clusters. (4-bit dense layers always stream INT4 weights widened into
    TMEM; the raw int_matmul ABI runs the INT8-operand kernel.)"""
    import paper_2310_09259_b200 as m

    lib = m.load_library()

    def force(cg, bn):
        lib.quik_set_gemm_multicast(1 if (request.param and cg == 2) else 0)
        return lib.quik_set_gemm_tile(cg, bn)

    yield force
    lib.quik_set_gemm_tile(0, 0)
    lib.quik_set_gemm_multicast(0)


@pytest.mark.parametrize("cg,bn", [(1, 32), (1, 64), (1, 128), (2, 128), (2, 192), (2, 256)])
def test_every_tile_config_exact(tile, cg, bn):
    """Forces each GEMM tile (1-CTA and CTA-pair) and checks the INT32 path and the
    O=0 f32 layer bit-exactly, with ragged M/N/K tails."""
    m = q()
    o = oracle()
    assert tile(cg, bn) == 0
    rng = np.random.default_rng(100 * cg + bn)
    for (t, k, n, bits) in [(300, 1000, 500, 4), (37, 259, 333, 8), (513, 640, 257, 4)]:
        lim = 7 if bits == 4 else 127
        xv = rng.integers(-lim - 1, lim + 1, size=(t, k))
        wv = rng.integers(-lim - 1, lim + 1, size=(n, k))
        got = m.int_matmul(m.pack_values(xv, t, k, bits), m.pack_values(wv, n, k, bits))
        np.testing.assert_array_equal(got, xv @ wv.T)
    # many tiles per persistent CTA in every configuration (f64 BLAS is exact here)
    t, k, n = 2048, 512, 3000
    xv = rng.integers(-8, 8, size=(t, k))
    wv = rng.integers(-8, 8, size=(n, k))
    got = m.int_matmul(m.pack_values(xv, t, k, 4), m.pack_values(wv, n, k, 4))
    np.testing.assert_array_equal(got, (xv.astype(np.float64) @ wv.T.astype(np.float64)).astype(np.int64))
    L, x, _ = make_layer(rng, 300, 700, 300, 4, 0, heavy_cols=2)
    st, want = o.quik_matmul(L, x, 2)
    got = m.quik_matmul(to_layer(L), x)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    L, x, _ = make_layer(rng, 260, 900, 520, 8, 64, heavy_cols=5)
    st, want = o.quik_matmul(L, x, 2)
    got = m.quik_matmul(to_layer(L), x)
    assert rel_frob(want, got) < 1e-5


def test_rtn_quantize_weights_device_bit_exact():
    """quantize-weights on the device vs the reference's rtn_quantize_weights
    (quantizer.cpp:339-371): codes, scales, wreduced and outlier columns bit-exact."""
    m = q()
    r = ref()
    rng = np.random.default_rng(53)
    for bits in (4, 8):
        for (N, K, O) in [(40, 96, 8), (257, 1001, 0), (64, 512, 64)]:
            w = rng.normal(0, 0.5, size=(N, K)).astype(np.float32)
            w[3] = 0.0  # all-zero row -> scale 1, q = 0
            idx = np.sort(rng.choice(K, O, replace=False)).astype(np.int64)
            want = r.rtn_quantize_weights(w, idx, bits)
            got = m.rtn_quantize_weights(w, m.OutlierSet.from_indices(K, idx), bits)
            np.testing.assert_array_equal(got.base.data, want["base"])
            np.testing.assert_array_equal(got.scales.view(np.uint32), want["scales"].view(np.uint32))
            np.testing.assert_array_equal(got.wreduced.view(np.uint32), want["wreduced"].view(np.uint32))
            np.testing.assert_array_equal(got.outlier_weights, want["outlier_weights"])


def test_quantizer_wide_rows_f32_and_f16():
    """K1 at the LLaMA-2-70B down-projection width (28672) with 896 outliers, both input types."""
    m = q()
    o = oracle()
    rng = np.random.default_rng(59)
    K = 28672
    x = rng.normal(0, 1, size=(3, K)).astype(np.float16).astype(np.float32)
    idx = np.sort(rng.choice(K, 896, replace=False)).astype(np.int64)
    st, pk, sc, ze, xo = o.quantize_fused(x, idx, 8)
    r, gxo = m.quantize_activations_fused(x, m.OutlierSet.from_indices(K, idx), 8)
    np.testing.assert_array_equal(r.packed.data, pk)
    np.testing.assert_array_equal(r.scale.view(np.uint32), sc.view(np.uint32))
    np.testing.assert_array_equal(gxo, xo)


# --------------------------------------------------------------------------- reference golden fixtures


def _golden():
    import json
    from pathlib import Path

    d = Path(__file__).resolve().parent / "golden"
    return np.load(d / "quik_golden.npz"), json.loads((d / "quik_golden.json").read_text())["cases"]


_G, _CASES = _golden()


@pytest.mark.parametrize("name", sorted(_CASES))
def test_device_matches_reference_golden(name):
    """Device path vs outputs of the reference sources themselves (tests/golden)."""
    m = q()
    meta = _CASES[name]
    g = lambda k: _G[f"{name}.{k}"]  # noqa: E731
    K, N, O, bits = meta["K"], meta["N"], meta["outliers"], meta["bits"]
    outl = m.OutlierSet.from_indices(K, g("idx"))
    x = g("x")
    r, xo = m.quantize_activations_fused(x, outl, bits)
    np.testing.assert_array_equal(r.packed.data, g("packed"))
    np.testing.assert_array_equal(r.scale.view(np.uint32), g("scale").view(np.uint32))
    np.testing.assert_array_equal(r.zero.view(np.uint32), g("zero").view(np.uint32))
    np.testing.assert_array_equal(xo, g("x_out"))
    w = m.QuantizedWeights(m.PackedIntMatrix(N, K - O, bits, g("base")), g("scales"), g("outlier_weights"),
                           g("wreduced"))
    np.testing.assert_array_equal(m.int_matmul(r.packed, w.base), g("acc"))
    layer = m.QuikLinearLayer(w, outl, g("bias"), bits)
    y = m.quik_matmul(layer, x)
    want = g("out_v3")
    if O == 0:
        np.testing.assert_array_equal(y.view(np.uint32), want.view(np.uint32))
    elif name.startswith("f16_"):  # f16-representable x / outlier weights: only summation order differs
        assert rel_frob(want, y) < 1e-5
    else:
        # f32 reference inputs: the device rounds the outlier operands to f16 (2 x 2^-11
        # relative per product) -- the bound is on the outlier term's magnitude
        S = np.abs(x[:, g("idx")]).astype(np.float64) @ np.abs(g("outlier_weights")).astype(np.float64).T
        assert np.all(np.abs(y - want) <= 2.0 ** -10 * S + 1e-5 * np.abs(want) + 1e-6)


def test_cpp_facade_parity_driver():
    """The C++ drop-in facade (include/quik_b200.hpp) driven like the reference's own
    unit tests (tests/cpp/facade_test.cpp, checked against the C oracle)."""
    import subprocess
    from pathlib import Path

    exe = Path(__file__).resolve().parent.parent / "build" / "tests" / "facade_test"
    assert exe.exists(), "build/tests/facade_test not built (__graft_entry__.build())"
    golden = Path(__file__).resolve().parent / "golden"
    r = subprocess.run([str(exe), str(golden)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failure(s)" in r.stdout


@pytest.mark.parametrize("xdt,ydt", [("f16", "f16"), ("f32", "f32"), ("f32", "f16")])
def test_forward_host_chunked_equals_device(xdt, ydt):
    """quik_linear_forward_host (host buffers, chunked copy/compute overlap) is
    bit-identical to the device-buffer forward for any chunking, pinned or not."""
    m = q()
    import torch

    dt = {"f16": torch.float16, "f32": torch.float32}
    rng = np.random.default_rng(41)
    L, x, _ = make_layer(rng, 1000, 1024, 384, 4, 64, heavy_cols=4)
    dev = m.QuikLinear(to_layer(L))
    xh = torch.from_numpy(x).to(dt[xdt])
    want = dev(xh.cuda(), out_dtype=dt[ydt]).cpu()
    for chunk, pin in [(0, True), (256, True), (100, False), (1000, True), (7, True)]:
        xin = xh.pin_memory() if pin else xh.clone()
        yh = torch.empty((1000, 384), dtype=dt[ydt])
        if pin:
            yh = yh.pin_memory()
        dev.forward_host(xin, yh, chunk_tokens=chunk)
        torch.cuda.synchronize()
        assert torch.equal(yh.view(torch.int16 if ydt == "f16" else torch.int32),
                           want.view(torch.int16 if ydt == "f16" else torch.int32)), (chunk, pin)


def _hot_k1_case(m, o, x16, idx, bits, N=8):
    """Runs the hot-path quantizer (GEMM layout) and checks it bit-exactly against
    the oracle's fused quantizer on the same (f16-representable) input."""
    import torch

    M, K = x16.shape
    x = x16.astype(np.float32)
    st, pk, sc, ze, xo = o.quantize_fused(x, idx, bits)
    assert st == 0
    kb = K - len(idx)
    want = o.unpack(pk, M, kb, bits).reshape(M, kb) if kb else np.zeros((M, 0), np.int8)
    rng = np.random.default_rng(5)
    L = dict(in_features=K, out_features=N, bits=bits, idx=np.asarray(idx, np.int64),
             base=np.zeros(N * row_bytes(kb, bits), np.uint8), scales=np.ones(N, np.float32),
             wreduced=np.zeros(N, np.float32), outlier_weights=np.zeros((N, len(idx)), np.float32), bias=None)
    dev = m.QuikLinear(to_layer(L))
    codes, s, z, xo16 = dev.quantize_gemm_layout(torch.from_numpy(x16).cuda())
    codes, s, z, xo16 = codes.cpu().numpy(), s.cpu().numpy(), z.cpu().numpy(), xo16.cpu().numpy()
    np.testing.assert_array_equal(codes[:, :kb], want.astype(np.int8))
    assert not codes[:, kb:].any()
    np.testing.assert_array_equal(s.view(np.uint32), sc.view(np.uint32))
    np.testing.assert_array_equal(z.view(np.uint32), ze.view(np.uint32))
    if len(idx):
        np.testing.assert_array_equal(xo16[:, :len(idx)].astype(np.float32), xo.reshape(M, -1))
    assert not xo16[:, len(idx):].astype(np.float32).any()


@pytest.mark.parametrize("bits", [4, 8])
def test_hot_quantizer_gemm_layout_bit_exact(bits):
    """The hot-path K1 (f16 rows, descriptor compaction) against the oracle: codes,
    scale, zero and outlier gather bit-exact, at random shapes and outlier sets
    (clustered outliers exercise the per-byte chunks, sparse ones the fast chunks)."""
    m = q()
    o = oracle()
    for seed in range(24):
        rng = np.random.default_rng(7000 + seed)
        K = int(rng.integers(1, 600)) * 8
        M = int(rng.integers(1, 12))
        x = rng.normal(0, 1.0, size=(M, K)).astype(np.float16)
        k = int(rng.integers(0, min(K, 300)))
        if seed % 3 == 0:
            start = int(rng.integers(0, K - k + 1))
            idx = np.arange(start, start + k, dtype=np.int64)  # one contiguous block
        else:
            idx = np.sort(rng.choice(K, size=k, replace=False)).astype(np.int64)
        x[:, idx] *= 30
        _hot_k1_case(m, o, x, idx, bits)


def test_hot_quantizer_ties_zeros_and_shapes():
    """Exact .5 ties (grid-aligned rows), signed zero minima, constant rows, and the
    BASELINE shapes' row widths (8192 / 11008 / 28672) through the hot kernel."""
    m = q()
    o = oracle()
    rng = np.random.default_rng(77)
    for bits in (4, 8):
        levels = (1 << bits) - 1
        # grid-aligned: (v - vmin) / scale lands on k + 0.5 exactly for many elements
        g = rng.integers(0, 2 * levels + 1, size=(6, 512)).astype(np.float32) * 0.5
        g[:, 0] = 0.0
        g[:, 1] = levels
        x = g.astype(np.float16)
        x[2, :] = 3.0                      # constant row -> scale 1
        x[3, 5] = -0.0                     # zero min with a negative zero first
        x[3, :5] = np.abs(x[3, :5]) + 1
        _hot_k1_case(m, o, x, np.array([], np.int64), bits)
        _hot_k1_case(m, o, x, np.array([3, 17, 100, 101, 102, 511], np.int64), bits)
    for K, O in [(8192, 256), (11008, 688), (28672, 896)]:
        x = rng.normal(0, 1, size=(3, K)).astype(np.float16)
        idx = np.sort(rng.choice(K, size=O, replace=False)).astype(np.int64)
        _hot_k1_case(m, o, x, idx, 4 if K == 8192 else 8)


def test_hot_quantizer_eight_vector_rows_outlier_fill():
    """Rows of eight 16-byte vectors per thread (K = 8192 / 11008 / 28672: the kernel that
    overwrites a row's outlier columns in shared memory with its first base value
    instead of holding lane masks in registers): outliers holding the row's extreme
    values, outliers before the first base column, zero minima whose first base zero is
    the first base column (-0 / +0) with zeros of the other sign at outlier columns and
    later base columns, constant rows, many rows per CTA."""
    m = q()
    o = oracle()
    rng = np.random.default_rng(7400)
    for K, O, bits, M in [(8192, 256, 4, 600), (11008, 688, 8, 300), (28672, 896, 8, 400)]:
        idx = np.sort(np.concatenate([np.arange(0, 5), rng.choice(np.arange(5, K), size=O - 5, replace=False)]))
        base = np.setdiff1d(np.arange(K), idx)
        x = rng.normal(0, 1, size=(M, K)).astype(np.float16)
        x[0, idx[7]] = -1000.0   # an outlier below every base value
        x[1, idx[9]] = 1000.0    # an outlier above every base value
        for r, (first, other) in ((2, (-0.0, 0.0)), (3, (0.0, -0.0))):
            x[r] = np.abs(x[r]) + np.float16(0.25)
            x[r, base[0]] = first                      # the first base column is the zero minimum
            x[r, base[len(base) // 2]] = other         # a later base zero of the other sign
            x[r, idx[:5]] = other                      # outlier zeros before it, other sign
        x[4] = np.float16(1.5)                         # constant row
        x[5, base] = np.float16(-0.0)                  # all-zero base row, -0 first
        x[5, idx] = np.float16(3.0)
        _hot_k1_case(m, o, x, idx.astype(np.int64), bits)


def test_wide_quantizer_cluster_slices_bit_exact():
    """K1 for wide rows (K > 32768: each row split over a thread-block cluster, one CTA
    per slice, min / max exchanged through distributed shared memory) against the oracle:
    OPT-66B fc2 (36864) and Falcon-180B fc2 (59392) widths and odd ones, outliers
    clustered on the slice boundaries, at the row ends, none at all; exact ties; zero
    minima whose first zero (and its sign) lies in a later slice; more rows than
    co-resident clusters."""
    m = q()
    o = oracle()
    rng = np.random.default_rng(7300)
    for K, M, bits, pattern in [(36864, 300, 8, "random"), (59392, 40, 8, "random"), (40000, 64, 4, "bounds"),
                                (49152, 50, 4, "bounds"), (36864, 30, 8, "ends"), (40960, 30, 4, "none"),
                                (36864, 1200, 4, "random")]:
        C = min(8, -(-K // 8192))
        if pattern == "random":
            idx = np.sort(rng.choice(K, size=K // 32, replace=False))
        elif pattern == "bounds":  # contiguous outlier runs straddling every slice boundary
            runs = [np.arange(max(0, c * K // C - 40), min(K, c * K // C + 25)) for c in range(1, C)]
            idx = np.unique(np.concatenate(runs + [rng.choice(K, size=64, replace=False)]))
        elif pattern == "ends":
            idx = np.concatenate([np.arange(0, 300), np.arange(K - 500, K)])
        else:
            idx = np.array([], np.int64)
        idx = np.asarray(idx, np.int64)
        x = rng.normal(0, 1, size=(M, K)).astype(np.float16)
        if len(idx):
            x[:, idx[::2]] *= 30
        base = np.setdiff1d(np.arange(K), idx)
        # row 0: exact ties on the quantization grid; rows 1-2: zero minimum, the first
        # zero in a late slice (-0 then +0, and +0 then -0); row 3: constant
        levels = (1 << bits) - 1
        g = rng.integers(0, 2 * levels + 1, size=K).astype(np.float32) * 0.5
        g[base[0]], g[base[1]] = 0.0, levels
        x[0] = g.astype(np.float16)
        for r, (s1, s2) in ((1, (-0.0, 0.0)), (2, (0.0, -0.0))):
            if M > r:
                x[r] = np.abs(x[r]) + np.float16(0.5)
                late = base[(len(base) * 3) // 4]
                later = base[(len(base) * 7) // 8]
                x[r, late], x[r, later] = s1, s2
        if M > 3:
            x[3] = np.float16(2.5)
        _hot_k1_case(m, o, x, idx, bits)


# --------------------------------------------------------------------------- 2:4 sparse base weights (cfg5)


def to_sparse_layer(L):
    layer = to_layer(L)
    layer.weights.mask = np.asarray(L["mask"], np.uint8)
    return layer


def test_hot_quantizer_ring_wrap_and_many_outliers():
    """The hot K1 with more rows than CTAs x ring stages (every ring slot refilled at
    barrier A of its row, several times per CTA) at the BASELINE row widths, and with
    more outlier columns than two per thread (the outlier gather from global memory)."""
    m = q()
    o = oracle()
    rng = np.random.default_rng(7100)
    for K, M, O, bits in [(1024, 20000, 600, 4), (2048, 3000, 700, 8), (8192, 2500, 256, 4), (28672, 700, 896, 8)]:
        x = rng.normal(0, 1, size=(M, K)).astype(np.float16)
        idx = np.sort(rng.choice(K, size=O, replace=False)).astype(np.int64)
        x[:, idx[::3]] *= 30
        _hot_k1_case(m, o, x, idx, bits)


def make_sparse_layer(rng, M, K, N, bits, O, heavy_cols=2):
    """RTN layer whose permuted base weights are pruned 2:4 by magnitude (the two
    smallest |w| of every aligned group of 4 base columns -> 0) before quantization."""
    o = oracle()
    L, x, w = make_layer(rng, M, K, N, bits, O, heavy_cols=heavy_cols)
    idx = np.asarray(L["idx"], np.int64)
    base_cols = np.setdiff1d(np.arange(K), idx)
    kb = base_cols.size
    wb = w[:, base_cols].copy()
    g = kb // 4 * 4
    grp = np.abs(wb[:, :g]).reshape(N, -1, 4)
    drop = np.argsort(grp, axis=-1, kind="stable")[..., :2]
    mask = np.ones((N, kb), np.uint8)
    mg = mask[:, :g].reshape(N, -1, 4)
    np.put_along_axis(mg, drop, 0, axis=-1)
    mask[:, :g] = mg.reshape(N, g)
    w2 = w.copy()
    w2[:, base_cols] = wb * mask
    q = o.rtn_quantize_weights(w2, idx, bits)
    L.update(base=q["base"], scales=q["scales"], wreduced=q["wreduced"], mask=mask)
    return L, x


@pytest.mark.parametrize("name", sorted(n for n in _CASES if n.startswith("sp24_")))
def test_sparse_device_matches_reference_golden(name):
    """2:4 sparse layers from the reference's sparsegpt_joint (tests/golden): the device
    compresses them and runs tcgen05.mma.sp; outputs vs the reference quik_matmul."""
    m = q()
    import torch

    meta = _CASES[name]
    g = lambda k: _G[f"{name}.{k}"]  # noqa: E731
    K, N, O, bits = meta["K"], meta["N"], meta["outliers"], meta["bits"]
    L = dict(in_features=K, out_features=N, bits=bits, base=g("base"), scales=g("scales"), wreduced=g("wreduced"),
             outlier_weights=g("outlier_weights"), idx=g("idx"), bias=g("bias"), mask=g("mask"))
    dev = m.QuikLinear(to_sparse_layer(L))
    # a trailing dense remainder group of 3 base columns is not 2:4 -> the layer stays dense
    assert dev.is_sparse == (not name.endswith("tail3")), name
    x = g("x")
    xt = torch.from_numpy(x).cuda()
    want = g("out_v3")
    for v in m.PipelineVariant:
        y = dev(xt, out_dtype=torch.float32, variant=v).cpu().numpy()
        if O == 0:
            np.testing.assert_array_equal(y.view(np.uint32), want.view(np.uint32))
        else:
            assert rel_frob(want, y) < 1e-5, (v, rel_frob(want, y))
    y16 = dev(xt.half()).float().cpu().numpy()
    assert rel_frob(want, y16) <= 5e-4


@pytest.mark.parametrize("cg,bn", [(1, 32), (1, 64), (1, 128), (2, 128), (2, 192)])
def test_sparse_every_tile_config_exact(tile, cg, bn):
    """Each sparse GEMM tile: O = 0 layers bit-exact (f32 out, so the INT32
    accumulators of the compressed MMAs are exact), outlier layers within tolerance,
    V1 = V2 = V3, ragged M / N / K."""
    m = q()
    o = oracle()
    import torch

    assert tile(cg, bn) == 0
    rng = np.random.default_rng(500 + 10 * cg + bn)
    for (M, K, N, bits, O) in [(300, 1024, 500, 4, 0), (77, 600, 257, 8, 0), (200, 1100, 384, 4, 64)]:
        L, x = make_sparse_layer(rng, M, K, N, bits, O)
        st, want = o.quik_matmul(L, x, 2)
        assert st == 0
        dev = m.QuikLinear(to_sparse_layer(L))
        assert dev.is_sparse
        xt = torch.from_numpy(x).cuda()
        outs = [dev(xt, out_dtype=torch.float32, variant=v).cpu().numpy() for v in m.PipelineVariant]
        for y in outs:
            np.testing.assert_array_equal(y.view(np.uint32), outs[2].view(np.uint32))
        if O == 0:
            np.testing.assert_array_equal(outs[2].view(np.uint32), want.view(np.uint32))
        else:
            assert rel_frob(want, outs[2]) < 1e-5
    # many tiles per persistent CTA: the oracle on a token / row subset (rows independent)
    M, K, N = 2048, 1024, 3000
    L, x = make_sparse_layer(rng, M, K, N, 4, 0)
    dev = m.QuikLinear(to_sparse_layer(L))
    assert dev.is_sparse
    y = dev(torch.from_numpy(x).cuda(), out_dtype=torch.float32).cpu().numpy()
    toks = np.unique(np.concatenate([rng.choice(M, 5, replace=False), [0, M - 1]]))
    rows = np.unique(np.concatenate([rng.choice(N, 200, replace=False), [0, N - 1]]))
    sub = dict(L)
    sub["out_features"] = rows.size
    sub["base"] = np.asarray(L["base"]).reshape(N, row_bytes(K, 4))[rows].reshape(-1)
    for key in ("scales", "wreduced", "bias"):
        sub[key] = np.asarray(L[key])[rows]
    sub["outlier_weights"] = np.zeros((rows.size, 0), np.float32)
    if "mask" in L:
        sub["mask"] = np.asarray(L["mask"]).reshape(N, -1)[rows]
    st, want = o.quik_matmul(sub, x[toks], 2)
    assert st == 0
    np.testing.assert_array_equal(y[np.ix_(toks, rows)].view(np.uint32), want.view(np.uint32))


def test_sparse_not_compressible_stays_dense():
    """A layer flagged sparse whose groups hold 3+ non-zero codes stays on the dense
    GEMM (no silent wrong answers)."""
    m = q()
    o = oracle()
    rng = np.random.default_rng(9)
    L, x, _ = make_layer(rng, 20, 256, 64, 4, 0)
    L["mask"] = np.ones((64, 256), np.uint8)
    dev = m.QuikLinear(to_sparse_layer(L))
    assert not dev.is_sparse
    st, want = o.quik_matmul(L, x, 2)
    got = m.quik_matmul(to_layer(L), x)
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


# --------------------------------------------------------------------------- weight-streaming path (M <= 64)


@pytest.mark.parametrize("bits", [4, 8])
def test_stream_gemm_bit_identical_to_fused(bits):
    """Small-M forwards: the decode kernel (default for dense layers at M <= 32: split-K
    GEMM on INT4 weights widened into TMEM (4-bit) or INT8 tiles (8-bit) + the fused
    epilogue finalised by the last CTA of each weight block) against the fused kernel.
    Integer sums are exact and the epilogue instructions are the fused kernel's, so both
    are bit-identical (f32 and f16 out, repeat calls: the workspace and counters are left
    zeroed), and equal to the reference when O = 0."""
    m = q()
    o = oracle()
    import torch

    lib = m.load_library()
    rng = np.random.default_rng(900 + bits)
    try:
        for (M, K, N, O) in [(1, 1024, 4096, 64), (7, 3000, 384, 32), (16, 4096, 1000, 128), (33, 640, 2048, 0),
                             (64, 2048, 512, 16), (20, 1000, 300, 8), (32, 8192, 2048, 256)]:
            L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=3)
            dev = m.QuikLinear(to_layer(L))
            xt = torch.from_numpy(x).cuda()
            for dt in (torch.float32, torch.float16):
                outs = []
                for decode in (0, 1, 1):
                    lib.quik_set_int4_decode(decode)
                    outs.append(dev(xt, out_dtype=dt).cpu().numpy())
                u = np.uint32 if dt == torch.float32 else np.uint16
                for y in outs[1:]:
                    np.testing.assert_array_equal(y.view(u), outs[0].view(u))
            if O == 0:
                lib.quik_set_int4_decode(1)
                st, want = o.quik_matmul(L, x, 2)
                got = dev(xt, out_dtype=torch.float32).cpu().numpy()
                np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    finally:
        lib.quik_set_int4_decode(1)


@pytest.mark.parametrize("name", ["f16_w4_o64", "sp24_w4_o16"])
def test_bundle_to_device_matches_reference(name):
    """Reference layer bundles (tests/golden/bundle_*, written by the reference's
    save_layer) loaded straight into the device layout (quik_layer_load_bundle): the
    forward matches the reference quik_matmul outputs of the same layer, the sparse
    bundle runs the 2:4 GEMM, and a row-shard load equals the slice of the full layer."""
    m = q()
    import torch
    from pathlib import Path

    d = Path(__file__).resolve().parent / "golden" / f"bundle_{name}"
    g = lambda k: _G[f"{name}.{k}"]  # noqa: E731
    dev = m.QuikLinear.from_bundle(d)
    assert dev.is_sparse == name.startswith("sp24")
    xt = torch.from_numpy(g("x")).cuda()
    y = dev(xt, out_dtype=torch.float32).cpu().numpy()
    assert rel_frob(g("out_v3"), y) < 1e-5
    N = dev.out_features
    r0, r1 = N // 3, N // 3 + 64
    shard = m.QuikLinear.from_bundle(d, row_begin=r0, row_end=r1)
    ys = shard(xt, out_dtype=torch.float32).cpu().numpy()
    np.testing.assert_array_equal(ys.view(np.uint32), y[:, r0:r1].view(np.uint32))
    host = m.load_layer(d)  # reference semantics: host arrays
    np.testing.assert_array_equal(m.quik_matmul(host, g("x")).view(np.uint32), y.view(np.uint32))


# --------------------------------------------------------------------------- gated MLP (§8f.2)


def _mlp_layers(rng, M, K, F, bits_ud, bits_down, O, O_down):
    """up / gate sharing the outlier set selected from x (the same input), and a down
    projection with its own outliers; RTN weights through the oracle. Weights are scaled
    so the hidden state h stays inside the f16 range of the outlier operands (the device
    path rounds outlier activations to f16, |x| <= 65504)."""
    o = oracle()
    up, x, w = make_layer(rng, M, K, F, bits_ud, O, heavy_cols=3)
    qu = o.rtn_quantize_weights(w * 0.02, up["idx"], bits_ud)
    up.update(base=qu["base"], scales=qu["scales"], wreduced=qu["wreduced"],
              outlier_weights=qu["outlier_weights"].astype(np.float16).astype(np.float32))
    wg = rng.normal(0.0, 0.01, size=(F, K)).astype(np.float32)
    qg = o.rtn_quantize_weights(wg, up["idx"], bits_ud)
    gate = dict(up, base=qg["base"], scales=qg["scales"], wreduced=qg["wreduced"],
                outlier_weights=qg["outlier_weights"].astype(np.float16).astype(np.float32),
                bias=rng.normal(0.0, 0.1, size=F).astype(np.float32))
    wd = rng.normal(0.0, 0.5, size=(K, F)).astype(np.float32)
    idx_d = np.sort(rng.choice(F, size=O_down, replace=False)).astype(np.int64)
    qd = o.rtn_quantize_weights(wd, idx_d, bits_down)
    down = dict(in_features=F, out_features=K, bits=bits_down, act_bits=bits_down, base=qd["base"],
                scales=qd["scales"], wreduced=qd["wreduced"],
                outlier_weights=qd["outlier_weights"].astype(np.float16).astype(np.float32), idx=idx_d,
                bias=rng.normal(0.0, 0.1, size=K).astype(np.float32))
    return up, gate, down, x


@pytest.mark.parametrize("bits", [4, 8])
def test_gated_projection_and_mlp_match_reference(bits):
    """h = silu(gate(x)) * up(x) from ONE fused layer (shared K1, interleaved up/gate
    rows, silu * up in the epilogue) and the whole block down(h) against the reference's
    forward_model(gated_mlp_ops) (runtime.cpp:325-388)."""
    m = q()
    r = ref()
    import torch

    rng = np.random.default_rng(600 + bits)
    for (M, K, F, O, Od) in [(40, 256, 160, 32, 16), (300, 512, 384, 64, 32), (7, 384, 96, 0, 0)]:
        up, gate, down, x = _mlp_layers(rng, M, K, F, bits, 8, O, Od)
        st, want, want_h = r.gated_mlp(up, gate, down, x)
        assert st == 0
        proj = m.QuikLinear.gated(to_layer(up), to_layer(gate))
        assert proj.out_features == F
        xt = torch.from_numpy(x).cuda()
        h32 = proj(xt, out_dtype=torch.float32).cpu().numpy()
        assert rel_frob(want_h, h32) < 1e-5, rel_frob(want_h, h32)  # exp ulps + f16 outlier order
        for v in m.PipelineVariant:  # V1 / V2 / V3 identical on the device
            hv = proj(xt, out_dtype=torch.float32, variant=v).cpu().numpy()
            np.testing.assert_array_equal(hv.view(np.uint32), h32.view(np.uint32))
        mlp = m.QuikGatedMLP(to_layer(up), to_layer(gate), to_layer(down))
        y32 = mlp(xt, out_dtype=torch.float32, hidden_dtype=torch.float32).cpu().numpy()
        # f32 h: the down projection's quantizer sees h within ~1e-6 relative of the
        # reference's h, which can move a code by one step (rounding discontinuity)
        assert rel_frob(want, y32) < 1e-3, rel_frob(want, y32)
        # f16 block: h is rounded to f16 between the projections (the reference keeps it
        # in f32), so each projection is checked against the reference on ITS input
        h16 = mlp.proj(xt.half())
        hh = h16.float().cpu().numpy()
        assert rel_frob(want_h, hh) <= 5e-4, rel_frob(want_h, hh)
        # the f16 epilogue rounds the same f32 value the f32 epilogue writes
        np.testing.assert_array_equal(h16.cpu().numpy().view(np.uint16),
                                      h32.astype(np.float16).view(np.uint16))
        y16 = mlp.down(h16).float().cpu().numpy()
        st, want_d = r.quik_matmul(down, hh, 2)
        assert st == 0
        assert np.all(np.abs(y16 - want_d) <= f16_output_bound(down, hh, want_d))
        assert rel_frob(want_d, y16) <= 5e-4
        if F % 64 == 0:  # 32-feature-aligned row shard == slice of the full projection
            sh = m.QuikLinear.gated(to_layer(up), to_layer(gate), row_begin=32, row_end=96)
            hs = sh(xt, out_dtype=torch.float32).cpu().numpy()
            np.testing.assert_array_equal(hs.view(np.uint32), h32[:, 32:96].view(np.uint32))


@pytest.mark.parametrize("cg,bn", [(1, 32), (1, 128), (2, 128), (2, 256)])
def test_gated_projection_every_tile(tile, cg, bn):
    m = q()
    import torch

    rng = np.random.default_rng(700 + bn)
    up, gate, down, x = _mlp_layers(rng, 260, 640, 320, 4, 8, 64, 16)
    proj = m.QuikLinear.gated(to_layer(up), to_layer(gate))
    xt = torch.from_numpy(x).cuda()
    want = proj(xt, out_dtype=torch.float32).cpu().numpy()
    assert tile(cg, bn) == 0
    got = proj(xt, out_dtype=torch.float32).cpu().numpy()
    np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))


# --------------------------------------------------------------------------- weight-only (§8f.3)


def _wo_bound(L, x, K_eff):
    """Per-element error bound of the weight-only kernel vs FP64: exact products, the
    f32 hi/lo split residuals (2^-22 relative) and an f32 summation over K terms
    (gamma_K = K 2^-24), all relative to S = sum_k |x_k| |w_k| (+ |bias|)."""
    from oracle_lib import oracle as _o

    chk = _o()
    K, N = L["in_features"], L["out_features"]
    idx = np.asarray(L["idx"], np.int64)
    kb = K - idx.size
    st, perm = chk.permutation(K, idx)
    qv = np.abs(chk.unpack(L["base"], N, kb, L["bits"]).astype(np.float64))
    w = np.zeros((N, K), np.float64)
    w[:, perm[:kb]] = qv * np.abs(np.asarray(L["scales"], np.float64))[:, None]
    if idx.size:
        w[:, idx] = np.abs(np.asarray(L["outlier_weights"], np.float64))
    S = np.abs(np.asarray(x, np.float64)) @ w.T
    if L.get("bias") is not None:
        S += np.abs(np.asarray(L["bias"], np.float64))[None, :]
    return (K_eff * 2.0 ** -24 + 2.0 ** -20) * S


@pytest.mark.parametrize("bits", [4, 8])
def test_weight_only_matches_reference(bits):
    """LayerMode::WeightOnly (runtime.cpp:115-136) on the device: f32 activations (two
    f16 planes) -> f32 out meets the reference test's bar (rel Frobenius < 1e-6 vs FP64,
    test_runtime.cpp:284-300) and a per-element bound; f16 activations -> f16 out within
    half an f16 ulp + the same bound. Shapes cover the direct-store path (one split),
    split-K + finalize, ragged N / K, O = 0, no bias, and M up to 300."""
    from oracle_lib import rel_frobenius, weight_only_f64

    m = q()
    import torch

    rng = np.random.default_rng(4100 + bits)
    cases = [(1, 4096, 4096, 64), (7, 64, 24, 8), (16, 3000, 1000, 128), (33, 640, 2048, 0), (5, 1024, 300, 16),
             (300, 2048, 512, 32), (1024, 512, 4096, 64), (2, 200, 129, 4)]
    for (M, K, N, O) in cases:
        L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=2, with_bias=(M % 2 == 1), fp16_inputs=False)
        dev = m.QuikLinear(to_layer(L))
        # f32 in -> f32 out
        y = dev.weight_only(torch.from_numpy(x).cuda(), out_dtype=torch.float32).cpu().numpy()
        want = weight_only_f64(L, x)
        assert rel_frobenius(want, y) < 1e-6, (M, K, N, O)
        assert np.all(np.abs(y - want) <= _wo_bound(L, x, K) + 1e-30), (M, K, N, O)
        # f16 in -> f16 out (the decode hot path)
        x16 = x.astype(np.float16)
        y16 = dev.weight_only(torch.from_numpy(x16).cuda()).cpu().numpy().astype(np.float64)
        want16 = weight_only_f64(L, x16.astype(np.float32))
        tol = F16_REL * np.abs(want16) + _wo_bound(L, x16.astype(np.float32), K) * 2 + 6.0e-8
        assert np.all(np.abs(y16 - want16) <= tol), (M, K, N, O)
        # deterministic (fixed-order split reduction)
        y2 = dev.weight_only(torch.from_numpy(x).cuda(), out_dtype=torch.float32).cpu().numpy()
        np.testing.assert_array_equal(y.view(np.uint32), y2.view(np.uint32))


def test_weight_only_keeps_activations_in_fp():
    """test_runtime.cpp:284-300 on the device: weight-only vs FP64 of the dequantized
    weights < 1e-6, and its error vs the FP product is no larger than quik mode's."""
    from oracle_lib import rel_frobenius, weight_only_f64

    m = q()
    import torch

    rng = np.random.default_rng(137)
    L, x, w = make_layer(rng, 7, 64, 24, 4, 8, heavy_cols=2, fp16_inputs=False)
    dev = m.QuikLinear(to_layer(L))
    xt = torch.from_numpy(x).cuda()
    out = dev.weight_only(xt, out_dtype=torch.float32).cpu().numpy()
    assert rel_frobenius(weight_only_f64(L, x), out) < 1e-6
    fp_ref = x.astype(np.float64) @ w.astype(np.float64).T + L["bias"].astype(np.float64)[None, :]
    quik_out = dev(xt, out_dtype=torch.float32).cpu().numpy()
    assert rel_frobenius(fp_ref, out) <= rel_frobenius(fp_ref, quik_out)


def test_weight_only_rejects_gated_and_compressed_layers():
    m = q()
    import torch

    rng = np.random.default_rng(9)
    up, x, _ = make_layer(rng, 4, 256, 64, 4, 16)
    gate = dict(up)
    g = m.QuikLinear.gated(to_layer(up), to_layer(gate))
    with pytest.raises(NotImplementedError):
        g.weight_only(torch.from_numpy(x).cuda())


# --------------------------------------------------------------------------- fused all-gather (§8e)


@pytest.mark.parametrize("M,stream", [(300, 0), (16, 0), (16, 1)])
def test_sharded_forward_fused_all_gather(M, stream):
    """quik_linear_forward_sharded: each output-row shard TMA-stores its tiles into
    EVERY destination (here two buffers on one GPU standing in for the local and a
    peer output). After both shards ran, each destination equals the unsharded forward
    bit for bit (the per-element arithmetic does not depend on the sharding)."""
    m = q()
    import torch

    lib = m.load_library()
    rng = np.random.default_rng(77 + M)
    L, x, _ = make_layer(rng, M, 1024, 768, 4, 32, heavy_cols=2)
    layer = to_layer(L)
    full = m.QuikLinear(layer)
    xt = torch.from_numpy(x).cuda().half()
    try:
        lib.quik_set_int4_decode(1 - stream)
        want = full(xt)
        ns = 768 // 3
        shards = [m.QuikLinear(layer, row_begin=r * ns, row_end=(r + 1) * ns) for r in range(3)]
        outs = [torch.full((M, 768), float("nan"), dtype=torch.float16, device="cuda") for _ in range(2)]
        for r, sh in enumerate(shards):
            sh.forward_sharded(xt, outs, r * ns)
        torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o.view(torch.int16), want.view(torch.int16))
    finally:
        lib.quik_set_int4_decode(1)
    with pytest.raises(NotImplementedError):  # pitch / offset not TMA-aligned
        shards[0].forward_sharded(xt, [torch.empty((M, 770), dtype=torch.float16, device="cuda")], 3)


def test_decode_path_under_graph_capture():
    """A small-M forward captured into a CUDA graph before the decode workspace exists
    (the warm-up ran the fused path) takes the fused path instead of allocating inside
    the capture; after a decode warm-up the captured forward runs the INT4 decode
    kernel. Both replay bit-identically to the eager fused forward."""
    m = q()
    import torch

    rng = np.random.default_rng(5)
    L, x, _ = make_layer(rng, 8, 2048, 4096, 4, 32, heavy_cols=2)
    lib = m.load_library()
    m.quik._ctxs.clear()  # a fresh context: no decode workspace yet
    dev = m.QuikLinear(to_layer(L))
    xt = torch.from_numpy(x).cuda().half()
    try:
        for warm_decode in (0, 1):
            lib.quik_set_int4_decode(warm_decode)
            want = dev(xt)  # warm-up (sizes K1 buffers; the decode workspace only when warm_decode)
            torch.cuda.synchronize()
            lib.quik_set_int4_decode(1)
            y = torch.empty_like(want)
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                dev(xt, out=y)
            y.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(y.view(torch.int16), want.view(torch.int16))
    finally:
        lib.quik_set_int4_decode(1)


# --------------------------------------------------------------------------- GPU GPTQ / SparseGPT (§8f.4)


def _gptq_case(rng, N, K, O, T, heavy=2):
    w = (rng.normal(0.0, 0.5, size=(N, K))).astype(np.float32)
    x = rng.normal(0.0, 1.0, size=(T, K)).astype(np.float32)
    for _ in range(heavy):
        x[:, int(rng.integers(0, K))] *= 20.0
    idx = np.sort(rng.choice(K, size=O, replace=False)).astype(np.int64)
    return w, x, idx


@pytest.mark.parametrize("sparse", [0, 1])
def test_gptq_identity_hessian_bit_exact(sparse):
    """H = I: no error compensation, so the device GPTQ / SparseGPT equal the
    reference's bit for bit (codes, scales, wreduced, outlier weights, 2:4 mask), with
    and without the clip search, 4 and 8 bits."""
    m = q()
    r = ref()
    rng = np.random.default_rng(31 + sparse)
    for bits in (4, 8):
        for clip in (False, True):
            N, K, O = 48, 200, 8
            w, _, idx = _gptq_case(rng, N, K, O, 1)
            st, want = r.gptq(w, idx, bits, None, 1, 0.01, clip, bool(sparse))
            assert st == 0
            got = m.gptq_quantize_device(w, m.OutlierSet.from_indices(K, idx), bits, np.eye(K), 0.01, clip, bool(sparse))
            np.testing.assert_array_equal(got.base.data, want["base"])
            np.testing.assert_array_equal(got.scales.view(np.uint32), want["scales"].view(np.uint32))
            np.testing.assert_array_equal(got.wreduced.view(np.uint32), want["wreduced"].view(np.uint32))
            np.testing.assert_array_equal(got.outlier_weights, want["outlier_weights"])
            if sparse:
                np.testing.assert_array_equal(got.mask, want["mask"])


@pytest.mark.parametrize("sparse", [0, 1])
def test_gptq_matches_reference(sparse):
    """Calibrated Hessians (heavy activation columns): the device GPTQ / SparseGPT vs
    the reference's gptq_quantize / sparsegpt_joint on the same Hessian. The Cholesky
    factor (cuSOLVER) and the blocked trailing updates (DGEMM) differ from the
    reference's loops only by FP64 rounding, so codes, masks and scales agree exactly
    and the outlier weights to float rounding; crossing a block boundary (K > 64) and
    a trailing partial block are covered."""
    m = q()
    r = ref()
    rng = np.random.default_rng(41 + sparse)
    for (N, K, O, T, bits, clip) in [(64, 96, 4, 256, 4, False), (40, 333, 16, 512, 4, True),
                                     (96, 256, 0, 300, 8, False), (33, 150, 10, 128, 8, True)]:
        w, x, idx = _gptq_case(rng, N, K, O, T)
        h = r.build_hessian(x)
        st, want = r.gptq(w, idx, bits, h, T, 0.01, clip, bool(sparse))
        assert st == 0
        got = m.gptq_quantize_device(w, m.OutlierSet.from_indices(K, idx), bits, h, 0.01, clip, bool(sparse))
        codes_got = m.unpack_values(got.base)
        codes_want = m.unpack_values(m.PackedIntMatrix(N, K - O, bits, want["base"]))
        agree = float((codes_got == codes_want).mean())
        assert agree == 1.0, (N, K, O, agree)
        np.testing.assert_array_equal(got.scales.view(np.uint32), want["scales"].view(np.uint32))
        np.testing.assert_array_equal(got.wreduced.view(np.uint32), want["wreduced"].view(np.uint32))
        np.testing.assert_allclose(got.outlier_weights, want["outlier_weights"], rtol=1e-6, atol=1e-6)
        if sparse:
            np.testing.assert_array_equal(got.mask, want["mask"])


def test_hessian_device_and_not_positive_definite():
    """The FP64 Hessian sum on the device equals the reference's to FP64 rounding; a
    Hessian that stays singular after damping (zero trace) raises NumericalError like
    the reference (quantizer.cpp:84-91)."""
    m = q()
    r = ref()
    rng = np.random.default_rng(5)
    x = rng.normal(size=(300, 72)).astype(np.float32)
    h = m.hessian_device([x[:100], x[100:]]).cpu().numpy()
    np.testing.assert_allclose(h, r.build_hessian(x), rtol=1e-12, atol=1e-9)
    w = rng.normal(size=(8, 72)).astype(np.float32)
    st, _ = r.gptq(w, np.array([], np.int64), 4, np.zeros((72, 72)), 1, 0.01)
    assert st == 3  # reference: NumericalError
    with pytest.raises(m.NumericalError):
        m.gptq_quantize_device(w, m.OutlierSet.from_indices(72, []), 4, np.zeros((72, 72)))


def test_sharded_quik_linear_nccl_world1():
    """The torch.distributed path of ShardedQuikLinear over NCCL on the device (world
    size 1 here: one GPU): shard upload, forward and all-gather equal the unsharded
    layer bit for bit."""
    import os

    import torch
    import torch.distributed as dist

    m = q()
    from paper_2310_09259_b200.sharded import ShardedQuikLinear

    rng = np.random.default_rng(12)
    L, x, _ = make_layer(rng, 96, 512, 384, 4, 16, heavy_cols=2)
    layer = to_layer(L)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29543")
    created = not dist.is_initialized()
    if created:
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        xt = torch.from_numpy(x).cuda().half()
        got = ShardedQuikLinear(layer, device=0).forward(xt)
        want = m.QuikLinear(layer)(xt)
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int16), want.view(torch.int16))
    finally:
        if created:
            dist.destroy_process_group()


def test_gated_projection_decode_kernel_bit_identical():
    """4-bit gated projections at M <= 32 run the INT4 decode kernel, whose finalisation
    pairs the gate / up quadrants like the fused epilogue: identical bits to the fused
    path (decode off), f32 and f16 out, full layer and a 64-feature row shard."""
    m = q()
    import torch

    lib = m.load_library()
    rng = np.random.default_rng(4242)
    try:
        for (M, K, F, O) in [(1, 512, 256, 32), (16, 1024, 640, 0), (29, 768, 384, 64)]:
            up, gate, down, x = _mlp_layers(rng, M, K, F, 4, 8, O, 0)
            xt = torch.from_numpy(x).cuda().half()
            for rb, re_ in [(0, 0), (64, 192)]:
                proj = m.QuikLinear.gated(to_layer(up), to_layer(gate), row_begin=rb, row_end=re_)
                for dt in (torch.float32, torch.float16):
                    lib.quik_set_int4_decode(0)
                    want = proj(xt, out_dtype=dt)
                    lib.quik_set_int4_decode(1)
                    got = proj(xt, out_dtype=dt)
                    u = torch.int32 if dt == torch.float32 else torch.int16
                    assert torch.equal(got.view(u), want.view(u)), (M, F, rb, dt)
    finally:
        lib.quik_set_int4_decode(1)


def test_decode_kernel_fuzz_bit_identical():
    """60 random small-M layers (M 1-32, ragged K / N, 0-256 outliers, 4 and 8 bits,
    with and without bias, f16 / f32 out): the decode kernel equals the fused kernel
    bit for bit, and repeated calls stay identical (workspace / counters reset)."""
    m = q()
    import torch

    lib = m.load_library()
    rng = np.random.default_rng(2024)
    try:
        for trial in range(60):
            bits = 4 if trial % 2 == 0 else 8
            M = int(rng.integers(1, 33))
            K = int(rng.integers(64, 3000))
            N = int(rng.integers(1, 1500))
            O = int(min(rng.choice([0, 8, 64, 256]), K // 4))
            L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=2, with_bias=bool(trial % 3))
            dev = m.QuikLinear(to_layer(L))
            xt = torch.from_numpy(x).cuda()
            dt = torch.float16 if trial % 4 < 2 else torch.float32
            lib.quik_set_int4_decode(0)
            want = dev(xt, out_dtype=dt)
            lib.quik_set_int4_decode(1)
            got1 = dev(xt, out_dtype=dt)
            got2 = dev(xt, out_dtype=dt)
            u = torch.int16 if dt == torch.float16 else torch.int32
            assert torch.equal(got1.view(u), want.view(u)), (trial, M, K, N, O, bits)
            assert torch.equal(got2.view(u), want.view(u)), (trial, "repeat")
        # more (weight block, K split) units than CTAs: several units per persistent CTA
        for (M, K, N, O, bits) in [(1, 4096, 8192, 128, 4), (16, 4096, 8192, 256, 8), (32, 2048, 12288, 64, 4)]:
            L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=2, with_bias=True)
            dev = m.QuikLinear(to_layer(L))
            xt = torch.from_numpy(x).cuda()
            lib.quik_set_int4_decode(0)
            want = dev(xt, out_dtype=torch.float32)
            lib.quik_set_int4_decode(1)
            got = dev(xt, out_dtype=torch.float32)
            assert torch.equal(got.view(torch.int32), want.view(torch.int32)), (M, K, N, O, bits)
    finally:
        lib.quik_set_int4_decode(1)


def test_weight_only_fuzz():
    """30 random layers through the weight-only kernel (M 1-40, ragged K / N, 0-128
    outliers, 4 / 8 bits, f32 in): rel Frobenius < 1e-6 vs FP64 (the reference test's
    bar) and repeat calls bit-identical."""
    from oracle_lib import rel_frobenius, weight_only_f64

    m = q()
    import torch

    rng = np.random.default_rng(77)
    for trial in range(30):
        bits = 4 if trial % 2 == 0 else 8
        M = int(rng.integers(1, 41))
        K = int(rng.integers(32, 2500))
        N = int(rng.integers(1, 1200))
        O = int(min(rng.choice([0, 4, 32, 128]), K // 4))
        L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=2, with_bias=bool(trial % 3), fp16_inputs=False)
        dev = m.QuikLinear(to_layer(L))
        xt = torch.from_numpy(x).cuda()
        y1 = dev.weight_only(xt, out_dtype=torch.float32).cpu().numpy()
        y2 = dev.weight_only(xt, out_dtype=torch.float32).cpu().numpy()
        assert rel_frobenius(weight_only_f64(L, x), y1) < 1e-6, (trial, M, K, N, O, bits)
        np.testing.assert_array_equal(y1.view(np.uint32), y2.view(np.uint32))
    # more (weight block, K split) units than CTAs
    for (M, K, N, O, bits) in [(1, 4096, 8192, 128, 4), (40, 2048, 12288, 32, 8)]:
        L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=2, with_bias=True, fp16_inputs=False)
        dev = m.QuikLinear(to_layer(L))
        y = dev.weight_only(torch.from_numpy(x).cuda(), out_dtype=torch.float32).cpu().numpy()
        assert rel_frobenius(weight_only_f64(L, x), y) < 1e-6, (M, K, N, O, bits)


# --------------------------------------------------------------------------- rest of the reference surface


@pytest.mark.parametrize("bits", [4, 8])
def test_rtn_clipping_compute_wreduced_dequantize_weights_vs_reference(bits):
    """rtn_quantize_weights(use_clipping) (clip_search, quantizer.cpp:266-290),
    compute_wreduced (:373-382) and dequantize_weights (:384-403) on the device against
    the reference's own sources, bit-exact."""
    m = q()
    r = ref()
    rng = np.random.default_rng(900 + bits)
    for (N, K, O) in [(33, 257, 7), (300, 4096, 128), (5, 40, 0)]:
        w = rng.normal(0, 0.5, size=(N, K)).astype(np.float32)
        w[0] = 0.0
        w[1, ::5] *= 30.0
        idx = np.sort(rng.choice(K, O, replace=False)).astype(np.int64)
        os_ = m.OutlierSet.from_indices(K, idx)
        want = r.rtn_quantize_weights(w, idx, bits, use_clipping=True)
        got = m.rtn_quantize_weights(w, os_, bits, use_clipping=True)
        np.testing.assert_array_equal(got.base.data, want["base"])
        np.testing.assert_array_equal(got.scales.view(np.uint32), want["scales"].view(np.uint32))
        np.testing.assert_array_equal(got.wreduced.view(np.uint32), want["wreduced"].view(np.uint32))
        np.testing.assert_array_equal(m.compute_wreduced(got).view(np.uint32), want["wreduced"].view(np.uint32))
        dq = m.dequantize_weights(got, os_)
        np.testing.assert_array_equal(dq.view(np.uint32), r.dequantize_weights(
            want["base"], N, K, idx, bits, want["scales"], want["outlier_weights"]).view(np.uint32))


def test_split_and_unpack_match_reference():
    """split_activations (runtime.cpp:169-186) and unpack_int4 / unpack_values
    (packed.cpp:68-91) through the device kernels."""
    m = q()
    o = oracle()
    rng = np.random.default_rng(905)
    x = rng.normal(size=(9, 300)).astype(np.float32)
    idx = np.sort(rng.choice(300, 20, replace=False))
    os_ = m.OutlierSet.from_indices(300, idx)
    xb, xo = m.split_activations(x, os_)
    np.testing.assert_array_equal(xb, x[:, os_.permutation[:280]])
    np.testing.assert_array_equal(xo, x[:, idx])
    with pytest.raises(ValueError):
        m.split_activations(x[:, :299], os_)
    for bits, cols in [(4, 7), (4, 64), (8, 33)]:
        v = rng.integers(-8 if bits == 4 else -128, 8 if bits == 4 else 128, size=(5, cols))
        pk = m.pack_values(v, 5, cols, bits)
        from paper_2310_09259_b200.quik import _unpack_device

        np.testing.assert_array_equal(_unpack_device(pk), v.astype(np.int8))
        np.testing.assert_array_equal(_unpack_device(pk), o.unpack(pk.data, 5, cols, bits))
        if bits == 4:
            np.testing.assert_array_equal(m.unpack_int4(pk), v.astype(np.int8))
        else:
            with pytest.raises(ValueError):
                m.unpack_int4(pk)


def test_stage_times_per_stage():
    """StageTimes (runtime.hpp:72-80): per-stage CUDA-event times with the reference's
    fused-stage convention; the timed forward equals the untimed one."""
    m = q()
    rng = np.random.default_rng(907)
    L, x, _ = make_layer(rng, 64, 1024, 768, 4, 32, heavy_cols=2)
    layer = to_layer(L)
    t3, t2, t1 = m.StageTimes(), m.StageTimes(), m.StageTimes()
    y3 = m.quik_matmul(layer, x, m.PipelineVariant.V3FusedEpilogue, t3)
    y2 = m.quik_matmul(layer, x, m.PipelineVariant.V2FusedQuant, t2)
    y1 = m.quik_matmul(layer, x, m.PipelineVariant.V1Unfused, t1)
    assert t3.quantize_fused and t3.dequantize_fused and t3.quantize_ms > 0 and t3.int_matmul_ms > 0
    assert t3.split_ms == 0 and t3.fp_matmul_ms == 0 and t3.dequantize_ms == 0
    assert t2.quantize_fused and t2.quantize_ms > 0 and t2.int_matmul_ms > 0 and t2.fp_matmul_ms > 0
    assert not t1.quantize_fused and t1.split_ms > 0 and t1.quantize_ms > 0 and t1.int_matmul_ms > 0
    for y in (y2, y1):
        np.testing.assert_array_equal(y.view(np.uint32), y3.view(np.uint32))
    np.testing.assert_array_equal(m.quik_matmul(layer, x).view(np.uint32), y3.view(np.uint32))


def test_forward_model_gated_mlp_ops_vs_reference():
    """forward_model(gated_mlp_ops) (runtime.cpp:325-382) with every value on the device
    against the reference's forward_model: the up / gate values bit-exact at O = 0, the
    block within the down layer's quantizer sensitivity."""
    m = q()
    r = ref()
    rng = np.random.default_rng(909)
    up, gate, down, x = _mlp_layers(rng, 24, 256, 128, 4, 8, 0, 8)
    layers = [to_layer(up), to_layer(gate), to_layer(down)]
    tr = m.forward_model_trace(layers, m.gated_mlp_ops(), x)
    assert len(tr) == 6
    st, want, want_h = r.gated_mlp(up, gate, down, x)
    assert st == 0
    for i, L in ((1, up), (2, gate)):
        s2, w2 = r.quik_matmul(L, x, 2)
        np.testing.assert_array_equal(tr[i].view(np.uint32), w2.view(np.uint32))
    assert rel_frob(want_h, tr[4]) < 1e-6
    assert rel_frob(want, tr[5]) < 1e-3
    np.testing.assert_array_equal(m.forward_model(layers, m.gated_mlp_ops(), x), tr[5])
    with pytest.raises(ValueError):
        m.forward_model(layers, [m.BlockOp(m.BlockOp.Kind.Linear, 0, -1, 5)], x)
    with pytest.raises(ValueError):
        m.forward_model(layers, [], x)


def test_forward_output_validation():
    """outputs of a wrong dtype, shape or device are rejected before the C ABI."""
    m = q()
    import torch

    rng = np.random.default_rng(911)
    L, x, _ = make_layer(rng, 8, 256, 128, 4, 16, heavy_cols=1)
    dev = m.QuikLinear(to_layer(L))
    xt = torch.from_numpy(x).cuda().half()
    for bad in (torch.empty((8, 128), dtype=torch.bfloat16, device="cuda"),
                torch.empty((8, 128), dtype=torch.int32, device="cuda"),
                torch.empty((7, 128), dtype=torch.float16, device="cuda"),
                torch.empty((8, 127), dtype=torch.float16, device="cuda"),
                torch.empty((8, 128), dtype=torch.float16)):
        with pytest.raises(ValueError):
            dev(xt, out=bad)
        with pytest.raises(ValueError):
            dev.weight_only(xt, out=bad)
    with pytest.raises(ValueError):
        dev(xt, out_dtype=torch.bfloat16)
    codes, scale, zero, xo = dev.quantize_gemm_layout(xt)
    kp, op = codes.shape[1], xo.shape[1]
    assert kp % 128 == 0 and kp >= 240 and op == 64


def test_streams_share_context_scratch_safely():
    """forwards through one context on two streams are ordered (the scratch is
    shared); every result equals the single-stream forward."""
    m = q()
    import torch

    rng = np.random.default_rng(913)
    L, x, _ = make_layer(rng, 512, 2048, 4096, 4, 64, heavy_cols=2)
    dev = m.QuikLinear(to_layer(L))
    xs = [torch.from_numpy(x).cuda().half(), torch.from_numpy(x[::-1].copy()).cuda().half()]
    want = [dev(v).clone() for v in xs]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    outs = []
    for i in range(8):
        s = s1 if i % 2 == 0 else s2
        with torch.cuda.stream(s):
            outs.append(dev(xs[i % 2]))
    torch.cuda.synchronize()
    for i, o_ in enumerate(outs):
        assert torch.equal(o_, want[i % 2]), i


def test_reserve_then_capture_and_numerics_flag():
    """quik_ctx_reserve sizes the scratch so a larger-M forward can be captured into a
    CUDA graph (scratch cannot grow under capture: clear error otherwise); the
    non-finite flag is reported by check_numerics and cleared."""
    m = q()
    import torch

    rng = np.random.default_rng(915)
    L, x, _ = make_layer(rng, 300, 512, 256, 4, 16, heavy_cols=1)
    dev = m.QuikLinear(to_layer(L))
    xt = torch.from_numpy(x).cuda().half()
    dev.reserve(300)
    want = dev(xt).clone()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    out = torch.empty_like(want)
    with torch.cuda.graph(g):
        dev(xt, out=out)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    bad = xt.clone()
    bad[3, 7] = float("nan")
    dev(bad)
    with pytest.raises(m.NumericalError):
        dev.check_numerics()
    dev(xt)
    dev.check_numerics()  # cleared by the previous check


# --------------------------------------------------------------------------- INT4-only weight mode


@pytest.mark.parametrize("cg,bn", [(0, 0), (1, 32), (1, 64), (1, 128), (2, 128), (2, 192)])
def test_int4_weight_mode_bit_identical(tile, cg, bn):
    """weights="int4" (one INT4 device copy, every GEMM widens INT4 tiles into TMEM, the
    MMAs sum 16 x the products and the epilogue shifts them back) gives the same bits as
    the INT8-weight path for every tile, V1 / V2 / V3, f16 and f32 out, ragged shapes,
    with and without outliers; and holds half the base-weight bytes."""
    m = q()
    o = oracle()
    import torch

    if cg:
        assert tile(cg, bn) == 0
    rng = np.random.default_rng(1300 + 10 * cg + bn)
    for (M, K, N, O) in [(300, 1000, 520, 24), (37, 2048, 384, 0), (513, 640, 1000, 64), (129, 4100, 257, 256)]:
        L, x, _ = make_layer(rng, M, K, N, 4, O, heavy_cols=2)
        fast = m.QuikLinear(to_layer(L))
        small = m.QuikLinear(to_layer(L), weights="int4")
        xt = torch.from_numpy(x).cuda()
        for v in m.PipelineVariant:
            a = fast(xt, out_dtype=torch.float32, variant=v).cpu().numpy()
            b = small(xt, out_dtype=torch.float32, variant=v).cpu().numpy()
            np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32), err_msg=f"{v} {M} {K} {N} {O}")
        np.testing.assert_array_equal(fast(xt.half()).cpu().numpy().view(np.uint16),
                                      small(xt.half()).cpu().numpy().view(np.uint16))
        if O == 0:
            st, want = o.quik_matmul(L, x, 2)
            got = small(xt, out_dtype=torch.float32).cpu().numpy()
            np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
        kpad = (K - O + 127) // 128 * 128
        assert fast.device_bytes - small.device_bytes >= N * kpad // 2  # the INT8 copy is gone


def test_int4_weight_mode_gated_and_decode():
    """INT4-only layers through the gated projection and the decode kernel (M <= 32)."""
    m = q()
    import torch

    rng = np.random.default_rng(1350)
    up, gate, down, x = _mlp_layers(rng, 200, 512, 256, 4, 8, 32, 16)
    a = m.QuikLinear.gated(to_layer(up), to_layer(gate))
    b = m.QuikLinear.gated(to_layer(up), to_layer(gate), weights="int4")
    xt = torch.from_numpy(x).cuda()
    for M in (200, 16, 1):
        np.testing.assert_array_equal(a(xt[:M], out_dtype=torch.float32).cpu().numpy().view(np.uint32),
                                      b(xt[:M], out_dtype=torch.float32).cpu().numpy().view(np.uint32))
