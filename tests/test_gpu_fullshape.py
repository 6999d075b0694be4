"""GPU parity at every BASELINE.json configuration's FULL shape, including the one
bench.py times (configs[2], LLaMA-2-70B up/gate 4096 x 8192 -> 28672, O = 256).

The layer is generated on the device (x ~ N(0,1) with heavy columns x50, outliers =
the O columns of largest max |x|, W ~ N(0, 0.5) RTN-quantized on the device,
which is bit-exact against the reference's rtn_quantize_weights; 2:4 layers are
magnitude-pruned over the permuted base columns first) and runs through the hot path
at full size. Tokens and output rows are independent, so the CPU oracle then checks
a subset of tokens x rows of that one full-size run:
  * the INT32 base accumulators / O = 0 layers: bit-exact (f32 out);
  * O > 0: the f32 output within the derived bound of oracle_lib.f16_output_bound
    (no f16 rounding) and rel_frobenius < 1e-5; the f16 output (the benched path)
    within the derived per-element f16 bound and rel_frobenius <= 5e-4.
"""
import zlib

import numpy as np
import pytest

from oracle_lib import f16_output_bound, oracle, rel_frobenius, row_bytes

pytestmark = pytest.mark.gpu

# (name, M, K, N, O, bits, sparse) -- BASELINE.json configs[1..4] at full shape
CONFIGS = [
    ("cfg3_70b_up", 4096, 8192, 28672, 256, 4, False),
    ("cfg3_70b_down_w8", 4096, 28672, 8192, 896, 8, False),
    ("cfg2_7b_qkvo", 2048, 4096, 4096, 256, 4, False),
    ("cfg2_7b_up", 2048, 4096, 11008, 256, 4, False),
    ("cfg2_7b_down_w8", 2048, 11008, 4096, 688, 8, False),
    ("cfg4_opt66b_fc1_m1", 1, 9216, 36864, 256, 4, False),
    ("cfg4_opt66b_fc1_m16", 16, 9216, 36864, 256, 4, False),
    ("cfg4_opt66b_fc1_m256", 256, 9216, 36864, 256, 4, False),
    ("cfg4_opt66b_fc1_m2048", 2048, 9216, 36864, 256, 4, False),
    ("cfg4_opt66b_fc2_m2048", 2048, 36864, 9216, 256, 4, False),
    ("cfg4_falcon180b_fc1_m2048", 2048, 14848, 59392, 256, 4, False),
    ("cfg4_falcon180b_fc2_w8_m2048", 2048, 59392, 14848, 1024, 8, False),
    ("cfg5_13b_up_24", 2048, 5120, 13824, 256, 4, True),
    ("cfg5_13b_q_24", 2048, 5120, 5120, 256, 4, True),
]


def q():
    import paper_2310_09259_b200 as m

    return m


def device_layer(M, K, N, O, bits, sparse, seed, bias=True, weights="speed"):
    """Full-size synthetic layer on the device. Returns (QuikLinear, x16 device tensor,
    host dict of the per-row reference-format weights, outlier indices)."""
    import torch

    from bench import prune_24

    m = q()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(seed)
    x = torch.randn((M, K), generator=g, device=dev)
    heavy = torch.unique(torch.randint(0, K, (max(O // 2, 1),), generator=g, device=dev))
    x[:, heavy] *= 50.0
    x16 = x.half()
    del x
    # outlier columns: the O columns of largest max |x| (ties to the lower index)
    score = x16.float().abs().amax(0)
    idx = torch.sort(score, descending=True, stable=True).indices[:O].sort().values.cpu().numpy()
    outliers = m.OutlierSet.from_indices(K, idx)
    W = torch.randn((N, K), generator=g, device=dev) * 0.5
    if sparse:
        prune_24(W, torch.as_tensor(outliers.permutation[: K - O], device=dev))
    base, sc, wr, ow = m.rtn_quantize_weights_device(W, outliers, bits)
    del W
    b = torch.randn(N, generator=g, device=dev) * 0.1 if bias else None
    layer = m.QuikLinear.from_device(outliers, base, sc, wr, ow, bits, bias=b, sparse=sparse, weights=weights)
    if sparse:
        assert layer.is_sparse
    host = dict(base=base.view(N, row_bytes(K - O, bits)), scales=sc, wreduced=wr,
                ow=ow.half().float() if O else ow, bias=b)
    torch.cuda.synchronize()
    return layer, x16, host, idx


def subset_layer(host, rows, K, O, bits, idx):
    import torch

    ri = torch.as_tensor(rows, device=host["scales"].device)
    t = lambda v: v[ri].cpu().numpy()  # noqa: E731
    return dict(in_features=K, out_features=rows.size, bits=bits, act_bits=bits,
                base=t(host["base"]).reshape(-1), scales=t(host["scales"]), wreduced=t(host["wreduced"]),
                outlier_weights=t(host["ow"]).reshape(rows.size, O) if O else np.zeros((rows.size, 0), np.float32),
                idx=np.asarray(idx, np.int64), bias=None if host["bias"] is None else t(host["bias"]))


# the INT4-only weight mode (one INT4 device copy, QuikLinear(weights="int4")) at full shape
INT4_CONFIGS = [(n + "_int4w",) + c[1:] for n, *_ in CONFIGS for c in [next(cc for cc in CONFIGS if cc[0] == n)]
                if n in ("cfg3_70b_up", "cfg2_7b_qkvo", "cfg4_opt66b_fc1_m256", "cfg4_opt66b_fc1_m16")]


@pytest.mark.parametrize("name,M,K,N,O,bits,sparse", CONFIGS + INT4_CONFIGS,
                         ids=[c[0] for c in CONFIGS + INT4_CONFIGS])
def test_baseline_config_full_shape(name, M, K, N, O, bits, sparse):
    import torch

    m = q()
    o = oracle()
    weights = "int4" if name.endswith("_int4w") else "speed"
    layer, x16, host, idx = device_layer(M, K, N, O, bits, sparse, seed=zlib.crc32(name.encode()) & 0xFFFF,
                                         weights=weights)
    if weights == "int4":  # one INT4 copy of the base weights (+ f16 outliers, per-row vectors, tables)
        kpad = (K - O + 127) // 128 * 128
        assert layer.device_bytes < N * kpad // 2 + N * ((O + 63) // 64 * 64) * 2 + 16 * N + 64 * K
    y16 = layer(x16)                                   # the benched path: f16 in, f16 out
    y32 = layer(x16, out_dtype=torch.float32)
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    toks = np.unique(np.concatenate([rng.choice(M, min(M, 6), replace=False), [0, M - 1]]))
    rows = np.unique(np.concatenate([rng.choice(N, 256, replace=False), [0, N - 1], np.arange(N - 128, N)]))
    L = subset_layer(host, rows, K, O, bits, idx)
    xs = x16[torch.as_tensor(toks, device=x16.device)].float().cpu().numpy()
    st, want = o.quik_matmul(L, xs, 2)
    assert st == 0
    ri = torch.as_tensor(rows, device=x16.device)
    ti = torch.as_tensor(toks, device=x16.device)
    got32 = y32[ti][:, ri].cpu().numpy()
    got16 = y16[ti][:, ri].float().cpu().numpy()
    if O == 0:
        np.testing.assert_array_equal(got32.view(np.uint32), want.view(np.uint32))
    err32 = np.abs(got32.astype(np.float64) - want)
    b32 = f16_output_bound(L, xs, want, y_is_f16=False)
    assert np.all(err32 <= b32), f"{name}: f32 out, worst err/bound {float((err32 / b32).max()):.3f}"
    assert rel_frobenius(want, got32) < 1e-5
    # the f16 epilogue rounds exactly the f32 value the f32 epilogue writes
    np.testing.assert_array_equal(y16[ti][:, ri].cpu().numpy().view(np.uint16),
                                  got32.astype(np.float16).view(np.uint16))
    err16 = np.abs(got16.astype(np.float64) - want)
    b16 = f16_output_bound(L, xs, want)
    assert np.all(err16 <= b16), f"{name}: f16 out, worst err/bound {float((err16 / b16).max()):.3f}"
    assert rel_frobenius(want, got16) <= 5e-4
    # the integer path alone at full shape: K1 codes of the sampled tokens, bit-exact
    codes, scale, zero, xo = layer.quantize_gemm_layout(x16[ti])
    st, pk, sc, ze, xo_ref = o.quantize_fused(xs, idx, bits)
    assert st == 0
    np.testing.assert_array_equal(scale.cpu().numpy().view(np.uint32), sc.view(np.uint32))
    np.testing.assert_array_equal(zero.cpu().numpy().view(np.uint32), ze.view(np.uint32))
    kb = K - O
    want_codes = o.unpack(pk, len(toks), kb, bits)
    np.testing.assert_array_equal(codes[:, :kb].cpu().numpy(), want_codes)
    del layer, y16, y32
    torch.cuda.empty_cache()
