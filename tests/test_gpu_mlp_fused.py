"""GPU: the gated MLP block with the down projection's quantizer reduction fused into the
gated GEMM's epilogue (C ABI quik_gated_mlp_forward, SURVEY.md §8f.2 second half).

The epilogue reduces, per token, the min / max of the down projection's base columns
over the f16 h it stores (order-preserving keys + atomics); the down K1 reads them
instead of its own reduction pass (runtime.cpp:36-50 split over two kernels). The bar
is bit-identity with the unfused block (gated forward, then the down forward on h),
which the reference-parity tests of test_gpu_parity.py pin against the reference's
forward_model(gated_mlp_ops): h, y (f16 and f32), repeated calls (the keys are
restored by the down K1), signed-zero minima, non-finite h, and the decode regime
(no statistics: the plain path).
"""
import numpy as np
import pytest

from oracle_lib import oracle
from test_gpu_parity import _mlp_layers, q, tile, to_layer  # noqa: F401 (tile: fixture)

pytestmark = pytest.mark.gpu


def _blocks(up, gate, down):
    m = q()
    return m.QuikGatedMLP(to_layer(up), to_layer(gate), to_layer(down))


def _check_block(mlp, xt, torch):
    for odt in (torch.float16, torch.float32):
        y_u, h_u = mlp.forward_with_hidden(xt, out_dtype=odt, hidden_dtype=torch.float16, fused=False)
        y_f, h_f = mlp.forward_with_hidden(xt, out_dtype=odt, hidden_dtype=torch.float16, fused=True)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(h_f.cpu().numpy().view(np.uint16), h_u.cpu().numpy().view(np.uint16))
        a, b = y_f.cpu().numpy(), y_u.cpu().numpy()
        np.testing.assert_array_equal(a.view(np.uint16 if odt == torch.float16 else np.uint32),
                                      b.view(np.uint16 if odt == torch.float16 else np.uint32))
    mlp.proj.check_numerics()


@pytest.mark.parametrize("bits_ud,bits_down", [(4, 8), (4, 4), (8, 8)])
def test_fused_mlp_bit_identical_to_unfused(bits_ud, bits_down):
    m = q()
    import torch

    rng = np.random.default_rng(1100 + 10 * bits_ud + bits_down)
    for (M, K, F, O, Od) in [(40, 256, 160, 32, 16), (300, 512, 384, 64, 32), (130, 384, 96, 0, 0),
                             (517, 640, 1024, 64, 0), (64, 256, 2048, 32, 96), (200, 256, 9216, 32, 300),
                             (48, 128, 36864, 0, 512)]:  # > 65535 gated rows; wide down rows: plain K1
        up, gate, down, x = _mlp_layers(rng, M, K, F, bits_ud, bits_down, O, Od)
        mlp = _blocks(up, gate, down)
        xt = torch.from_numpy(x).cuda()
        _check_block(mlp, xt, torch)
        _check_block(mlp, xt.half(), torch)
        # keys restored between calls: fresh inputs through the same context
        for s in range(3):
            x2 = torch.from_numpy(rng.normal(0, 1 + s, size=x.shape).astype(np.float32)).cuda().half()
            _check_block(mlp, x2, torch)
    assert m is not None


def test_fused_mlp_decode_regime_and_every_tile(tile):
    """M <= 32 runs the gated projection on the decode kernel (no statistics, plain
    down K1); every GEMM tile configuration of the fused path emits the same keys."""
    import torch

    rng = np.random.default_rng(1200)
    up, gate, down, x = _mlp_layers(rng, 260, 640, 320, 4, 8, 64, 16)
    mlp = _blocks(up, gate, down)
    xt = torch.from_numpy(x).cuda().half()
    for M in (1, 7, 16, 32, 33):
        _check_block(mlp, xt[:M].contiguous(), torch)
    for cg, bn in [(1, 32), (1, 128), (2, 128), (2, 256)]:
        assert tile(cg, bn) == 0
        _check_block(mlp, xt, torch)


def test_fused_mlp_int4_weights_mode():
    """Both projections with one INT4 weight copy (weights="int4": the W4 GEMM tiles emit
    the statistics) equal the speed-mode block bit for bit."""
    m = q()
    import torch

    rng = np.random.default_rng(1700)
    up, gate, down, x = _mlp_layers(rng, 300, 512, 384, 4, 4, 64, 32)
    xt = torch.from_numpy(x).cuda().half()
    a = _blocks(up, gate, down)
    b = m.QuikGatedMLP(to_layer(up), to_layer(gate), to_layer(down), weights="int4")
    _check_block(b, xt, torch)
    ya, yb = a(xt), b(xt)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ya.cpu().numpy().view(np.uint16), yb.cpu().numpy().view(np.uint16))


def test_fused_mlp_signed_zero_minimum():
    """h == +-0 everywhere (zero up weights and bias): the down quantizer's minimum is a
    zero whose sign is the first base column's (runtime.cpp:44-48 strict comparisons),
    tracked by the epilogue as the first zero's column."""
    import torch

    rng = np.random.default_rng(1300)
    o = oracle()
    up, gate, down, x = _mlp_layers(rng, 96, 256, 192, 4, 8, 32, 16)
    zq = o.rtn_quantize_weights(np.zeros((192, 256), np.float32), up["idx"], 4)
    up = dict(up, base=zq["base"], scales=zq["scales"], wreduced=zq["wreduced"],
              outlier_weights=np.zeros_like(up["outlier_weights"]), bias=np.zeros(192, np.float32))
    mlp = _blocks(up, gate, down)
    xt = torch.from_numpy(x).cuda().half()
    y, h = mlp.forward_with_hidden(xt, hidden_dtype=torch.float16)
    hh = h.cpu().numpy()
    assert np.all(hh == 0) and np.any(np.signbit(hh)) and np.any(~np.signbit(hh))
    _check_block(mlp, xt, torch)
    # h >= 0 with a zero minimum: features 0..63 are -0 (zero up rows, silu(gate) < 0),
    # the rest positive (up bias +5, gate bias +50): zero = -0 from the first base column
    w = rng.normal(0.0, 1e-3, size=(192, 256)).astype(np.float32)
    w[:64] = 0.0
    lq = o.rtn_quantize_weights(w, up["idx"], 4)
    up2 = dict(up, base=lq["base"], scales=lq["scales"], wreduced=lq["wreduced"],
               outlier_weights=lq["outlier_weights"].astype(np.float16).astype(np.float32),
               bias=np.r_[np.zeros(64), np.full(128, 5.0)].astype(np.float32))
    gate2 = dict(gate, bias=np.r_[np.full(64, -50.0), np.full(128, 50.0)].astype(np.float32))
    mlp2 = _blocks(up2, gate2, down)
    y, h = mlp2.forward_with_hidden(xt, hidden_dtype=torch.float16)
    hh = h.cpu().numpy()
    assert np.all(hh[:, :64] == 0) and np.all(np.signbit(hh[:, :64])) and np.all(hh[:, 64:] > 0)
    _check_block(mlp2, xt, torch)


def test_fused_mlp_nonfinite_hidden_raises():
    """|h| beyond the f16 range in a base column of the down projection: both paths raise
    NumericalError at the next check (reference runtime.cpp:52)."""
    m = q()
    import torch

    rng = np.random.default_rng(1400)
    up, gate, down, x = _mlp_layers(rng, 64, 256, 128, 4, 8, 32, 16)
    up = dict(up, bias=np.full(128, 3.0e4, np.float32))
    gate = dict(gate, bias=np.full(128, 10.0, np.float32))
    mlp = _blocks(up, gate, down)
    xt = torch.from_numpy(x).cuda().half()
    for fused in (False, True):
        mlp.forward(xt, hidden_dtype=torch.float16, fused=fused)
        with pytest.raises(m.NumericalError):
            mlp.proj.check_numerics()
    # a clean block afterwards on the same context: no stale flag, keys restored
    up3, gate3, down3, x3 = _mlp_layers(rng, 64, 256, 128, 4, 8, 32, 16)
    _check_block(_blocks(up3, gate3, down3), torch.from_numpy(x3).cuda().half(), torch)


def test_fused_mlp_llama7b_shape():
    """LLaMA-2-7B MLP (4096 -> 11008 -> 4096, W4A4 up / gate, W8A8 down with 688 outliers)
    at 512 tokens: the prescaled hot down K1 at its 11008-wide rows."""
    import torch

    rng = np.random.default_rng(1500)
    up, gate, down, x = _mlp_layers(rng, 512, 4096, 11008, 4, 8, 256, 688)
    mlp = _blocks(up, gate, down)
    _check_block(mlp, torch.from_numpy(x).cuda().half(), torch)


def test_fused_mlp_cuda_graph_replay():
    """The block captured into a CUDA graph after quik_ctx_reserve (gated layer + down):
    every replay consumes and restores the statistics keys, so replays with new inputs in
    the captured buffer equal the unfused block."""
    import torch

    rng = np.random.default_rng(1600)
    up, gate, down, x = _mlp_layers(rng, 192, 512, 640, 4, 8, 32, 48)
    mlp = _blocks(up, gate, down)
    xt = torch.from_numpy(x).cuda().half()
    mlp.proj.reserve(xt.shape[0])
    mlp.down.reserve(xt.shape[0])
    y = torch.empty(xt.shape[0], down["out_features"], device="cuda", dtype=torch.float16)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        mlp.forward(xt, out=y)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        mlp.forward(xt, out=y)
    for k in range(3):
        xt.copy_(torch.from_numpy(rng.normal(0, 1 + k, size=x.shape).astype(np.float16)).cuda())
        g.replay()
        torch.cuda.synchronize()
        want = mlp.forward(xt, hidden_dtype=torch.float16, fused=False)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(y.cpu().numpy().view(np.uint16), want.cpu().numpy().view(np.uint16))


def test_fused_mlp_hidden_row_pitch():
    """h in a caller buffer with a row pitch > F (16-byte multiple: the statistics and the
    prescaled down K1 at that pitch; not a multiple: the plain path)."""
    import torch

    rng = np.random.default_rng(1800)
    up, gate, down, x = _mlp_layers(rng, 200, 512, 384, 4, 8, 64, 32)
    mlp = _blocks(up, gate, down)
    xt = torch.from_numpy(x).cuda().half()
    want, hw = mlp.forward_with_hidden(xt, fused=False)
    for pad in (40, 4):
        buf = torch.full((xt.shape[0], 384 + pad), 7.0, device="cuda", dtype=torch.float16)
        y, h = mlp.forward_with_hidden(xt, hidden=buf[:, :384])
        torch.cuda.synchronize()
        assert h.stride(0) == 384 + pad
        np.testing.assert_array_equal(h.cpu().numpy().view(np.uint16), hw.cpu().numpy().view(np.uint16))
        np.testing.assert_array_equal(y.cpu().numpy().view(np.uint16), want.cpu().numpy().view(np.uint16))
        assert torch.all(buf[:, 384:] == 7.0)
