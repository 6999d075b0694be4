"""Gated MLP block (reference gated_mlp_ops: down(silu(gate(x)) * up(x))) on one GPU:
the fused QuikGatedMLP (shared quantizer + one up/gate GEMM with the silu * up
epilogue, then down) vs the unfused device path (three QuikLinear layers + torch
silu / multiply) vs cuBLAS f16 (three matmuls + silu / multiply). CUDA-graph replay.

  python tools/mlp_bench.py [--only 7b]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2310_09259_b200 as q

SHAPES = [  # name, M, hidden, ffn, O (up/gate), O (down), bits up/gate, bits down
    ("LLaMA-2-7B MLP", 2048, 4096, 11008, 256, 688, 4, 8),
    ("LLaMA-2-70B MLP", 4096, 8192, 28672, 256, 896, 4, 8),
]


def device_layer(dev, K, N, O, bits, g, idx=None):
    if idx is None:
        idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy()
    outl = q.OutlierSet.from_indices(K, idx)
    W = torch.randn(N, K, device=dev, generator=g) * 0.02
    base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, bits)
    return outl, (base, sc, wr, ow)


def host_layer(outl, t, bits):
    base, sc, wr, ow = (a.cpu().numpy() for a in t)
    N = sc.shape[0]
    w = q.QuantizedWeights(q.PackedIntMatrix(N, outl.base_count(), bits, base), sc, ow.reshape(N, -1), wr)
    return q.QuikLinearLayer(w, outl, None, bits)


def timeit(fn, iters=20):
    g = torch.cuda.CUDAGraph()
    fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--tokens", type=int, default=0, help="override M (e.g. 1 / 16 for decode)")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    for name, M, H, F, O, Od, b_ud, b_d in SHAPES:
        if args.only and args.only not in name:
            continue
        if args.tokens:
            M = args.tokens
        g = torch.Generator(device=dev).manual_seed(5)
        outl, tu = device_layer(dev, H, F, O, b_ud, g)
        _, tg = device_layer(dev, H, F, O, b_ud, g, idx=outl.indices)
        outl_d, td = device_layer(dev, F, H, Od, b_d, g)
        up, gate, down = host_layer(outl, tu, b_ud), host_layer(outl, tg, b_ud), host_layer(outl_d, td, b_d)
        del tu, tg, td
        fused = q.QuikGatedMLP(up, gate, down)
        l_up, l_gate, l_down = q.QuikLinear(up), q.QuikLinear(gate), q.QuikLinear(down)
        x = torch.randn(M, H, device=dev, dtype=torch.float16)
        y = torch.empty(M, H, device=dev, dtype=torch.float16)
        h = torch.empty(M, F, device=dev, dtype=torch.float16)
        u = torch.empty(M, F, device=dev, dtype=torch.float16)
        gt = torch.empty(M, F, device=dev, dtype=torch.float16)

        def run_fused():
            fused.proj(x, out=h)
            fused.down(h, out=y)

        def run_unfused():
            l_up(x, out=u)
            l_gate(x, out=gt)
            torch.mul(torch.nn.functional.silu(gt), u, out=h)
            l_down(h, out=y)

        Wu = torch.randn(F, H, device=dev, dtype=torch.float16)
        Wg = torch.randn(F, H, device=dev, dtype=torch.float16)
        Wd = torch.randn(H, F, device=dev, dtype=torch.float16)

        def run_cublas():
            torch.matmul(x, Wu.t(), out=u)
            torch.matmul(x, Wg.t(), out=gt)
            torch.mul(torch.nn.functional.silu(gt), u, out=h)
            torch.matmul(h, Wd.t(), out=y)

        def run_block():  # quik_gated_mlp_forward: down K1 reduction fused into the gated epilogue
            fused.forward(x, out=y)

        tb, t2, tu_, tc = timeit(run_block), timeit(run_fused), timeit(run_unfused), timeit(run_cublas)
        tproj = timeit(lambda: fused.proj(x, out=h))
        tf = tb
        ops = 2.0 * M * H * F * 3
        print(json.dumps(dict(name=name, M=M, hidden=H, ffn=F, fused_ms=tf, two_forwards_ms=t2, unfused_ms=tu_,
                              cublas_f16_ms=tc, gated_proj_ms=tproj, fused_tops=ops / tf / 1e9,
                              speedup_vs_two_forwards=t2 / tf, speedup_vs_unfused=tu_ / tf,
                              speedup_vs_cublas_f16=tc / tf)), flush=True)
        del fused, l_up, l_gate, l_down, Wu, Wg, Wd
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
