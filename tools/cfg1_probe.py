"""cfg1 (16 x 4096 -> 4096, O = 128, W4A4) forward composition: graph-replayed step,
K1 alone, decode kernel alone, cuBLAS f16 — for the single-launch work.
  python tools/cfg1_probe.py [--once]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2310_09259_b200 as q


def timeit(fn, iters=200, warm=20):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--m", default="1,16,32")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    K, N, O = 4096, 4096, 128
    g = torch.Generator(device=dev).manual_seed(3)
    idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy()
    outl = q.OutlierSet.from_indices(K, idx)
    W = torch.randn(N, K, device=dev, generator=g)
    base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, 4)
    layer = q.QuikLinear.from_device(outl, base, sc, wr, ow, 4)
    W16 = W.half()
    for m in [int(v) for v in args.m.split(",")]:
        x = torch.randn(m, K, device=dev, dtype=torch.float16)
        y = torch.empty(m, N, device=dev, dtype=torch.float16)
        if args.once:
            for _ in range(3):
                layer.forward(x, out=y)
            torch.cuda.synchronize()
            continue
        eager = timeit(lambda: layer.forward(x, out=y))
        gr = torch.cuda.CUDAGraph()
        layer.forward(x, out=y)
        with torch.cuda.graph(gr):
            layer.forward(x, out=y)
        graph = timeit(gr.replay)
        g10 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g10):
            for _ in range(10):
                layer.forward(x, out=y)
        graph10 = timeit(g10.replay, iters=50) / 10
        o16 = torch.empty(m, N, device=dev, dtype=torch.float16)
        g16 = torch.cuda.CUDAGraph()
        torch.matmul(x, W16.t(), out=o16)
        with torch.cuda.graph(g16):
            torch.matmul(x, W16.t(), out=o16)
        f16 = timeit(g16.replay)
        g16b = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g16b):
            for _ in range(10):
                torch.matmul(x, W16.t(), out=o16)
        f16_10 = timeit(g16b.replay, iters=50) / 10
        print(json.dumps(dict(M=m, eager_us=eager, graph_us=graph, graph_back_to_back_us=graph10,
                              cublas_f16_graph_us=f16, cublas_f16_back_to_back_us=f16_10,
                              speedup_single=f16 / graph, speedup_back_to_back=f16_10 / graph10)), flush=True)


if __name__ == "__main__":
    main()
