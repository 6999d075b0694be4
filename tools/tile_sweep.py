"""Forward time per GEMM tile configuration (quik_set_gemm_tile) at the mid-size
BASELINE shapes: is the default tile choice right where the tile count is a poor
multiple of the SM count? 10 forwards per CUDA graph.

  python tools/tile_sweep.py
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2310_09259_b200 as q
from paper_2310_09259_b200 import _lib

SHAPES = [("7B qkvo", 2048, 4096, 4096, 256, 4), ("7B up", 2048, 4096, 11008, 256, 4),
          ("7B down W8A8", 2048, 11008, 4096, 688, 8), ("13B up", 2048, 5120, 13824, 256, 4),
          ("Falcon qkv", 2048, 14848, 14848, 256, 4)]
TILES = [(0, 0), (1, 128), (2, 128), (2, 256)]


def timeit(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def main():
    dev = torch.device("cuda", 0)
    lib = q.load_library()
    for name, M, K, N, O, bits in SHAPES:
        g = torch.Generator(device=dev).manual_seed(1)
        idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy()
        outl = q.OutlierSet.from_indices(K, idx)
        W = torch.randn(N, K, device=dev, generator=g)
        base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, bits)
        del W
        layer = q.QuikLinear.from_device(outl, base, sc, wr, ow, bits)
        x = torch.randn(M, K, device=dev, dtype=torch.float16)
        y = torch.empty(M, N, device=dev, dtype=torch.float16)
        res = dict(name=name)
        for cfg in TILES:
            _lib.check(lib.quik_set_gemm_tile(*cfg))
            layer.forward(x, out=y)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                for _ in range(10):
                    layer.forward(x, out=y)
            res[f"{cfg[0]}x{cfg[1]}_us"] = round(timeit(gr.replay) / 10 * 1e3, 1)
        lib.quik_set_gemm_tile(0, 0)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
