"""Shape sweep on one GPU: QUIK layer step time (K1 + fused GEMM) vs cuBLAS f16 of
the same shape, for the BASELINE.json configs and the cfg4 token sweep.

  python tools/sweep.py [--quick] > sweep.json
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2310_09259_b200 as q

SHAPES = [
    # name, M, K, N, O, bits
    ("cfg1 oracle 4096->4096", 16, 4096, 4096, 128, 4),
    ("cfg2 7B qkvo", 2048, 4096, 4096, 256, 4),
    ("cfg2 7B up/gate", 2048, 4096, 11008, 256, 4),
    ("cfg2 7B down W8A8", 2048, 11008, 4096, 688, 8),
    ("cfg3 70B up/gate", 4096, 8192, 28672, 256, 4),
    ("cfg3 70B down W8A8", 4096, 28672, 8192, 896, 8),
    ("cfg5-shape 13B up", 2048, 5120, 13824, 256, 4),
    ("cfg5 13B up 2:4", 2048, 5120, 13824, 256, 4, True),
    ("cfg5 13B q 2:4", 2048, 5120, 5120, 256, 4, True),
    ("cfg3 70B up/gate 2:4", 4096, 8192, 28672, 256, 4, True),
    ("cfg4 OPT fc1 M=16 2:4", 16, 9216, 36864, 256, 4, True),
    ("cfg4 OPT-66B fc2 M=2048", 2048, 36864, 9216, 256, 4),
    # Falcon-180B (hidden 14848, FFN 59392; public model card), FC2 INT8 with the
    # proportional outlier count 256 * 59392 / 14848 = 1024
    ("cfg4 Falcon-180B fc1 M=2048", 2048, 14848, 59392, 256, 4),
    ("cfg4 Falcon-180B fc2 W8A8 M=2048", 2048, 59392, 14848, 1024, 8),
    ("cfg4 Falcon-180B qkv M=2048", 2048, 14848, 14848, 256, 4),
    # decode regime (M <= 32): the INT4 decode kernel
    ("decode cfg1 M=32", 32, 4096, 4096, 128, 4),
    ("decode 70B up/gate M=1", 1, 8192, 28672, 256, 4),
    ("decode 70B up/gate M=16", 16, 8192, 28672, 256, 4),
    ("decode 70B up/gate M=32", 32, 8192, 28672, 256, 4),
    ("decode OPT-66B fc1 M=32", 32, 9216, 36864, 256, 4),
    ("decode 7B up/gate M=16", 16, 4096, 11008, 256, 4),
    ("decode 7B up/gate M=32", 32, 4096, 11008, 256, 4),
    ("decode 7B qkvo M=32", 32, 4096, 4096, 256, 4),
    ("decode 70B down W8A8 M=16", 16, 28672, 8192, 896, 8),
]
OPT_FC1 = [(m, 9216, 36864, 256, 4) for m in (1, 16, 64, 128, 256, 512, 1024, 2048, 4096, 8192)]
FALCON_FC1 = [(m, 14848, 59392, 256, 4) for m in (1, 16, 128, 512, 2048, 8192)]


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


WEIGHTS = "speed"
REPS = 10  # forwards per CUDA graph


def run(name, M, K, N, O, bits, layers, sparse=False):
    dev = torch.device("cuda", 0)
    key = (K, N, O, bits, sparse)
    if key not in layers:
        layers.clear()
        torch.cuda.empty_cache()
        g = torch.Generator(device=dev).manual_seed(7)
        idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy()
        outl = q.OutlierSet.from_indices(K, idx)
        W = torch.randn(N, K, device=dev, generator=g)
        if sparse:
            from bench import prune_24

            prune_24(W, torch.as_tensor(outl.permutation[: K - O], device=dev))
        base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, bits)
        del W
        layers[key] = (q.QuikLinear.from_device(outl, base, sc, wr, ow, bits, sparse=sparse, weights=WEIGHTS),
                       torch.randn(N, K, device=dev, dtype=torch.float16))
    layer, W16 = layers[key]
    x = torch.randn(M, K, device=dev, dtype=torch.float16)
    y = torch.empty(M, N, device=dev, dtype=torch.float16)
    mid = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for e in mid:  # materialise the raw cudaEvent handles
        e.record()
    t_step_eager = timeit(lambda: layer.forward(x, out=y))
    # CUDA graph of REPS back-to-back forwards (removes host launch overhead; a graph of
    # one small forward is timed at the graph-launch granularity, ~2 us steps, instead)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(REPS):
            layer.forward(x, out=y)
    t_step = timeit(g.replay) / REPS
    # kernel split from one instrumented call
    for _ in range(3):
        mid[0].record()
        layer.forward(x, out=y, mid_event=mid[1])
        mid[2].record()
    torch.cuda.synchronize()
    t_k1, t_gemm = mid[0].elapsed_time(mid[1]), mid[1].elapsed_time(mid[2])
    out16 = torch.empty(M, N, device=dev, dtype=torch.float16)
    g16 = torch.cuda.CUDAGraph()
    torch.matmul(x, W16.t(), out=out16)
    with torch.cuda.graph(g16):
        for _ in range(REPS):
            torch.matmul(x, W16.t(), out=out16)
    t16 = timeit(g16.replay) / REPS
    ops = 2.0 * M * N * K
    return dict(name=name, M=M, K=K, N=N, O=O, bits=bits, sparse=layer.is_sparse, weights=WEIGHTS,
                layer_mb=layer.device_bytes / 1e6, step_ms=t_step, step_eager_ms=t_step_eager,
                k1_ms=t_k1, gemm_ms=t_gemm,
                tops=ops / t_step / 1e9, cublas_f16_ms=t16, speedup_vs_f16=t16 / t_step)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--opt-m", default="", help="comma list of OPT fc1 token counts (default: all)")
    ap.add_argument("--falcon", action="store_true", help="also the Falcon-180B fc1 token sweep")
    ap.add_argument("--weights", default="speed", choices=["speed", "int4"],
                    help="device copy of 4-bit weights (QuikLinear weights=)")
    args = ap.parse_args()
    global WEIGHTS
    WEIGHTS = args.weights
    layers = {}
    res = []
    for s in SHAPES:
        if args.only and args.only not in s[0]:
            continue
        res.append(run(*s[:6], layers, *s[6:]))
    opt = OPT_FC1[::3] if args.quick else OPT_FC1
    if args.opt_m:
        opt = [o for o in OPT_FC1 if str(o[0]) in args.opt_m.split(",")]
    for m, K, N, O, bits in ([] if args.only and not args.opt_m else opt):
        res.append(run(f"cfg4 OPT-66B fc1 M={m}", m, K, N, O, bits, layers))
    if args.falcon:
        for m, K, N, O, bits in FALCON_FC1:
            res.append(run(f"cfg4 Falcon-180B fc1 M={m}", m, K, N, O, bits, layers))
    for r in res:
        print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
