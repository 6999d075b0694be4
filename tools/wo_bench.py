"""Weight-only (LayerMode::WeightOnly) decode timing: the INT4/INT8
weight-streaming wo_gemm_kernel (f16 activations, A operand widened into TMEM) vs the
QUIK W4A4 forward of the same layer vs cuBLAS f16 of the same shape. CUDA-graph replay,
weights (> L2) streamed from HBM every call.

  python tools/wo_bench.py [--only 70b] [--bits 4]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2310_09259_b200 as q

SHAPES = [  # name, K, N, O
    ("LLaMA-2-70B up 8192->28672", 8192, 28672, 256),
    ("OPT-66B fc1 9216->36864", 9216, 36864, 256),
    ("LLaMA-2-7B qkv 4096->4096", 4096, 4096, 128),
]


def timeit(fn, iters=50):
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
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--tokens", default="1,4,16,64")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    peaks = {}
    try:
        peaks = json.load(open(Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"))
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6548.8))
    for name, K, N, O in SHAPES:
        if args.only and args.only not in name:
            continue
        g = torch.Generator(device=dev).manual_seed(11)
        idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy()
        outl = q.OutlierSet.from_indices(K, idx)
        W = torch.randn(N, K, device=dev, generator=g) * 0.02
        base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, args.bits)
        del W
        layer = q.QuikLinear.from_device(outl, base, sc, wr, ow, args.bits)
        del base, sc, wr, ow
        Wf = torch.randn(N, K, device=dev, dtype=torch.float16)
        kb = K - O
        wbytes = N * kb * args.bits / 8 + N * O * 4  # codes + f16 hi/lo outlier planes
        for M in (int(t) for t in args.tokens.split(",")):
            x = torch.randn(M, K, device=dev, dtype=torch.float16)
            y = torch.empty(M, N, device=dev, dtype=torch.float16)
            t_wo = timeit(lambda: layer.weight_only(x, out=y))
            t_q = timeit(lambda: layer(x, out=y))
            t_c = timeit(lambda: torch.matmul(x, Wf.t(), out=y))
            print(json.dumps(dict(name=name, M=M, bits=args.bits, weight_only_us=1e3 * t_wo, quik_us=1e3 * t_q,
                                  cublas_f16_us=1e3 * t_c, wo_weight_gbs=wbytes / (t_wo * 1e-3) / 1e9,
                                  wo_hbm_frac=wbytes / (t_wo * 1e-3) / 1e9 / hbm,
                                  speedup_vs_cublas_f16=t_c / t_wo)), flush=True)
        del layer, Wf
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
