"""Diagnostics for the fused GEMM at a workload shape: library baselines
(cuBLASLt int8 via torch._int_mm, cuBLAS f16) and our kernel per tile config,
with and without the output epilogue stores (quik_set_probe_mode)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2310_09259_b200 as q
from paper_2310_09259_b200 import _lib


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


def main(M=4096, K=8192, N=28672, O=256):
    dev = torch.device("cuda", 0)
    res = {}
    A = torch.randint(-8, 8, (M, K), dtype=torch.int8, device=dev)
    B = torch.randint(-8, 8, (N, K), dtype=torch.int8, device=dev)
    t = timeit(lambda: torch._int_mm(A, B.t()))
    res["cublaslt_int8_ms"] = t
    res["cublaslt_int8_tops"] = 2 * M * N * K / t / 1e9
    x16 = torch.randn(M, K, device=dev, dtype=torch.float16)
    W16 = torch.randn(N, K, device=dev, dtype=torch.float16)
    t = timeit(lambda: torch.matmul(x16, W16.t()))
    res["cublas_f16_ms"] = t
    res["cublas_f16_tflops"] = 2 * M * N * K / t / 1e9
    del A, B, W16
    g = torch.Generator(device=dev).manual_seed(1)
    idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy()
    outl = q.OutlierSet.from_indices(K, idx)
    W = torch.randn(N, K, device=dev, generator=g)
    base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, 4)
    del W
    layer = q.QuikLinear.from_device(outl, base, sc, wr, ow, 4)
    y = torch.empty(M, N, device=dev, dtype=torch.float16)
    lib = q.load_library()
    ev = torch.cuda.Event(enable_timing=True)
    for cfg in [(1, 128), (2, 128), (2, 256)]:
        _lib.check(lib.quik_set_gemm_tile(*cfg))
        for probe in (0, 1):
            lib.quik_set_probe_mode(probe)
            t = timeit(lambda: layer.forward(x16, out=y))
            res[f"quik_{cfg[0]}x{cfg[1]}_{'probe' if probe else 'full'}_ms"] = t
    lib.quik_set_probe_mode(0)
    lib.quik_set_gemm_tile(0, 0)
    # K1 alone: the fused quantizer into the layer scratch (ABI fused quantize, ABI outputs)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
