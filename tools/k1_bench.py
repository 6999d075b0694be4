"""K1 (activation quantizer) alone: device time per launch and achieved HBM GB/s
at the BASELINE shapes (CUDA-graph replay, inputs larger than L2 rotate).

  python tools/k1_bench.py            # timing table (JSON lines)
  python tools/k1_bench.py --once     # one launch per shape (for ncu)
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch

import paper_2310_09259_b200 as q

SHAPES = [  # name, M, K, O, bits
    ("cfg3 70B up/gate", 4096, 8192, 256, 4),
    ("cfg3 70B down W8A8", 4096, 28672, 896, 8),
    ("cfg2 7B qkvo", 2048, 4096, 256, 4),
    ("cfg2 7B down W8A8", 2048, 11008, 688, 8),
    ("cfg1", 16, 4096, 128, 4),
    ("cfg5 13B up", 2048, 5120, 256, 4),
    ("cfg4 OPT-66B fc2 W4", 2048, 36864, 256, 4),
    ("cfg4 Falcon-180B fc2 W8A8", 2048, 59392, 1024, 8),
    ("cfg4 OPT-66B fc1", 2048, 9216, 256, 4),
    ("cfg4 Falcon-180B fc1 / qkv", 2048, 14848, 256, 4),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    for name, M, K, O, bits in SHAPES:
        if args.only and args.only not in name:
            continue
        rng = np.random.default_rng(1)
        idx = np.sort(rng.choice(K, size=O, replace=False)).astype(np.int64)
        outl = q.OutlierSet.from_indices(K, idx)
        N = 128
        kb = K - O
        base = torch.zeros(N * (kb // 2 if bits == 4 else kb), dtype=torch.uint8, device=dev)
        ones = torch.ones(N, device=dev)
        layer = q.QuikLinear.from_device(outl, base, ones, torch.zeros(N, device=dev),
                                         torch.zeros(N, O, device=dev), bits)
        nbuf = max(1, int(np.ceil(3 * 128e6 / (M * K * 2))))  # rotate inputs past L2
        xs = [torch.randn(M, K, device=dev).half() for _ in range(nbuf)]
        kpad = (kb + 127) // 128 * 128
        opad = (O + 63) // 64 * 64
        codes = torch.empty((M, kpad), dtype=torch.int8, device=dev)
        sc = torch.empty(M, device=dev)
        ze = torch.empty(M, device=dev)
        xo = torch.empty((M, opad), dtype=torch.float16, device=dev)
        lib = q._lib.load()
        import ctypes as C

        def run(x):
            s = torch.cuda.current_stream(dev).cuda_stream
            q._lib.check(lib.quik_quantize_activations_gemm(
                layer.ctx.handle, layer.handle, C.c_void_p(x.data_ptr()), q._lib.QUIK_F16, M,
                C.c_void_p(codes.data_ptr()), C.c_void_p(sc.data_ptr()), C.c_void_p(ze.data_ptr()),
                C.c_void_p(xo.data_ptr()), C.c_void_p(s)))

        if args.once:
            run(xs[0])
            torch.cuda.synchronize()
            continue
        for x in xs:
            run(x)
        g = torch.cuda.CUDAGraph()
        reps = 8
        with torch.cuda.graph(g):
            for r in range(reps):
                run(xs[r % nbuf])
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        iters = 10
        for _ in range(iters):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / (iters * reps)
        nbytes = M * K * 2 + M * kpad + M * opad * 2 + 8 * M  # the kernel's own (int8 code) layout
        alg = M * K * 2 + M * ((kb + 1) // 2 if bits == 4 else kb) + M * O * 2 + 8 * M  # SURVEY §8(d) bytes
        peak = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
            if (Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").exists() else 6650.0
        print(json.dumps(dict(name=name, M=M, K=K, O=O, bits=bits, us=us, gbs=nbytes / us * 1e-3,
                              frac_device_layout=nbytes / us * 1e-3 / peak, alg_bytes=alg,
                              frac=alg / us * 1e-3 / peak, peak_gbs=peak)), flush=True)


if __name__ == "__main__":
    main()
