"""GPU GPTQ / SparseGPT (quik_gptq_quantize) timing vs the reference's
CPU implementation (oracle/_ref, OpenMP on all host cores) on the same layer, plus the
device Hessian. Synthetic weights / calibration tokens.

  python tools/gptq_bench.py [--shapes 4096x4096,28672x8192] [--cpu-max 4096]
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np
import torch

import paper_2310_09259_b200 as q


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="4096x4096,28672x8192")
    ap.add_argument("--tokens", type=int, default=1024)
    ap.add_argument("--cpu-max", type=int, default=4096, help="largest in_features also run on the CPU reference")
    ap.add_argument("--sparse", action="store_true")
    args = ap.parse_args()
    rng = np.random.default_rng(0)
    for shp in args.shapes.split(","):
        N, K = (int(v) for v in shp.split("x"))
        O = 256 if K >= 4096 else 16
        w = rng.normal(0.0, 0.02, size=(N, K)).astype(np.float32)
        x = rng.normal(0.0, 1.0, size=(args.tokens, K)).astype(np.float32)
        x[:, rng.choice(K, 8, replace=False)] *= 20.0
        idx = np.sort(rng.choice(K, O, replace=False)).astype(np.int64)
        outl = q.OutlierSet.from_indices(K, idx)
        xt = torch.from_numpy(x).cuda()
        wt = torch.from_numpy(w).cuda()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        h = q.hessian_device([xt])
        torch.cuda.synchronize()
        t_h = time.perf_counter() - t0
        q.gptq_quantize_device(wt[:64], outl, 4, h, sparse=args.sparse)  # warm-up (handles, kernels)
        t0 = time.perf_counter()
        got = q.gptq_quantize_device(wt, outl, 4, h, sparse=args.sparse)
        t_g = time.perf_counter() - t0
        res = dict(shape=f"{N}x{K}", outliers=O, tokens=args.tokens, sparse=args.sparse, gpu_hessian_s=t_h,
                   gpu_gptq_s=t_g)
        if K <= args.cpu_max:
            from oracle_lib import REF_SO, ref

            if REF_SO.exists():
                r = ref()
                t0 = time.perf_counter()
                hr = r.build_hessian(x)
                t_hr = time.perf_counter() - t0
                t0 = time.perf_counter()
                st, want = r.gptq(w, idx, 4, hr, args.tokens, 0.01, False, args.sparse)
                t_gr = time.perf_counter() - t0
                codes = q.unpack_values(got.base)
                codes_ref = q.unpack_values(q.PackedIntMatrix(N, K - O, 4, want["base"]))
                res.update(cpu_hessian_s=t_hr, cpu_gptq_s=t_gr, cpu_threads=os.cpu_count(),
                           code_agreement=float((codes == codes_ref).mean()),
                           scales_equal=bool(np.array_equal(got.scales, want["scales"])),
                           speedup_gptq=t_gr / t_g)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
