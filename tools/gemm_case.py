"""One fused-GEMM case for tuning / ncu: builds a synthetic layer (optionally 2:4
sparse) and times K1 + GEMM (graph replay) with variations.

  python tools/gemm_case.py --M 2048 --K 5120 --N 13824 --O 256 [--sparse] [--tile 2,192]
                            [--probe] [--once]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch

import paper_2310_09259_b200 as q
from bench import prune_24


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--M", type=int, default=2048)
    ap.add_argument("--K", type=int, default=5120)
    ap.add_argument("--N", type=int, default=13824)
    ap.add_argument("--O", type=int, default=256)
    ap.add_argument("--bits", type=int, default=4)
    ap.add_argument("--sparse", action="store_true")
    ap.add_argument("--tile", default="")
    ap.add_argument("--probe", action="store_true", help="GEMM without output stores")
    ap.add_argument("--once", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = q.load_library()
    if a.tile:
        cg, bn = (int(v) for v in a.tile.split(","))
        q._lib.check(lib.quik_set_gemm_tile(cg, bn))
    g = torch.Generator(device=dev).manual_seed(3)
    idx = torch.randperm(a.K, generator=g, device=dev)[: a.O].sort().values.cpu().numpy()
    outl = q.OutlierSet.from_indices(a.K, idx)
    W = torch.randn(a.N, a.K, device=dev, generator=g)
    if a.sparse:
        prune_24(W, torch.as_tensor(outl.permutation[: a.K - a.O], device=dev))
    base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, a.bits)
    del W
    layer = q.QuikLinear.from_device(outl, base, sc, wr, ow, a.bits, sparse=a.sparse)
    x = torch.randn(a.M, a.K, device=dev, dtype=torch.float16)
    y = torch.empty(a.M, a.N, device=dev, dtype=torch.float16)
    if a.probe:
        lib.quik_set_probe_mode(1)
    if a.once:
        layer.forward(x, out=y)
        torch.cuda.synchronize()
        return
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for e in ev:  # materialise the raw cudaEvent handles (the C ABI records ev[1])
        e.record()
    ks, gs = [], []
    for i in range(25):
        ev[0].record()
        layer.forward(x, out=y, mid_event=ev[1])
        ev[2].record()
        torch.cuda.synchronize()
        if i >= 5:
            ks.append(ev[0].elapsed_time(ev[1]))
            gs.append(ev[1].elapsed_time(ev[2]))
    gemm = sorted(gs)[len(gs) // 2]
    ops = 2.0 * a.M * a.N * a.K
    print(json.dumps(dict(M=a.M, K=a.K, N=a.N, O=a.O, sparse=layer.is_sparse, tile=a.tile, probe=a.probe,
                          k1_us=1e3 * sorted(ks)[len(ks) // 2], gemm_us=1e3 * gemm, gemm_tops=ops / gemm / 1e9)))


if __name__ == "__main__":
    main()
