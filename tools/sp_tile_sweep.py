"""2:4 sparse GEMM tile sweep at cfg5 (LLaMA-2-13B up 5120 -> 13824 and q 5120 -> 5120,
2048 tokens, W4A4, 256 outliers): forward time per tile configuration, with and without
4-CTA TMA-multicast clusters (quik_set_gemm_multicast), against the dense layer.
10 forwards per CUDA graph."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2310_09259_b200 as q  # noqa: E402
from paper_2310_09259_b200 import _lib  # noqa: E402
from bench import prune_24  # noqa: E402
from tile_sweep import timeit  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    lib = q.load_library()
    for name, M, K, N, O in [("13B up", 2048, 5120, 13824, 256), ("13B q", 2048, 5120, 5120, 256)]:
        g = torch.Generator(device=dev).manual_seed(1)
        idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy()
        outl = q.OutlierSet.from_indices(K, idx)
        W = torch.randn(N, K, device=dev, generator=g)
        dense = q.QuikLinear.from_device(outl, *q.rtn_quantize_weights_device(W, outl, 4), 4)
        prune_24(W, torch.as_tensor(outl.permutation[: K - O], device=dev))
        sp = q.QuikLinear.from_device(outl, *q.rtn_quantize_weights_device(W, outl, 4), 4, sparse=True)
        del W
        x = torch.randn(M, K, device=dev, dtype=torch.float16)
        y = torch.empty(M, N, device=dev, dtype=torch.float16)
        res = dict(name=name, sparse=sp.is_sparse)
        for lname, layer in (("dense", dense), ("sp", sp)):
            for cfg in [(0, 0), (1, 128), (2, 128), (2, 192), (2, 256)]:
                for mc in (0, 1):
                    if mc and cfg[0] != 2:
                        continue
                    lib.quik_set_gemm_multicast(mc)
                    if lib.quik_set_gemm_tile(*cfg) != 0:
                        continue
                    try:
                        layer.forward(x, out=y)
                        gr = torch.cuda.CUDAGraph()
                        with torch.cuda.graph(gr):
                            for _ in range(10):
                                layer.forward(x, out=y)
                        res[f"{lname}_{cfg[0]}x{cfg[1]}{'_mc' if mc else ''}_us"] = round(timeit(gr.replay) / 10 * 1e3, 1)
                    except Exception as e:  # unsupported tile for this path
                        res[f"{lname}_{cfg[0]}x{cfg[1]}{'_mc' if mc else ''}_us"] = str(e)[:60]
        lib.quik_set_gemm_tile(0, 0)
        lib.quik_set_gemm_multicast(0)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
