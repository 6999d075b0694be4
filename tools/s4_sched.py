"""Decode-kernel schedule check: for each shape, the decode-regime forward (stream4.cu,
schedule from QUIK_S4_SPLITS / the cost model) must equal the V1 (unfused) forward bit
for bit; prints the time of one forward (10 per CUDA graph, median of 5 replays)."""
import json
import os
import statistics
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2310_09259_b200 as q  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(11)
for name, K, N, O in [("70B up", 8192, 28672, 256), ("OPT-66B fc1", 9216, 36864, 256), ("Falcon fc1", 14848, 59392, 256),
                      ("odd", 2048, 20480 + 384, 64)]:
    idx = torch.randperm(K, generator=g, device=dev)[:O].sort().values.cpu().numpy()
    outl = q.OutlierSet.from_indices(K, idx)
    W = torch.randn(N, K, device=dev, generator=g)
    base, sc, wr, ow = q.rtn_quantize_weights_device(W, outl, 4)
    del W
    L = q.QuikLinear.from_device(outl, base, sc, wr, ow, 4)
    for M in (1, 16):
        x = torch.randn(M, K, device=dev, dtype=torch.float16, generator=g)
        y = L(x, out_dtype=torch.float32)
        y1 = L(x, out_dtype=torch.float32, variant=q.PipelineVariant.V1Unfused)
        torch.cuda.synchronize()
        same = bool(torch.equal(y.view(torch.int32), y1.view(torch.int32)))
        yt = torch.empty(M, N, device=dev, dtype=torch.float16)
        L(x, out=yt)
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            for _ in range(10):
                L(x, out=yt)
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gr.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 100)
        print(json.dumps(dict(sched=os.environ.get("QUIK_S4_SPLITS", "auto"), name=name, M=M, us=round(statistics.median(ts), 2),
                              bit_identical_to_v1=same)), flush=True)
    del L, base, ow
    torch.cuda.empty_cache()
