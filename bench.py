#!/usr/bin/env python
"""bench.py — QUIK linear-layer throughput on B200 (BASELINE.json metric:
"QUIK linear TOPS & speedup vs FP16 cuBLAS at LLaMA-2-70B shapes, 1/2/4/8 GPU").

One step = one QUIK linear forward (K1 fused quantizer + fused tcgen05 INT/FP16
GEMM with the dequantisation epilogue) over a synthetic activation batch of the
workload shape, inputs resident in HBM. Default workload: BASELINE configs[2],
the LLaMA-2-70B MLP up/gate layer 8192 -> 28672, 256 outliers, W4A4, 4096 tokens
(fits one GPU). For N > 1 (torchrun, or self-launched by --gpus N) the output
features are sharded over the ranks and every rank's GEMM epilogue stores its f16
shard into every rank's [M][N] output through CUDA IPC (the all-gather fused into
the GEMM; NCCL all-gather timed beside it; strong scaling: total work fixed).
value = whole-job TOPS = 2*M*N*K / step time (max over ranks).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3]
  python bench.py --impl reference ...   # the reference's own CPU quik_matmul
                                         # (oracle/_ref: the unmodified sources)

Extra keys: roofline (GEMM kernel vs tensor peak), cpu_baseline (reference CPU
path on this host), e2e (host buffers through the public API, H2D/D2H inside the
timed region), fp16_cublas (torch.matmul f16 of the same shape), clocks,
gpu_launches.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "QUIK linear TOPS & speedup vs FP16 cuBLAS at LLaMA-2-70B shapes, 1/2/4/8 GPU"

WORKLOADS = {
    # BASELINE.json configs[2] (headline): LLaMA-2-70B MLP up/gate (arch/llama2-70b.json:16-17)
    "cfg3": dict(desc="LLaMA-2-70B MLP up/gate 8192->28672, 256 outliers, W4A4, 4096 tokens",
                 M=4096, K=8192, N=28672, O=256, bits=4),
    "cfg3-down": dict(desc="LLaMA-2-70B MLP down 28672->8192, 896 outliers, W8A8, 4096 tokens",
                      M=4096, K=28672, N=8192, O=896, bits=8),
    "cfg1": dict(desc="QUIK W4A4 4096->4096, 128 outliers, 16 tokens (oracle shape)", M=16, K=4096, N=4096, O=128,
                 bits=4),
    "cfg2-qkvo": dict(desc="LLaMA-2-7B q/k/v/o 4096->4096, 256 outliers, W4A4, 2048 tokens", M=2048, K=4096,
                      N=4096, O=256, bits=4),
    "cfg2-up": dict(desc="LLaMA-2-7B up/gate 4096->11008, 256 outliers, W4A4, 2048 tokens", M=2048, K=4096,
                    N=11008, O=256, bits=4),
    "cfg2-down": dict(desc="LLaMA-2-7B down 11008->4096, 688 outliers, W8A8, 2048 tokens", M=2048, K=11008,
                      N=4096, O=688, bits=8),
    "cfg4-opt-fc1": dict(desc="OPT-66B fc1 9216->36864, 256 outliers, W4A4, 2048 tokens", M=2048, K=9216,
                         N=36864, O=256, bits=4),
    # BASELINE.json configs[4]: W4A4 + 2:4 structured-sparse base weights, LLaMA-2-13B
    # (hidden 5120, intermediate 13824; public model card), 2048 tokens
    "cfg5-up": dict(desc="LLaMA-2-13B up/gate 5120->13824, 256 outliers, W4A4 + 2:4 sparse, 2048 tokens", M=2048,
                    K=5120, N=13824, O=256, bits=4, sparse=True),
    "cfg5-q": dict(desc="LLaMA-2-13B q/k/v/o 5120->5120, 256 outliers, W4A4 + 2:4 sparse, 2048 tokens", M=2048,
                   K=5120, N=5120, O=256, bits=4, sparse=True),
}


def prune_24(W, base_cols):
    """2:4 magnitude pruning over the permuted base columns (the two smallest |w| of
    every aligned group of 4 -> 0): the structure sparsegpt_joint produces
    (quantizer.cpp:299-337) with an identity Hessian. W: torch or numpy [N][K]."""
    import torch

    t = torch.as_tensor(W)
    cols = torch.as_tensor(base_cols, device=t.device)
    wb = t[:, cols]
    g = wb.shape[1] // 4 * 4
    grp = wb[:, :g].reshape(t.shape[0], -1, 4)
    drop = grp.abs().argsort(dim=-1, stable=True)[..., :2]
    grp.scatter_(-1, drop, 0.0)
    wb[:, :g] = grp.reshape(t.shape[0], g)
    t[:, cols] = wb
    return W

CPU_SAMPLE_TOKENS = 256  # bounded sample of the workload for the CPU reference (~1 s per call at cfg3)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm_gbs=float(d["hbm_gbs"]), bf16=float(d["bf16_tflops"]),
                    bf16_sustained=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), source="measured")
    return dict(hbm_gbs=6650.0, bf16=1590.0, bf16_sustained=1400.0, source="fallback")


def emit(obj):
    print(json.dumps(obj), flush=True)


# =============================================================================== reference arm


def synth_host(w, seed, tokens):
    """CPU synthetic layer for the reference arm, bench.cpp:51-72 style: W, x ~ N(0,1),
    O random heavy columns x50, outliers = select_outliers(x), RTN weights — all with
    the reference's own functions (oracle/_ref)."""
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import ref  # the reference's compiled sources (TEST/BASELINE infrastructure)

    r = ref()
    rng = np.random.default_rng(seed)
    W = rng.standard_normal((w["N"], w["K"]), dtype=np.float32)
    x = rng.standard_normal((tokens, w["K"]), dtype=np.float32)
    heavy = np.unique(rng.integers(0, w["K"], size=max(w["O"], 1)))
    if w["O"]:
        x[:, heavy] *= 50.0
    x = x.astype(np.float16).astype(np.float32)
    idx = r.select_outliers(x, w["O"])
    if w.get("sparse"):
        prune_24(W, np.setdiff1d(np.arange(w["K"]), idx))  # the reference runs it densely over the zeros
    q = r.rtn_quantize_weights(W, idx, w["bits"])
    del W
    L = dict(in_features=w["K"], out_features=w["N"], bits=w["bits"], act_bits=w["bits"], base=q["base"],
             scales=q["scales"], wreduced=q["wreduced"], outlier_weights=q["outlier_weights"], idx=idx, bias=None)
    return r, L, x


def run_reference(args, w):
    """The reference's own CPU implementation (oracle/_ref = proj/src compiled unchanged,
    OpenMP on all host threads), each step one quik_matmul V3 call on a bounded token
    sample of the workload. With --layer-npz (bench.py's own cpu_baseline leg) the layer
    and the sampled tokens come from the GPU arm's run and the output is saved to
    --ref-out as the parity checker."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    if args.layer_npz:
        sys.path.insert(0, str(ROOT / "tests"))
        from oracle_lib import ref  # the reference's compiled sources (the cpu_baseline leg)

        r = ref()
        z = np.load(args.layer_npz)
        x = z["x"]
        L = dict(in_features=int(z["in_features"]), out_features=int(z["out_features"]), bits=int(z["bits"]),
                 act_bits=int(z["bits"]), base=z["base"], scales=z["scales"], wreduced=z["wreduced"],
                 outlier_weights=z["outlier_weights"], idx=z["idx"], bias=z["bias"] if "bias" in z else None)
        n_out = L["out_features"]
    else:
        r, L, x = synth_host(w, args.seed, args.cpu_tokens)
        n_out = w["N"]
    M_s = x.shape[0]
    h, keep = r.layer_create(L)
    times = np.zeros(6)
    for _ in range(args.warmup):
        st, _ = r.layer_forward(h, x, n_out, 2)
        assert st == 0, st
    per = []
    stage = np.zeros(6)
    y = None
    for _ in range(args.steps):
        t0 = time.perf_counter()
        st, y = r.layer_forward(h, x, n_out, 2, times)
        per.append(time.perf_counter() - t0)
        assert st == 0, st
        stage += times
    r.layer_destroy(h)
    if args.ref_out:
        np.save(args.ref_out, y)
    med = statistics.median(per)
    ops = 2.0 * M_s * n_out * w["K"]
    value = ops / med / 1e12
    sample = (f"{M_s} of {w['M']} tokens of {args.workload} ({w['desc']}); quik_matmul V3 per step (median of "
              f"{args.steps}), OpenMP threads={os.environ.get('OMP_NUM_THREADS')}")
    out = dict(metric=METRIC, value=value, unit="TOPS", n_gpus=args.gpus, steps=args.steps, warmup=args.warmup,
               ms_per_step=1e3 * med, higher_is_better=True, scaling="strong", vs_baseline=None,
               dtype="int8", data="synthetic", impl="reference",
               config=dict(workload=args.workload, M=w["M"], K=w["K"], N=w["N"], outliers=w["O"], bits=w["bits"],
                           sample_tokens=M_s),
               cpu_baseline=dict(value=value, unit="TOPS", cores=int(os.environ.get("OMP_NUM_THREADS", cores)),
                                 kind="reference", sample=sample,
                                 stage_ms_mean=dict(zip(["split", "quantize", "int_matmul", "fp_matmul",
                                                         "dequantize", "add"],
                                                        (stage / args.steps).round(3).tolist()))),
               e2e=dict(value=value, unit="TOPS", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    emit(out)


# =============================================================================== our arm


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        self.proc = None
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            p = [s.strip() for s in line.split(",")]
            if len(p) < 9:
                continue
            try:
                rows.append(dict(sm=float(p[1]), smax=float(p[2]), power=float(p[3]), hw=p[5], hwt=p[6], swt=p[7],
                                 swp=p[8]))
            except ValueError:
                continue
        os.unlink(self.path)
        if not rows:
            return None
        load = [r for r in rows if r["power"] > 300.0] or rows
        reasons = sorted({name for r in load for name, key in (("hw_slowdown", "hw"),
                                                                 ("hw_thermal_slowdown", "hwt"),
                                                                 ("sw_thermal_slowdown", "swt"),
                                                                 ("sw_power_cap", "swp")) if r[key] == "Active"})
        return dict(sm_mhz=statistics.median(r["sm"] for r in load), sm_max_mhz=max(r["smax"] for r in rows),
                    reasons=reasons, samples=len(rows), samples_under_load=len(load),
                    power_w_max=max(r["power"] for r in rows))


L2_BYTES = 126 * 1024 * 1024  # B200 L2


def cublaslt_int8_peak(dev):
    """Live dense INT8 tensor-core throughput of this GPU: cuBLASLt (torch._int_mm)
    int8 x int8 -> int32 at 8192^3, best of 5 (tools/int8_peak.py is the standalone
    version whose output is committed under profiles/)."""
    import torch

    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t()
    for _ in range(2):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch._int_mm(a, b)
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def f16_output_bound(want, xs_o, ow, bias):
    """Per-element bound on |y_f16 - reference| (the same formula as
    tests/oracle_lib.f16_output_bound): 2^-11|r| + 2^-25 + (1 + 2^-11)(1.125 O + 3) 2^-24 T,
    T = |r| + 2|bias| + 2 sum|x_o w_o|."""
    O = xs_o.shape[1]
    r = np.abs(want.astype(np.float64))
    T = r.copy()
    if O:
        T += 2.0 * (np.abs(xs_o.astype(np.float64)) @ np.abs(ow.astype(np.float64)).T)
    if bias is not None:
        T += 2.0 * np.abs(bias.astype(np.float64))[None, :]
    return 2.0 ** -11 * r + 2.0 ** -25 + (1.0 + 2.0 ** -11) * (1.125 * O + 3.0) * 2.0 ** -24 * T


def cpu_leg(args, w, host, xs16, y_sample):
    """cpu_baseline + parity: the reference's own quik_matmul (oracle/_ref, the unmodified
    sources, OpenMP on every host core; a subprocess so OMP_NUM_THREADS applies) on the
    SAME layer and the sampled tokens of this run's input. Returns (cpu_baseline, parity):
    the reference's output on those tokens is the checker for this run's y."""
    tmp = tempfile.mkdtemp(prefix="quik_bench_")
    lp, op = os.path.join(tmp, "layer.npz"), os.path.join(tmp, "ref_out.npy")
    xs = xs16.astype(np.float32)
    np.savez(lp, x=xs, **host)
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", args.workload,
           "--steps", "3", "--warmup", "1", "--layer-npz", lp, "--ref-out", op]
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "LOCAL_WORLD_SIZE"):
        env.pop(k, None)
    env["OMP_NUM_THREADS"] = str(os.cpu_count() or 1)
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
        line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
        cpu = json.loads(line)["cpu_baseline"]
        want = np.load(op)
    except Exception as exc:  # reported, never silently replaced
        return (dict(value=None, unit="TOPS", cores=os.cpu_count(), kind="reference",
                     sample=f"failed: {type(exc).__name__}: {exc}"[:300]),
                dict(status="not run", reason=f"reference leg failed: {type(exc).__name__}"))
    finally:
        for f in (lp, op):
            if os.path.exists(f):
                os.unlink(f)
        os.rmdir(tmp)
    idx = host["idx"]
    bound = f16_output_bound(want, xs[:, idx], host["outlier_weights"], host.get("bias"))
    err = np.abs(y_sample.astype(np.float64) - want)
    ratio = float((err / bound).max())
    rel = float(np.linalg.norm(y_sample.astype(np.float64) - want) / max(np.linalg.norm(want), 1e-300))
    ok = ratio <= 1.0 and rel <= 5e-4 and bool(np.all(np.isfinite(y_sample)))
    parity = dict(status="ok" if ok else "fail", tokens=int(xs.shape[0]), rows=int(want.shape[1]),
                  max_err_over_bound=ratio, rel_frobenius=rel,
                  checker="reference quik_matmul V3 (oracle/_ref: proj/src compiled unchanged) on the same layer and "
                          "the sampled tokens of this run's x; f16 y vs the f32 reference within the derived per-element "
                          "bound (DESIGN.md §4) and rel_frobenius <= 5e-4")
    return cpu, parity


def run_ours(args, w):
    import torch
    import torch.distributed as dist

    import paper_2310_09259_b200 as q

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # QUIK_BENCH_DIST_BACKEND=gloo + fewer GPUs than ranks: a functional check of the
    # N > 1 code path on a one-GPU box (ranks share the device); never a bench number
    backend = os.environ.get("QUIK_BENCH_DIST_BACKEND", "nccl")
    ndev = torch.cuda.device_count()
    if backend == "nccl" and world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if backend != "nccl" and ndev < world:
        local = local % ndev
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    def max_over_ranks(t):
        """In-place max over the ranks (device tensor with NCCL, through host memory with
        the gloo check backend)."""
        if backend == "nccl":
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        else:
            h = t.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MAX)
            t.copy_(h)

    M, K, N, O, bits = w["M"], w["K"], w["N"], w["O"], w["bits"]
    if N % world:
        raise SystemExit(f"out_features {N} not divisible by {world} GPUs")
    ns = N // world
    kb = K - O

    # ---- synthetic layer, generated on the device (same seed on every rank)
    g = torch.Generator(device=dev)
    g.manual_seed(args.seed)
    x = torch.randn((M, K), generator=g, device=dev, dtype=torch.float32)
    heavy = torch.unique(torch.randint(0, K, (max(O, 1),), generator=g, device=dev))
    if O:
        x[:, heavy] *= 50.0
    x16 = x.half()
    maxabs = x16.float().abs().amax(0)
    order = torch.sort(maxabs, descending=True, stable=True).indices[:O]
    outliers = q.OutlierSet.from_indices(K, order.cpu().numpy())
    del x, maxabs
    Wt = torch.randn((ns, K), generator=torch.Generator(device=dev).manual_seed(args.seed * 1000 + rank), device=dev,
                     dtype=torch.float32)
    sparse = bool(w.get("sparse"))
    if sparse:
        prune_24(Wt, torch.as_tensor(outliers.permutation[:kb], device=dev))
    base, sc, wr, ow = q.rtn_quantize_weights_device(Wt, outliers, bits)
    del Wt
    layer = q.QuikLinear.from_device(outliers, base, sc, wr, ow, bits, sparse=sparse)
    if sparse and not layer.is_sparse:
        raise SystemExit("2:4 workload: layer did not compress")
    # the same layer with ONE INT4 weight copy in HBM (weights="int4": every GEMM tile
    # widens the INT4 tiles into TMEM), reported beside the headline's speed mode
    layer4 = (q.QuikLinear.from_device(outliers, base, sc, wr, ow, bits, weights="int4")
              if bits == 4 and not sparse and world == 1 and not args.no_cublas else None)
    check_cpu = rank == 0 and world == 1 and not args.no_cpu
    host = None
    if check_cpu:  # reference-format copy of the layer for the CPU reference leg (cpu_baseline + parity)
        host = dict(base=base.cpu().numpy(), scales=sc.cpu().numpy(), wreduced=wr.cpu().numpy(),
                    outlier_weights=ow.half().float().cpu().numpy().reshape(ns, O), idx=outliers.indices,
                    in_features=np.int64(K), out_features=np.int64(ns), bits=np.int64(bits))
    del base, ow
    torch.cuda.synchronize()

    # inputs rotated over enough copies of x that the set exceeds L2 (x is only read by
    # K1; the weights and y are each larger than L2 at the headline shape)
    nbuf = max(1, -(-3 * L2_BYTES // 2 // (M * K * 2)))
    nbuf = min(nbuf, 8)
    xs_dev = [x16] + [x16.clone() for _ in range(nbuf - 1)]
    footprint = nbuf * M * K * 2 + ns * ((kb + 127) // 128 * 128) + M * ns * 2
    flush = footprint < 2 * L2_BYTES
    flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if flush else None

    def all_gather(out, inp):
        if backend == "nccl":
            dist.all_gather_into_tensor(out, inp)
        else:  # gloo check mode: through host memory
            parts = [torch.empty_like(inp, device="cpu") for _ in range(world)]
            dist.all_gather(parts, inp.cpu())
            out.copy_(torch.stack(parts))

    y_local = torch.empty((M, ns), dtype=torch.float16, device=dev)
    fused, fused_err = None, None
    if world > 1:
        gathered = torch.empty((world, M, ns), dtype=torch.float16, device=dev)
        y = torch.empty((M, N), dtype=torch.float16, device=dev)
        # N > 1 exchange: the all-gather fused into the GEMM epilogue (CUDA IPC peer
        # stores into every rank's [M][N] output + a one-element NCCL all-reduce as the
        # completion fence); NCCL all-gather + transpose is measured beside it
        try:
            from paper_2310_09259_b200.sharded import FusedShardedQuikLinear

            def gloo_fence():
                torch.cuda.synchronize()
                dist.barrier()

            fused = FusedShardedQuikLinear(None, M, local=layer, n_total=N,
                                           barrier_fn=None if backend == "nccl" else gloo_fence)
        except Exception as exc:  # reported in the JSON line; the NCCL exchange is used instead
            fused, fused_err = None, f"{type(exc).__name__}: {exc}"[:300]

    def step_nccl(i):
        layer.forward(xs_dev[i % nbuf], out=y_local)
        all_gather(gathered, y_local)
        y.view(M, world, ns).copy_(gathered.permute(1, 0, 2))

    def step(i, mid_event=None):
        if world == 1:
            layer.forward(xs_dev[i % nbuf], out=y_local, mid_event=mid_event)
        elif fused is not None:
            fused(xs_dev[i % nbuf])
        else:
            step_nccl(i)

    steps, warm = args.steps, args.warmup
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    ev_step = [(ev(), ev()) for _ in range(steps)]
    ev_mid = [(ev(), ev(), ev()) for _ in range(steps)]
    for e in [e for t in ev_step + ev_mid for e in t]:  # materialise the raw cudaEvent handles
        e.record()
    for i in range(warm):
        step(i)
    torch.cuda.synchronize()

    # ---- timed region: K steps, max over ranks. Large workloads: back to back with no
    # event inside (the PDL chain K1 -> GEMM -> next K1 runs as in production);
    # L2-resident workloads: each step bracketed by events with an L2 flush in between
    sampler = ClockSampler(local) if not args.no_clocks else None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start, end = ev(), ev()
    if not flush:
        start.record()
        for i in range(steps):
            step(i)
        end.record()
        torch.cuda.synchronize()
        total_ms = start.elapsed_time(end)
    else:
        for i in range(steps):
            flush_buf.fill_(float(i))
            ev_step[i][0].record()
            step(i)
            ev_step[i][1].record()
        torch.cuda.synchronize()
        total_ms = sum(a.elapsed_time(b) for a, b in ev_step)
    if world > 1:
        dist.barrier()

    # ---- per-step and per-kernel passes (outside the headline region): the median step
    # and the K1 / GEMM split (an event between the two kernels)
    for i in range(steps):
        if flush:
            flush_buf.fill_(float(i))
        ev_step[i][0].record()
        step(i)
        ev_step[i][1].record()
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in ev_step]
    for i in range(steps):
        if flush:
            flush_buf.fill_(float(i))
        ev_mid[i][0].record()
        layer.forward(xs_dev[i % nbuf], out=y_local, mid_event=ev_mid[i][1])
        ev_mid[i][2].record()
    torch.cuda.synchronize()
    quant_ms = [a.elapsed_time(b) for a, b, _ in ev_mid]
    gemm_ms = [b.elapsed_time(c) for _, b, c in ev_mid]

    exchange = None
    if world > 1:
        # the same K steps with the other exchange, and compute only (no exchange)
        def timed(fn):
            torch.cuda.synchronize()
            dist.barrier()
            a, b = ev(), ev()
            a.record()
            for i in range(steps):
                fn(i)
            b.record()
            torch.cuda.synchronize()
            t = torch.tensor([a.elapsed_time(b) / steps], device=dev, dtype=torch.float64)
            max_over_ranks(t)
            return float(t.item())

        exchange = dict(headline="fused all-gather (CUDA IPC peer stores in the GEMM epilogue + NCCL fence)"
                        if fused is not None else "NCCL all-gather + transpose", fused_error=fused_err,
                        nccl_allgather_ms=timed(step_nccl),
                        compute_only_ms=timed(lambda i: layer.forward(xs_dev[i % nbuf], out=y_local)))
        if fused is not None:
            exchange["fused_ms"] = timed(lambda i: fused(xs_dev[i % nbuf]))

    sustained = None
    if args.soak_s > 0:
        # sustained continuation (power-cap steady state), reported next to the value
        s0, s1 = ev(), ev()
        n_sus = 0
        t_end = time.perf_counter() + args.soak_s
        s0.record()
        while time.perf_counter() < t_end:
            for j in range(20):
                step(j)
            n_sus += 20
            torch.cuda.synchronize()
        s1.record()
        torch.cuda.synchronize()
        ts = torch.tensor([s0.elapsed_time(s1) / n_sus], device=dev, dtype=torch.float64)
        if world > 1:
            max_over_ranks(ts)
        ts = float(ts.item())
        sustained = dict(value=2.0 * M * N * K / (ts * 1e-3) / 1e12, unit="TOPS", ms_per_step=ts, steps=n_sus,
                         note="same step repeated back to back for --soak-s seconds after the timed region")
    clocks = sampler.stop() if sampler else None

    stats = torch.tensor([total_ms, statistics.median(step_ms), statistics.median(gemm_ms),
                          statistics.median(quant_ms), statistics.mean(gemm_ms), statistics.mean(quant_ms)],
                         device=dev, dtype=torch.float64)
    if world > 1:
        max_over_ranks(stats)
    total_ms, step_med, gemm_med, quant_med, gemm_mean, quant_mean = stats.tolist()
    ms_per_step = total_ms / steps
    ops = 2.0 * M * N * K
    value = ops / (ms_per_step * 1e-3) / 1e12

    # ---- roofline of the dominant kernel (fused GEMM), per launch on this rank
    pk = peaks()
    p_f16 = pk["bf16"]
    i8_live = cublaslt_int8_peak(dev) if not args.no_cublas else None
    # INT8 peak: the larger of 2x the measured bf16 rate (B200 dense INT8 = 2x FP16) and
    # the live cuBLASLt INT8 rate (conservative: the larger peak gives the lower frac)
    p_i8 = max(2.0 * p_f16, i8_live or 0.0)
    if sparse:
        p_i8 *= 2.0  # 2:4 sparse INT8 (tcgen05.mma.sp) = 2x dense INT8
    ops_rank = 2.0 * M * ns * K
    t_ideal_s = 2.0 * M * ns * kb / (p_i8 * 1e12) + 2.0 * M * ns * O / (p_f16 * 1e12)
    mixed_peak = ops_rank / t_ideal_s / 1e12
    achieved = ops_rank / (gemm_med * 1e-3) / 1e12
    a_bytes = (lambda n: (n + 1) // 2) if bits == 4 else (lambda n: n)
    w_bytes = ns * a_bytes(kb) if not sparse else ns * a_bytes(kb) // 2 + ns * kb // 8
    gemm_bytes = M * a_bytes(kb) + w_bytes + ns * O * 2 + M * O * 2 + 12 * ns + 8 * M + M * ns * 2
    traffic = None
    tp = ROOT / "profiles" / "ncu_gemm_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get(args.workload)
        except Exception:
            traffic = None
    roofline = dict(bound="tensor", achieved=achieved, peak=mixed_peak, unit="TFLOP/s", frac=achieved / mixed_peak,
                    traffic=traffic, algorithmic_bytes=gemm_bytes,
                    traffic_ratio=(traffic / gemm_bytes) if traffic else None,
                    kernel="quik_gemm_kernel (fused int8 GEMM%s + f16 outlier GEMM + dequant epilogue)"
                           % (" on 2:4-compressed weights, tcgen05.mma.sp" if sparse else ""),
                    kernel_ms_median=gemm_med, kernel_ms_mean=gemm_mean,
                    peak_basis=(f"{pk['source']} bf16 burst {p_f16:.1f} TF/s (MEASURED_PEAKS.json) for the {O} f16 "
                                f"outlier columns; INT8 peak = max(2 x bf16, live cuBLASLt int8 "
                                f"{(i8_live or 0):.1f} TOPS) = {p_i8 / (2 if sparse else 1):.1f} TOPS"
                                f"{' x2 for 2:4 sparse' if sparse else ''} for the {kb} int columns (dense-equivalent "
                                "ops); mixed peak = ops / (int_ops/P_i8 + f16_ops/P_f16); achieved from the median "
                                "GEMM launch (CUDA events on the launch stream)"),
                    int8_peak_cublaslt_tops=i8_live, int8_only_frac=achieved / p_i8,
                    nominal_frac=achieved / (ops_rank / (2.0 * M * ns * kb / ((9000.0 if sparse else 4500.0) * 1e12)
                                                         + 2.0 * M * ns * O / (2250.0 * 1e12)) / 1e12),
                    note="denominators are a cuBLAS-derived measured peak (a kernel can read a little above 1.0, "
                         "B200_PROFILING.md); nominal_frac is against the nominal dense 4.5 POPS int8 / 2.25 PFLOPS "
                         "f16 at the boost clock")
    # K1 algorithmic bytes per SURVEY.md §8(d): x f16 in, the codes at the reference's
    # width (INT4: ceil(K_b/2) per token), x_outlier f16, scale + zero
    bytes_q = M * K * 2 + M * a_bytes(kb) + M * O * 2 + 8 * M
    quant = dict(kernel="quantize_hot_kernel (K1, persistent TMA ring)", ms_median=quant_med, ms_mean=quant_mean,
                 algorithmic_bytes=bytes_q, achieved_gbs=bytes_q / (quant_med * 1e-3) / 1e9,
                 peak_gbs=pk["hbm_gbs"], frac=(bytes_q / (quant_med * 1e-3) / 1e9) / pk["hbm_gbs"],
                 device_layout_bytes=M * K * 2 + M * ((kb + 127) // 128 * 128) + M * ((O + 63) // 64 * 64) * 2 + 8 * M,
                 note="§8(d) bytes (codes at the INT%d width); the kernel writes int8 GEMM-layout codes" % bits)

    # ---- FP16 cuBLAS GEMM of the same (sharded) shape, same x
    fp16 = None
    int4_weights = None
    if not args.no_cublas:
        Wf = torch.randn((ns, K), device=dev, dtype=torch.float16)
        out16 = torch.empty((M, ns), device=dev, dtype=torch.float16)
        for _ in range(3):
            torch.matmul(x16, Wf.t(), out=out16)
        torch.cuda.synchronize()
        t16s = []
        for i in range(steps):
            if flush:
                flush_buf.fill_(float(i))
            ev_step[i][0].record()
            torch.matmul(xs_dev[i % nbuf], Wf.t(), out=out16)
            ev_step[i][1].record()
        torch.cuda.synchronize()
        t16s = [a.elapsed_time(b) for a, b in ev_step]
        t16 = torch.tensor([statistics.median(t16s)], device=dev, dtype=torch.float64)
        if world > 1:
            max_over_ranks(t16)
        t16 = float(t16.item())
        fp16 = dict(ms_median=t16, tflops=2.0 * M * ns * K / (t16 * 1e-3) / 1e12, speedup_step=t16 / step_med,
                    speedup_gemm=t16 / gemm_med,
                    note="torch.matmul f16 (cuBLAS) of the per-rank shape, same x; medians of per-step events")
        decode = decode_regime(torch, layer, xs_dev[0], Wf, ns, K, kb, O, bits, pk) if world == 1 else None
        del Wf, out16
        if layer4 is not None:
            for i in range(3):
                layer4.forward(xs_dev[i % nbuf], out=y_local)
            torch.cuda.synchronize()
            for i in range(steps):
                if flush:
                    flush_buf.fill_(float(i))
                ev_step[i][0].record()
                layer4.forward(xs_dev[i % nbuf], out=y_local)
                ev_step[i][1].record()
            torch.cuda.synchronize()
            t4 = statistics.median(a.elapsed_time(b) for a, b in ev_step)
            int4_weights = dict(ms_median=t4, tops=ops_rank / (t4 * 1e-3) / 1e12, speedup_vs_cublas_f16=t16 / t4,
                                device_bytes=layer4.device_bytes, speed_mode_device_bytes=layer.device_bytes,
                                note="the same layer built with weights='int4' (one INT4 weight copy in HBM, widened "
                                     "into TMEM inside every GEMM tile; quik_layer_create QUIK_WEIGHTS_INT4): "
                                     "K1 + GEMM per step, median of per-step events; the headline runs speed mode "
                                     "(an INT8 copy for prefill GEMMs)")
        del layer4
    else:
        decode = None
        del layer4

    # ---- e2e: host (pinned) buffers through the public API, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        xh = x16.cpu().pin_memory()
        yh = torch.empty((M, N if world > 1 else ns), dtype=torch.float16).pin_memory()
        xd = torch.empty_like(x16)
        e2e_steps = max(3, min(steps, 10))

        def e2e_step():
            if world == 1:
                # the host-buffer entry point: chunked H2D / kernels / D2H overlap
                layer.forward_host(xh, yh)
                return
            xd.copy_(xh, non_blocking=True)
            if fused is not None:
                yy = fused(xd)
            else:
                layer.forward(xd, out=y_local)
                all_gather(gathered, y_local)
                y.view(M, world, ns).copy_(gathered.permute(1, 0, 2))
                yy = y
            if rank == 0:
                yh.copy_(yy, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = ev(), ev()
        a.record()
        for _ in range(e2e_steps):
            e2e_step()
        b.record()
        torch.cuda.synchronize()
        te = torch.tensor([a.elapsed_time(b) / e2e_steps], device=dev, dtype=torch.float64)
        if world > 1:
            max_over_ranks(te)
        te = float(te.item())
        e2e = dict(value=ops / (te * 1e-3) / 1e12, unit="TOPS", h2d_bytes_per_step=M * K * 2 * world,
                   d2h_bytes_per_step=M * N * 2, ms_per_step=te, steps=e2e_steps,
                   path=("QuikLinear.forward_host (C ABI quik_linear_forward_host: chunked, H2D/kernels/D2H overlapped)"
                         if world == 1 else ("FusedShardedQuikLinear (C ABI quik_linear_forward_sharded, IPC peer stores)"
                                             if fused is not None else "QuikLinear.forward + NCCL all-gather"))
                   + " with pinned host f16 x -> y")
        if world == 1:
            # the reference-facing drop-in call (C++ facade quik::b200::quik_matmul on an
            # FpMatrix): f32 host x in, f32 host y out, same C ABI entry point
            xh32 = x16.float().cpu().pin_memory()
            yh32 = torch.empty((M, ns), dtype=torch.float32).pin_memory()
            layer.forward_host(xh32, yh32)
            torch.cuda.synchronize()
            a2, b2 = ev(), ev()
            a2.record()
            for _ in range(e2e_steps):
                layer.forward_host(xh32, yh32)
            b2.record()
            torch.cuda.synchronize()
            tf = a2.elapsed_time(b2) / e2e_steps
            e2e["f32_drop_in"] = dict(value=ops / (tf * 1e-3) / 1e12, unit="TOPS", ms_per_step=tf,
                                      h2d_bytes_per_step=M * K * 4, d2h_bytes_per_step=M * ns * 4,
                                      path="quik_linear_forward_host with pinned host f32 x -> f32 y (the facade's "
                                           "quik_matmul(FpMatrix) semantics)")
            del xh32, yh32

    # ---- CPU reference leg (rank 0, N = 1): cpu_baseline timing and the parity check of
    # this run's y, both from the reference's own code on the same layer and tokens
    cpu, parity = None, dict(status="not run", reason="N > 1 or --no-cpu")
    if check_cpu:
        rs = np.random.default_rng(args.seed)
        toks = np.sort(rs.choice(M, min(M, args.cpu_tokens), replace=False))
        ti = torch.as_tensor(toks, device=dev)
        layer.forward(xs_dev[0], out=y_local)  # y of the first input buffer
        y_sample = y_local[ti].float().cpu().numpy()
        xs16 = xs_dev[0][ti].cpu().numpy()
        cpu, parity = cpu_leg(args, w, host, xs16, y_sample)
        if cpu.get("sample"):
            cpu["sample"] += f"; tokens = {toks.size} sampled rows of this run's x (the same layer)"

    if rank == 0:
        out = dict(metric=METRIC, value=value, unit="TOPS", n_gpus=world, steps=steps, warmup=warm,
                   ms_per_step=ms_per_step, ms_per_step_median=step_med, higher_is_better=True, scaling="strong",
                   vs_baseline=None, dtype="int8", data="synthetic",
                   config=dict(workload=args.workload, desc=w["desc"], M=M, K=K, N=N, outliers=O, bits=bits,
                               parallelism=f"output-feature shards x{world}" + (
                                   "" if world == 1 else (" + all-gather fused into the GEMM epilogue (CUDA IPC)"
                                                          if fused is not None else " + NCCL all-gather")),
                               l2=(f"L2 flushed between steps (workload {footprint / 1e6:.0f} MB < 2 x L2); value = "
                                   "sum of per-step event times" if flush else
                                   f"inputs larger than L2: x rotated over {nbuf} buffers ({nbuf * M * K * 2 / 1e6:.0f} "
                                   f"MB), int8 weights {ns * ((kb + 127) // 128 * 128) / 1e6:.0f} MB, y "
                                   f"{M * ns * 2 / 1e6:.0f} MB; no flush")),
                   parity=parity, exchange=exchange, roofline=roofline, cpu_baseline=cpu, e2e=e2e, fp16_cublas=fp16, quantizer=quant,
                   sustained=sustained, decode=decode, int4_weights=int4_weights,
                   clocks=clocks, gpu_launches=steps * q.QuikLinear.launches(),
                   precision="W%dA%d integer codes on tcgen05 kind::i8 (s32 accumulate) + f16 outliers (f32 accumulate), f16 out"
                             % (bits, bits))
        emit(out)
    if world > 1:
        dist.destroy_process_group()


def decode_regime(torch, layer, x, Wf, ns, K, kb, O, bits, pk):
    """The same layer in the decode regime (1 and 16 tokens: K1 + the weight-streaming
    decode kernel, stream4.cu) against cuBLAS f16 of the same shape: 10 forwards per
    CUDA graph, median of 5 replays. HBM fraction over the bytes a forward must stream:
    the INT4 weights and the f16 outlier weights (x and y are < 1 MB)."""
    out = {}
    wbytes = ns * ((kb + 127) // 128 * 128) // (2 if bits == 4 else 1) + ns * ((O + 63) // 64 * 64) * 2

    def graph_us(fn):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(10):
                fn()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / 10)
        return statistics.median(ts)

    for t in (1, 16):
        xt = x[:t].contiguous()
        yt = torch.empty((t, ns), device=x.device, dtype=torch.float16)
        o16 = torch.empty((t, ns), device=x.device, dtype=torch.float16)
        us = graph_us(lambda: layer.forward(xt, out=yt))
        us16 = graph_us(lambda: torch.matmul(xt, Wf.t(), out=o16))
        out[f"tokens_{t}"] = dict(us=us, hbm_gbs=wbytes / (us * 1e-6) / 1e9, hbm_frac=wbytes / (us * 1e-6) / 1e9 / pk["hbm_gbs"],
                                  cublas_f16_us=us16, speedup=us16 / us)
    out["weight_bytes"] = wbytes
    out["note"] = ("same layer, first 1 / 16 tokens of x: K1 + the INT4 decode kernel; 10 forwards per CUDA graph, "
                   "median of 5 replays; HBM fraction of the INT4 + f16 outlier weight bytes")
    return out


def spawn_ranks(args) -> int:
    """--gpus N > 1 without a torchrun environment: launch N ranks of this script (one
    process per GPU, rendezvous on 127.0.0.1) and return their exit status."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(WORKLOADS))
    ap.add_argument("--seed", type=int, default=2310)
    ap.add_argument("--cpu-tokens", type=int, default=CPU_SAMPLE_TOKENS)
    ap.add_argument("--soak-s", type=float, default=1.5)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--layer-npz", default="", help=argparse.SUPPRESS)  # internal: the cpu_baseline leg
    ap.add_argument("--ref-out", default="", help=argparse.SUPPRESS)
    ap.add_argument("--tile", default="", help="force the GEMM tile 'cta_group,block_n' (tuning)")
    args = ap.parse_args()
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if args.tile and args.impl == "ours":
        import paper_2310_09259_b200 as q

        cg, bn = (int(v) for v in args.tile.split(","))
        from paper_2310_09259_b200 import _lib

        _lib.check(q.load_library().quik_set_gemm_tile(cg, bn))
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    w = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference(args, w)
    else:
        run_ours(args, w)


if __name__ == "__main__":
    main()
