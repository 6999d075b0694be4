"""The fused all-gather across PROCESSES through CUDA IPC (sharded.FusedShardedQuikLinear):
two ranks (gloo for the handle exchange, both on cuda:0 — CUDA IPC works between
processes on one device, which is what this box has) each own half of the output rows;
each rank's GEMM epilogue stores its shard into both ranks' outputs. Both outputs must
equal the unsharded forward bit for bit."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_09259_b200 as q
        from paper_2310_09259_b200.sharded import FusedShardedQuikLinear
        from oracle_lib import make_layer

        res = []
        for (M, K, N, bits, O) in [(300, 1024, 768, 4, 32), (16, 2048, 1024, 4, 64), (200, 1024, 512, 8, 16)]:
            rng = np.random.default_rng(1234 + M)
            L, x, _ = make_layer(rng, M, K, N, bits, O, heavy_cols=2)
            kb = K - O
            layer = q.QuikLinearLayer(
                q.QuantizedWeights(q.PackedIntMatrix(N, kb, bits, L["base"]), L["scales"], L["outlier_weights"],
                                   L["wreduced"]), q.OutlierSet.from_indices(K, L["idx"]), L["bias"], bits)
            xt = torch.from_numpy(x).cuda().half()
            want = q.QuikLinear(layer)(xt)
            fused = FusedShardedQuikLinear(layer, max_tokens=M, barrier=False)
            for step in range(3):  # round-robin buffers
                y = fused(xt)
                torch.cuda.synchronize()
                dist.barrier()  # every rank's peer stores are complete (stands in for the NCCL fence)
                res.append(bool(torch.equal(y.view(torch.int16), want.view(torch.int16))))
                dist.barrier()
            fused.out.close()
        out_q.put((rank, res))
    except Exception as e:  # reported to the parent
        out_q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_fused_all_gather_cuda_ipc_two_processes():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    qout = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qout)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(qout.get(timeout=280) for _ in procs)
    for p in procs:
        p.join(30)
    assert res == {0: [True] * 9, 1: [True] * 9}, res


@pytest.mark.timeout(300)
def test_fused_all_gather_cpp_two_processes():
    """The same exchange from C++ (quik::b200::FusedShardedLayer, tests/cpp/ipc_test.cpp):
    two forked processes, IPC handles and barriers over pipes, every step of both ranks
    bit-identical to the unsharded layer."""
    import subprocess
    from pathlib import Path

    from paper_2310_09259_b200 import build

    exe = build.build_ipc_test()
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=280, cwd=Path(exe).parent)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
