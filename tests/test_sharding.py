"""Multi-process CPU tests (gloo, world_size 2) of the N-sharded layer's host logic:
shard bounds, per-rank weight slicing, all-gather and reassembly. The per-shard
compute is the CPU oracle here (the device path is covered by the GPU tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_09259_b200.sharded import ShardedQuikLinear, assemble, max_shard, shard_bounds


def test_shard_bounds_cover_and_balance():
    for n in (1, 7, 11008, 28672, 1376 * 8 + 3):
        for w in (1, 2, 3, 4, 8):
            if n < w:
                continue
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(w - 1))
            sizes = [e - b for b, e in spans]
            assert max(sizes) - min(sizes) <= 1 and max(sizes) == max_shard(n, w)


def test_assemble_numpy():
    n, w, M = 11, 3, 4
    full = np.arange(M * n).reshape(M, n)
    g = np.zeros((w, M, max_shard(n, w)), full.dtype)
    for r in range(w):
        b, e = shard_bounds(n, w, r)
        g[r, :, : e - b] = full[:, b:e]
    assert np.array_equal(assemble(g, n, w), full)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice_layer(L, b, e):
    from oracle_lib import row_bytes

    kb = L["in_features"] - len(L["idx"])
    rb = row_bytes(kb, L["bits"])
    S = dict(L)
    S["out_features"] = e - b
    S["base"] = np.asarray(L["base"]).reshape(L["out_features"], rb)[b:e].reshape(-1)
    for k in ("scales", "wreduced", "bias"):
        S[k] = None if L[k] is None else np.asarray(L[k])[b:e]
    S["outlier_weights"] = np.asarray(L["outlier_weights"])[b:e]
    return S


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2310_09259_b200 as q
        from oracle_lib import make_layer, oracle

        rng = np.random.default_rng(99)
        L, x, _ = make_layer(rng, 6, 96, 37, 4, 8, heavy_cols=2)
        layer = q.QuikLinearLayer(
            q.QuantizedWeights(q.PackedIntMatrix(37, 88, 4, L["base"]), L["scales"], L["outlier_weights"],
                               L["wreduced"]), q.OutlierSet.from_indices(96, L["idx"]), L["bias"], 4)

        def compute(xt):
            b, e = shard_bounds(37, world, rank)
            st, y = oracle().quik_matmul(_slice_layer(L, b, e), xt.numpy(), 2)
            assert st == 0
            return torch.from_numpy(y)

        sh = ShardedQuikLinear(layer, compute=compute)
        y = sh(torch.from_numpy(x))
        st, want = oracle().quik_matmul(L, x, 2)
        out_q.put((rank, bool(np.array_equal(y.numpy().view(np.uint32), want.view(np.uint32)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_sharded_forward_gloo_world2_matches_unsharded():
    ctx = mp.get_context("spawn")
    qout = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, qout)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(qout.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(30)
    assert res == {0: True, 1: True}


def _ipc_worker(rank, world, port, out_q):
    """Handle exchange of the fused all-gather (sharded.FusedAllGatherOutput) with
    stand-in handles: every rank serialises one handle per output buffer, gathers all of
    them, 'opens' the others' and builds its destination list [own, others in rank order]."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2310_09259_b200.sharded import gather_handles, peer_destinations

        mine = [bytes([rank, b]) * 36 for b in range(2)]  # 72-byte stand-ins (64 handle + 8 offset)
        allh = gather_handles(mine)
        ok = len(allh) == world and all(allh[r][b] == bytes([r, b]) * 36 for r in range(world) for b in range(2))
        opened_of = lambda raw: 1000 * raw[0] + raw[1]  # noqa: E731  "open" -> a fake device pointer
        dests = [peer_destinations(rank, world, opened_of(mine[b]),
                                   {r: opened_of(allh[r][b]) for r in range(world) if r != rank}) for b in range(2)]
        want = [[1000 * rank + b] + [1000 * r + b for r in range(world) if r != rank] for b in range(2)]
        out_q.put((rank, ok and dests == want))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_fused_all_gather_handle_exchange_gloo_world3():
    ctx = mp.get_context("spawn")
    qout = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 3, port, qout)) for r in range(3)]
    for p in procs:
        p.start()
    res = dict(qout.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(30)
    assert res == {0: True, 1: True, 2: True}


def test_peer_destinations_rejects_missing_ranks():
    from paper_2310_09259_b200.sharded import peer_destinations

    assert peer_destinations(1, 3, "own", {0: "a", 2: "c"}) == ["own", "a", "c"]
    with pytest.raises(ValueError):
        peer_destinations(1, 3, "own", {0: "a"})
