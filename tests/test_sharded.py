"""Sequence sharding of the decode step.

CPU (no GPU): the block-cyclic ownership masks partition every position
exactly once, and a world_size-2 / 3 gloo run of the sharded decomposition --
per-rank threshold selection over owned blocks, rank-0 dense merge, ONE
all_gather of the packed (out, lse) partials, rank-order P-way merge -- equals
the unsharded reference engine (oracle port) on the same inputs: outputs
within 1e-5 relative, shard contexts disjoint and their union equal to the
unsharded context bit for bit.

GPU: world 1/2/4 shards of ShardedHybridEngine simulated in one process on
cuda:0 (decode_partial -> concatenated partials -> merge, the exact buffers
the NCCL all_gather moves) against the single-GPU HybridEngine and the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import port
from paper_2507_03153_b200.sharded import packed_stride, shard_owner
from paper_2507_03153_b200.sparsifier import ownership_words


def test_ownership_partitions_positions():
    for blk in (1, 8, 32):
        for world in (1, 2, 3, 8):
            words = 40
            masks = [ownership_words(words, blk, r, world) for r in range(world)]
            acc = np.zeros(words, np.uint64)
            for m in masks:
                assert not (acc & m).any(), "two ranks own one position"
                acc |= m
            assert (acc == 0xFFFFFFFF).all()
            pos = np.arange(words * 32)
            for r, m in enumerate(masks):
                bits = (m[pos // 32] >> (pos % 32).astype(np.uint32)) & 1
                want = np.array([shard_owner(p // blk, world) == r for p in pos])
                assert (bits.astype(bool) == want).all()


def test_layer_state_keep_bits_on_cpu():
    import paper_2507_03153_b200 as hg

    cfg = hg.EngineConfig(layers=1, heads=4, head_dim=64, cache=hg.CacheConfig(blk_num=4, blk_size=16),
                          core_count=64, shard_rank=1, shard_world=2)
    ls = hg.LayerState(cfg, 256, torch.device("cpu"))
    got = ls.keep.numpy().view(np.uint32)
    assert (got == ownership_words(8, 16, 1, 2)).all()
    # block-cyclic 16-position blocks over 32-bit words: rank 1 owns the high half
    assert got[0] == 0xFFFF0000


def test_sharded_config_contract():
    import paper_2507_03153_b200 as hg

    with pytest.raises(hg.ContractError):
        hg.EngineConfig(shard_rank=2, shard_world=2)
    with pytest.raises(hg.ContractError):
        hg.EngineConfig(heads=8, core_count=1, shard_world=2)  # padding groups
    with pytest.raises(hg.ContractError):
        hg.EngineConfig(selection="topk", topk=4, core_count=64, shard_world=2)


def _inputs(steps, H, d, seed):
    rng = np.random.default_rng(seed)
    return [(rng.standard_normal((H, 1, d)).astype(np.float32),
             rng.standard_normal((H, 1, d)).astype(np.float32),
             rng.standard_normal((H, 1, d)).astype(np.float32)) for _ in range(steps)]


GEOM = dict(heads=4, head_dim=32, blk_num=4, blk_size=8, beta=1.0, core_count=64, max_len=640)
STEPS = 400


def _make_oracle(shard):
    g = GEOM
    return port.OracleEngine(g["heads"], g["head_dim"], g["blk_num"], g["blk_size"], beta=g["beta"],
                             core_count=g["core_count"], max_len=g["max_len"], shard=shard)


def _gloo_worker(rank, world, port_no, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        eng = _make_oracle((rank, world))
        H, d = GEOM["heads"], GEOM["head_dim"]
        rows = H
        outs, lses = [], []
        for qq, kk, vv in _inputs(STEPS, H, d, 5):
            r = eng.step("decode", qq, kk, vv)
            mine_out = r.output if rank == 0 else r.s_out
            mine_lse = r.lse if rank == 0 else r.s_lse
            # one packed buffer per rank, exactly as the device path sends it
            send = np.zeros(packed_stride(rows, d), np.uint8)
            send[: rows * d * 4] = np.ascontiguousarray(mine_out[:, 0], np.float32).view(np.uint8).ravel()
            send[rows * d * 4:] = np.ascontiguousarray(mine_lse[:, 0], np.float64).view(np.uint8)
            parts = [torch.empty(send.size, dtype=torch.uint8) for _ in range(world)]
            dist.all_gather(parts, torch.from_numpy(send))
            po = np.stack([p.numpy()[: rows * d * 4].view(np.float32).reshape(rows, d) for p in parts])
            pl = np.stack([p.numpy()[rows * d * 4:].view(np.float64) for p in parts])
            o, l = port.merge_packed(po, pl)
            outs.append(o)
            lses.append(l)
        q.put((rank, np.stack(outs), np.stack(lses), [c.copy() for c in eng.context], eng.lo))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_decode_equals_unsharded(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port_no, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r[1:]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = _make_oracle((0, 1))
    H, d = GEOM["heads"], GEOM["head_dim"]
    ref_o, ref_l = [], []
    for qq, kk, vv in _inputs(STEPS, H, d, 5):
        r = full.step("decode", qq, kk, vv)
        ref_o.append(r.output[:, 0])
        ref_l.append(r.lse[:, 0])
    ref_o, ref_l = np.stack(ref_o), np.stack(ref_l)
    assert full.lo > 10 * GEOM["blk_size"], "the archive must span several shards' blocks"
    for rank in range(world):
        o, l, ctxs, lo = res[rank]
        assert lo == full.lo
        err = np.abs(o - ref_o).max() / np.abs(ref_o).max()
        assert err <= 1e-5, f"rank {rank}: sharded output rel err {err:.3e}"
        np.testing.assert_allclose(l, ref_l, rtol=1e-12, atol=1e-12)
    # selection: disjoint shards whose union is the unsharded context, bit for bit
    for h in range(H):
        parts = [res[r][2][h] for r in range(world)]
        allp = np.concatenate(parts)
        assert len(np.unique(allp)) == len(allp)
        np.testing.assert_array_equal(np.sort(allp), full.context[h])
        for r, p in enumerate(parts):
            assert all(shard_owner(int(x) // GEOM["blk_size"], world) == r for x in p)


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
@pytest.mark.parametrize("world,dtype", [(1, "float32"), (2, "float32"), (4, "float32"), (4, "bfloat16")])
def test_gpu_sharded_shards_match_single_engine(cuda, world, dtype):
    hg = cuda
    H, Hkv, d, B = 8, 2, 128, 2
    cfg = hg.EngineConfig(layers=1, heads=H, kv_heads=Hkv, head_dim=d, batch=B, dtype=dtype,
                          cache=hg.CacheConfig(blk_num=4, blk_size=32, beta=1.0),
                          core_count=64, max_positions=1024)
    single = hg.HybridEngine(cfg)
    shards = [hg.ShardedHybridEngine(cfg, rank=r, world=world) for r in range(world)]
    oracles = [port.OracleEngine(H, d, 4, 32, core_count=64, batch=B, max_len=1024) for _ in range(B)]
    rng = np.random.default_rng(11)
    out = torch.empty((B * H, d), dtype=torch.float32, device="cuda")
    lse = torch.empty(B * H, dtype=torch.float64, device="cuda")
    worst_single = worst_oracle = 0.0
    tol = 1e-4 if dtype == "float32" else 1e-2
    for t in range(700):
        q = rng.standard_normal((B, H, 1, d)).astype(np.float32)
        k = rng.standard_normal((B, Hkv, 1, d)).astype(np.float32)
        v = rng.standard_normal((B, Hkv, 1, d)).astype(np.float32)
        if dtype == "bfloat16":
            q, k, v = port.bf16_round(q), port.bf16_round(k), port.bf16_round(v)
        tq, tk, tv = (torch.from_numpy(x).cuda().to(single.tdtype) for x in (q, k, v))
        so, sl, _ = single.decode_device(0, tq, tk, tv)
        for e in shards:
            e.decode_partial(0, tq, tk, tv)
        parts = torch.cat([e.send for e in shards])
        shards[0].merge(parts, out, lse)
        got = out.cpu().numpy()
        ref = so.cpu().numpy()
        worst_single = max(worst_single, float(np.abs(got - ref).max() / np.abs(ref).max()))
        for b in range(B):
            o = oracles[b].step("decode", q[b], port.expand_gqa(k[b], H), port.expand_gqa(v[b], H))
            worst_oracle = max(worst_oracle, float(np.abs(got.reshape(B, H, d)[b] - o.output[:, 0]).max()
                                                   / np.abs(o.output).max()))
    torch.cuda.synchronize()
    assert single.layers[0].archive_size > 400
    assert worst_single <= tol, f"sharded vs single-GPU rel err {worst_single:.3e}"
    assert worst_oracle <= tol, f"sharded vs reference oracle rel err {worst_oracle:.3e}"
    # every archived row is selected on exactly the rank that owns its block
    ctx_single = single.context_indices()
    ctx_sh = [e.context_indices() for e in shards]
    for row in range(B * H):
        allp = np.concatenate([c[row] for c in ctx_sh])
        assert len(np.unique(allp)) == len(allp)
        np.testing.assert_array_equal(np.sort(allp), ctx_single[row])


@pytest.mark.gpu
@pytest.mark.parametrize("world,dtype,split", [(2, "bfloat16", False), (3, "float32", False), (2, "bfloat16", True)])
def test_gpu_push_exchange_matches_allgather(cuda, world, dtype, split):
    """exchange="push" with `world` ranks in one process (one stream each, the
    peers' boxes as plain device pointers): the merge kernels push their packed
    partials into every box and the flag-waiting merge folds them -- bit-equal
    to the all-gather exchange of the same partials, on every rank. split: the
    split merge (several CTAs per head, the combining one pushes) on both."""
    hg = cuda
    H, Hkv, d, B = 8, 2, 128, 2
    cfg = hg.EngineConfig(layers=1, heads=H, kv_heads=Hkv, head_dim=d, batch=B, dtype=dtype,
                          cache=hg.CacheConfig(blk_num=4, blk_size=32, beta=1.0),
                          core_count=64, max_positions=1024)
    push = [hg.ShardedHybridEngine(cfg, rank=r, world=world, exchange="push") for r in range(world)]
    bases = [e.xchg.base for e in push]
    for e in push:
        e.xchg.connect_local(bases)
    ref = [hg.ShardedHybridEngine(cfg, rank=r, world=world) for r in range(world)]
    if split:
        for e in push + ref:
            e.merge_items = 4
    streams = [torch.cuda.Stream() for _ in range(world)]
    outs = [(torch.empty((B * H, d), dtype=torch.float32, device="cuda"),
             torch.empty(B * H, dtype=torch.float64, device="cuda")) for _ in range(world)]
    rout = torch.empty((B * H, d), dtype=torch.float32, device="cuda")
    rlse = torch.empty(B * H, dtype=torch.float64, device="cuda")
    g = torch.Generator(device="cuda").manual_seed(3)
    tdt = push[0].tdtype
    for t in range(300):
        qq = torch.randn((B, H, 1, d), generator=g, device="cuda").to(tdt)
        kk = torch.randn((B, Hkv, 1, d), generator=g, device="cuda").to(tdt)
        vv = torch.randn((B, Hkv, 1, d), generator=g, device="cuda").to(tdt)
        main = torch.cuda.current_stream()
        for r, e in enumerate(push):  # every rank's partial (and push) first ...
            streams[r].wait_stream(main)
            with torch.cuda.stream(streams[r]):
                e.push_partial(0, qq, kk, vv)
        for r, e in enumerate(push):  # ... then the flag-waiting merges
            with torch.cuda.stream(streams[r]):
                e.push_merge(outs[r][0], outs[r][1])
        for s_ in streams:
            main.wait_stream(s_)
        for e in ref:
            e.decode_partial(0, qq, kk, vv)
        ref[0].merge(torch.cat([e.send for e in ref]), rout, rlse)
        for r in range(world):
            assert torch.equal(outs[r][0], rout) and torch.equal(outs[r][1], rlse), (t, r)
    torch.cuda.synchronize()
    for e in push:
        e.check_exchange()
        assert e.collectives == 300
    assert push[0].layers[0].archive_size > 100
    if split:
        assert push[0].layers[0].merge_split > 1, "the split merge never engaged"
    for e in push:
        e.close()


def _gpu_worker(rank, world, port_no, q, exchange="allgather", steps=400, own_device=False):
    import torch.distributed as dist

    import paper_2507_03153_b200 as hg

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    if own_device:  # one physical GPU per rank: NCCL over NVLink, CUDA IPC between devices
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if not own_device:
            torch.cuda.set_device(0)
        cfg = hg.EngineConfig(layers=1, heads=8, kv_heads=2, head_dim=128, batch=2, dtype="bfloat16",
                              cache=hg.CacheConfig(blk_num=4, blk_size=32, beta=1.0), core_count=64,
                              max_positions=1024)
        # rank / world from the process group (push: IPC handles exchanged through it)
        eng = hg.ShardedHybridEngine(cfg, exchange=exchange, push_timeout_ms=20000)
        g = torch.Generator(device="cuda").manual_seed(5)
        outs = []
        for _ in range(steps):
            qq = torch.randn((2, 8, 1, 128), generator=g, device="cuda").to(torch.bfloat16)
            kk = torch.randn((2, 2, 1, 128), generator=g, device="cuda").to(torch.bfloat16)
            o, l, _ = eng.decode_device(0, qq, kk, -kk)
            outs.append(o.cpu().numpy().copy())
        eng.check_exchange()
        torch.cuda.synchronize()
        dist.barrier()
        eng.close()
        q.put((rank, np.stack(outs), eng.collectives, eng.layers[0].archive_size))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("exchange,steps", [("allgather", 400), ("push", 200)])
def test_gpu_sharded_engine_two_processes(cuda, exchange, steps):
    """ShardedHybridEngine.decode_device end to end in two processes (gloo
    process group, both on cuda:0): every rank returns the same output, equal
    to the single-GPU engine's within bf16 tolerance. exchange="push": the
    receive boxes are mapped across the processes with CUDA IPC and the merge
    kernels push into them (the two contexts time-slice one GPU here, so the
    flag waits are slow but bounded)."""
    import torch.multiprocessing as mp

    hg = cuda
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port_no, q, exchange, steps)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = hg.EngineConfig(layers=1, heads=8, kv_heads=2, head_dim=128, batch=2, dtype="bfloat16",
                          cache=hg.CacheConfig(blk_num=4, blk_size=32, beta=1.0), core_count=64, max_positions=1024)
    single = hg.HybridEngine(cfg)
    g = torch.Generator(device="cuda").manual_seed(5)
    ref = []
    for _ in range(steps):
        qq = torch.randn((2, 8, 1, 128), generator=g, device="cuda").to(torch.bfloat16)
        kk = torch.randn((2, 2, 1, 128), generator=g, device="cuda").to(torch.bfloat16)
        o, _, _ = single.decode_device(0, qq, kk, -kk)
        ref.append(o.cpu().numpy().copy())
    ref = np.stack(ref)
    assert res[0][1] == steps and res[0][2] == single.layers[0].archive_size > 0
    np.testing.assert_array_equal(res[0][0], res[1][0])
    err = np.abs(res[0][0] - ref).max() / np.abs(ref).max()
    assert err <= 1e-2, err


@pytest.mark.gpu
@pytest.mark.skipif(not (torch.cuda.is_available() and torch.cuda.device_count() >= 2),
                    reason="needs two physical GPUs")
@pytest.mark.parametrize("exchange", ["allgather", "push"])
def test_multi_gpu_sharded_engine(cuda, exchange):
    """Two ranks on two physical GPUs (NCCL process group): the NCCL all-gather
    and the one-shot push over NVLink (receive boxes mapped across devices with
    CUDA IPC) both return, on every rank, the single-GPU engine's output within
    bf16 tolerance -- identical on both ranks."""
    import torch.multiprocessing as mp

    hg = cuda
    steps = 300
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port_no, q, exchange, steps, True)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=600) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = hg.EngineConfig(layers=1, heads=8, kv_heads=2, head_dim=128, batch=2, dtype="bfloat16",
                          cache=hg.CacheConfig(blk_num=4, blk_size=32, beta=1.0), core_count=64, max_positions=1024)
    single = hg.HybridEngine(cfg)
    g = torch.Generator(device="cuda").manual_seed(5)
    ref = []
    for _ in range(steps):
        qq = torch.randn((2, 8, 1, 128), generator=g, device="cuda").to(torch.bfloat16)
        kk = torch.randn((2, 2, 1, 128), generator=g, device="cuda").to(torch.bfloat16)
        o, _, _ = single.decode_device(0, qq, kk, -kk)
        ref.append(o.cpu().numpy().copy())
    ref = np.stack(ref)
    np.testing.assert_array_equal(res[0][0], res[1][0])
    assert np.abs(res[0][0] - ref).max() / np.abs(ref).max() <= 1e-2
