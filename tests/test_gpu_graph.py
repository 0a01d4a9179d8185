"""Graph mode of the decode step (hgca_decode_desc.state, engine.DecodeGraph).

One captured CUDA graph (decode + merge per layer, chained by programmatic
dependent launch) replays step after step while the merge kernel advances the
device step state; the host mirrors the positions and runs evictions eagerly
between replays. The replayed steps must be BIT-identical to the eager
decode_device steps of a second engine fed the same inputs: same kernels,
same data, only where the window range comes from differs. Covered across
evictions (ingest + union rebuild between replays), for both storage dtypes,
GQA, two layers, and a switch back and forth between eager and graph steps.
"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _pair(cuda, dtype, layers=1, B=2, Hq=8, Hkv=2, D=128, bn=4, bs=32, arch=200, T=1024, seed=3):
    cfg = cuda.EngineConfig(layers=layers, heads=Hq, kv_heads=Hkv, head_dim=D, batch=B, dtype=dtype,
                            cache=cuda.CacheConfig(blk_num=bn, blk_size=bs, alpha=0.5, beta=1.0),
                            core_count=10 ** 6, max_positions=T)
    engs = [cuda.HybridEngine(cfg), cuda.HybridEngine(cfg)]
    g = torch.Generator(device="cuda").manual_seed(seed)
    tdt = engs[0].tdtype
    for li in range(layers):
        k = torch.randn((B, Hkv, arch, D), generator=g, device="cuda").to(tdt)
        v = torch.randn((B, Hkv, arch, D), generator=g, device="cuda").to(tdt)
        u = torch.rand((B, Hq, arch), generator=g, device="cuda", dtype=torch.float64)
        maw = torch.where(u < 0.2, (1.0 / (bn * bs)) * (1.0 + u), 1e-6 * u)
        for e in engs:
            e.bulk_ingest(li, k, v, maw, bn * bs)
    return engs, g


def _inputs(eng, g, n):
    tdt = eng.tdtype
    q = torch.randn((n, eng.B, eng.Hq, 1, eng.D), generator=g, device="cuda").to(tdt)
    k = torch.randn((n, eng.B, eng.Hkv, 1, eng.D), generator=g, device="cuda").to(tdt)
    v = torch.randn((n, eng.B, eng.Hkv, 1, eng.D), generator=g, device="cuda").to(tdt)
    return q, k, v


@pytest.mark.parametrize("dtype,Hq,Hkv", [("float32", 8, 8), ("float32", 8, 2), ("bfloat16", 32, 8),
                                          ("bfloat16", 8, 8)])
def test_graph_steps_bit_equal_eager(cuda, dtype, Hq, Hkv):
    (ea, eb), g = _pair(cuda, dtype, Hq=Hq, Hkv=Hkv)
    steps = 300  # ~9 evictions of a 4 x 32 window
    q, k, v = _inputs(ea, g, steps)
    gr = cuda.DecodeGraph(eb, layers=[0])
    for t in range(steps):
        oa, la, _ = ea.decode_device(0, q[t], k[t], v[t])
        gr.q[0, 0].copy_(q[t])
        gr.k[0, 0].copy_(k[t])
        gr.v[0, 0].copy_(v[t])
        ob, lb = gr.step()
        torch.cuda.synchronize()
        assert torch.equal(oa, ob[0, 0]), f"step {t}: graph output differs from eager"
        assert torch.equal(la, lb[0, 0]), f"step {t}: graph lse differs from eager"
    la_, lb_ = ea.layers[0], eb.layers[0]
    assert (la_.lo, la_.nxt) == (lb_.lo, lb_.nxt) and la_.lo > 200
    assert torch.equal(la_.maw, lb_.maw), "MAW (EMA'd in the merge kernel) differs"
    assert torch.equal(la_.ctx, lb_.ctx), "context sets differ"
    assert torch.equal(la_.KV, lb_.KV), "kv_in rows written by the graph's decode kernel differ"


def test_graph_two_layers_and_mode_switches(cuda):
    (ea, eb), g = _pair(cuda, "bfloat16", layers=2, B=1, Hq=16, Hkv=4)
    steps = 120
    q, k, v = _inputs(ea, g, steps)
    gr = cuda.DecodeGraph(eb)
    for t in range(steps):
        ref = [ea.decode_device(li, q[t], k[t], v[t])[:2] for li in range(2)]
        if t % 40 < 30:  # graph steps (both layers in one replay)
            for li in range(2):
                gr.q[0, li].copy_(q[t])
                gr.k[0, li].copy_(k[t])
                gr.v[0, li].copy_(v[t])
            ob, lb = gr.step()
            got = [(ob[0, li], lb[0, li]) for li in range(2)]
        else:  # eager steps on the graph's engine: the device state must re-sync afterwards
            got = [eb.decode_device(li, q[t], k[t], v[t])[:2] for li in range(2)]
        torch.cuda.synchronize()
        for li in range(2):
            assert torch.equal(ref[li][0], got[li][0]) and torch.equal(ref[li][1], got[li][1]), \
                f"step {t} layer {li} differs"
    for li in range(2):
        assert torch.equal(ea.layers[li].maw, eb.layers[li].maw)
        assert (ea.layers[li].lo, ea.layers[li].nxt) == (eb.layers[li].lo, eb.layers[li].nxt)


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_multi_step_graph_bit_equal_eager(cuda, dtype):
    """A graph of 8 consecutive steps x 2 layers (16 decode + 16 merge kernels
    chained by PDL, the state advanced on device between them), replayed up to
    each eviction; eager steps fill the gaps the graph cannot cover."""
    (ea, eb), g = _pair(cuda, dtype, layers=2, B=2, Hq=8, Hkv=2)
    n, steps = 8, 260
    q, k, v = _inputs(ea, g, steps)
    gr = cuda.DecodeGraph(eb, steps=n)
    t = 0
    replays = 0
    while t < steps:
        if gr.room() >= n and t + n <= steps:
            for j in range(n):
                for li in range(2):
                    gr.q[j, li].copy_(q[t + j])
                    gr.k[j, li].copy_(k[t + j])
                    gr.v[j, li].copy_(v[t + j])
            ob, lb = gr.step()
            replays += 1
            got = [[(ob[j, li].clone(), lb[j, li].clone()) for li in range(2)] for j in range(n)]
        else:
            got = [[eb.decode_device(li, q[t], k[t], v[t])[:2] for li in range(2)]]
        for j, row in enumerate(got):
            for li in range(2):
                oa, la, _ = ea.decode_device(li, q[t + j], k[t + j], v[t + j])
                torch.cuda.synchronize()
                assert torch.equal(oa, row[li][0]) and torch.equal(la, row[li][1]), f"token {t + j} layer {li}"
        t += len(got)
    assert replays >= 20
    for li in range(2):
        assert torch.equal(ea.layers[li].maw, eb.layers[li].maw)
        assert torch.equal(ea.layers[li].KV, eb.layers[li].KV)
        assert (ea.layers[li].lo, ea.layers[li].nxt) == (eb.layers[li].lo, eb.layers[li].nxt)


def test_graph_refuses_eager_only_features(cuda):
    cfg = cuda.EngineConfig(layers=1, heads=4, head_dim=64, keep_weights=True,
                            cache=cuda.CacheConfig(blk_num=2, blk_size=32), core_count=10 ** 6, max_positions=256)
    with pytest.raises(cuda.ContractError):
        cuda.DecodeGraph(cuda.HybridEngine(cfg))


@pytest.mark.parametrize("dtype,Hq,Hkv", [("float32", 8, 2), ("bfloat16", 32, 8)])
def test_split_merge_matches_single_cta_merge(cuda, dtype, Hq, Hkv):
    """Split merge (hgca_decode_desc.merge_split: several CTAs per query head
    fold shares of the item list, the last one combines them in share order)
    against the one-CTA-per-head merge on the same inputs: outputs and lse to
    the rounding of the re-associated fold (fp64 on the fp32 path, fp32 fold
    weights on the bf16 path), the window MAW and the context sets (dense
    stats stay in one share) identical. Shares of 4 items force
    the split on this small shape."""
    (ea, eb), g = _pair(cuda, dtype, Hq=Hq, Hkv=Hkv, arch=600, T=2048)
    ea.merge_items, eb.merge_items = 10 ** 9, 4
    steps = 160
    q, k, v = _inputs(ea, g, steps)
    splits = set()
    for t in range(steps):
        oa, la, _ = ea.decode_device(0, q[t], k[t], v[t])
        ob, lb, _ = eb.decode_device(0, q[t], k[t], v[t])
        torch.cuda.synchronize()
        splits.add(eb.layers[0].merge_split)
        # fp32 path: fp64 folds (re-association only); bf16 path: fp32 fold weights
        o_tol, l_tol = (1e-5, 1e-12) if dtype == "float32" else (1e-4, 1e-6)
        assert torch.allclose(oa, ob, rtol=o_tol, atol=o_tol), f"step {t}: split-merge output differs"
        assert torch.allclose(la, lb, rtol=l_tol, atol=l_tol), f"step {t}: split-merge lse differs"
    assert max(splits) > 1, "the split merge never engaged"
    la_, lb_ = ea.layers[0], eb.layers[0]
    assert torch.equal(la_.ctx, lb_.ctx), "context sets differ"
    assert torch.allclose(la_.maw, lb_.maw, rtol=1e-15, atol=0), "MAW differs"


def test_split_merge_keep_weights_window_weights_equal(cuda):
    """keep_weights with the split merge: the dense share writes the window
    weights (a_gpu) and the MAW exactly as the one-CTA merge does."""
    cfg = cuda.EngineConfig(layers=1, heads=8, kv_heads=2, head_dim=128, batch=2, dtype="float32",
                            cache=cuda.CacheConfig(blk_num=4, blk_size=32, alpha=0.5, beta=1.0),
                            core_count=10 ** 6, max_positions=2048, keep_weights=True)
    ea, eb = cuda.HybridEngine(cfg), cuda.HybridEngine(cfg)
    ea.merge_items, eb.merge_items = 10 ** 9, 4
    g = torch.Generator(device="cuda").manual_seed(9)
    arch = 600
    k = torch.randn((2, 2, arch, 128), generator=g, device="cuda")
    v = torch.randn((2, 2, arch, 128), generator=g, device="cuda")
    u = torch.rand((2, 8, arch), generator=g, device="cuda", dtype=torch.float64)
    maw = torch.where(u < 0.2, (1.0 / 128) * (1.0 + u), 1e-6 * u)
    for e in (ea, eb):
        e.bulk_ingest(0, k, v, maw, 128)
    splits = set()
    for t in range(100):
        q = torch.randn((2, 8, 1, 128), generator=g, device="cuda")
        kk = torch.randn((2, 2, 1, 128), generator=g, device="cuda")
        oa, la, wa = ea.decode_device(0, q, kk, -kk)
        ob, lb, wb = eb.decode_device(0, q, kk, -kk)
        torch.cuda.synchronize()
        splits.add(eb.layers[0].merge_split)
        assert torch.equal(wa, wb), f"step {t}: window weights differ"
        assert torch.allclose(oa, ob, rtol=1e-5, atol=1e-6) and torch.allclose(la, lb, rtol=1e-12, atol=1e-12)
    assert max(splits) > 1
    assert torch.equal(ea.layers[0].maw, eb.layers[0].maw)
