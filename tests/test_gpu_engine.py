"""GPU parity of the device-resident decode engine against the reference.

* golden runs of the reference HybridEngine (tests/golden/engine.npz):
  outputs within 1e-4 relative (fp32 path), MAW and context index sets
  bit-exact;
* the oracle port (oracle/port.py, itself pinned bitwise to the reference by
  tests/test_oracle.py) for batch / GQA / bf16 extensions via the SURVEY.md
  F8 adapters (bf16 tolerance 1e-2);
* size-independent properties at BASELINE sizes (determinism, merge identity
  with an empty store, conservation of window + archive).
"""

import math

import numpy as np
import pytest
import torch

from oracle import port
from oracle import workload as owl
from test_oracle import ENGINE_CASES

from conftest import host  # noqa: E402

pytestmark = pytest.mark.gpu

REL_FP32 = 1e-4   # north star: outputs within 1e-4 relative on the fp32 path
REL_BF16 = 1e-2   # ... and 1e-2 on the bf16 path


def rel_err(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def make_engine(cuda, H, d, bn, bs, alpha, beta, cores, total, **kw):
    cfg = cuda.EngineConfig(layers=1, heads=H, head_dim=d,
                            cache=cuda.CacheConfig(blk_num=bn, blk_size=bs, alpha=alpha, beta=beta),
                            core_count=cores, max_positions=total, **kw)
    return cuda.HybridEngine(cfg)


@pytest.mark.parametrize("name", sorted(ENGINE_CASES))
def test_engine_vs_reference_golden(cuda, name, golden):
    g = golden("engine.npz")
    H, d, bn, bs, alpha, beta, cores, spec_kw = ENGINE_CASES[name]
    steps = owl.gen_workload(owl.WorkloadSpec(**spec_kw), H, d, 1 / math.sqrt(d), 1)
    total = sum(s.n_q for s in steps)
    eng = make_engine(cuda, H, d, bn, bs, alpha, beta, cores, total)
    outs, lses = [], []
    for s in steps:
        r = eng.step(0, cuda.StepInput(s.mode, s.q[0], s.keys[0], s.values[0]))
        outs.append(host(r.output[:, -1, :]))
        lses.append(host(r.lse[:, -1]))
    sel = g[f"{name}_steps"]
    go, gl = g[f"{name}_out"], g[f"{name}_lse"]
    worst = max(rel_err(outs[i], go[j]) for j, i in enumerate(sel))
    assert worst <= REL_FP32, f"max relative output error {worst:.3e}"
    np.testing.assert_allclose(np.stack([lses[i] for i in sel]), gl, rtol=1e-9, atol=1e-9)
    ls = eng.layers[0]
    w_size, n = g[f"{name}_sizes"]
    assert (ls.window_size, ls.archive_size) == (w_size, n)
    maw = eng.maw_host()
    np.testing.assert_array_equal(maw[:, :n], g[f"{name}_store_maw"])
    np.testing.assert_array_equal(maw[:, n:n + w_size], g[f"{name}_window_maw"])
    ctx = np.zeros((H, n), bool)
    for h, idx in enumerate(eng.context_indices()):
        ctx[h, idx] = True
    np.testing.assert_array_equal(ctx, g[f"{name}_ctx"])


def _run_batched(cuda, B, Hq, Hkv, d, dtype, beta, cores, steps_n, seed):
    """Device engine with batch/GQA/dtype vs B oracle engines on adapted inputs."""
    rng = np.random.default_rng(seed)
    bn, bs = 4, 16
    prefill = 24
    total = prefill + steps_n
    cfg = dict(kv_heads=Hkv, batch=B, dtype=dtype)
    eng = make_engine(cuda, Hq, d, bn, bs, 0.5, beta, cores, total, **cfg)
    oracles = [port.OracleEngine(Hq, d, bn, bs, 0.5, beta, core_count=cores, batch=B, max_len=total)
               for _ in range(B)]
    rnd = port.bf16_round if dtype == "bfloat16" else (lambda x: x)
    worst = 0.0
    for t in range(-1, steps_n):
        n = prefill if t < 0 else 1
        mode = "append" if t < 0 else "decode"
        q = rnd(rng.standard_normal((B, Hq, n, d)).astype(np.float32))
        k = rnd(rng.standard_normal((B, Hkv, n, d)).astype(np.float32))
        v = rnd(rng.standard_normal((B, Hkv, n, d)).astype(np.float32))
        r = eng.step(0, cuda.StepInput(mode, q, k, v))
        got = host(r.output)
        for b in range(B):
            o = oracles[b].step(mode, q[b], port.expand_gqa(k[b], Hq), port.expand_gqa(v[b], Hq))
            worst = max(worst, rel_err(got[b, :, -1], o.output[:, -1]))
    return eng, oracles, worst


def test_engine_gqa_batch_fp32(cuda):
    eng, oracles, worst = _run_batched(cuda, B=3, Hq=8, Hkv=2, d=128, dtype="float32", beta=1.0,
                                       cores=64, steps_n=150, seed=1)
    assert worst <= REL_FP32, worst
    # selections stay per query head and match the per-sequence reference bitwise
    ctx = eng.context_indices()
    for b, o in enumerate(oracles):
        for h in range(8):
            np.testing.assert_array_equal(ctx[b * 8 + h], o.context[h])


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_engine_soak_vs_oracle(cuda, dtype):
    """3000 decode steps (~185 evictions + re-selections, archive ~3000 entries)
    against the oracle: no drift in positions, windows, unions or MAW; fp32
    selections stay bit-exact to the end."""
    eng, oracles, worst = _run_batched(cuda, B=2, Hq=8, Hkv=2, d=64, dtype=dtype, beta=1.0,
                                       cores=64, steps_n=3000, seed=9)
    assert eng.layers[0].archive_size > 2500
    assert worst <= (REL_BF16 if dtype == "bfloat16" else REL_FP32), worst
    if dtype == "float32":
        ctx = eng.context_indices()
        for b, o in enumerate(oracles):
            for h in range(8):
                np.testing.assert_array_equal(ctx[b * 8 + h], o.context[h])


def test_engine_append_events_soak_bf16(cuda):
    """bf16, G = 4, D = 128: 16-query appends every 150 steps (the tcgen05 append
    passes: MAW re-evaluation and re-selection) interleaved with decode steps,
    every step's output against the oracle."""
    B, Hq, Hkv, d = 2, 8, 2, 128
    rng = np.random.default_rng(12)
    bn, bs, prefill, steps_n, nq = 4, 16, 24, 900, 16
    total = prefill + steps_n + (steps_n // 150) * nq + nq
    eng = make_engine(cuda, Hq, d, bn, bs, 0.5, 1.0, 64, total, kv_heads=Hkv, batch=B, dtype="bfloat16")
    oracles = [port.OracleEngine(Hq, d, bn, bs, 0.5, 1.0, core_count=64, batch=B, max_len=total) for _ in range(B)]
    worst, appends = 0.0, 0
    for t in range(-1, steps_n):
        if t < 0:
            mode, n = "append", prefill
        elif t % 150 == 149:
            mode, n = "append", nq
            appends += 1
        else:
            mode, n = "decode", 1
        q = port.bf16_round(rng.standard_normal((B, Hq, n, d)).astype(np.float32))
        k = port.bf16_round(rng.standard_normal((B, Hkv, n, d)).astype(np.float32))
        v = port.bf16_round(rng.standard_normal((B, Hkv, n, d)).astype(np.float32))
        r = eng.step(0, cuda.StepInput(mode, q, k, v))
        got = host(r.output)
        for b in range(B):
            o = oracles[b].step(mode, q[b], port.expand_gqa(k[b], Hq), port.expand_gqa(v[b], Hq))
            for i in range(n):
                worst = max(worst, rel_err(got[b, :, i], o.output[:, i]))
    assert appends == steps_n // 150 and eng.layers[0].archive_size > 800
    assert worst <= REL_BF16, worst


def test_engine_gqa_batch_bf16(cuda):
    eng, oracles, worst = _run_batched(cuda, B=2, Hq=32, Hkv=8, d=128, dtype="bfloat16", beta=1.0,
                                       cores=64, steps_n=120, seed=2)
    assert worst <= REL_BF16, worst


def test_engine_gqa_padding_groups(cuda):
    # batch*heads/core_count = 2*8/4 -> groups of 4 heads padded to the group max
    eng, oracles, worst = _run_batched(cuda, B=2, Hq=8, Hkv=4, d=64, dtype="float32", beta=1.0,
                                       cores=4, steps_n=130, seed=3)
    assert worst <= REL_FP32, worst
    entries, flags = eng.store_entries()
    for b, o in enumerate(oracles):
        want = o.sparse_entries()
        for h in range(8):
            np.testing.assert_array_equal(entries[b * 8 + h], want[h])


def test_engine_empty_store_equals_dense(cuda, rng):
    """test_engine.py:50-64: with an empty archive the step is dense attention."""
    eng = make_engine(cuda, 4, 64, 4, 16, 0.5, 1.0, 8, 64)
    hk, hv = [], []
    for _ in range(20):
        q, k, v = (rng.standard_normal((4, 1, 64)).astype(np.float32) for _ in range(3))
        hk.append(k)
        hv.append(v)
        r = eng.step(0, cuda.StepInput("decode", q, k, v))
        dense = cuda.attend(q, np.concatenate(hk, 1), np.concatenate(hv, 1), cuda.HeadShape(4, 64))
        np.testing.assert_allclose(host(r.output), dense.output, rtol=0, atol=2e-6)
        np.testing.assert_allclose(host(r.lse), dense.lse, rtol=0, atol=1e-9)
    assert eng.layers[0].archive_size == 0


def test_engine_conservation_and_eviction_arithmetic(cuda, rng):
    """test_engine.py:190-210 replayed on the device engine."""
    eng = make_engine(cuda, 2, 64, 4, 16, 0.5, 1.0, 2, 256)
    size = archived = 0
    for _ in range(200):
        q, k, v = (rng.standard_normal((2, 1, 64)).astype(np.float32) for _ in range(3))
        eng.step(0, cuda.StepInput("decode", q, k, v))
        if size + 1 >= 64:
            evict = -((size + 1 - 64 + 1) // -16) * 16
            size -= evict
            archived += evict
        size += 1
    ls = eng.layers[0]
    assert (ls.window_size, ls.archive_size) == (size, archived)
    assert ls.archive_size % 16 == 0


def _big_engine(cuda, dtype, B=4, Hq=32, Hkv=8, ctx=8192, frac=0.1, seed=0):
    """Stage a long archive with a threshold selecting ~frac per query head."""
    cfg = cuda.EngineConfig(layers=1, heads=Hq, kv_heads=Hkv, head_dim=128, batch=B, dtype=dtype,
                            cache=cuda.CacheConfig(blk_num=16, blk_size=32, beta=1.0),
                            core_count=10 ** 6, max_positions=ctx + 64)
    eng = cuda.HybridEngine(cfg)
    g = torch.Generator(device="cuda").manual_seed(seed)
    tdt = torch.bfloat16 if dtype == "bfloat16" else torch.float32
    n = ctx - 512
    k = torch.randn((B, Hkv, n, 128), generator=g, device="cuda").to(tdt)
    v = torch.randn((B, Hkv, n, 128), generator=g, device="cuda").to(tdt)
    divisor = 512
    thr = 1.0 / divisor
    u = torch.rand((B, Hq, n), generator=g, device="cuda", dtype=torch.float64)
    maw = torch.where(u < frac, thr * (1 + u), thr * u)  # exactly the u < frac entries pass
    eng.bulk_ingest(0, k, v, maw, divisor)
    for _ in range(512):
        q = torch.randn((B, Hq, 1, 128), generator=g, device="cuda").to(tdt)
        kk = torch.randn((B, Hkv, 1, 128), generator=g, device="cuda").to(tdt)
        vv = torch.randn((B, Hkv, 1, 128), generator=g, device="cuda").to(tdt)
        eng.step(0, cuda.StepInput("decode", q, kk, vv))
    return eng, g, tdt


@pytest.mark.parametrize("dtype", ["bfloat16", "float32"])
def test_engine_long_context_vs_oracle(cuda, dtype):
    """A long staged archive: the decode step of batch element 0 vs the oracle
    (sparse over the selected entries + dense window + merge)."""
    B, Hq, Hkv = 2, 32, 8
    eng, g, tdt = _big_engine(cuda, dtype, B=B, ctx=8192)
    ls = eng.layers[0]
    q = torch.randn((B, Hq, 1, 128), generator=g, device="cuda").to(tdt)
    kk = torch.randn((B, Hkv, 1, 128), generator=g, device="cuda").to(tdt)
    vv = torch.randn((B, Hkv, 1, 128), generator=g, device="cuda").to(tdt)
    lo, nxt = ls.lo, ls.nxt
    entries, _ = eng.store_entries()
    K = ls.K.float().cpu().numpy()
    V = ls.V.float().cpu().numpy()
    r = eng.step(0, cuda.StepInput("decode", q, kk, vv))
    got = host(r.output)
    qh = q.float().cpu().numpy()
    kn = kk.float().cpu().numpy()
    vn = vv.float().cpu().numpy()
    G = Hq // Hkv
    for b in range(B):
        for h in range(0, Hq, 5):
            kvh = b * Hkv + h // G
            so, sl, _ = port.attend_indexed(qh[b, h], K[kvh, :lo], V[kvh, :lo], entries[b * Hq + h],
                                            1 / math.sqrt(128), False)
            dk = np.concatenate([K[kvh, lo:nxt], kn[b, h // G]], 0)[None]
            dv = np.concatenate([V[kvh, lo:nxt], vn[b, h // G]], 0)[None]
            do, dl, _ = port.attend_dense(qh[b, h][None], dk, dv, 1 / math.sqrt(128), False)
            o, _ = port.merge_states(so, sl, do[0], dl[0])
            assert rel_err(got[b, h, 0], o[0]) <= (REL_BF16 if dtype == "bfloat16" else REL_FP32)


def test_engine_decode_is_deterministic(cuda):
    outs = []
    for _ in range(2):
        eng, g, tdt = _big_engine(cuda, "bfloat16", B=2, ctx=4096, seed=5)
        q = torch.randn((2, 32, 1, 128), generator=g, device="cuda").to(tdt)
        kk = torch.randn((2, 8, 1, 128), generator=g, device="cuda").to(tdt)
        r = eng.step(0, cuda.StepInput("decode", q, kk, kk))
        outs.append((host(r.output), host(r.lse), eng.maw_host()))
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)


# every (storage dtype, head_dim, GQA group) instantiation of the decode kernels
@pytest.mark.parametrize("dtype", ["bfloat16", "float32"])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("Hq,Hkv", [(4, 4), (8, 4), (8, 2), (8, 1)])
def test_engine_kernel_instantiations(cuda, dtype, d, Hq, Hkv):
    eng, oracles, worst = _run_batched(cuda, B=2, Hq=Hq, Hkv=Hkv, d=d, dtype=dtype, beta=1.0,
                                       cores=64, steps_n=90, seed=d + Hq + Hkv)
    assert eng.layers[0].archive_size > 0
    assert worst <= (REL_BF16 if dtype == "bfloat16" else REL_FP32), worst
    if dtype == "float32":  # reference-exact path: selections bit-exact per query head
        ctx = eng.context_indices()
        for b, o in enumerate(oracles):
            for h in range(Hq):
                np.testing.assert_array_equal(ctx[b * Hq + h], o.context[h])


def test_bf16_rows_rotated_and_union_classes(cuda):
    """bf16 K|V rows are stored position-rotated (hgca_write_rows) and the
    union lists are class-interleaved per 32-entry window: the logical K/V views
    give back exactly what was written, every selected archive row appears once
    in its (batch, kv-head) union with the right query-head mask, each aligned
    window of 32 holds exactly the position-ordered list's entries there, in
    (rank within class p & 7, class) order."""
    B, Hq, Hkv = 2, 8, 2
    eng, g, tdt = _big_engine(cuda, "bfloat16", B=B, Hq=Hq, Hkv=Hkv, ctx=2048, seed=9)
    ls = eng.layers[0]
    kv = ls.rows()
    # rows written by the staged decode steps round-trip through the rotation
    src = torch.randn((B, Hkv, 1, 128), generator=g, device="cuda").to(tdt)
    pos = ls.nxt
    eng.step(0, cuda.StepInput("decode", torch.randn((B, Hq, 1, 128), generator=g, device="cuda").to(tdt),
                               src, -src))
    kv = ls.rows()
    torch.testing.assert_close(kv[:, pos, 0].view(B, Hkv, 128), src[:, :, 0], rtol=0, atol=0)
    torch.testing.assert_close(kv[:, pos, 1].view(B, Hkv, 128), -src[:, :, 0], rtol=0, atol=0)
    G = Hq // Hkv
    sel = eng.store_entries()[0]
    ent = ls.u_ent.cpu().numpy().view(np.uint32)
    cnt = ls.u_cnt.cpu().numpy()
    for bk in range(B * Hkv):
        e = ent[bk, :cnt[bk]]
        p, qm = e & 0xFFFFFF, e >> 24
        b, kvh = divmod(bk, Hkv)
        want = {}
        for gi in range(G):
            for x in sel[b * Hq + kvh * G + gi]:
                want[int(x)] = want.get(int(x), 0) | (1 << gi)
        assert len(p) == len(set(p.tolist())) == len(want)
        assert all(want[int(x)] == int(m) for x, m in zip(p, qm))
        ps = np.sort(p)
        for w0 in range(0, len(p), 32):
            win = p[w0:w0 + 32]
            np.testing.assert_array_equal(np.sort(win), ps[w0:w0 + 32])  # same entries as position order
            cls = win % 8
            rank = np.array([int((ps[w0:w0 + 32] % 8 == c)[: np.searchsorted(ps[w0:w0 + 32], x)].sum())
                             for x, c in zip(win, cls)])
            key = rank * 16 + cls
            assert (np.diff(key) > 0).all()  # (rank, class) order inside the window


def test_decode_host_packed_matches_device_path(cuda):
    """The end-to-end host-buffer entry point (one H2D of q|k|v; out|lse written
    by the merge kernel straight into the pinned, mapped host buffer -- or, for a
    pageable buffer, staged and copied) computes exactly what the device-tensor
    path computes."""
    outs = []
    for packed in (False, "pinned", "pageable"):
        eng, g, tdt = _big_engine(cuda, "bfloat16", B=2, ctx=2048, seed=21)
        B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
        res = []
        for _ in range(40):  # crosses an eviction + re-selection
            q = torch.randn((B, Hq, 1, D), generator=g, device="cuda").to(tdt)
            k = torch.randn((B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
            v = torch.randn((B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
            if packed:
                in_h = torch.cat([q.reshape(-1), k.reshape(-1), v.reshape(-1)]).cpu().pin_memory()
                out_h = torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8)
                if packed == "pinned":
                    out_h = out_h.pin_memory()
                eng.decode_host_packed(0, in_h, out_h)
                o = out_h[: B * Hq * D * 4].view(torch.float32).numpy().copy()
                l = out_h[B * Hq * D * 4:].view(torch.float64).numpy().copy()
            else:
                ot, lt, _ = eng.decode_device(0, q, k, v)
                o, l = ot.cpu().numpy().ravel(), lt.cpu().numpy()
            res.append((o, l))
        outs.append(res)
    for other in outs[1:]:
        for (o1, l1), (o2, l2) in zip(outs[0], other):
            np.testing.assert_array_equal(o1, o2)
            np.testing.assert_array_equal(l1, l2)


@pytest.mark.parametrize("nq,Hq,Hkv,d", [(16, 8, 2, 128), (5, 8, 4, 128), (1, 4, 4, 64), (40, 8, 2, 64),
                                         (8, 8, 2, 128), (1, 8, 2, 128), (3, 8, 2, 128), (12, 8, 2, 128), (1, 4, 4, 128), (2, 4, 4, 128),  # split keys
                                         (32, 8, 2, 128), (64, 8, 2, 128),  # tcgen05 pass 1
                                         (160, 8, 2, 128), (200, 4, 4, 128), (150, 4, 4, 64)])  # > 128: chunks
def test_bf16_append_tensor_core_path_matches_reference_path(cuda, nq, Hq, Hkv, d):
    """hgca_append_bf16 (tensor cores, row-mean weights in-kernel) against the
    reference-order fp64 path (keep_weights=True) on the same staged state: the
    step output, lse, and the re-evaluated archive / EMA'd window MAW."""
    res = []
    for keep in (True, False):
        cfg = cuda.EngineConfig(layers=1, heads=Hq, kv_heads=Hkv, head_dim=d, batch=2, dtype="bfloat16",
                                cache=cuda.CacheConfig(blk_num=8, blk_size=32, beta=1.0),
                                core_count=10 ** 6, max_positions=6000, keep_weights=keep)
        eng = cuda.HybridEngine(cfg)
        g = torch.Generator(device="cuda").manual_seed(77)
        n = 4096 + 37  # archive not a multiple of the 4096-key chunk
        k = torch.randn((2, Hkv, n, d), generator=g, device="cuda").to(torch.bfloat16)
        v = torch.randn((2, Hkv, n, d), generator=g, device="cuda").to(torch.bfloat16)
        maw = torch.rand((2, Hq, n), generator=g, device="cuda", dtype=torch.float64) / 256
        eng.bulk_ingest(0, k, v, maw, 256)
        for _ in range(100):
            q = torch.randn((2, Hq, 1, d), generator=g, device="cuda").to(torch.bfloat16)
            kk = torch.randn((2, Hkv, 1, d), generator=g, device="cuda").to(torch.bfloat16)
            eng.step(0, cuda.StepInput("decode", q, kk, kk))
        q = torch.randn((2, Hq, nq, d), generator=g, device="cuda").to(torch.bfloat16)
        kk = torch.randn((2, Hkv, nq, d), generator=g, device="cuda").to(torch.bfloat16)
        ls = eng.layers[0]
        lo, nxt = ls.lo, ls.nxt
        r = eng.step(0, cuda.StepInput("append", q, kk, -kk))
        torch.cuda.synchronize()
        res.append((host(r.output), host(r.lse), ls.maw[:, :nxt + nq].cpu().numpy(), lo, nxt))
    (o1, l1, m1, lo, nxt), (o2, l2, m2, _, _) = res
    assert rel_err(o2, o1) <= 1e-3
    np.testing.assert_allclose(l2, l1, rtol=0, atol=1e-4)
    # archive MAW = re-evaluated row means; window = EMA / init from the window weights
    np.testing.assert_allclose(m2[:, :lo], m1[:, :lo], rtol=2e-3, atol=1e-9)
    np.testing.assert_allclose(m2[:, lo:], m1[:, lo:], rtol=2e-3, atol=1e-9)


def test_accuracy_metrics_full_selection_and_top1(cuda, rng):
    """accuracy.step_metrics (harness.py:147-160 on the GPU): with beta = 0 every
    archived entry is selected, so the hybrid step equals full attention (eps ~ 0,
    no bound violation); with a 1-entry top-k context the dropped mass is large
    but the error stays within 2*eps*max|V| (the reference's guarantee)."""
    from paper_2507_03153_b200 import accuracy

    for kw in (dict(cache=cuda.CacheConfig(blk_num=4, blk_size=16, beta=0.0)),
               dict(cache=cuda.CacheConfig(blk_num=4, blk_size=16, beta=1.0), selection="topk", topk=1)):
        cfg = cuda.EngineConfig(layers=1, heads=4, kv_heads=2, head_dim=64, batch=2, core_count=64,
                                max_positions=512, **kw)
        eng = cuda.HybridEngine(cfg)
        for _ in range(300):
            q, k, v = (torch.from_numpy(rng.standard_normal(s).astype(np.float32)).cuda()
                       for s in ((2, 4, 1, 64), (2, 2, 1, 64), (2, 2, 1, 64)))
            eng.decode_device(0, q, k, v)
        ls = eng.layers[0]
        n = ls.nxt + 1
        mask = accuracy.attended_mask(eng, 0, n)
        q, k, v = (torch.from_numpy(rng.standard_normal(s).astype(np.float32)).cuda()
                   for s in ((2, 4, 1, 64), (2, 2, 1, 64), (2, 2, 1, 64)))
        out, _, _ = eng.decode_device(0, q, k, v)
        m = accuracy.step_metrics(eng, 0, out, q, mask, n)
        assert m["bound_violations"] == 0, m
        if kw["cache"].beta == 0.0:
            assert m["eps_max"] < 1e-6 and m["max_err"] < 1e-5, m
        else:
            assert m["eps_mean"] > 0.1, m
