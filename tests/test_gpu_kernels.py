"""GPU parity: plugin kernels (attend / attend_indexed / merge_states /
selection) through the C ABI against the reference's outputs (golden) and the
oracle. Mirrors the reference's test_attention.py / test_backends.py /
test_sparsifier.py cases."""

import math

import numpy as np
import pytest

from cases import DENSE_CASES, INDEXED_CASES, dense_inputs, indexed_inputs
from conftest import reference_attention
from oracle import port

pytestmark = pytest.mark.gpu


def tol(dt):
    return 1e-10 if np.dtype(dt) == np.float64 else 1e-6


@pytest.mark.parametrize("key", sorted(DENSE_CASES))
def test_attend_dense_vs_reference(cuda, key, golden):
    g = golden("kernels.npz")
    q, k, v, scale = dense_inputs(key)
    o, l, w = cuda.CUDA.attend_dense(q, k, v, scale, True)
    assert o.dtype == q.dtype and l.dtype == np.float64 and w.dtype == q.dtype
    t = tol(q.dtype)
    go, gl, gw = g[f"{key}_out"], g[f"{key}_lse"], g[f"{key}_w"]
    np.testing.assert_allclose(o, go, atol=t * max(1.0, np.abs(go).max()), rtol=0)
    np.testing.assert_allclose(l, gl, atol=t * max(1.0, np.abs(gl[np.isfinite(gl)]).max(initial=1)), rtol=0)
    np.testing.assert_allclose(w, gw, atol=t, rtol=0)
    if w.size and q.dtype == np.float32:
        # weights feed the MAW: fp64 softmax rounded to fp32
        assert (w != gw).mean() < 1e-4


@pytest.mark.parametrize("key", sorted(INDEXED_CASES))
def test_attend_indexed_vs_reference(cuda, key, golden):
    g = golden("kernels.npz")
    q, k, v, idx, scale = indexed_inputs(key)
    o, l, w = cuda.CUDA.attend_indexed(q, k, v, idx, scale, True)
    np.testing.assert_allclose(o, g[f"{key}_out"], atol=1e-6, rtol=0)
    np.testing.assert_allclose(l, g[f"{key}_lse"], atol=1e-6, rtol=0)
    np.testing.assert_allclose(w, g[f"{key}_w"], atol=1e-7, rtol=0)


def test_frozen_vector(cuda):
    """test_attention.py:94-111."""
    rng = np.random.default_rng(2024)
    q, k, v = (rng.standard_normal(s) for s in ((2, 3), (4, 3), (4, 3)))
    res = cuda.attend(q, k, v, cuda.HeadShape(1, 3))
    np.testing.assert_allclose(res.output, [[-1.1711360815114202, -0.6485395437336913, 0.603185579921532],
                                            [-0.22046775538466243, -0.4585035040865019, 0.2588060306723151]],
                               atol=1e-12)
    np.testing.assert_allclose(res.lse, [2.583235965688748, 1.1851014276031953], atol=1e-12)


def test_random_cases_match_brute_force(cuda, rng):
    """test_attention.py:113-124 (1e-12 on float64)."""
    for _ in range(25):
        nq, n, d = rng.integers(1, 5), rng.integers(1, 9), rng.integers(1, 6)
        q, k, v = (rng.standard_normal(s) for s in ((nq, d), (n, d), (n, d)))
        shape = cuda.HeadShape(1, int(d))
        res = cuda.attend(q, k, v, shape, keep_weights=True)
        ro, rl, rw = reference_attention(q, k, v, shape.scale)
        np.testing.assert_allclose(res.output, ro, atol=1e-12)
        np.testing.assert_allclose(res.lse, rl, atol=1e-12)
        np.testing.assert_allclose(res.weights, rw, atol=1e-12)


def test_attend_contract_edges(cuda, rng):
    """test_attention.py:77-166: single key, ties, empty set, sums, stability, dtypes."""
    HS = cuda.HeadShape
    q, k, v = rng.standard_normal((1, 3)), rng.standard_normal((1, 3)), rng.standard_normal((1, 3))
    res = cuda.attend(q, k, v, HS(1, 3), keep_weights=True)
    np.testing.assert_allclose(res.weights, [[1.0]])
    np.testing.assert_allclose(res.output, v, rtol=1e-6)
    k2 = np.repeat(rng.standard_normal((1, 3)), 2, axis=0)
    v2 = rng.standard_normal((2, 3))
    res = cuda.attend(q, k2, v2, HS(1, 3), keep_weights=True)
    np.testing.assert_allclose(res.weights, [[0.5, 0.5]], atol=1e-7)
    res = cuda.attend(np.ones((2, 4)), np.zeros((0, 4)), np.zeros((0, 4)), HS(1, 4), keep_weights=True)
    assert np.isneginf(res.lse).all() and not res.output.any() and res.weights.shape == (2, 0)
    q3 = rng.standard_normal((4, 3, 8)).astype(np.float32)
    k3 = rng.standard_normal((4, 17, 8)).astype(np.float32)
    v3 = rng.standard_normal((4, 17, 8)).astype(np.float32)
    res = cuda.attend(q3, k3, v3, HS(4, 8), keep_weights=True)
    np.testing.assert_allclose(res.weights.sum(axis=-1), 1.0, atol=1e-6)
    assert res.output.dtype == np.float32 and res.weights.dtype == np.float32 and res.lse.dtype == np.float64
    res = cuda.attend(np.full((1, 2), 100.0), np.array([[100.0, 100.0], [-100.0, -100.0], [95.0, 100.0]]),
                      np.eye(3, 2), HS(1, 2, scale=1.0))
    assert np.isfinite(res.output).all() and np.isfinite(res.lse).all()
    with pytest.raises(cuda.ContractError):
        cuda.attend(q, rng.standard_normal((2, 4)), rng.standard_normal((2, 4)), HS(1, 3))
    with pytest.raises(cuda.ContractError):
        cuda.attend(q, rng.standard_normal((2, 3)), rng.standard_normal((3, 3)), HS(1, 3))


def test_attend_indexed_equals_gathered(cuda, rng):
    """test_attention.py:169-190."""
    k, v, q = rng.standard_normal((10, 4)), rng.standard_normal((10, 4)), rng.standard_normal((2, 4))
    idx = np.array([7, 1, 4], dtype=np.int64)
    shape = cuda.HeadShape(1, 4)
    a = cuda.attend_indexed(q, k, v, idx, shape.scale, keep_weights=True)
    b = cuda.attend(q, k[idx], v[idx], shape, keep_weights=True)
    np.testing.assert_allclose(a.output, b.output, atol=1e-12)
    np.testing.assert_allclose(a.lse, b.lse, atol=1e-12)
    np.testing.assert_allclose(a.weights, b.weights, atol=1e-12)
    res = cuda.attend_indexed(rng.standard_normal((1, 4)), rng.standard_normal((5, 4)),
                              rng.standard_normal((5, 4)), [], 0.5)
    assert np.isneginf(res.lse).all() and not res.output.any()
    with pytest.raises(cuda.ContractError):
        cuda.attend_indexed(rng.standard_normal((1, 4)), rng.standard_normal((5, 4)),
                            rng.standard_normal((5, 4)), [5], 0.5)


def test_merge_states_vs_reference(cuda, golden):
    g = golden("kernels.npz")
    for ci in range(3):
        key = f"merge{ci}"
        a = cuda.AttentionResult(g[f"{key}_oa"], g[f"{key}_la"], g[f"{key}_wa"])
        b = cuda.AttentionResult(g[f"{key}_ob"], g[f"{key}_lb"], g[f"{key}_wb"])
        m = cuda.merge_states(a, b)
        np.testing.assert_allclose(m.output, g[f"{key}_out"], atol=1e-14, rtol=1e-14)
        np.testing.assert_allclose(m.lse, g[f"{key}_lse"], atol=1e-13)
        np.testing.assert_allclose(m.weights, g[f"{key}_w"], atol=1e-14)


def test_merge_properties(cuda, rng):
    """test_attention.py:193-295: identity, both-empty, +ln2, split 5/3,
    random partitions at magnitudes {1, 10, 1e3}, associativity, fp32."""
    HS = cuda.HeadShape
    shape = HS(1, 4)
    q = rng.standard_normal((3, 4))
    a = cuda.attend(q, rng.standard_normal((6, 4)), rng.standard_normal((6, 4)), shape)
    b = cuda.attend(q, np.zeros((0, 4)), np.zeros((0, 4)), shape)
    for m in (cuda.merge_states(a, b), cuda.merge_states(b, a)):
        np.testing.assert_allclose(m.output, a.output, atol=1e-12)
        np.testing.assert_allclose(m.lse, a.lse, atol=1e-12)
    e = cuda.AttentionResult(np.zeros((1, 2)), np.full(1, -np.inf))
    m = cuda.merge_states(e, e)
    assert np.isneginf(m.lse).all() and not m.output.any()
    k, v = rng.standard_normal((5, 4)), rng.standard_normal((5, 4))
    a = cuda.attend(q[:2], k, v, shape)
    m = cuda.merge_states(a, a)
    np.testing.assert_allclose(m.output, a.output, atol=1e-12)
    np.testing.assert_allclose(m.lse, a.lse + math.log(2), atol=1e-12)
    for seed in range(40):
        r = np.random.default_rng(seed)
        heads, n, d = int(r.integers(1, 5)), int(r.integers(1, 25)), int(r.integers(1, 17))
        mag = [1.0, 10.0, 1e3][seed % 3]
        sh = HS(heads, d)
        qq = mag * r.standard_normal((heads, 2, d))
        kk, vv = r.standard_normal((heads, n, d)), r.standard_normal((heads, n, d))
        cut = int(r.integers(0, n + 1))
        perm = r.permutation(n)
        merged = cuda.merge_states(cuda.attend(qq, kk[:, perm[:cut]], vv[:, perm[:cut]], sh),
                                   cuda.attend(qq, kk[:, perm[cut:]], vv[:, perm[cut:]], sh))
        full = cuda.attend(qq, kk[:, perm], vv[:, perm], sh)
        np.testing.assert_allclose(merged.output, full.output, atol=1e-10)
        np.testing.assert_allclose(merged.lse, full.lse, atol=1e-10)
    sh = HS(2, 8)
    q32 = rng.standard_normal((2, 1, 8)).astype(np.float32)
    k32 = rng.standard_normal((2, 50, 8)).astype(np.float32)
    v32 = rng.standard_normal((2, 50, 8)).astype(np.float32)
    merged = cuda.merge_states(cuda.attend(q32, k32[:, :20], v32[:, :20], sh), cuda.attend(q32, k32[:, 20:], v32[:, 20:], sh))
    assert merged.output.dtype == np.float32
    np.testing.assert_allclose(merged.output, cuda.attend(q32, k32, v32, sh).output, atol=1e-5)
    with pytest.raises(cuda.ContractError):
        cuda.merge_states(cuda.AttentionResult(np.zeros((1, 2)), np.zeros(1)),
                          cuda.AttentionResult(np.zeros((1, 3)), np.zeros(1)))


def test_select_salient_vs_reference(cuda, golden):
    g = golden("selection.npz")
    for i in range(4):
        sel = cuda.select_salient(g[f"sal{i}_maw"], float(g[f"sal{i}_beta"]), int(g[f"sal{i}_div"]))
        got = np.stack([np.isin(np.arange(g[f"sal{i}_maw"].shape[1]), s) for s in sel])
        np.testing.assert_array_equal(got, g[f"sal{i}_mask"])
    assert cuda.select_salient(np.array([[0.5, 0.3, 0.1, 0.05, 0.05]]), 1.0, 5)[0].tolist() == [0, 1]
    assert cuda.select_salient(np.full((1, 5), 0.2), 1.0, 5)[0].size == 0
    with pytest.raises(cuda.ContractError):
        cuda.select_salient(np.zeros((1, 3)), 1.0, 0)


@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 40000])
def test_select_topk_vs_lexsort(cuda, n):
    r = np.random.default_rng(n)
    maw = np.round(r.random((6, n)) * 50) / 50       # heavy exact ties
    maw[1] = 0.0                                      # all tied
    maw[2, ::2] = -0.0                                # signed zeros tie with +0
    for k in (0, 1, n // 3, n - 1, n, n + 5):
        got = cuda.select_topk(maw, k)
        want = port.select_topk(maw, k)
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)


def test_pack_head_groups_vs_reference(cuda, golden):
    g = golden("selection.npz")

    class Store:  # duck-typed reference StoreTier
        pass

    for i in range(4):
        maw, ctx_mask = g[f"pack{i}_maw"], g[f"pack{i}_ctx"]
        st = Store()
        st.shape = cuda.HeadShape(maw.shape[0], 4)
        st.maw = maw
        st.archive_size = maw.shape[1]
        st.context = Store()
        st.context.indices = [np.nonzero(r)[0].astype(np.int64) for r in ctx_mask]
        tasks = cuda.pack_head_groups(st, batch=int(g[f"pack{i}_batch"]), core_count=int(g[f"pack{i}_cores"]))
        ent = np.zeros_like(ctx_mask)
        pad = np.zeros_like(ctx_mask)
        for t in tasks:
            for hd, e, p in zip(t.heads, t.entries, t.padding):
                assert (np.diff(e) > 0).all()
                ent[hd, e] = True
                pad[hd, e[p]] = True
        np.testing.assert_array_equal(ent, g[f"pack{i}_entries"])
        np.testing.assert_array_equal(pad, g[f"pack{i}_padding"])
