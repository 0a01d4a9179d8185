"""CPU: pin the oracle (oracle/) against the reference's own outputs.

The golden fixtures in tests/golden/ were produced by running the reference
package (tierkv, compiled backend) via tests/golden/make_golden.py. Every
check here is bitwise unless a tolerance is written next to it.
"""

import math

import numpy as np
import pytest

from cases import DENSE_CASES, INDEXED_CASES, dense_inputs, indexed_inputs
from conftest import reference_attention
from oracle import port
from oracle import workload as owl


def test_oracle_library_builds_and_loads():
    assert port.lib() is not None


@pytest.mark.parametrize("key", sorted(DENSE_CASES))
def test_dense_matches_reference_bitwise(key, golden):
    g = golden("kernels.npz")
    q, k, v, scale = dense_inputs(key)
    o, l, w = port.attend_dense(q, k, v, scale, True)
    np.testing.assert_array_equal(o, g[f"{key}_out"])
    np.testing.assert_array_equal(l, g[f"{key}_lse"])
    np.testing.assert_array_equal(w, g[f"{key}_w"])


@pytest.mark.parametrize("key", sorted(INDEXED_CASES))
def test_indexed_matches_reference_bitwise(key, golden):
    g = golden("kernels.npz")
    q, k, v, idx, scale = indexed_inputs(key)
    o, l, w = port.attend_indexed(q, k, v, idx, scale, True)
    np.testing.assert_array_equal(o, g[f"{key}_out"])
    np.testing.assert_array_equal(l, g[f"{key}_lse"])
    np.testing.assert_array_equal(w, g[f"{key}_w"])


def test_frozen_reference_vector():
    """test_attention.py:94-111 frozen case (seed 2024, 2x4x3), tol 1e-12."""
    rng = np.random.default_rng(2024)
    q = rng.standard_normal((2, 3))
    k = rng.standard_normal((4, 3))
    v = rng.standard_normal((4, 3))
    frozen_out = np.array([
        [-1.1711360815114202, -0.6485395437336913, 0.603185579921532],
        [-0.22046775538466243, -0.4585035040865019, 0.2588060306723151],
    ])
    frozen_lse = np.array([2.583235965688748, 1.1851014276031953])
    o, l, _ = port.attend_dense(q[None], k[None], v[None], 1 / math.sqrt(3), False)
    np.testing.assert_allclose(o[0], frozen_out, atol=1e-12)
    np.testing.assert_allclose(l[0], frozen_lse, atol=1e-12)
    ref_out, ref_lse, _ = reference_attention(q, k, v, 1 / math.sqrt(3))
    np.testing.assert_allclose(ref_out, frozen_out, atol=1e-15)


def test_merge_matches_reference_bitwise(golden):
    g = golden("kernels.npz")
    for ci in range(3):
        key = f"merge{ci}"
        out, lse = port.merge_states(g[f"{key}_oa"], g[f"{key}_la"], g[f"{key}_ob"], g[f"{key}_lb"])
        np.testing.assert_array_equal(out, g[f"{key}_out"])
        np.testing.assert_array_equal(lse, g[f"{key}_lse"])


def test_select_salient_matches_reference(golden):
    g = golden("selection.npz")
    for i in range(4):
        sel = port.select_salient(g[f"sal{i}_maw"], float(g[f"sal{i}_beta"]), int(g[f"sal{i}_div"]))
        got = np.stack([np.isin(np.arange(g[f"sal{i}_maw"].shape[1]), s) for s in sel])
        np.testing.assert_array_equal(got, g[f"sal{i}_mask"])


def test_select_salient_kats():
    """test_sparsifier.py:27-43."""
    assert [s.tolist() for s in port.select_salient(np.array([[0.1, 0.2], [0.3, 0.4]]), 0.0, 10)] == [[0, 1], [0, 1]]
    assert port.select_salient(np.full((1, 5), 0.2), 1.0, 5)[0].size == 0
    assert port.select_salient(np.array([[0.5, 0.3, 0.1, 0.05, 0.05]]), 1.0, 5)[0].tolist() == [0, 1]


def test_pack_head_groups_matches_reference(golden):
    g = golden("selection.npz")
    for i in range(4):
        maw, ctx_mask = g[f"pack{i}_maw"], g[f"pack{i}_ctx"]
        n = maw.shape[1]
        ctx = [np.nonzero(r)[0].astype(np.int64) for r in ctx_mask]
        entries, padding = port.pack_head_groups(ctx, maw, n, int(g[f"pack{i}_batch"]), int(g[f"pack{i}_cores"]))
        ent = np.zeros_like(ctx_mask)
        pad = np.zeros_like(ctx_mask)
        for h in range(len(ctx)):
            ent[h, entries[h]] = True
            pad[h, entries[h][padding[h]]] = True
        np.testing.assert_array_equal(ent, g[f"pack{i}_entries"])
        np.testing.assert_array_equal(pad, g[f"pack{i}_padding"])


def test_padding_kats():
    """test_sparsifier.py:176-199: pad [4, 6]; zero-selected head -> [1, 2, 3, 4]."""
    maw = np.array([[0.9, 0.9, 0.9, 0.9, 0.9, 0.0, 0.0, 0.0],
                    [0.9, 0.9, 0.9, 0.0, 0.08, 0.02, 0.05, 0.0]])
    ctx = port.select_salient(maw, 1.0, 2)
    e, p = port.pack_head_groups(ctx, maw, 8, 1, 1)
    assert sorted(e[1][p[1]].tolist()) == [4, 6]
    maw = np.array([[0.9, 0.9, 0.9, 0.9, 0.0, 0.0, 0.0, 0.0],
                    [0.0, 0.01, 0.02, 0.03, 0.04, 0.0, 0.0, 0.0]])
    ctx = port.select_salient(maw, 1.0, 2)
    e, p = port.pack_head_groups(ctx, maw, 8, 1, 1)
    assert sorted(e[1].tolist()) == [1, 2, 3, 4] and p[1].all()


def test_workload_restatement_bit_identical(golden):
    g = golden("workload.npz")
    steps = owl.gen_workload(owl.WorkloadSpec(seed=3, steps=40, prefill_len=8, append_events=((20, 4),)),
                             2, 8, 1 / math.sqrt(8), 2)
    np.testing.assert_array_equal(np.concatenate([s.q for s in steps], axis=2), g["small_q"])
    np.testing.assert_array_equal(np.concatenate([s.keys for s in steps], axis=2), g["small_k"])
    np.testing.assert_array_equal(np.concatenate([s.values for s in steps], axis=2), g["small_v"])


ENGINE_CASES = {
    "e1_g1": (4, 64, 4, 16, 0.5, 1.0, 8, dict(seed=7, steps=300, prefill_len=16)),
    "e2_pad": (4, 64, 4, 16, 0.5, 1.0, 1, dict(seed=7, steps=300, prefill_len=16, append_events=((150, 8),))),
    "e3_d128": (8, 128, 8, 32, 0.5, 0.5, 8, dict(seed=11, steps=400, prefill_len=64, append_events=((200, 16),))),
}


def run_oracle_engine(name, threads=1):
    H, d, bn, bs, alpha, beta, cores, spec_kw = ENGINE_CASES[name]
    spec = owl.WorkloadSpec(**spec_kw)
    steps = owl.gen_workload(spec, H, d, 1 / math.sqrt(d), 1)
    eng = port.OracleEngine(H, d, bn, bs, alpha, beta, core_count=cores, batch=1,
                            max_len=sum(s.n_q for s in steps), threads=threads)
    outs = []
    for s in steps:
        r = eng.step(s.mode, s.q[0], s.keys[0], s.values[0])
        outs.append((r.output[:, -1, :].copy(), r.lse[:, -1].copy()))
    return eng, outs


@pytest.mark.parametrize("name", sorted(ENGINE_CASES))
def test_engine_port_matches_reference_bitwise(name, golden):
    g = golden("engine.npz")
    eng, outs = run_oracle_engine(name)
    sel = g[f"{name}_steps"]
    np.testing.assert_array_equal(np.stack([outs[i][0] for i in sel]), g[f"{name}_out"])
    np.testing.assert_array_equal(np.stack([outs[i][1] for i in sel]), g[f"{name}_lse"])
    w_size, n = g[f"{name}_sizes"]
    assert (eng.window_size, eng.archive_size) == (w_size, n)
    np.testing.assert_array_equal(eng.maw[:, :n], g[f"{name}_store_maw"])
    np.testing.assert_array_equal(eng.maw[:, n:n + w_size], g[f"{name}_window_maw"])
    ctx = np.zeros((eng.H, n), bool)
    for h in range(eng.H):
        ctx[h, eng.context[h]] = True
    np.testing.assert_array_equal(ctx, g[f"{name}_ctx"])


def test_threaded_sparse_loop_is_bitwise_serial():
    _, a = run_oracle_engine("e1_g1", threads=1)
    _, b = run_oracle_engine("e1_g1", threads=4)
    for (o1, l1), (o2, l2) in zip(a, b):
        np.testing.assert_array_equal(o1, o2)
        np.testing.assert_array_equal(l1, l2)


@pytest.mark.skipif(not port.ref_core(), reason="oracle/_ref not built (make -C oracle ref)")
def test_c_restatement_equals_reference_core(rng):
    """The C restatement is bit-identical to the reference's compiled _core."""
    for nkv in (0, 1, 33, 700):
        q = (50 * rng.standard_normal((3, 2, 64))).astype(np.float32)
        k = (50 * rng.standard_normal((3, nkv, 64))).astype(np.float32)
        v = rng.standard_normal((3, nkv, 64)).astype(np.float32)
        a = port.attend_dense(q, k, v, 0.125, True)
        b = port.attend_dense(q, k, v, 0.125, True, kernels="reference")
        for x, y in zip(a, b):
            np.testing.assert_array_equal(x, y)


@pytest.mark.parametrize("beta,cores", [(1.0, 8), (0.0, 32)])
def test_engine_port_matches_reference_c1_prefix(beta, cores, golden):
    """BASELINE config 1 (32 heads d128, gen_workload seed 7, window 16x32): the
    first 640 steps of the reference's own run (tests/golden/c1.npz), bitwise --
    outputs, lse, context sizes and attended (context + padding) counts."""
    g = golden("c1.npz")
    name = f"c1_b{beta}_c{cores}"
    spec = owl.WorkloadSpec(seed=7, steps=3968, prefill_len=128)
    steps = owl.gen_workload(spec, 32, 128, 1 / math.sqrt(128), 1)[:641]
    eng = port.OracleEngine(32, 128, 16, 32, 0.5, beta, core_count=cores, batch=1, max_len=4096, threads=4)
    out_idx = {int(s): j for j, s in enumerate(g[f"{name}_out_steps"])}
    lse_idx = {int(s): j for j, s in enumerate(g[f"{name}_lse_steps"])}
    checked = 0
    for i, s in enumerate(steps):
        r = eng.step(s.mode, s.q[0], s.keys[0], s.values[0])
        if i in lse_idx:
            j = lse_idx[i]
            np.testing.assert_array_equal(r.lse[:, -1], g[f"{name}_lse"][j])
            np.testing.assert_array_equal([c.size for c in eng.context], g[f"{name}_ctx_sizes"][j])
            np.testing.assert_array_equal([e.size for e in r.store_entries], g[f"{name}_attended"][j])
        if i in out_idx:
            np.testing.assert_array_equal(r.output[:, -1, :], g[f"{name}_out"][out_idx[i]])
            checked += 1
    assert checked == 6 and eng.archive_size > 0


HARNESS_CASES = {
    # (layers, heads, head_dim, blk_num, blk_size, alpha, beta, core_count, spec kwargs) = make_golden.HARNESS_CASES
    "h1": (1, 4, 64, 4, 16, 0.5, 1.0, 8, dict(seed=5, steps=300, prefill_len=16, append_events=((150, 8),))),
    "h2": (2, 4, 64, 3, 8, 0.7, 0.5, 2, dict(seed=6, steps=200, prefill_len=8, heavy_hitter_boost=0.6,
                                             append_events=((90, 4),))),
}


@pytest.mark.parametrize("name", sorted(HARNESS_CASES))
def test_harness_restatement_matches_reference(name, golden):
    """oracle/harness.py over the oracle port reproduces tierkv.harness.run_experiment's
    per-head metric rows and summary (tests/golden/harness.npz) bitwise."""
    from oracle import harness as oh

    g = golden("harness.npz")
    L, H, d, bn, bs, alpha, beta, cores, spec_kw = HARNESS_CASES[name]
    steps = owl.gen_workload(owl.WorkloadSpec(**spec_kw), H, d, 1 / math.sqrt(d), L)
    total = sum(s.n_q for s in steps)
    engines = [port.OracleEngine(H, d, bn, bs, alpha, beta, core_count=cores, batch=1, max_len=total)
               for _ in range(L)]
    probe = oh.MetricsProbe(L, H, d, total, 1 / math.sqrt(d))
    oh.run_port_sequence(engines, steps, probe.on_step)
    np.testing.assert_array_equal(np.array(probe.rows, np.float64), g[f"{name}_rows"])
    summ = probe.summary()
    ref = dict(zip(g[f"{name}_summary_keys"].tolist(), g[f"{name}_summary"].tolist()))
    assert set(summ) == set(ref)
    for k, v in summ.items():
        assert float(v) == ref[k], (k, v, ref[k])
