"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
package (tierkv, /root/reference/pkg) with its compiled Cython backend.

Run in the build container only (the reference does not exist on the GPU
box); the resulting .npz files are committed. Usage:

    python tests/golden/make_golden.py [--ref-src /tmp/refbuild/pkg/src]

If --ref-src has no built tierkv._core, the reference package is copied to
/tmp/refbuild and built there (`python setup.py build_ext --inplace`);
/root/reference itself is never written to.
"""

from __future__ import annotations

import argparse
import glob
import hashlib
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def ensure_ref(src):
    if glob.glob(os.path.join(src, "tierkv", "_core*.so")):
        return src
    pkg = "/tmp/refbuild/pkg"
    if not os.path.exists(pkg):
        os.makedirs("/tmp/refbuild", exist_ok=True)
        shutil.copytree("/root/reference/pkg", pkg)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=pkg, check=True,
                   capture_output=True)
    return os.path.join(pkg, "src")


def kernels(tk, out):
    """Reference outputs for the kernel cases of tests/golden/cases.py (inputs
    are regenerated from per-case seeds, so only outputs are stored)."""
    from cases import DENSE_CASES, INDEXED_CASES, dense_inputs, indexed_inputs

    be = tk.backends.get_backend("compiled")
    rec = {}
    for key in DENSE_CASES:
        q, k, v, scale = dense_inputs(key)
        o, l, w = be.attend_dense(q, k, v, scale, True)
        rec.update({f"{key}_out": o, f"{key}_lse": l, f"{key}_w": w})
    for key in INDEXED_CASES:
        q, k, v, idx, scale = indexed_inputs(key)
        o, l, w = be.attend_indexed(q, k, v, idx, scale, True)
        rec.update({f"{key}_out": o, f"{key}_lse": l, f"{key}_w": w})
    rng = np.random.default_rng(0xC0FFEE)
    # merge_states: random partitions at magnitudes {1, 10, 1e3} (test_attention.py:238-262)
    for ci, mag in enumerate((1.0, 10.0, 1e3)):
        H, n, d = 3, 24, 16
        q = mag * rng.standard_normal((H, 2, d))
        k = rng.standard_normal((H, n, d))
        v = rng.standard_normal((H, n, d))
        cut = 9
        shape = tk.HeadShape(H, d)
        a = tk.attend(q, k[:, :cut], v[:, :cut], shape, keep_weights=True)
        b = tk.attend(q, k[:, cut:], v[:, cut:], shape, keep_weights=True)
        m = tk.merge_states(a, b)
        key = f"merge{ci}"
        rec.update({f"{key}_oa": a.output, f"{key}_la": a.lse, f"{key}_wa": a.weights,
                    f"{key}_ob": b.output, f"{key}_lb": b.lse, f"{key}_wb": b.weights,
                    f"{key}_out": m.output, f"{key}_lse": m.lse, f"{key}_w": m.weights})
    np.savez_compressed(out, **rec)


def selection(tk, out):
    rng = np.random.default_rng(2027)
    rec = {}
    # select_salient: random rows incl. exact ties at the threshold
    maw = rng.random((4, 300))
    maw[:, ::7] = 1.0 / 13.0
    for i, (beta, div) in enumerate([(1.0, 13), (0.5, 40), (0.0, 5), (2.0, 300)]):
        sel = tk.select_salient(maw, beta, div)
        rec[f"sal{i}_maw"] = maw
        rec[f"sal{i}_beta"] = np.array(beta)
        rec[f"sal{i}_div"] = np.array(div)
        rec[f"sal{i}_mask"] = np.stack([np.isin(np.arange(300), s) for s in sel])
    # pack_head_groups over a StoreTier with quantized MAW (many exact ties)
    shape = tk.HeadShape(8, 4)
    for i, (cores, batch, n) in enumerate([(1, 1, 200), (2, 1, 333), (4, 3, 64), (8, 1, 50)]):
        st = tk.StoreTier(shape)
        mw = np.round(rng.random((8, n)) * 20) / 20 * rng.choice([0.0, 1.0], size=(8, n), p=[0.2, 0.8])
        kv = np.zeros((8, n, 4), np.float32)
        blk = tk.KvBlock(keys=kv, values=kv.copy(), maw=mw, start=0, occupancy=n)
        st.ingest_evicted([blk], beta=1.0, window_size=int(rng.integers(2, 12)))
        tasks = tk.pack_head_groups(st, batch=batch, core_count=cores)
        ent = np.zeros((8, n), bool)
        pad = np.zeros((8, n), bool)
        for t in tasks:
            for hd, e, p in zip(t.heads, t.entries, t.padding):
                ent[hd, e] = True
                pad[hd, e[p]] = True
        ctx = np.stack([np.isin(np.arange(n), st.context.indices[h]) for h in range(8)])
        rec.update({f"pack{i}_maw": st.maw, f"pack{i}_ctx": ctx, f"pack{i}_entries": ent,
                    f"pack{i}_padding": pad, f"pack{i}_cores": np.array(cores),
                    f"pack{i}_batch": np.array(batch)})
    np.savez_compressed(out, **rec)


ENGINE_CASES = {
    # name: (layers, heads, head_dim, blk_num, blk_size, alpha, beta, core_count, spec kwargs, stride)
    "e1_g1": (1, 4, 64, 4, 16, 0.5, 1.0, 8, dict(seed=7, steps=300, prefill_len=16), 1),
    "e2_pad": (1, 4, 64, 4, 16, 0.5, 1.0, 1, dict(seed=7, steps=300, prefill_len=16,
                                                   append_events=((150, 8),)), 1),
    "e3_d128": (1, 8, 128, 8, 32, 0.5, 0.5, 8, dict(seed=11, steps=400, prefill_len=64,
                                                    append_events=((200, 16),)), 10),
}


def engine(tk, out):
    rec = {}
    for name, (L, H, d, bn, bs, alpha, beta, cores, spec_kw, stride) in ENGINE_CASES.items():
        cfg = tk.EngineConfig(layers=L, heads=H, head_dim=d,
                              cache=tk.CacheConfig(blk_num=bn, blk_size=bs, alpha=alpha, beta=beta),
                              core_count=cores)
        wl = tk.gen_workload(tk.WorkloadSpec(**spec_kw), cfg.head_shape, cfg.layers)
        eng, outs = tk.run_sequence(cfg, wl, collect=True)
        sel = [i for i in range(len(outs)) if i % stride == 0 or i == len(outs) - 1]
        o = np.stack([np.ascontiguousarray(outs[i][0].output[:, -1, :]) for i in sel])
        l = np.stack([outs[i][0].lse[:, -1] for i in sel])
        st = eng.layers[0].store
        win = eng.layers[0].window
        n = st.archive_size
        ctx = np.stack([np.isin(np.arange(n), st.context.indices[h]) for h in range(H)])
        rec.update({f"{name}_steps": np.array(sel), f"{name}_out": o, f"{name}_lse": l,
                    f"{name}_store_maw": st.maw, f"{name}_window_maw": win.maw_matrix(),
                    f"{name}_ctx": ctx, f"{name}_sizes": np.array([win.size, n])})
    np.savez_compressed(out, **rec)


def workload(tk, out):
    rec = {}
    spec = tk.WorkloadSpec(seed=3, steps=40, prefill_len=8, append_events=((20, 4),))
    wl = tk.gen_workload(spec, tk.HeadShape(2, 8), 2)
    rec["small_q"] = np.concatenate([s.q for s in wl], axis=2)
    rec["small_k"] = np.concatenate([s.keys for s in wl], axis=2)
    rec["small_v"] = np.concatenate([s.values for s in wl], axis=2)
    spec = tk.WorkloadSpec(seed=7, steps=3968, prefill_len=128)
    wl = tk.gen_workload(spec, tk.HeadShape(32, 128), 1)
    h = hashlib.sha256()
    for s in wl:
        h.update(s.q.tobytes())
        h.update(s.keys.tobytes())
        h.update(s.values.tobytes())
    rec["c1_sha256"] = np.frombuffer(h.digest(), dtype=np.uint8)
    np.savez_compressed(out, **rec)


def workload_file(tk, out):
    """A small file written by the reference's own save_workload (workload.py:189-210):
    pins paper_2507_03153_b200.workload's reader and writer to the format."""
    spec = tk.WorkloadSpec(seed=3, steps=12, prefill_len=4, append_events=((5, 3),))
    tk.save_workload(tk.gen_workload(spec, tk.HeadShape(2, 16), 2), out)


def perf_model(tk, out):
    """Reference perf_model.py values at a few cells: pins costmodel's reference layer."""
    import json
    from tierkv import perf_model as pm
    shape = pm.WorkloadShape(batch=1, heads=32, head_dim=128, n_q=1, bytes_per_elem=2)
    rec = {"merge_bytes": pm.merge_bytes(shape), "kv_bytes_1000": pm.kv_bytes(1000, shape),
           "cost_gpu_1025": pm.attention_cost(1025, shape.with_(n_window=1024), pm.DEFAULT_GPU),
           "cost_cpu_8192_q64": pm.attention_cost(8192, shape.with_(n_q=64, batch=3), pm.DEFAULT_CPU)}
    cell = shape.with_(n_window=256, n_store=4096, n_selected=819)
    b = pm.time_offload_baseline(cell, pm.DEFAULT_GPU, pm.DEFAULT_LINK)
    h = pm.time_hybrid(cell, pm.DEFAULT_GPU, pm.DEFAULT_CPU, pm.DEFAULT_LINK, 0.7)
    rec.update(baseline=[b.transfer, b.compute], hybrid=[h.gpu_part, h.cpu_part, h.merge])
    rec["heatmap"] = pm.speedup_heatmap([256, 512, 1024], [0, 1024, 16384], shape).tolist()
    rec["rows"] = pm.heatmap_rows([256, 1024], [0, 4096], [1, 4], shape, core_efficiency=0.25,
                                  retention_fraction=0.1)
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)


C1_BETAS = (0.0, 0.5, 1.0, 2.0)
C1_CORES = (32, 8)          # g = 1 and g = 4 (padding) at batch 1, 32 heads
C1_FULL = "c1_b1.0_c32"     # the run whose final MAW is stored in full (the rest: sha256)
C1_OUT_EVERY, C1_LSE_EVERY = 128, 8


def c1_name(beta, cores):
    return f"c1_b{beta}_c{cores}"


def _c1_run(args):
    """One BASELINE config-1 run of the reference (SURVEY.md §8(d) Config 1):
    gen_workload(seed=7, steps=3968, prefill_len=128), HeadShape(32, 128),
    CacheConfig(16, 32, 0.5, beta), core_count `cores`, compiled backend."""
    src, beta, cores = args
    sys.path.insert(0, src)
    os.environ["TIERKV_BACKEND"] = "compiled"
    import tierkv as tk

    cfg = tk.EngineConfig(layers=1, heads=32, head_dim=128,
                          cache=tk.CacheConfig(blk_num=16, blk_size=32, alpha=0.5, beta=beta),
                          core_count=cores)
    wl = tk.gen_workload(tk.WorkloadSpec(seed=7, steps=3968, prefill_len=128), cfg.head_shape, 1)
    eng = tk.HybridEngine(cfg)
    ck_out, outs, ck_lse, lses, ctx_sizes, attended = [], [], [], [], [], []
    n_steps = len(wl)
    for i, s in enumerate(wl):
        r = eng.step(0, tk.StepInput(s.mode, s.q[0], s.keys[0], s.values[0]))
        last = i == n_steps - 1
        if i % C1_LSE_EVERY == 0 or last:
            ck_lse.append(i)
            lses.append(r.lse[:, -1].copy())
            ctx_sizes.append(eng.layers[0].store.context.sizes())
            attended.append([p.size for p in r.store_positions])
        if i % C1_OUT_EVERY == 0 or last:
            ck_out.append(i)
            outs.append(np.ascontiguousarray(r.output[:, -1, :]))
    st, win = eng.layers[0].store, eng.layers[0].window
    n = st.archive_size
    ctx = np.stack([np.isin(np.arange(n), st.context.indices[h]) for h in range(32)])
    name = c1_name(beta, cores)
    rec = {f"{name}_out_steps": np.array(ck_out), f"{name}_out": np.stack(outs).astype(np.float32),
           f"{name}_lse_steps": np.array(ck_lse), f"{name}_lse": np.stack(lses),
           f"{name}_ctx_sizes": np.array(ctx_sizes, np.int32), f"{name}_attended": np.array(attended, np.int32),
           f"{name}_ctx_bits": np.packbits(ctx, axis=1), f"{name}_sizes": np.array([win.size, n]),
           f"{name}_store_maw_sha": np.frombuffer(hashlib.sha256(np.ascontiguousarray(st.maw).tobytes()).digest(), np.uint8),
           f"{name}_window_maw_sha": np.frombuffer(hashlib.sha256(np.ascontiguousarray(win.maw_matrix()).tobytes()).digest(), np.uint8)}
    if name == C1_FULL:
        rec[f"{name}_store_maw"] = st.maw
        rec[f"{name}_window_maw"] = win.maw_matrix()
    return rec


def c1(src, out):
    """BASELINE config 1 at full size, every beta x {g=1, g=4}: outputs every 128
    steps, lse / context sizes / attended counts every 8 steps, the final context
    bitmasks and MAW (sha256; full arrays for one run). 8 processes."""
    import multiprocessing as mp

    jobs = [(src, b, c) for b in C1_BETAS for c in C1_CORES]
    with mp.get_context("spawn").Pool(min(len(jobs), os.cpu_count() or 1)) as pool:
        recs = pool.map(_c1_run, jobs)
    rec = {}
    for r in recs:
        rec.update(r)
    np.savez_compressed(out, **rec)


HARNESS_CASES = {
    # name: (layers, heads, head_dim, blk_num, blk_size, alpha, beta, core_count, spec kwargs)
    "h1": (1, 4, 64, 4, 16, 0.5, 1.0, 8, dict(seed=5, steps=300, prefill_len=16,
                                              append_events=((150, 8),))),
    "h2": (2, 4, 64, 3, 8, 0.7, 0.5, 2, dict(seed=6, steps=200, prefill_len=8, heavy_hitter_boost=0.6,
                                             append_events=((90, 4),))),
}


def harness(tk, out):
    """tierkv.harness.run_experiment (harness.py:123-192) per-head metric rows
    and summary: pins accuracy.step_metrics and the harness restatement."""
    from tierkv.harness import run_experiment

    rec = {}
    for name, (L, H, d, bn, bs, alpha, beta, cores, spec_kw) in HARNESS_CASES.items():
        cfg = tk.EngineConfig(layers=L, heads=H, head_dim=d,
                              cache=tk.CacheConfig(blk_num=bn, blk_size=bs, alpha=alpha, beta=beta),
                              core_count=cores)
        wl = tk.gen_workload(tk.WorkloadSpec(**spec_kw), cfg.head_shape, cfg.layers)
        rep = run_experiment(cfg, tk.PerfConfig(), wl)
        rows = np.array([[float(x) for x in r] for r in rep.per_head_rows], np.float64)
        rec[f"{name}_rows"] = rows
        rec[f"{name}_summary_keys"] = np.array(list(rep.summary.keys()))
        rec[f"{name}_summary"] = np.array([float(v) for v in rep.summary.values()])
    np.savez_compressed(out, **rec)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-src", default="/tmp/refbuild/pkg/src")
    ap.add_argument("--only", default=None, help="regenerate one fixture (e.g. workload_file)")
    args = ap.parse_args()
    src = ensure_ref(args.ref_src)
    sys.path.insert(0, src)
    sys.path.insert(0, HERE)
    os.environ["TIERKV_BACKEND"] = "compiled"
    import tierkv as tk

    assert tk.backends.active.name == "compiled"
    if args.only == "workload_file":
        workload_file(tk, os.path.join(HERE, "workload_small.tkv"))
        return
    if args.only == "perf_model":
        perf_model(tk, os.path.join(HERE, "perf_model.json"))
        return
    if args.only == "c1":
        c1(src, os.path.join(HERE, "c1.npz"))
        return
    if args.only == "harness":
        harness(tk, os.path.join(HERE, "harness.npz"))
        return
    workload_file(tk, os.path.join(HERE, "workload_small.tkv"))
    perf_model(tk, os.path.join(HERE, "perf_model.json"))
    kernels(tk, os.path.join(HERE, "kernels.npz"))
    selection(tk, os.path.join(HERE, "selection.npz"))
    engine(tk, os.path.join(HERE, "engine.npz"))
    workload(tk, os.path.join(HERE, "workload.npz"))
    harness(tk, os.path.join(HERE, "harness.npz"))
    c1(src, os.path.join(HERE, "c1.npz"))
    for f in sorted(glob.glob(os.path.join(HERE, "*.npz"))):
        print(f, os.path.getsize(f))


if __name__ == "__main__":
    main()
