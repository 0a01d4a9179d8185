"""TEST INFRASTRUCTURE ONLY — the reference's CPU hot path, timed for
bench.py's cpu_baseline leg and its `--impl reference` arm.

One sequence's decode layer-step exactly as the reference executes it
(engine.py:134-169): per query head one attend_indexed over that head's
selected archive entries (engine.py:139-148), one stacked-head attend_dense
over the window plus the new entry (engine.py:161-164), then merge_states
(attention.py:153-188), plus the MAW EMA of the window (kv_cache.py:186).
The attention loops are the reference's own compiled core (oracle/_ref, built
from /root/reference/pkg/src/tierkv/_core.pyx) when present
(kind="reference"), else the C restatement (kind="port"). GQA uses the
SURVEY.md F8 adapter (query head h reads KV head h // G); bf16 workloads are
run on their bf16-rounded values upcast to float32 (F4).

The sample deliberately omits the reference's per-step pack_head_groups /
window gather / concatenation overheads (~35% of its step time, SURVEY.md
§3), so the CPU number is, if anything, favourable to the CPU.
"""

from __future__ import annotations

import math
import multiprocessing as mp
import os
import time

import numpy as np

from . import port

_SHARED = {}


def kind():
    return "reference" if port.ref_core() is not None else "port"


def make_sequence(Hq, Hkv, D, n_arch, W, frac, seed):
    """Synthetic single-sequence state shaped like one batch element of C2."""
    rng = np.random.default_rng(seed)
    K = port.bf16_round(rng.standard_normal((Hkv, n_arch + W, D), dtype=np.float32))
    V = port.bf16_round(rng.standard_normal((Hkv, n_arch + W, D), dtype=np.float32))
    q = port.bf16_round(rng.standard_normal((Hq, D), dtype=np.float32))
    sel = [np.sort(np.nonzero(rng.random(n_arch) < frac)[0]).astype(np.int64) for _ in range(Hq)]
    maw = rng.random((Hq, W))
    return dict(K=K, V=V, q=q, sel=sel, maw=maw, n_arch=n_arch, W=W, Hq=Hq, Hkv=Hkv, D=D)


def sequence_step(s, kernels, h0=0, h1=None):
    """One reference hot-path layer-step for one sequence (query heads
    [h0, h1), default all); returns output."""
    Hq, Hkv, D, n, W = s["Hq"], s["Hkv"], s["D"], s["n_arch"], s["W"]
    h1 = Hq if h1 is None else h1
    G = Hq // Hkv
    scale = 1.0 / math.sqrt(D)
    K, V, q = s["K"], s["V"], s["q"]
    H = h1 - h0
    s_out = np.zeros((H, 1, D), np.float32)
    s_lse = np.full((H, 1), -np.inf)
    for h in range(h0, h1):
        o, l, _ = port.attend_indexed(q[h][None], K[h // G, :n], V[h // G, :n], s["sel"][h], scale, True,
                                      kernels=kernels)
        s_out[h - h0], s_lse[h - h0] = o, l
    heads = np.arange(h0, h1) // G
    kw = np.ascontiguousarray(K[heads, n:n + W])
    vw = np.ascontiguousarray(V[heads, n:n + W])
    d_out, d_lse, a_gpu = port.attend_dense(q[h0:h1, None], kw, vw, scale, True, kernels=kernels)
    out, lse = port.merge_states(s_out, s_lse, d_out, d_lse)
    a_mean = a_gpu.mean(axis=1, dtype=np.float64)
    s["maw"][h0:h1] = 0.5 * s["maw"][h0:h1] + 0.5 * a_mean
    return out


def _worker(args):
    idx, kernels, h0, h1 = args
    s = _SHARED["seqs"][idx % len(_SHARED["seqs"])]
    t0 = time.perf_counter()
    sequence_step(s, kernels, h0, h1)
    return time.perf_counter() - t0


def time_single(Hq, Hkv, D, n_arch, W, frac, sequences=2, reps=2, seed=0):
    """cpu_baseline: sequences x reps single-threaded layer-steps; tokens/s."""
    kernels = kind()
    s = make_sequence(Hq, Hkv, D, n_arch, W, frac, seed)
    sequence_step(s, kernels)  # warm caches / page in
    t0 = time.perf_counter()
    for _ in range(reps):
        for _ in range(sequences):
            sequence_step(s, kernels)
    dt = time.perf_counter() - t0
    return dict(value=sequences * reps / dt, unit="tokens/s", cores=1, kind=kernels,
                sample=f"{sequences} sequence(s) x {reps} rep(s) of one decode layer-step "
                       f"(Hq={Hq}, Hkv={Hkv}, d={D}, archive {n_arch}, window {W}, "
                       f"{frac:.0%} selected per head), 1 thread, {dt:.2f} s")


def pool_bench(Hq, Hkv, D, n_arch, W, frac, batch, steps, warmup, workers=None, seed=0):
    """--impl reference: all host cores. Each step runs the full batch: every
    sequence's layer-step split into per-head-group tasks (the reference's
    HeadGroupTask unit, sparsifier.py:90-102; each task runs the reference's
    own per-head loops), spread over a process pool so B * groups >= cores;
    returns per-step wall times."""
    kernels = kind()
    workers = workers or len(os.sched_getaffinity(0))
    groups = max(1, min(Hq, -(-workers // batch)))          # head groups per sequence
    bounds = np.linspace(0, Hq, groups + 1).astype(int)
    tasks = [(b, kernels, int(bounds[i]), int(bounds[i + 1])) for b in range(batch) for i in range(groups)
             if bounds[i + 1] > bounds[i]]
    _SHARED["seqs"] = [make_sequence(Hq, Hkv, D, n_arch, W, frac, seed + i) for i in range(batch)]
    ctx = mp.get_context("fork")
    times = []
    procs = min(workers, len(tasks))
    with ctx.Pool(processes=procs) as pool:
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_worker, tasks, chunksize=1)
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
    return dict(times=times, workers=procs, kind=kernels, tasks=len(tasks))
