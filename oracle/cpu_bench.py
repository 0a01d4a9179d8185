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


def sequence_step(s, kernels):
    """One reference hot-path layer-step for one sequence; returns output."""
    Hq, Hkv, D, n, W = s["Hq"], s["Hkv"], s["D"], s["n_arch"], s["W"]
    G = Hq // Hkv
    scale = 1.0 / math.sqrt(D)
    K, V, q = s["K"], s["V"], s["q"]
    s_out = np.zeros((Hq, 1, D), np.float32)
    s_lse = np.full((Hq, 1), -np.inf)
    for h in range(Hq):
        o, l, _ = port.attend_indexed(q[h][None], K[h // G, :n], V[h // G, :n], s["sel"][h], scale, True,
                                      kernels=kernels)
        s_out[h], s_lse[h] = o, l
    kw = np.repeat(K[:, n:n + W], G, axis=0)
    vw = np.repeat(V[:, n:n + W], G, axis=0)
    d_out, d_lse, a_gpu = port.attend_dense(q[:, None], kw, vw, scale, True, kernels=kernels)
    out, lse = port.merge_states(s_out, s_lse, d_out, d_lse)
    a_mean = a_gpu.mean(axis=1, dtype=np.float64)
    s["maw"] = 0.5 * s["maw"] + 0.5 * a_mean
    return out


def _worker(args):
    idx, kernels = args
    s = _SHARED["seqs"][idx % len(_SHARED["seqs"])]
    t0 = time.perf_counter()
    sequence_step(s, kernels)
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
    """--impl reference: all host cores, one process per sequence slot.
    Each step runs the full batch (B sequences) across the pool; returns
    per-step wall times."""
    kernels = kind()
    workers = workers or len(os.sched_getaffinity(0))
    n_seq = min(batch, workers)
    _SHARED["seqs"] = [make_sequence(Hq, Hkv, D, n_arch, W, frac, seed + i) for i in range(n_seq)]
    ctx = mp.get_context("fork")
    times = []
    with ctx.Pool(processes=min(workers, batch)) as pool:
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_worker, [(b, kernels) for b in range(batch)], chunksize=1)
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
    return dict(times=times, workers=min(workers, batch), kind=kernels)
