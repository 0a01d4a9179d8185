"""TEST INFRASTRUCTURE ONLY — restatement of the reference's synthetic
workload generator (/root/reference/pkg/src/tierkv/workload.py:124-182), so
parity tests and the bench can build the reference's Q/K/V streams on a box
without the reference installed. Same numpy Generator call order, so the
arrays are bit-identical to tierkv.gen_workload (pinned by
tests/test_oracle.py against tests/golden/workload_*.npz).

Frame per (layer, head): orthonormal (u, w);
  q_p = (lam p) u + w ; k_j = (lam j) w + noise ; sink k = u + noise ;
  i-th heavy hitter k = u + (i+1) ln(boost)/scale w + noise ; lam = ln(1/decay)/scale.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class WorkloadSpec:
    """workload.py:40-74 (defaults identical)."""

    seed: int = 0
    steps: int = 2048
    prefill_len: int = 128
    append_events: tuple = ()
    sink_count: int = 4
    heavy_hitter_count: int = 8
    heavy_hitter_boost: float = 0.75
    recency_decay: float = 0.98
    noise_scale: float = 0.05

    def __post_init__(self):
        object.__setattr__(self, "append_events",
                           tuple(sorted((int(s), int(n)) for s, n in self.append_events)))


@dataclass
class StepData:
    index: int
    mode: str
    start: int
    q: np.ndarray       # [layers, heads, n_q, head_dim] float32
    keys: np.ndarray
    values: np.ndarray

    @property
    def n_q(self):
        return self.q.shape[2]


def step_lengths(spec):
    """workload.py:111-121."""
    events = dict(spec.append_events)
    lengths = []
    if spec.prefill_len:
        lengths.append(("append", spec.prefill_len))
    for s in range(spec.steps):
        lengths.append(("append", events[s]) if s in events else ("decode", 1))
    return lengths


def gen_streams(spec, heads, head_dim, scale, layers):
    """Full [layers, heads, total, d] float32 q / k / v streams (workload.py:128-169)."""
    rng = np.random.default_rng(spec.seed)
    plan = step_lengths(spec)
    total = sum(n for _, n in plan)
    h, d = heads, head_dim
    lam = math.log(1.0 / spec.recency_decay) / scale
    u_coeff = np.zeros(total, np.float64)
    w_coeff = lam * np.arange(total, dtype=np.float64)
    u_coeff[:min(spec.sink_count, total)] = 1.0
    w_coeff[:min(spec.sink_count, total)] = 0.0
    early_lo = spec.sink_count
    early_hi = max(early_lo + 1, total // 4)
    if (spec.heavy_hitter_count and spec.heavy_hitter_boost > 0
            and early_hi > early_lo and total > early_lo):
        pool = np.arange(early_lo, min(early_hi, total))
        count = min(spec.heavy_hitter_count, pool.size)
        hh_pos = np.sort(rng.choice(pool, size=count, replace=False))
        u_coeff[hh_pos] = 1.0
        w_coeff[hh_pos] = np.arange(1, count + 1) * math.log(spec.heavy_hitter_boost) / scale
    pos = np.arange(total, dtype=np.float64)
    keys = np.empty((layers, h, total, d), np.float32)
    queries = np.empty((layers, h, total, d), np.float32)
    values = rng.standard_normal((layers, h, total, d)).astype(np.float32)
    for li in range(layers):
        for hd in range(h):
            u = rng.standard_normal(d)
            u /= np.linalg.norm(u)
            w = rng.standard_normal(d)
            w -= (w @ u) * u
            w /= np.linalg.norm(w)
            noise = rng.standard_normal((total, d))
            noise -= np.outer(noise @ u, u)
            k = np.outer(u_coeff, u) + np.outer(w_coeff, w)
            keys[li, hd] = k + spec.noise_scale * noise
            queries[li, hd] = np.outer(lam * pos, u) + w
    return plan, queries, keys, values


def gen_workload(spec, heads, head_dim, scale, layers):
    """workload.py:124-182: list of StepData."""
    plan, queries, keys, values = gen_streams(spec, heads, head_dim, scale, layers)
    steps, cursor = [], 0
    for idx, (mode, n) in enumerate(plan):
        sl = slice(cursor, cursor + n)
        steps.append(StepData(idx, mode, cursor,
                              np.ascontiguousarray(queries[:, :, sl]),
                              np.ascontiguousarray(keys[:, :, sl]),
                              np.ascontiguousarray(values[:, :, sl])))
        cursor += n
    return steps
