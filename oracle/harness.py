"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference harness's
accuracy metrics (/root/reference/pkg/src/tierkv/harness.py:59-192) and its
fp64 full-attention oracle (oracle.py:27-55).

Drives any engine through a workload with the reference's run_sequence
contract (engine.py:198-224): on_step(step_idx, layer_idx, inp, out,
layer_state) with out.output / out.dense_positions / out.store_positions and
layer_state.store.context.sizes() / .archive_size. Produces the per-head rows
[step, layer, head, ctx_size, store_attended, eps, retained_min, max_err,
mean_err, bound_gap] (harness.py:31-34, 147-160) and the summary of
MetricsReport.finalize (harness.py:65-80). The cost-model columns of the
per-step rows are not restated (they do not depend on the engine).
"""

from __future__ import annotations

import numpy as np


def full_attention_oracle(q, keys, values, scale):
    """oracle.py:27-55: exact f64 softmax attention over the whole history ->
    (output [h, nq, d], lse [h, nq], weights [h, nq, n])."""
    q = np.asarray(q, dtype=np.float64)
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    h, nq, d = q.shape
    if keys.shape[1] == 0:
        return np.zeros((h, nq, d)), np.full((h, nq), -np.inf), np.zeros((h, nq, 0))
    scores = scale * (q @ keys.transpose(0, 2, 1))
    m = scores.max(axis=2, keepdims=True)
    e = np.exp(scores - m)
    z = e.sum(axis=2, keepdims=True)
    w = e / z
    return w @ values, m[:, :, 0] + np.log(z[:, :, 0]), w


class MetricsProbe:
    """harness.py:101-192 for one run: per-layer history, running max|V| and
    the per-head metric rows."""

    def __init__(self, layers, heads, head_dim, total_entries, scale):
        self.scale = scale
        self.keys = [np.empty((heads, total_entries, head_dim)) for _ in range(layers)]
        self.values = [np.empty((heads, total_entries, head_dim)) for _ in range(layers)]
        self.v_absmax = [np.zeros((heads, head_dim)) for _ in range(layers)]
        self.lengths = [0] * layers
        self.heads = heads
        self.rows = []

    def _extend(self, layer, keys, values):
        n = keys.shape[1]
        lo = self.lengths[layer]
        self.keys[layer][:, lo:lo + n] = keys
        self.values[layer][:, lo:lo + n] = values
        self.v_absmax[layer] = np.maximum(self.v_absmax[layer], np.abs(values.astype(np.float64)).max(axis=1))
        self.lengths[layer] += n
        return self.lengths[layer]

    def on_step(self, step_idx, layer_idx, inp, out, layer_state):
        """harness.py:135-160."""
        n = self._extend(layer_idx, np.asarray(inp.keys), np.asarray(inp.values))
        o_out, _, o_w = full_attention_oracle(inp.q, self.keys[layer_idx][:, :n], self.values[layer_idx][:, :n],
                                              self.scale)
        err = np.abs(np.asarray(out.output).astype(np.float64) - o_out)
        v_absmax = self.v_absmax[layer_idx]
        ctx_sizes = layer_state.store.context.sizes()
        store_pos = out.store_positions
        for h in range(self.heads):
            attended = np.concatenate([out.dense_positions, store_pos[h]])
            retained_rows = o_w[h][:, attended].sum(axis=1)
            eps_rows = np.maximum(1.0 - retained_rows, 0.0)
            bound = 2.0 * eps_rows[:, None] * v_absmax[h][None, :]
            gap = float((err[h] - bound).max())
            self.rows.append([step_idx, layer_idx, h, ctx_sizes[h], store_pos[h].size, float(eps_rows.max()),
                              float(retained_rows.min()), float(err[h].max()), float(err[h].mean()), gap])

    def summary(self, bound_slack=1e-5):
        """MetricsReport.finalize (harness.py:65-80)."""
        head = np.array([[r[5], r[6], r[7], r[9]] for r in self.rows], dtype=np.float64)
        eps, retained, max_err, gap = head.T
        return {
            "steps": int(max(r[0] for r in self.rows)) + 1 if self.rows else 0,
            "max_err": float(max_err.max()),
            "p95_err": float(np.percentile(max_err, 95)),
            "mean_eps": float(eps.mean()),
            "max_eps": float(eps.max()),
            "bound_violations": int((gap > bound_slack).sum()),
            "worst_bound_gap": float(gap.max()),
            "mass_accounting_err": float(np.abs(retained + eps - 1.0).max()),
            "mean_ctx_size": float(np.mean([r[3] for r in self.rows])),
        }


class _PortStore:
    """StoreTier read API over an oracle port engine (archive index == position)."""

    def __init__(self, eng):
        self._eng = eng

    @property
    def archive_size(self):
        return self._eng.archive_size

    @property
    def context(self):
        return self

    def sizes(self):
        return [int(c.size) for c in self._eng.context]


class _PortLayer:
    def __init__(self, eng):
        self.store = _PortStore(eng)


class _PortOut:
    def __init__(self, r, dense_positions, store_positions):
        self.output, self.lse = r.output, r.lse
        self.dense_positions, self.store_positions = dense_positions, store_positions


class _Inp:
    def __init__(self, mode, q, keys, values):
        self.mode, self.q, self.keys, self.values = mode, q, keys, values


def run_port_sequence(engines, steps, on_step):
    """run_sequence (engine.py:198-224) over one oracle port engine per layer."""
    for step_idx, s in enumerate(steps):
        for li, eng in enumerate(engines):
            lo, nxt = eng.lo, eng.nxt
            r = eng.step(s.mode, s.q[li], s.keys[li], s.values[li])
            dense = np.arange(lo, nxt + s.n_q, dtype=np.int64)
            store = [np.asarray(e, np.int64) for e in r.store_entries]
            on_step(step_idx, li, _Inp(s.mode, s.q[li], s.keys[li], s.values[li]), _PortOut(r, dense, store),
                    _PortLayer(eng))
