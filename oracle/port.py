"""TEST INFRASTRUCTURE ONLY — CPU restatement of the reference hot path.

This module is the parity oracle and the CPU-baseline leg. Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import it; the product package never does.

What it restates (reference = /root/reference/pkg/src/tierkv):
  * the attention loops  -> oracle/hgca_oracle.c (C, same loop order as
    _core.pyx:22-150), or the reference's own compiled _core from oracle/_ref
    (kernels="reference");
  * merge_states           attention.py:153-188
  * select_salient         sparsifier.py:32-42
  * pack_head_groups       sparsifier.py:198-235
  * WindowCache arithmetic kv_cache.py:171-221 (update_maw, evict_if_full),
    kv_cache.py:122-169 (append_kv)
  * StoreTier              sparsifier.py:127-177 (ingest_evicted, reevaluate)
  * HybridEngine._run_step engine.py:116-195
over flat arrays: one [H, T, d] buffer per tensor holding every position, the
archive being positions [0, lo) and the window [lo, nxt). Because the
reference's archive is position-ordered from position 0 and its window blocks
start at multiples of blk_size, archive index == position and this layout is a
re-indexing of the reference's deque-of-blocks, not a change of algorithm.

Extensions the reference does not define, with the adapters
named there: batch B = B independent engines with EngineConfig(batch=B);
GQA = KV expanded per query head (q-head h reads kv-head h // (Hq/Hkv));
bf16 = the bf16-rounded values upcast to fp32; topk(k) = the first k entries of
the (-maw, +position) lexsort order used by the padding rule
(sparsifier.py:219-226).
"""

from __future__ import annotations

import ctypes
import glob
import importlib.util
import math
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_REF_CORE = None


class OracleError(ValueError):
    """Mirror of tierkv.errors.ContractError (errors.py:1-2)."""


def lib():
    """The C restatement (oracle/_build/libhgca_oracle.so), built by `make -C oracle`."""
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "_build", "libhgca_oracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"oracle library missing: {path} (run make -C oracle)")
        L = ctypes.CDLL(path)
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        for name in ("or_attend_dense_f32", "or_attend_dense_f64"):
            f = getattr(L, name)
            f.argtypes = [P, P, P, I64, I64, I64, I64, D, I, P, P, P, I]
            f.restype = I
        for name in ("or_attend_indexed_f32", "or_attend_indexed_f64"):
            f = getattr(L, name)
            f.argtypes = [P, P, P, P, I64, I64, I64, D, I, P, P, P]
            f.restype = I
        f = L.or_attend_indexed_tasks_f32
        f.argtypes = [P, P, P, P, P, P, I64, I64, I64, D, I, P, P, P, P, I]
        f.restype = I
        _LIB = L
    return _LIB


def ref_core():
    """The reference's own compiled _core (oracle/_ref), or None if not built."""
    global _REF_CORE
    if _REF_CORE is None:
        hits = glob.glob(os.path.join(HERE, "_ref", "_core*.so"))
        if not hits:
            return None
        spec = importlib.util.spec_from_file_location("_core", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _REF_CORE = mod
    return _REF_CORE


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


# ---------------------------------------------------------------- kernels
def attend_dense(q, k, v, scale, keep_weights, threads=1, kernels="port"):
    """Backend contract of backends.py:8-20 / _core.pyx:22-84."""
    if kernels == "reference":
        core = ref_core()
        if core is None:
            raise RuntimeError("oracle/_ref not built")
        return core.attend_dense(q, k, v, float(scale), bool(keep_weights))
    q, k, v = (np.ascontiguousarray(a) for a in (q, k, v))
    dt = q.dtype
    H, nq, d = q.shape
    nkv = k.shape[1]
    out = np.zeros((H, nq, d), dt)
    lse = np.full((H, nq), -np.inf)
    w = np.zeros((H, nq, nkv), dt) if keep_weights else None
    if nkv == 0:
        return out, lse, w
    fn = lib().or_attend_dense_f32 if dt == np.float32 else lib().or_attend_dense_f64
    fn(_ptr(q), _ptr(k), _ptr(v), H, nq, nkv, d, float(scale), int(keep_weights),
       _ptr(out), _ptr(lse), _ptr(w), int(threads))
    return out, lse, w


def attend_indexed(q, k, v, idx, scale, keep_weights, kernels="port"):
    """Backend contract of _core.pyx:87-150 (single head)."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    if kernels == "reference":
        core = ref_core()
        if core is None:
            raise RuntimeError("oracle/_ref not built")
        return core.attend_indexed(q, k, v, idx, float(scale), bool(keep_weights))
    q, k, v = (np.ascontiguousarray(a) for a in (q, k, v))
    dt = q.dtype
    nq, d = q.shape
    n = idx.size
    out = np.zeros((nq, d), dt)
    lse = np.full(nq, -np.inf)
    w = np.zeros((nq, n), dt) if keep_weights else None
    if n == 0:
        return out, lse, w
    fn = lib().or_attend_indexed_f32 if dt == np.float32 else lib().or_attend_indexed_f64
    fn(_ptr(q), _ptr(k), _ptr(v), _ptr(idx), n, nq, d, float(scale), int(keep_weights),
       _ptr(out), _ptr(lse), _ptr(w))
    return out, lse, w


def merge_states(out_a, lse_a, out_b, lse_b):
    """attention.py:153-188 (outputs only; weight-row concat not needed here)."""
    lse_a = np.asarray(lse_a, dtype=np.float64)
    lse_b = np.asarray(lse_b, dtype=np.float64)
    m = np.maximum(lse_a, lse_b)
    both_empty = np.isneginf(m)
    m_safe = np.where(both_empty, 0.0, m)
    wa = np.exp(lse_a - m_safe)
    wb = np.exp(lse_b - m_safe)
    z = wa + wb
    z_safe = np.where(both_empty, 1.0, z)
    lse = np.where(both_empty, -np.inf, m_safe + np.log(z_safe))
    dtype = np.result_type(out_a, out_b)
    ca = (wa / z_safe).astype(dtype)[..., None]
    cb = (wb / z_safe).astype(dtype)[..., None]
    out = ca * out_a.astype(dtype, copy=False) + cb * out_b.astype(dtype, copy=False)
    return out, lse


# ---------------------------------------------------------------- selection
def select_salient(maw, beta, divisor):
    """sparsifier.py:32-42: strict maw > beta/divisor, per-head sorted int64."""
    if divisor < 1:
        raise OracleError(f"divisor must be >= 1, got {divisor}")
    maw = np.asarray(maw, dtype=np.float64)
    threshold = beta / divisor
    return [np.nonzero(row > threshold)[0].astype(np.int64) for row in maw]


def topk_order(maw_row, cand):
    """(-maw, +position) order of candidate entries (sparsifier.py:224-225)."""
    return cand[np.lexsort((cand, -maw_row[cand]))]


def select_topk(maw, k):
    """F1 extension: per head the first k entries of the padding order, sorted."""
    maw = np.asarray(maw, dtype=np.float64)
    out = []
    for row in maw:
        cand = np.arange(row.size, dtype=np.int64)
        out.append(np.sort(topk_order(row, cand)[:k]).astype(np.int64))
    return out


def group_size(batch, heads, core_count):
    """sparsifier.py:209."""
    return max(1, int(batch * heads / core_count + 0.5))


def pack_head_groups(context, maw, archive_size, batch, core_count):
    """sparsifier.py:198-235. context: per-head sorted int64 index arrays.

    Returns per head (entries, padding flags), grouped exactly like the
    reference (the grouping only decides each head's padding target)."""
    if core_count < 1:
        raise OracleError(f"core_count must be >= 1, got {core_count}")
    h = len(context)
    g = group_size(batch, h, core_count)
    entries, padding = [None] * h, [None] * h
    for lo in range(0, h, g):
        heads = list(range(lo, min(lo + g, h)))
        target = max((context[hd].size for hd in heads), default=0)
        for hd in heads:
            idx = context[hd]
            need = target - idx.size
            pad_idx = np.zeros(0, np.int64)
            if need > 0:
                mask = np.ones(archive_size, dtype=bool)
                mask[idx] = False
                cand = np.nonzero(mask)[0]
                if cand.size:
                    order = np.lexsort((cand, -maw[hd, cand]))
                    pad_idx = cand[order[:need]].astype(np.int64)
            merged = np.concatenate([idx, pad_idx])
            sort = np.argsort(merged, kind="stable")
            flags = np.concatenate([np.zeros(idx.size, bool), np.ones(pad_idx.size, bool)])
            entries[hd] = merged[sort]
            padding[hd] = flags[sort]
    return entries, padding


# ---------------------------------------------------------------- engine
@dataclass
class OracleStep:
    output: np.ndarray       # [H, nq, d] f32
    lse: np.ndarray          # [H, nq] f64
    a_gpu: np.ndarray        # [H, nq, w + nq] f32
    store_entries: list      # per head attended archive indices
    a_cpu: list              # per head [nq, n_h] f32 weights
    s_out: np.ndarray = None  # sparse partial [H, nq, d] f32
    s_lse: np.ndarray = None  # sparse partial lse [H, nq] f64


class OracleEngine:
    """One layer of engine.py's HybridEngine over flat position-indexed arrays.

    Single sequence, MHA heads, fp32 storage (kv_cache.py:73-75,
    sparsifier.py:117-118). max_len bounds the total positions.
    """

    def __init__(self, heads, head_dim, blk_num, blk_size, alpha=0.5, beta=1.0,
                 core_count=8, batch=1, scale=None, max_len=4096, kernels="port",
                 threads=1, selection="threshold", topk=0, shard=(0, 1)):
        if blk_num < 2 or blk_size < 1:
            raise OracleError("bad cache geometry")
        self.H, self.d = heads, head_dim
        self.blk_num, self.blk_size = blk_num, blk_size
        self.cap = blk_num * blk_size
        self.alpha, self.beta = float(alpha), float(beta)
        self.core_count, self.batch = core_count, batch
        self.scale = 1.0 / math.sqrt(head_dim) if scale is None else float(scale)
        self.kernels, self.threads = kernels, threads
        self.selection, self.topk = selection, topk
        # sequence sharding (not in the reference): this
        # engine selects only archive blocks j with j % world == rank
        self.shard_rank, self.shard_world = shard
        self.keys = np.zeros((heads, max_len, head_dim), np.float32)
        self.values = np.zeros((heads, max_len, head_dim), np.float32)
        self.maw = np.zeros((heads, max_len), np.float64)
        self.context = [np.zeros(0, np.int64) for _ in range(heads)]
        self.lo = 0    # archive = [0, lo), window = [lo, nxt)
        self.nxt = 0

    @property
    def window_size(self):
        return self.nxt - self.lo

    @property
    def archive_size(self):
        return self.lo

    # -- store tier (sparsifier.py:127-177) --
    def _ingest(self, lo, hi, divisor):
        """ingest_evicted of positions [lo, hi) at beta/divisor."""
        if self.selection == "topk":
            self._select_topk_all(hi)
            return
        picked = select_salient(self.maw[:, lo:hi], self.beta, divisor)
        for h in range(self.H):
            p = self._owned(picked[h] + lo)
            if p.size:
                self.context[h] = np.sort(np.concatenate([self.context[h], p]))

    def _owned(self, pos):
        if self.shard_world == 1:
            return pos
        return pos[(pos // self.blk_size) % self.shard_world == self.shard_rank]

    def _select_topk_all(self, n):
        self.context = select_topk(self.maw[:, :n], min(self.topk, n))

    def _reevaluate(self, a_cpu_mean):
        """sparsifier.py:158-177."""
        n = self.lo
        if n == 0:
            return
        self.maw[:, :n] = a_cpu_mean
        if self.selection == "topk":
            self._select_topk_all(n)
            return
        self.context = [self._owned(c) for c in select_salient(self.maw[:, :n], self.beta, n)]

    def bulk_ingest(self, keys, values, maw, divisor):
        """Archive positions [nxt, nxt+n) directly (one ingest_evicted call
        with a single divisor, sparsifier.py:127-156); used to stage long
        contexts. keys/values [H, n, d], maw [H, n]. Window must be empty."""
        if self.window_size:
            raise OracleError("bulk_ingest requires an empty window")
        n = keys.shape[1]
        lo = self.nxt
        self.keys[:, lo:lo + n] = keys
        self.values[:, lo:lo + n] = values
        self.maw[:, lo:lo + n] = maw
        self.nxt += n
        self.lo = self.nxt
        self._ingest(lo, lo + n, divisor)

    def sparse_entries(self):
        """Per-head attended archive entries in decode mode (engine.py:139)."""
        entries, _ = pack_head_groups(self.context, self.maw, self.lo, self.batch, self.core_count)
        return entries

    # -- engine.py:151-195 --
    def step(self, mode, q, k, v):
        q = np.ascontiguousarray(q, np.float32)
        k = np.ascontiguousarray(k, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        H, nq, d = q.shape
        if mode == "decode" and nq != 1:
            raise OracleError("decode steps take exactly one query row")
        lo, nxt = self.lo, self.nxt
        w_size = nxt - lo
        kr = self.kernels
        # 1. sparse partial (engine.py:116-149)
        if lo == 0:
            s_out = np.zeros((H, nq, d), np.float32)
            s_lse = np.full((H, nq), -np.inf)
            a_cpu = [np.zeros((nq, 0), np.float32) for _ in range(H)]
            entries = [np.zeros(0, np.int64) for _ in range(H)]
        elif mode == "append":
            s_out, s_lse, wts = attend_dense(q, self.keys[:, :lo], self.values[:, :lo],
                                             self.scale, True, self.threads, kr)
            a_cpu = [wts[h] for h in range(H)]
            entries = [np.arange(lo, dtype=np.int64) for _ in range(H)]
        else:
            entries = self.sparse_entries()
            s_out = np.zeros((H, nq, d), np.float32)
            s_lse = np.full((H, nq), -np.inf)
            a_cpu = [None] * H
            if kr == "port" and self.threads > 1:
                self._sparse_tasks(q, entries, s_out, s_lse, a_cpu)
            else:
                for h in range(H):
                    o, l, w = attend_indexed(q[h], self.keys[h, :lo], self.values[h, :lo],
                                             entries[h], self.scale, True, kr)
                    s_out[h], s_lse[h], a_cpu[h] = o, l, w
        # 2. dense over window + kv_in (engine.py:161-164)
        dk = np.concatenate([self.keys[:, lo:nxt], k], axis=1)
        dv = np.concatenate([self.values[:, lo:nxt], v], axis=1)
        d_out, d_lse, a_gpu = attend_dense(q, dk, dv, self.scale, True, self.threads, kr)
        # 3. merge (engine.py:166-169)
        out, lse = merge_states(s_out, s_lse, d_out, d_lse)
        # 4. maintenance (engine.py:175-186)
        a_mean = a_gpu.mean(axis=1, dtype=np.float64)
        if w_size:
            self.maw[:, lo:nxt] = (1.0 - self.alpha) * self.maw[:, lo:nxt] + self.alpha * a_mean[:, :w_size]
        ev_lo, ev_hi = self._evict_if_full(nq)
        if mode == "append" and lo:
            a_cpu_mean = np.stack([w.mean(axis=0, dtype=np.float64) for w in a_cpu])
            self._reevaluate(a_cpu_mean)
        if ev_hi > ev_lo:
            self.lo = ev_hi
            self._ingest(ev_lo, ev_hi, w_size + nq)
        # append_kv (kv_cache.py:122-169)
        if self.window_size + nq > self.cap:
            raise OracleError("append overflows window capacity")
        if self.nxt + nq > self.keys.shape[1]:
            raise OracleError("max_len exceeded")
        self.keys[:, self.nxt:self.nxt + nq] = k
        self.values[:, self.nxt:self.nxt + nq] = v
        self.maw[:, self.nxt:self.nxt + nq] = a_mean[:, w_size:]
        self.nxt += nq
        return OracleStep(out, lse, a_gpu, entries, a_cpu, s_out, s_lse)

    def _evict_if_full(self, incoming):
        """kv_cache.py:189-221 -> evicted position range [lo, lo + freed)."""
        if incoming > self.cap:
            raise OracleError("a single step exceeds the whole window")
        size = self.nxt - self.lo
        l_cur = size + incoming
        if l_cur < self.cap:
            return self.lo, self.lo
        n_blocks = math.ceil((l_cur - self.cap + 1) / self.blk_size)
        full_blocks = size // self.blk_size
        n_blocks = min(n_blocks, full_blocks)
        freed = n_blocks * self.blk_size
        if self.cap - (size - freed) < incoming:
            raise OracleError("cannot free room for the incoming entries")
        return self.lo, self.lo + freed

    def _sparse_tasks(self, q, entries, s_out, s_lse, a_cpu):
        """Same per-head attend_indexed loops, heads spread over threads."""
        H, nq, d = q.shape
        lo = self.lo
        T = self.keys.shape[1]
        kv_off = np.arange(H, dtype=np.int64) * T
        sizes = np.array([e.size for e in entries], np.int64)
        idx_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        idx_cat = np.concatenate(entries).astype(np.int64) if H else np.zeros(0, np.int64)
        w_off = idx_off * nq
        wts = np.zeros(max(int(w_off[-1]), 1), np.float32)
        lib().or_attend_indexed_tasks_f32(
            _ptr(q), _ptr(self.keys), _ptr(self.values), _ptr(kv_off), _ptr(idx_cat),
            _ptr(idx_off), H, nq, d, self.scale, 1, _ptr(s_out), _ptr(s_lse), _ptr(wts),
            _ptr(w_off), int(self.threads))
        for h in range(H):
            a_cpu[h] = wts[w_off[h]:w_off[h + 1]].reshape(nq, sizes[h])
        del lo


def merge_packed(outs, lses):
    """P-way fold of sharded partials in rank order, restating the product's
    hgca_merge_packed arithmetic (max, sum of exp(lse - M), weighted mean in
    fp64, fp32 output). outs [P, rows, d] f32, lses [P, rows] f64."""
    outs = np.asarray(outs, np.float32)
    lses = np.asarray(lses, np.float64)
    P, rows, d = outs.shape
    M = lses.max(axis=0)
    empty = M == -np.inf
    Ms = np.where(empty, 0.0, M)
    w = np.exp(lses - Ms[None])
    w[:, empty] = 0.0
    Z = np.zeros(rows)
    acc = np.zeros((rows, d))
    for p in range(P):
        Z = Z + w[p]
        acc = acc + w[p][:, None] * outs[p].astype(np.float64)
    Zs = np.where(empty, 1.0, Z)
    out = np.where(empty[:, None], 0.0, acc / Zs[:, None]).astype(np.float32)
    lse = np.where(empty, -np.inf, Ms + np.log(Zs))
    return out, lse


def expand_gqa(x, q_heads):
    """GQA adapter: [..., Hkv, n, d] -> [..., Hq, n, d]."""
    hkv = x.shape[-3]
    return np.repeat(x, q_heads // hkv, axis=-3)


def bf16_round(x):
    """Round fp32 values to bf16 (nearest-even) and return them as fp32."""
    a = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0x7FFF + ((a >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(np.shape(x))
