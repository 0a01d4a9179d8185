"""Store-tier selection on the B200 (tierkv/sparsifier.py:32-42, 198-235).

Selections are kept on the device as per-head bit masks ([rows, words]
uint32, bit p = archive position p): the strict threshold rule fills a mask
in one pass, padding / top-k are a radix select over the fp64 MAW keyed by
(maw descending, position ascending), and index lists are a compaction of
the mask. The list-returning functions here keep the reference signatures.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._dev import as_device, device, stream_handle
from .errors import ContractError

__all__ = ["HeadGroupTask", "ContextCache", "StoreTier", "select_salient", "select_topk", "renormalize",
           "pack_head_groups", "group_size", "indices_to_mask", "mask_to_lists", "words_for"]


def words_for(n: int) -> int:
    return max(1, (int(n) + 31) // 32)


def group_size(batch: int, heads: int, core_count: int) -> int:
    """sparsifier.py:209."""
    return max(1, int(batch * heads / core_count + 0.5))


@dataclass
class HeadGroupTask:
    """sparsifier.py:90-102."""

    heads: list
    entries: list
    padding: list = field(default_factory=list)


def _maw_dev(maw):
    t, is_np = as_device(maw)
    t = t.to(torch.float64)
    if t.dim() != 2:
        raise ContractError(f"maw must be [num_heads, n], got {tuple(t.shape)}")
    return t.contiguous(), is_np


def ownership_words(words, blk_size, rank, world):
    """Position mask [words] uint32 of the archive blocks rank owns under
    block-cyclic sequence sharding: block j = positions [j*blk, (j+1)*blk)
    belongs to rank j % world."""
    pos = np.arange(words * 32, dtype=np.int64)
    own = ((pos // blk_size) % world == rank).astype(np.uint64)
    return (own.reshape(words, 32) << np.arange(32, dtype=np.uint64)).sum(axis=1).astype(np.uint32)


def threshold_mask(maw_t, beta, divisor, p0=0, p1=None, mask=None, assign=True):
    """Device mask of maw > beta/divisor over [p0, p1) (sparsifier.py:41-42)."""
    rows, n = maw_t.shape
    p1 = n if p1 is None else p1
    words = words_for(n)
    if mask is None:
        mask = torch.zeros((rows, words), dtype=torch.int32, device=maw_t.device)
    _lib.call("hgca_select_threshold", maw_t.data_ptr(), rows, maw_t.stride(0), p0, p1, float(beta),
              int(divisor), mask.data_ptr(), mask.shape[1], int(assign), None, stream_handle(maw_t.device))
    return mask


def mask_to_lists(mask_a, n, mask_b=None, want_flags=False):
    """Compact masks (a | b) over [0, n) into per-row ascending int64 lists."""
    rows = mask_a.shape[0]
    dev = mask_a.device
    idx = torch.empty((rows, max(n, 1)), dtype=torch.int64, device=dev)
    cnt = torch.zeros(rows, dtype=torch.int64, device=dev)
    flags = torch.empty((rows, max(n, 1)), dtype=torch.uint8, device=dev) if want_flags else None
    if rows:
        _lib.call("hgca_mask_to_indices", mask_a.data_ptr(), mask_b.data_ptr() if mask_b is not None else None,
                  rows, mask_a.shape[1], n, idx.data_ptr(), idx.shape[1],
                  flags.data_ptr() if flags is not None else None, cnt.data_ptr(), stream_handle(dev))
    cnt_h = cnt.cpu().numpy()
    idx_h = idx.cpu().numpy()
    lists = [idx_h[r, : cnt_h[r]].copy() for r in range(rows)]
    if not want_flags:
        return lists
    fl_h = flags.cpu().numpy().astype(bool)
    return lists, [fl_h[r, : cnt_h[r]].copy() for r in range(rows)]


def indices_to_mask(index_lists, n, dev=None):
    """Per-row index lists -> device bit mask [rows, words] (host packing)."""
    rows = len(index_lists)
    words = words_for(n)
    bits = np.zeros((rows, words * 32), dtype=bool)
    for r, idx in enumerate(index_lists):
        idx = np.asarray(idx.detach().cpu() if isinstance(idx, torch.Tensor) else idx, dtype=np.int64)
        if idx.size:
            bits[r, idx] = True
    packed = np.packbits(bits, axis=1, bitorder="little").view(np.uint32).view(np.int32)
    return torch.from_numpy(np.ascontiguousarray(packed)).to(dev or device())


def _out(lists, like_numpy, dev):
    if like_numpy:
        return [a.astype(np.int64) for a in lists]
    return [torch.from_numpy(a).to(dev) for a in lists]


def select_salient(maw, beta: float, divisor: int):
    """Per-head sorted int64 indices with maw > beta/divisor (sparsifier.py:32-42)."""
    if divisor < 1:
        raise ContractError(f"divisor must be >= 1, got {divisor}")
    maw_t, is_np = _maw_dev(maw)
    n = maw_t.shape[1]
    mask = threshold_mask(maw_t, beta, divisor)
    return _out(mask_to_lists(mask, n), is_np, maw_t.device)


def topk_mask(maw_t, k, n=None, exclude=None, out=None):
    """OR into `out` the top-k[row] of [0, n) by (maw desc, position asc), skipping `exclude`."""
    rows, ld = maw_t.shape
    n = ld if n is None else n
    dev = maw_t.device
    if out is None:
        out = torch.zeros((rows, words_for(ld)), dtype=torch.int32, device=dev)
    if not isinstance(k, torch.Tensor):
        k = torch.as_tensor(np.broadcast_to(np.asarray(k, dtype=np.int64), (rows,)).copy())
    k = k.to(device=dev, dtype=torch.int64).contiguous()
    if rows and n:
        _lib.call("hgca_select_topk", maw_t.data_ptr(), rows, maw_t.stride(0), n, k.data_ptr(),
                  exclude.data_ptr() if exclude is not None else None, out.data_ptr(), out.shape[1],
                  stream_handle(dev))
    return out


def select_topk(maw, k: int):
    """F1 extension: per head the k highest-MAW entries, ties by
    ascending position (the order of sparsifier.py:224-225), sorted."""
    maw_t, is_np = _maw_dev(maw)
    mask = topk_mask(maw_t, int(k))
    return _out(mask_to_lists(mask, maw_t.shape[1]), is_np, maw_t.device)


def pack_head_groups(store, batch: int, core_count: int) -> list:
    """sparsifier.py:198-235 on the device.

    `store` is duck-typed like the reference StoreTier: `.shape.num_heads`,
    `.context.indices` (per-head position-sorted lists), `.maw` [H, N] and
    `.archive_size`. Each head is padded up to its group's longest selection
    with its own highest-MAW below-threshold entries (ties by position).
    """
    if core_count < 1:
        raise ContractError(f"core_count must be >= 1, got {core_count}")
    h = store.shape.num_heads
    g = group_size(batch, h, core_count)
    n = int(store.archive_size)
    dev = device()
    if n == 0:
        empty = np.zeros(0, np.int64)
        return [HeadGroupTask(heads=list(range(lo, min(lo + g, h))),
                              entries=[empty.copy() for _ in range(lo, min(lo + g, h))],
                              padding=[np.zeros(0, bool) for _ in range(lo, min(lo + g, h))])
                for lo in range(0, h, g)]
    ctx = indices_to_mask(store.context.indices, n, dev)
    maw_t, _ = _maw_dev(store.maw)
    maw_t = maw_t[:, :n].contiguous()
    counts = torch.zeros(h, dtype=torch.int64, device=dev)
    _lib.call("hgca_popcount_rows", ctx.data_ptr(), h, ctx.shape[1], n, counts.data_ptr(), stream_handle(dev))
    need = torch.zeros(h, dtype=torch.int64, device=dev)
    _lib.call("hgca_group_need", counts.data_ptr(), 1, h, g, need.data_ptr(), stream_handle(dev))
    pad = topk_mask(maw_t, need, n=n, exclude=ctx)
    lists, flags = mask_to_lists(ctx, n, mask_b=pad, want_flags=True)
    tasks = []
    for lo in range(0, h, g):
        heads = list(range(lo, min(lo + g, h)))
        tasks.append(HeadGroupTask(heads=heads, entries=[lists[x] for x in heads],
                                   padding=[flags[x] for x in heads]))
    return tasks


def renormalize(weights):
    """sparsifier.py:45-55: weights / sum (float64); ValueError for an empty or
    all-zero set."""
    w, is_np = as_device(weights)
    w = w.to(torch.float64)
    total = float(w.sum()) if w.numel() else 0.0
    if w.numel() == 0 or total <= 0.0:
        raise ValueError("cannot renormalize an empty or all-zero weight set")
    out = w / total
    return out.cpu().numpy() if is_np else out


class ContextCache:
    """sparsifier.py:58-87: per-head salient subset of the archive -- sorted
    archive indices (host int64 arrays, the reference's type), their
    renormalized MAW (metadata only) and contiguous device copies of the
    selected keys / values."""

    def __init__(self, num_heads: int, head_dim: int):
        dev = device()
        self.num_heads = num_heads
        self.head_dim = head_dim
        self.indices = [np.zeros(0, np.int64) for _ in range(num_heads)]
        self.weights = [np.zeros(0, np.float64) for _ in range(num_heads)]
        self.keys = [torch.zeros((0, head_dim), dtype=torch.float32, device=dev) for _ in range(num_heads)]
        self.values = [torch.zeros((0, head_dim), dtype=torch.float32, device=dev) for _ in range(num_heads)]

    def sizes(self) -> list:
        return [int(idx.size) for idx in self.indices]

    def set_head(self, head: int, idx, archive_keys, archive_values, maw_source):
        """Replace one head's selection; renormalizes maw_source over idx."""
        idx = np.sort(np.asarray(idx.cpu() if isinstance(idx, torch.Tensor) else idx, dtype=np.int64))
        self.indices[head] = idx
        ti = torch.from_numpy(idx).to(archive_keys.device)
        self.keys[head] = archive_keys[head].index_select(0, ti).contiguous()
        self.values[head] = archive_values[head].index_select(0, ti).contiguous()
        sel = maw_source[head].index_select(0, ti.to(maw_source.device))
        if idx.size and float(sel.sum()) > 0.0:
            self.weights[head] = renormalize(sel.cpu().numpy())
        else:
            self.weights[head] = np.zeros(idx.size, np.float64)


class StoreTier:
    """sparsifier.py:105-195: per-layer archive of evicted KV blocks (device
    tensors keys / values [H, N, d] float32, maw [H, N] float64, host
    positions) plus the context cache. Selection runs on the device
    (hgca_select_threshold: strict maw > beta / divisor with an IEEE fp64
    divide)."""

    def __init__(self, shape, layer_id: int = 0):
        dev = device()
        self.shape = shape
        self.layer_id = layer_id
        h, d = shape.num_heads, shape.head_dim
        self.keys = torch.zeros((h, 0, d), dtype=torch.float32, device=dev)
        self.values = torch.zeros((h, 0, d), dtype=torch.float32, device=dev)
        self.maw = torch.zeros((h, 0), dtype=torch.float64, device=dev)
        self.positions = np.zeros(0, np.int64)
        self.context = ContextCache(h, d)

    @property
    def archive_size(self) -> int:
        return int(self.positions.size)

    def _picked(self, maw_t, beta, divisor):
        n = maw_t.shape[1]
        mask = threshold_mask(maw_t.contiguous(), beta, divisor)
        return mask_to_lists(mask, n)

    def ingest_evicted(self, blocks, beta: float, window_size: int) -> None:
        """sparsifier.py:127-156: archive the blocks (eviction order) and admit
        per head the entries with maw > beta / window_size."""
        if not blocks:
            return
        new_keys = torch.cat([b.keys[:, : b.occupancy] for b in blocks], dim=1)
        new_values = torch.cat([b.values[:, : b.occupancy] for b in blocks], dim=1)
        new_maw = torch.cat([b.maw[:, : b.occupancy] for b in blocks], dim=1)
        new_pos = np.concatenate([b.positions for b in blocks])
        if self.positions.size and new_pos[0] <= self.positions[-1]:
            raise ContractError(f"blocks out of eviction order: position {new_pos[0]} after {self.positions[-1]}")
        if window_size < 1:
            raise ContractError(f"divisor must be >= 1, got {window_size}")
        base = self.archive_size
        self.keys = torch.cat([self.keys, new_keys], dim=1)
        self.values = torch.cat([self.values, new_values], dim=1)
        self.maw = torch.cat([self.maw, new_maw], dim=1)
        self.positions = np.concatenate([self.positions, new_pos])
        picked = self._picked(new_maw, beta, window_size)
        for h in range(self.shape.num_heads):
            if picked[h].size == 0:
                continue
            merged = np.concatenate([self.context.indices[h], picked[h] + base])
            self.context.set_head(h, merged, self.keys, self.values, self.maw)

    def reevaluate(self, a_cpu, beta: float) -> None:
        """sparsifier.py:158-177: MAW := a_cpu [num_heads, archive_size]; the
        context becomes the entries passing beta / archive_size."""
        a, _ = as_device(a_cpu)
        a = a.to(torch.float64)
        if tuple(a.shape) != (self.shape.num_heads, self.archive_size):
            raise ContractError(f"a_cpu shape {tuple(a.shape)} != ({self.shape.num_heads}, {self.archive_size})")
        if self.archive_size == 0:
            return
        self.maw = a.clone().contiguous()
        picked = self._picked(self.maw, beta, self.archive_size)
        for h in range(self.shape.num_heads):
            self.context.set_head(h, picked[h], self.keys, self.values, self.maw)

    def context_dump(self, tasks=None) -> str:
        """sparsifier.py:179-195: per head, one line per archive entry."""
        padded = [set() for _ in range(self.shape.num_heads)]
        if tasks:
            for task in tasks:
                for h, entries, pad in zip(task.heads, task.entries, task.padding):
                    padded[h].update(np.asarray(entries)[np.asarray(pad, bool)].tolist())
        maw = self.maw.cpu().numpy()
        lines = []
        for h in range(self.shape.num_heads):
            selected = set(self.context.indices[h].tolist())
            for i in range(self.archive_size):
                lines.append(f"layer={self.layer_id} head={h} pos={self.positions[i]} maw={maw[h, i]:.6e} "
                             f"selected={int(i in selected)} padding={int(i in padded[h])}")
        return "\n".join(lines)
