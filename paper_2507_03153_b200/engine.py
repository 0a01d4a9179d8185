"""Device-resident hybrid two-tier decode engine (tierkv/engine.py on the B200).

HybridEngine keeps every tier in HBM and mirrors the reference step driver
(engine.py:87-195) with its configuration, step input/output types and
maintenance order, extended the way SURVEY.md F8 describes:
  * batch B = B lock-step sequences, each an independent reference engine
    built with EngineConfig(batch=B) (batch only feeds the padding group size);
  * grouped-query attention: `kv_heads` KV heads, query head h reading KV head
    h // (heads // kv_heads); MAW and selection stay per query head;
  * storage dtype float32 (the reference's working precision) or bfloat16.

HBM layout per layer (positions are absolute, so the window tier and the
store tier share one buffer and eviction is a pointer move, not a copy):
  KV         [B*Hkv, T, 2, D] storage dtype, K row then V row of each position
                              (one contiguous gather per selected entry);
                              archive = [0, lo), window = [lo, nxt)
  maw        [B*Hq, T]        float64 per (query head, position)     kv_cache.py:73-75
  ctx        [B*Hq, T/32]     context-cache membership bits          sparsifier.py:58-87
  sel        [B*Hq, T/32]     attended set = ctx | padding           sparsifier.py:198-235
  u_ent      [B*Hkv, T]       per-KV-head union of `sel`: position | query-head mask << 24
The decode step is one call of hgca_decode_step (dense window + sparse union
+ merge + MAW EMA); selection changes (ingest / re-evaluation) rebuild the
masks and the union with the selection kernels.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _lib
from ._dev import DTYPE_CODE, device, stream_handle
from .attention import HeadShape
from .errors import ContractError
from .kv_cache import CacheConfig, KvBlock
from .sparsifier import HeadGroupTask, group_size, mask_to_lists, ownership_words, topk_mask

__all__ = ["CacheConfig", "EngineConfig", "StepInput", "StepOutput", "LayerState", "HybridEngine", "WindowView",
           "StoreView", "run_sequence"]

MODES = ("decode", "append")


# Step-adaptive work items (hgca_union_build_items_w): items of small steps
# are shortened (down to one 32-row stage) so that the union and the window
# give every decode warp about HGCA_ITEMS_PER_WARP items (0.75 measured best
# once the window counts: 0.5 shortchanges mid-size steps, 1 small ones), and the dense window parts follow the
# same granularity at half length (the decode kernel reads it from item_off);
# big steps keep 256-row items. (An earlier A/B that shortened only the sparse items showed
# no gain -- profiles/r02_item_ab.txt: the 256-row dense items stayed the
# critical path of small steps.)
MIN_ITEM_ROWS = int(os.environ.get("HGCA_MIN_ITEM_ROWS", "32"))
# Split merge (hgca_decode_desc.merge_split): per-head item lists longer than
# MERGE_ITEMS are folded by ceil(items / MERGE_ITEMS) CTAs per query head (at
# most MERGE_SPLIT_MAX) whose partials the last one combines; the host takes
# the item counts from an asynchronous copy of each union rebuild's item table.
MERGE_ITEMS = int(os.environ.get("HGCA_MERGE_ITEMS", "96"))
MERGE_SPLIT_MAX = 8
COUNT_WINDOW = os.environ.get("HGCA_ITEMS_COUNT_WINDOW", "1") != "0"  # A/B knob: window in the item sizing
ITEMS_PER_WARP = float(os.environ.get("HGCA_ITEMS_PER_WARP", "0.75"))


def item_target(dtype: str, G: int, D: int, dev) -> int:
    """Sparse work items a union rebuild aims for: ITEMS_PER_WARP per decode
    warp (hgca_decode_config consumer warps x SMs), so small steps spread over
    the whole GPU while big steps keep long items (hgca_union_build_items)."""
    cfg = (ctypes.c_int64 * 5)()
    _lib.call("hgca_decode_config", DTYPE_CODE[torch.bfloat16 if dtype == "bfloat16" else torch.float32], D, G, cfg)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count if torch.device(dev).type == "cuda" else 148
    return int(ITEMS_PER_WARP * int(cfg[0]) * nsm)


def sparse_capacity(BK: int, T: int, max_rows: int, target: int) -> int:
    """Upper bound on sparse items (hgca_decode_step's partials check): fixed
    max_rows items (tail items of max_rows / 4) or adaptive ones."""
    return BK * (-(-4 * T // max_rows) + 2) + (5 * target + 2) // 3 + 5 * BK


def item_rows(dtype: str) -> tuple[int, int]:
    """(window rows per dense item, union rows per sparse item) of the decode
    kernel for a storage dtype (hgca_item_rows)."""
    out = (ctypes.c_int64 * 2)()
    _lib.call("hgca_item_rows", DTYPE_CODE[torch.bfloat16 if dtype == "bfloat16" else torch.float32], out)
    return int(out[0]), int(out[1])


@dataclass(frozen=True)
class EngineConfig:
    """config.py:24-51 plus the B200 extensions (kv_heads, dtype, max_positions,
    selection policy)."""

    layers: int = 2
    heads: int = 8
    head_dim: int = 64
    scale: float | None = None
    cache: CacheConfig = field(default_factory=lambda: CacheConfig(blk_num=8, blk_size=32))
    core_count: int = 8
    batch: int = 1
    seed: int = 0
    kv_heads: int | None = None       # None: = heads (the reference's 1:1 heads)
    dtype: str = "float32"            # storage: "float32" | "bfloat16"
    max_positions: int = 4096         # HBM capacity per sequence (positions)
    selection: str = "threshold"      # "threshold" (reference) | "topk" (F1 extension)
    topk: int = 0                     # entries per head for selection="topk"
    keep_weights: bool = False        # materialize a_gpu in StepOutput
    shard_rank: int = 0               # sequence sharding: this rank ...
    shard_world: int = 1              # ... of shard_world owns archive blocks j with j % world == rank

    def __post_init__(self):
        if self.layers < 1:
            raise ContractError(f"layers must be >= 1, got {self.layers}")
        if self.core_count < 1:
            raise ContractError(f"core_count must be >= 1, got {self.core_count}")
        if self.batch < 1:
            raise ContractError(f"batch must be >= 1, got {self.batch}")
        kvh = self.heads if self.kv_heads is None else self.kv_heads
        if kvh < 1 or self.heads % kvh or self.heads // kvh not in (1, 2, 4, 8):
            raise ContractError(f"heads/kv_heads must be 1, 2, 4 or 8 (heads={self.heads}, kv_heads={kvh})")
        if self.dtype not in ("float32", "bfloat16"):
            raise ContractError(f"dtype must be float32 or bfloat16, got {self.dtype}")
        if self.selection not in ("threshold", "topk"):
            raise ContractError(f"selection must be threshold or topk, got {self.selection}")
        if self.shard_world < 1 or not 0 <= self.shard_rank < self.shard_world:
            raise ContractError(f"bad shard {self.shard_rank}/{self.shard_world}")
        if self.shard_world > 1:
            # threshold selection is per entry, so it shards locally; padding and
            # top-k need a global order (an allreduce at ingest) -- not built yet
            if self.selection != "threshold":
                raise ContractError("sequence sharding supports threshold selection only")
            if group_size(self.batch, self.heads, self.core_count) != 1:
                raise ContractError("sequence sharding needs padding group size 1 (raise core_count)")

    @property
    def head_shape(self) -> HeadShape:
        return HeadShape(self.heads, self.head_dim, self.scale)

    @property
    def n_kv_heads(self) -> int:
        return self.heads if self.kv_heads is None else self.kv_heads

    def with_(self, **kw) -> "EngineConfig":
        return replace(self, **kw)


@dataclass
class StepInput:
    """engine.py:31-58. q [B, Hq, n_q, D] (or [Hq, n_q, D] when batch == 1);
    keys/values [B, Hkv, n_q, D] (or [Hkv, n_q, D]). numpy or torch."""

    mode: str
    q: object
    keys: object
    values: object

    def __post_init__(self):
        if self.mode not in MODES:
            raise ContractError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.q.ndim not in (3, 4):
            raise ContractError(f"q must be [(batch,) heads, n_q, head_dim], got {tuple(self.q.shape)}")
        if self.mode == "decode" and self.n_q != 1:
            raise ContractError(f"decode steps take exactly one query row, got {self.n_q}")
        if self.n_q < 1:
            raise ContractError("append steps take at least one query row")
        if tuple(self.keys.shape) != tuple(self.values.shape) or self.keys.shape[-2] != self.n_q \
                or self.keys.shape[-1] != self.q.shape[-1] or self.keys.ndim != self.q.ndim:
            raise ContractError("kv_in must align with q")

    @property
    def n_q(self) -> int:
        return int(self.q.shape[-2])


class StepOutput:
    """engine.py:61-78. Arrays come back in the caller's kind: numpy when the
    StepInput held numpy arrays (the reference's contract), device tensors
    otherwise.

      output  [B, Hq, n_q, D] float32 (or [Hq, n_q, D] when batch == 1)
      lse     [B, Hq, n_q] float64
      a_gpu   window-tier weights [B, Hq, n_q, W] (append steps, or decode
              with keep_weights), else None
      a_cpu   per (b*Hq + h) store-tier weight rows [n_q, n_h] over the
              attended entries (append: the whole archive; decode: context +
              padding, keep_weights only), else None
      dense_positions   window-tier positions attended (int64)
      store_positions   per (b*Hq + h) attended store positions (int64),
                        computed on first access from the selection the step
                        attended
    """

    __slots__ = ("output", "lse", "a_gpu", "a_cpu", "dense_positions", "_store", "_store_fn")

    def __init__(self, output, lse, a_gpu, a_cpu, dense_positions, store_positions=None, store_fn=None):
        self.output, self.lse, self.a_gpu, self.a_cpu = output, lse, a_gpu, a_cpu
        self.dense_positions = dense_positions
        self._store, self._store_fn = store_positions, store_fn

    @property
    def store_positions(self):
        if self._store is None and self._store_fn is not None:
            self._store = self._store_fn()
            self._store_fn = None
        return self._store


APPEND_MAX_NQ = 128  # queries per hgca_append_bf16 call (include/hgca_b200.h)


def _np(x):
    return x.detach().cpu().numpy() if isinstance(x, torch.Tensor) else x


class LayerState:
    """HBM-resident window + store tiers of one layer (see module docstring)."""

    def __init__(self, cfg: EngineConfig, T: int, dev, layer_id: int = 0):
        self.cfg, self.layer_id = cfg, layer_id
        B, Hq, Hkv, D = cfg.batch, cfg.heads, cfg.n_kv_heads, cfg.head_dim
        tdt = torch.bfloat16 if cfg.dtype == "bfloat16" else torch.float32
        self.KV = torch.zeros((B * Hkv, T, 2, D), dtype=tdt, device=dev)
        self.maw = torch.zeros((B * Hq, T), dtype=torch.float64, device=dev)
        words = T // 32
        self.ctx = torch.zeros((B * Hq, words), dtype=torch.int32, device=dev)
        self.sel = torch.zeros((B * Hq, words), dtype=torch.int32, device=dev)
        self.u_ent = torch.zeros((B * Hkv, T), dtype=torch.int32, device=dev)
        self.u_cnt = torch.zeros(B * Hkv, dtype=torch.int32, device=dev)
        self.item_off = torch.zeros(2 * (B * Hkv + 1) + 1, dtype=torch.int32, device=dev)
        self.sparse_rows = item_rows(cfg.dtype)[1]   # the longest sparse item; shorter when the union is small
        self.item_target = item_target(cfg.dtype, Hq // Hkv, D, dev)
        self.item_tab = torch.zeros((sparse_capacity(B * Hkv, T, self.sparse_rows, self.item_target), 4),
                                    dtype=torch.int32, device=dev)
        self.lo = 0    # archive size
        self.nxt = 0   # next position
        self.desc = None  # cached hgca_decode_desc (engine-owned)
        self.merge_split = 1       # CTAs per query head in the merge kernel (split merge)
        self.off_host = None       # pinned copy of the item table offsets of the last union rebuild
        self.off_event = None      # ... and the event that says it has landed
        self.state = None  # graph mode: device step state {dlo, dhi, epoch, arrivals} (DecodeGraph)
        self.state_mirror = None  # (dlo, dhi) the device state holds, as far as the host knows
        self.keep = None
        if cfg.shard_world > 1:
            # ownership bits: archive block j (positions [j*blk, (j+1)*blk)) lives on rank j % world
            bits = ownership_words(words, cfg.cache.blk_size, cfg.shard_rank, cfg.shard_world)
            self.keep = torch.from_numpy(bits.view(np.int32)).to(dev)

    def rows(self):
        """Logical [B*Hkv, T, 2, D] copy of KV, whose rows are stored
        position-rotated: 16-byte chunk c of the row pair of position p at
        chunk (c & ~7) | ((c ^ p) & 7) (hgca_write_rows)."""
        BH, T, _, D = self.KV.shape
        epc = 16 // self.KV.element_size()   # elements per 16-byte chunk
        ch = 2 * D // epc
        c = torch.arange(ch, device=self.KV.device)
        p = torch.arange(T, device=self.KV.device)
        phys = (c[None, :] & ~7) | ((c[None, :] ^ p[:, None]) & 7)          # [T, ch]
        flat = self.KV.view(BH, T, ch, epc)
        idx = phys[None, :, :, None].expand(BH, T, ch, epc)
        return torch.gather(flat, 2, idx).view(BH, T, 2, D)

    @property
    def K(self):
        return self.rows()[:, :, 0]

    @property
    def V(self):
        return self.rows()[:, :, 1]

    @property
    def window_size(self):
        return self.nxt - self.lo

    @property
    def archive_size(self):
        return self.lo

    @property
    def window(self) -> "WindowView":
        """The reference's LayerState.window (engine.py:81-84): WindowCache read API."""
        return WindowView(self)

    @property
    def store(self) -> "StoreView":
        """The reference's LayerState.store (engine.py:81-84): StoreTier read API."""
        return StoreView(self)


class WindowView:
    """WindowCache's read API (kv_cache.py:102-255) over one layer's window
    tier, positions [lo, nxt) of the engine's HBM buffer. K/V rows are
    (b*Hkv + kv-head), MAW rows (b*Hq + h); with batch 1 and kv_heads == heads
    the shapes are the reference's [num_heads, ...]. Mutation goes through
    HybridEngine.step, which keeps the tiers consistent."""

    def __init__(self, ls: LayerState):
        self._ls = ls
        self.layer_id = ls.layer_id
        self.config = ls.cfg.cache

    @property
    def shape(self):
        return self._ls.cfg.head_shape

    @property
    def capacity(self) -> int:
        return self.config.capacity

    @property
    def size(self) -> int:
        return self._ls.window_size

    @property
    def next_position(self) -> int:
        return self._ls.nxt

    @property
    def blocks(self) -> list:
        """KvBlocks (float32 device copies) of the window, oldest first."""
        ls, blk = self._ls, self.config.blk_size
        rows = ls.rows()
        out = []
        for start in range(ls.lo, ls.nxt, blk):
            occ = min(blk, ls.nxt - start)
            kv = rows[:, start:start + blk].float()
            if kv.shape[1] < blk:
                kv = torch.cat([kv, kv.new_zeros((kv.shape[0], blk - kv.shape[1]) + tuple(kv.shape[2:]))], dim=1)
            maw = ls.maw[:, start:start + blk]
            if maw.shape[1] < blk:
                maw = torch.cat([maw, maw.new_zeros((maw.shape[0], blk - maw.shape[1]))], dim=1)
            out.append(KvBlock(keys=kv[:, :, 0].contiguous(), values=kv[:, :, 1].contiguous(), maw=maw.clone(),
                               start=start, occupancy=occ))
        return out

    def gather(self):
        """kv_cache.py:223-230: ([rows, size, D], [rows, size, D]) float32 device copies."""
        ls = self._ls
        kv = ls.rows()[:, ls.lo:ls.nxt].float()
        return kv[:, :, 0].contiguous(), kv[:, :, 1].contiguous()

    def maw_matrix(self) -> np.ndarray:
        ls = self._ls
        return ls.maw[:, ls.lo:ls.nxt].cpu().numpy()

    def positions(self) -> np.ndarray:
        return np.arange(self._ls.lo, self._ls.nxt, dtype=np.int64)

    def dump(self) -> str:
        """kv_cache.py:243-255."""
        ls, blk = self._ls, self.config.blk_size
        maw = self.maw_matrix()
        lines = []
        for i, start in enumerate(range(ls.lo, ls.nxt, blk)):
            occ = min(blk, ls.nxt - start)
            col = start - ls.lo
            mm = " ".join(f"{m:.6f}" for m in maw[:, col:col + occ].mean(axis=1))
            lines.append(f"layer={self.layer_id} block={i} pos={start}..{start + occ - 1} "
                         f"occ={occ}/{blk} maw_mean=[{mm}]")
        return "\n".join(lines)


class ContextView:
    """ContextCache's read API (sparsifier.py:58-87) over the engine's
    context-cache bitmask of one layer (rows b*Hq + h)."""

    def __init__(self, ls: LayerState):
        self._ls = ls
        self.num_heads = ls.ctx.shape[0]
        self.head_dim = ls.cfg.head_dim

    @property
    def indices(self) -> list:
        return mask_to_lists(self._ls.ctx, self._ls.lo)

    def sizes(self) -> list:
        ls = self._ls
        counts = torch.zeros(ls.ctx.shape[0], dtype=torch.int64, device=ls.ctx.device)
        if ls.lo:
            _lib.call("hgca_popcount_rows", ls.ctx.data_ptr(), ls.ctx.shape[0], ls.ctx.shape[1], ls.lo,
                      counts.data_ptr(), stream_handle(ls.ctx.device))
        return counts.cpu().tolist()

    @property
    def weights(self) -> list:
        """Renormalized MAW over each head's context (metadata, sparsifier.py:83-87)."""
        maw = self._ls.maw[:, : self._ls.lo].cpu().numpy()
        out = []
        for r, idx in enumerate(self.indices):
            sel = maw[r, idx]
            out.append(sel / sel.sum() if idx.size and sel.sum() > 0.0 else np.zeros(idx.size, np.float64))
        return out

    def _rows(self, which):
        ls = self._ls
        G = ls.cfg.heads // ls.cfg.n_kv_heads
        rows = ls.rows()
        out = []
        for r, idx in enumerate(self.indices):
            bk = (r // ls.cfg.heads) * ls.cfg.n_kv_heads + (r % ls.cfg.heads) // G
            out.append(rows[bk, torch.from_numpy(idx).to(rows.device), which].float())
        return out

    @property
    def keys(self) -> list:
        return self._rows(0)

    @property
    def values(self) -> list:
        return self._rows(1)


class StoreView:
    """StoreTier's read API (sparsifier.py:105-195) over the engine's archive
    tier of one layer: positions [0, lo) of the HBM buffer."""

    def __init__(self, ls: LayerState):
        self._ls = ls
        self.layer_id = ls.layer_id
        self.context = ContextView(ls)

    @property
    def shape(self):
        return self._ls.cfg.head_shape

    @property
    def archive_size(self) -> int:
        return self._ls.lo

    @property
    def positions(self) -> np.ndarray:
        return np.arange(self._ls.lo, dtype=np.int64)

    @property
    def maw(self):
        """[rows, archive_size] float64 device view."""
        return self._ls.maw[:, : self._ls.lo]

    @property
    def keys(self):
        return self._ls.rows()[:, : self._ls.lo, 0].float()

    @property
    def values(self):
        return self._ls.rows()[:, : self._ls.lo, 1].float()

    def context_dump(self, tasks=None) -> str:
        """sparsifier.py:179-195."""
        ls = self._ls
        rows = ls.ctx.shape[0]
        padded = [set() for _ in range(rows)]
        if tasks:
            for task in tasks:
                for h, entries, pad in zip(task.heads, task.entries, task.padding):
                    padded[h].update(np.asarray(entries)[np.asarray(pad, bool)].tolist())
        maw = self.maw.cpu().numpy()
        idx = self.context.indices
        lines = []
        for h in range(rows):
            selected = set(idx[h].tolist())
            for i in range(ls.lo):
                lines.append(f"layer={self.layer_id} head={h} pos={i} maw={maw[h, i]:.6e} "
                             f"selected={int(i in selected)} padding={int(i in padded[h])}")
        return "\n".join(lines)


class HybridEngine:
    """engine.py:87-195 on the B200, for `layers` layers.

    Streams: every launch goes to torch's current stream on the engine's
    device, and the layers share one set of per-step scratch (dense scores,
    item partials, the work counter), so all calls on one engine must be
    issued in order on ONE stream (the reference engine is single-threaded
    too, engine.py:10-11). Run independent engines for concurrent streams.
    """

    def __init__(self, config: EngineConfig, dev=None):
        self.config = config
        self.shape = config.head_shape
        self.dev = torch.device(dev) if dev is not None else device()
        if self.dev.type == "cuda" and self.dev.index is None:
            self.dev = torch.device("cuda", torch.cuda.current_device())
        c = config
        self.B, self.Hq, self.Hkv, self.D = c.batch, c.heads, c.n_kv_heads, c.head_dim
        self.G = self.Hq // self.Hkv
        if self.D not in (64, 128):
            raise ContractError("the device engine supports head_dim 64 or 128")
        self.T = int(math.ceil(c.max_positions / 32) * 32)
        if self.T >= 1 << 24:
            raise ContractError("max_positions must be below 2^24 (union entries pack 24-bit positions)")
        self.cap = c.cache.capacity
        self.tdtype = torch.bfloat16 if c.dtype == "bfloat16" else torch.float32
        self.dcode = DTYPE_CODE[self.tdtype]
        self.g_pad = group_size(c.batch, c.heads, c.core_count)
        self.layers = [LayerState(c, self.T, self.dev, i) for i in range(c.layers)]
        # shared per-step scratch (steps run in stream order)
        BHq = self.B * self.Hq
        self.dsc_ld = self.cap + 1
        self.dsc = torch.zeros((BHq, self.dsc_ld), dtype=torch.float64, device=self.dev)
        dense_rows, sparse_rows = item_rows(c.dtype)
        n_dense = self.B * self.Hkv * math.ceil(self.dsc_ld / dense_rows)
        n_sparse = sparse_capacity(self.B * self.Hkv, self.T, sparse_rows, self.layers[0].item_target)
        self.max_items = n_dense + n_sparse
        # per-item partials, head-major ([G, max_items] / [G, max_items, D])
        self.part_m = torch.empty(self.G * self.max_items, dtype=torch.float64, device=self.dev)
        self.part_z = torch.empty(self.G * self.max_items, dtype=torch.float64, device=self.dev)
        self.part_acc = torch.empty(self.max_items * self.G * self.D, dtype=torch.float32, device=self.dev)
        self.counter = torch.zeros(4, dtype=torch.int32, device=self.dev)  # decode work counter
        nb = int(_lib.load().hgca_merge_scratch_bytes(self.B, self.Hq, self.D, MERGE_SPLIT_MAX))
        self.merge_scratch = torch.zeros(nb // 8 + 1, dtype=torch.int64, device=self.dev)  # split-merge partials
        self.merge_items = MERGE_ITEMS  # items per merge CTA share (split merge)
        self.launches = 0          # kernels of libhgca_b200 launched by this engine
        self.step_events = None     # list -> (start, end) CUDA events around the decode kernel
        self._push = None           # per-step push descriptor (ShardedHybridEngine, exchange="push")

    # ------------------------------------------------------------ helpers
    def _stream(self):
        return stream_handle(self.dev)

    @staticmethod
    def _keep_ptr(ls: LayerState):
        return ls.keep.data_ptr() if ls.keep is not None else None

    def _as_dev(self, x, heads):
        """[B, heads, n, D] (or [heads, n, D] when B == 1) -> contiguous device tensor."""
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
        if t.dim() == 3:
            if self.B != 1:
                raise ContractError(f"3-D step input needs batch == 1 (batch={self.B})")
            t = t[None]
        if tuple(t.shape[:2]) != (self.B, heads) or t.shape[-1] != self.D:
            raise ContractError(f"step tensor shape {tuple(t.shape)} does not match "
                                f"({self.B}, {heads}, n, {self.D})")
        return t.to(device=self.dev, dtype=self.tdtype, non_blocking=True).contiguous()

    def _refresh_selection(self, ls: LayerState):
        """Padding / top-k and the union lists after the context changed."""
        n = ls.lo
        s = self._stream()
        words = ls.ctx.shape[1]
        if self.config.selection == "topk":
            ls.ctx.zero_()
            if n:
                topk_mask(ls.maw, min(self.config.topk, n), n=n, out=ls.ctx)
        if self.g_pad > 1 and n:
            counts = torch.zeros(self.B * self.Hq, dtype=torch.int64, device=self.dev)
            _lib.call("hgca_popcount_rows", ls.ctx.data_ptr(), self.B * self.Hq, words, n,
                      counts.data_ptr(), s)
            need = torch.zeros_like(counts)
            _lib.call("hgca_group_need", counts.data_ptr(), self.B, self.Hq, self.g_pad,
                      need.data_ptr(), s)
            ls.sel = ls.ctx.clone()  # a fresh tensor: a StepOutput may hold the old one
            topk_mask(ls.maw, need, n=n, exclude=ls.ctx, out=ls.sel)
        else:
            ls.sel = ls.ctx.clone()  # a fresh tensor: a StepOutput may hold the old one
        self.launches += 2 + (3 if (self.g_pad > 1 and n) else 0) + (1 if self.config.selection == "topk" and n else 0)
        # fp32 kernel: union rows grouped by query-head mask (single-head
        # sub-chunks), bf16 kernel: position order; both then position-class
        # interleaved per 32-entry window (conflict-free shared-memory reads of
        # the position-rotated rows)
        grouped = 3 if self.tdtype == torch.float32 else 2
        _lib.call("hgca_union_build_items_w", ls.sel.data_ptr(), self.B, self.Hq, self.Hkv, words, n, self.T,
                  ls.u_ent.data_ptr(), ls.u_cnt.data_ptr(), ls.item_off.data_ptr(), ls.item_tab.data_ptr(),
                  ls.sparse_rows, min(MIN_ITEM_ROWS, ls.sparse_rows), ls.item_target,
                  min(self.cap, self.T) if COUNT_WINDOW else 0, grouped, s)
        # the new item counts, for the merge's split factor: copied behind the rebuild and
        # picked up by a later step once the copy has landed (no host synchronization)
        nbk = 2 * self.B * self.Hkv + 3
        if ls.off_host is None:
            ls.off_host = torch.empty(nbk, dtype=torch.int32).pin_memory()
        ls.off_host.copy_(ls.item_off[:nbk], non_blocking=True)
        ls.off_event = torch.cuda.Event()
        ls.off_event.record()

    def _ingest(self, ls: LayerState, lo, hi, divisor):
        """StoreTier.ingest_evicted of positions [lo, hi) (sparsifier.py:127-156)."""
        if self.config.selection == "threshold" and hi > lo:
            self.launches += 1
            _lib.call("hgca_select_threshold", ls.maw.data_ptr(), self.B * self.Hq, self.T, lo, hi,
                      float(self.config.cache.beta), int(divisor), ls.ctx.data_ptr(), ls.ctx.shape[1], 0,
                      self._keep_ptr(ls), self._stream())
        ls.lo = hi
        self._refresh_selection(ls)

    def _evict_range(self, ls: LayerState, incoming):
        """WindowCache.evict_if_full (kv_cache.py:189-221) -> [lo, lo+freed)."""
        cap, blk = self.cap, self.config.cache.blk_size
        if incoming < 0:
            raise ContractError("incoming_count must be >= 0")
        if incoming > cap:
            raise ContractError(f"a single step of {incoming} entries exceeds the whole window ({cap}); unsupported")
        size = ls.window_size
        l_cur = size + incoming
        if l_cur < cap:
            return ls.lo, ls.lo
        n_blocks = math.ceil((l_cur - cap + 1) / blk)
        full_blocks = size // blk
        n_blocks = min(n_blocks, full_blocks)
        freed = n_blocks * blk
        if cap - (size - freed) < incoming:
            raise ContractError(f"cannot free room for {incoming} entries: only {full_blocks} full blocks are evictable")
        return ls.lo, ls.lo + freed

    # ------------------------------------------------------------ staging
    def bulk_ingest(self, layer_idx, keys, values, maw, divisor):
        """Archive n positions at once: StoreTier.ingest_evicted(blocks, beta,
        window_size=divisor) with the blocks' keys/values/MAW given directly
        (sparsifier.py:127-156). keys/values [B, Hkv, n, D], maw [B, Hq, n].
        Requires an empty window (stages long contexts)."""
        ls = self.layers[layer_idx]
        if ls.window_size:
            raise ContractError("bulk_ingest requires an empty window")
        k = self._as_dev(keys, self.Hkv)
        v = self._as_dev(values, self.Hkv)
        n = k.shape[2]
        if ls.nxt + n > self.T:
            raise ContractError("max_positions exceeded")
        m = maw if isinstance(maw, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(maw))
        m = m.to(device=self.dev, dtype=torch.float64).reshape(self.B * self.Hq, n)
        p0 = ls.nxt
        _lib.call("hgca_write_rows", self.dcode, ls.KV.data_ptr(), self.B * self.Hkv,
                  self.T, self.D, p0, k.data_ptr(), v.data_ptr(), n, self._stream())
        ls.maw[:, p0:p0 + n].copy_(m)
        ls.nxt = p0 + n
        self._ingest(ls, p0, p0 + n, divisor)

    # ------------------------------------------------------------ steps
    def step(self, layer_idx: int, inp: StepInput) -> StepOutput:
        if inp.mode == "decode":
            return self.decode_step(layer_idx, inp)
        return self.append_step(layer_idx, inp)

    def decode_step(self, layer_idx: int, inp: StepInput) -> StepOutput:
        if inp.mode != "decode":
            raise ContractError(f"decode_step got mode {inp.mode!r}")
        return self._decode(layer_idx, inp)

    def append_step(self, layer_idx: int, inp: StepInput) -> StepOutput:
        if inp.mode != "append":
            raise ContractError(f"append_step got mode {inp.mode!r}")
        return self._append(layer_idx, inp)

    def _decode(self, layer_idx, inp, out=None, lse=None):
        ls = self.layers[layer_idx]
        to_np = not isinstance(inp.q, torch.Tensor)
        squeeze = inp.q.ndim == 3
        q = self._as_dev(inp.q, self.Hq)
        k = self._as_dev(inp.keys, self.Hkv)
        v = self._as_dev(inp.values, self.Hkv)
        lo, sel = ls.lo, ls.sel  # the selection this step attends (refreshes replace ls.sel)
        a_cpu = self._store_weights(ls, q, sel, lo, 1) if (self.config.keep_weights and lo) else None
        o, l, w = self.decode_device(layer_idx, q, k, v, out=out, lse=lse)
        o = o.view(self.B, self.Hq, 1, self.D)
        l = l.view(self.B, self.Hq, 1)
        if w is not None:
            w = w.view(self.B, self.Hq, 1, -1)
        if squeeze:
            o, l = o[0], l[0]
            w = w[0] if w is not None else None
        rows = self.B * self.Hq

        def store_positions():
            if lo == 0:
                return [np.zeros(0, np.int64) for _ in range(rows)]
            return mask_to_lists(sel, lo)

        return self._output(to_np, o, l, w, a_cpu, np.arange(*self._last_dense_range, dtype=np.int64),
                            store_fn=store_positions)

    @staticmethod
    def _output(to_np, o, l, w, a_cpu, dense, store=None, store_fn=None):
        if to_np:
            o, l, w = _np(o), _np(l), _np(w)
            a_cpu = [_np(x) for x in a_cpu] if a_cpu is not None else None
        return StepOutput(o, l, w, a_cpu, dense, store_positions=store, store_fn=store_fn)

    def _store_weights(self, ls, q, sel, lo, nq):
        """Decode a_cpu (engine.py:139-148, keep_weights only): per query head the
        softmax weights [nq, n_h] over its attended store entries (context +
        padding), through hgca_attend_gqa_indexed on the engine's KV."""
        rows, dev, s = self.B * self.Hq, self.dev, self._stream()
        idx = torch.empty((rows, lo), dtype=torch.int64, device=dev)
        cnt = torch.zeros(rows, dtype=torch.int64, device=dev)
        _lib.call("hgca_mask_to_indices", sel.data_ptr(), None, rows, sel.shape[1], lo, idx.data_ptr(), lo, None,
                  cnt.data_ptr(), s)
        off = torch.arange(rows, dtype=torch.int64, device=dev) * lo
        o = torch.empty((rows, nq, self.D), dtype=torch.float32, device=dev)
        l = torch.empty((rows, nq), dtype=torch.float64, device=dev)
        w = torch.zeros((rows, nq, lo), dtype=torch.float32, device=dev)
        ws = torch.empty(rows * nq * lo, dtype=torch.float64, device=dev)
        _lib.call("hgca_attend_gqa_indexed", self.dcode, q.data_ptr(), ls.KV.data_ptr(), self.B, self.Hq, self.Hkv,
                  self.T, idx.data_ptr(), off.data_ptr(), cnt.data_ptr(), lo, nq, self.D, float(self.shape.scale),
                  o.data_ptr(), l.data_ptr(), w.data_ptr(), ws.data_ptr(), s)
        self.launches += 2
        cnt_h = cnt.cpu().tolist()
        return [w[r, :, : cnt_h[r]] for r in range(rows)]

    def decode_device(self, layer_idx, q, k, v, out=None, lse=None, wts=None, out_sparse=None, lse_sparse=None):
        """The decode hot path on device tensors: q [B, Hq, 1, D], k/v
        [B, Hkv, 1, D] (storage dtype). Returns (out [B*Hq, D] f32,
        lse [B*Hq] f64, a_gpu or None). Launches only; no host sync.
        out_sparse / lse_sparse (optional) receive the sparse-only partial
        (the per-rank contribution under sequence sharding)."""
        ls = self.layers[layer_idx]
        BHq = self.B * self.Hq
        nq_el, nk_el = BHq * self.D, self.B * self.Hkv * self.D
        for name, t, n in (("q", q, nq_el), ("k", k, nk_el), ("v", v, nk_el)):
            if not isinstance(t, torch.Tensor) or t.dtype != self.tdtype or not t.is_contiguous() \
                    or t.device != self.dev or t.numel() != n:
                raise ContractError(f"decode_device: {name} must be a contiguous {self.tdtype} tensor of {n} "
                                    f"elements on {self.dev}")
        for name, t, dt, n in (("out", out, torch.float32, BHq * self.D), ("lse", lse, torch.float64, BHq)):
            if t is not None and (t.dtype != dt or not t.is_contiguous() or t.device != self.dev or t.numel() != n):
                raise ContractError(f"decode_device: {name} must be a contiguous {dt} tensor of {n} elements")
        if out is None:
            out = torch.empty((BHq, self.D), dtype=torch.float32, device=self.dev)
        if lse is None:
            lse = torch.empty(BHq, dtype=torch.float64, device=self.dev)
        if wts is None and self.config.keep_weights:
            wts = torch.empty((BHq, ls.window_size + 1), dtype=torch.float32, device=self.dev)
        d = self._step_desc(ls, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), lse.data_ptr(),
                            wts.data_ptr() if wts is not None else None,
                            out_sparse.data_ptr() if out_sparse is not None else None,
                            lse_sparse.data_ptr() if lse_sparse is not None else None)
        s = self._stream()
        if self.step_events is None:
            _lib.call("hgca_decode_step", d, s)
        else:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.call("hgca_decode_step", d, s)
            e1.record()
            self.step_events.append((e0, e1))
        self._step_done(ls)
        return out, lse, wts

    def _step_desc(self, ls, q, k, v, out, lse, wts=None, out_sparse=None, lse_sparse=None):
        """Fill the layer's cached hgca_decode_desc for this step (raw device pointers)."""
        if ls.nxt + 1 > self.T:
            raise ContractError("max_positions exceeded")
        d = ls.desc
        if d is None:  # per-layer descriptor: the static fields once
            d = ls.desc = _lib.DecodeDesc()
            d.dtype = self.dcode
            d.B, d.Hq, d.Hkv, d.D, d.T = self.B, self.Hq, self.Hkv, self.D, self.T
            d.KV = ls.KV.data_ptr()
            d.scale = float(self.shape.scale)
            d.sparse_rows, d.item_target = ls.sparse_rows, ls.item_target
            d.u_ent, d.u_cnt, d.item_off = ls.u_ent.data_ptr(), ls.u_cnt.data_ptr(), ls.item_off.data_ptr()
            d.item_tab = ls.item_tab.data_ptr()
            d.dsc, d.dsc_ld = self.dsc.data_ptr(), self.dsc_ld
            d.part_m, d.part_z, d.part_acc = self.part_m.data_ptr(), self.part_z.data_ptr(), self.part_acc.data_ptr()
            d.max_items = self.max_items
            d.counter = self.counter.data_ptr()
            d.maw, d.alpha = ls.maw.data_ptr(), float(self.config.cache.alpha)
            d.merge_scratch = self.merge_scratch.data_ptr()
        if ls.off_event is not None and ls.off_event.query():
            ls.merge_split = self._merge_split(ls)
            ls.off_event = None
        d.merge_split = ls.merge_split
        # per step: the queries, kv_in (the kernel writes it at position nxt, append_kv's slot,
        # before the dense pass), the window range and the outputs
        d.q, d.k_new, d.v_new = q, k, v
        d.dlo, d.dhi, d.w_old = ls.lo, ls.nxt + 1, ls.nxt - ls.lo
        d.out, d.lse, d.wts_out = out, lse, wts
        d.out_sparse, d.lse_sparse = out_sparse, lse_sparse
        push = self._push  # one-shot exchange of the sharded engine (sharded.PeerExchange), else off
        d.push_n = 0
        if push is not None:
            d.push_sparse = push["sparse"]
            for i, (dst, flag) in enumerate(zip(push["dst"], push["flag"])):
                d.push_dst[i], d.push_flag[i] = dst, flag
            d.epoch, d.push_cnt = push["epoch"], push["cnt"]
            d.push_n = len(push["dst"])
        return d

    def _merge_split(self, ls):
        """CTAs per query head for the merge: the longest per-(batch, kv-head)
        item list of the last rebuild (full + tail sparse items + window parts)
        in shares of MERGE_ITEMS."""
        off = ls.off_host.numpy().astype(np.int64)
        BK = self.B * self.Hkv
        rows = max(int(off[2 * (BK + 1)]), 16)
        items = (off[1:BK + 1] - off[:BK]) + (off[BK + 2:2 * BK + 2] - off[BK + 1:2 * BK + 1])
        dense_rows = max(min(rows, 32), rows // 2)  # window parts: half the item length (HGCA_DENSE_DIV)
        n = int(items.max()) + -(-self.cap // dense_rows) if BK else 0
        return int(min(MERGE_SPLIT_MAX, max(1, -(-n // self.merge_items))))

    def _step_done(self, ls):
        """Host bookkeeping after a launched decode step (engine.py:175-191): the
        MAW EMA / init ran in the kernel; eviction -> ingest here; append_kv is
        the position move."""
        self.launches += 2  # decode kernel (writes kv_in), merge kernel
        self._last_dense_range = (ls.lo, ls.nxt + 1)
        w_size = ls.window_size
        ev_lo, ev_hi = self._evict_range(ls, 1)
        ls.nxt += 1
        if ev_hi > ev_lo:
            self._ingest(ls, ev_lo, ev_hi, w_size + 1)

    def decode_host_packed(self, layer_idx, in_host, out_host, staging=None):
        """End-to-end decode in ONE library call: in_host is a pinned buffer
        holding q [B,Hq,D] | k [B,Hkv,D] | v [B,Hkv,D] in the storage dtype back
        to back; out_host a pinned uint8 buffer of B*Hq*(4*D + 8) bytes that
        receives out f32 [B*Hq, D] followed by lse f64 [B*Hq].
        hgca_decode_step_host_async copies in, runs the step and delivers out
        | lse; the host bookkeeping of the step (eviction / ingest) is issued
        while the GPU runs it, then the stream is synchronized (the host owns
        the result on return)."""
        B, Hq, Hkv, D = self.B, self.Hq, self.Hkv, self.D
        nq, nk = B * Hq * D, B * Hkv * D
        if in_host.numel() != nq + 2 * nk or in_host.dtype != self.tdtype:
            raise ContractError("in_host must hold q | k | v in the storage dtype")
        nout = B * Hq * (4 * D + 8)
        if out_host.numel() != nout or out_host.dtype != torch.uint8:
            raise ContractError(f"out_host must be a uint8 buffer of {nout} bytes")
        if staging is None:
            staging = (torch.empty(nq + 2 * nk, dtype=self.tdtype, device=self.dev),
                       torch.empty(nout, dtype=torch.uint8, device=self.dev))
        dev_in, dev_out = staging
        ls = self.layers[layer_idx]
        e = self.tdtype.itemsize
        pi, po = dev_in.data_ptr(), dev_out.data_ptr()
        d = self._step_desc(ls, pi, pi + nq * e, pi + (nq + nk) * e, po, po + B * Hq * D * 4)
        # enqueue the step, do this step's host bookkeeping (eviction / ingest
        # launches go behind it on the stream) while the GPU runs it, then wait
        _lib.call("hgca_decode_step_host_async", d, in_host.data_ptr(), pi, (nq + 2 * nk) * e, out_host.data_ptr(),
                  po, nout, self._stream())
        self._step_done(ls)
        torch.cuda.current_stream(self.dev).synchronize()
        return out_host

    def decode_host(self, layer_idx, q_host, k_host, v_host, out_host, lse_host, staging=None):
        """End-to-end decode through the C ABI with HOST buffers: pinned
        q [B,Hq,1,D] / k, v [B,Hkv,1,D] are copied to HBM, the step runs, and
        out [B*Hq, D] f32 / lse [B*Hq] f64 are copied back and synchronized
        (the host reads the step's result)."""
        if staging is None:
            staging = (torch.empty(q_host.shape, dtype=self.tdtype, device=self.dev),
                       torch.empty(k_host.shape, dtype=self.tdtype, device=self.dev),
                       torch.empty(v_host.shape, dtype=self.tdtype, device=self.dev))
        q, k, v = staging
        q.copy_(q_host, non_blocking=True)
        k.copy_(k_host, non_blocking=True)
        v.copy_(v_host, non_blocking=True)
        out, lse, _ = self.decode_device(layer_idx, q, k, v)
        out_host.copy_(out, non_blocking=True)
        lse_host.copy_(lse, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        return out_host, lse_host

    def _append(self, layer_idx, inp):
        """Append step (engine.py:111-114 -> _run_step with the full archive)."""
        ls = self.layers[layer_idx]
        squeeze = inp.q.ndim == 3
        q = self._as_dev(inp.q, self.Hq)
        k = self._as_dev(inp.keys, self.Hkv)
        v = self._as_dev(inp.values, self.Hkv)
        nq = q.shape[2]
        s = self._stream()
        if ls.nxt + nq > self.T:
            raise ContractError("max_positions exceeded")
        _lib.call("hgca_write_rows", self.dcode, ls.KV.data_ptr(), self.B * self.Hkv,
                  self.T, self.D, ls.nxt, k.data_ptr(), v.data_ptr(), nq, s)
        BHq = self.B * self.Hq
        lo, nxt = ls.lo, ls.nxt
        w_size = nxt - lo
        W = w_size + nq
        odt = torch.float32
        if self.tdtype == torch.bfloat16 and not self.config.keep_weights:
            return self._append_tc(ls, q, nq, squeeze, not isinstance(inp.q, torch.Tensor))
        # sparse partial over the whole archive, with weights (engine.py:127-132)
        s_out = torch.zeros((BHq, nq, self.D), dtype=odt, device=self.dev)
        s_lse = torch.full((BHq, nq), -math.inf, dtype=torch.float64, device=self.dev)
        a_cpu = None
        if lo:
            a_cpu = torch.empty((BHq, nq, lo), dtype=odt, device=self.dev)
            ws = torch.empty(BHq * nq * lo, dtype=torch.float64, device=self.dev)
            _lib.call("hgca_attend_gqa", self.dcode, q.data_ptr(), ls.KV.data_ptr(),
                      self.B, self.Hq, self.Hkv, self.T, 0, lo, nq, self.D, float(self.shape.scale),
                      s_out.data_ptr(), s_lse.data_ptr(), a_cpu.data_ptr(), lo, ws.data_ptr(), s)
        # dense over window + kv_in (engine.py:161-164)
        d_out = torch.empty((BHq, nq, self.D), dtype=odt, device=self.dev)
        d_lse = torch.empty((BHq, nq), dtype=torch.float64, device=self.dev)
        a_gpu = torch.empty((BHq, nq, W), dtype=odt, device=self.dev)
        ws = torch.empty(BHq * nq * W, dtype=torch.float64, device=self.dev)
        _lib.call("hgca_attend_gqa", self.dcode, q.data_ptr(), ls.KV.data_ptr(),
                  self.B, self.Hq, self.Hkv, self.T, lo, W, nq, self.D, float(self.shape.scale),
                  d_out.data_ptr(), d_lse.data_ptr(), a_gpu.data_ptr(), W, ws.data_ptr(), s)
        # merge (engine.py:166-169)
        out = torch.empty_like(d_out)
        lse = torch.empty_like(d_lse)
        _lib.call("hgca_merge_states", _lib.DTYPE_F32, s_out.data_ptr(), s_lse.data_ptr(), d_out.data_ptr(),
                  d_lse.data_ptr(), BHq * nq, self.D, out.data_ptr(), lse.data_ptr(), None, None, 0, 0,
                  None, s)
        # maintenance (engine.py:175-186)
        _lib.call("hgca_maw_update", a_gpu.data_ptr(), BHq, nq, W, W, ls.maw.data_ptr(), self.T, lo, w_size,
                  float(self.config.cache.alpha), 0, s)
        ev_lo, ev_hi = self._evict_range(ls, nq)
        if lo:
            # StoreTier.reevaluate(mean_rows(a_cpu), beta) (sparsifier.py:158-177)
            _lib.call("hgca_maw_update", a_cpu.data_ptr(), BHq, nq, lo, lo, ls.maw.data_ptr(), self.T, 0, 0,
                      float(self.config.cache.alpha), 1, s)
            if self.config.selection == "threshold":
                _lib.call("hgca_select_threshold", ls.maw.data_ptr(), BHq, self.T, 0, lo,
                          float(self.config.cache.beta), int(lo), ls.ctx.data_ptr(), ls.ctx.shape[1], 1,
                          self._keep_ptr(ls), s)
        if ev_hi > ev_lo:
            self._ingest(ls, ev_lo, ev_hi, w_size + nq)
        elif lo:
            self._refresh_selection(ls)
        if ls.window_size + nq > self.cap:
            raise ContractError(f"append of {nq} entries overflows window capacity {self.cap}")
        ls.nxt += nq
        o = out.view(self.B, self.Hq, nq, self.D)
        l = lse.view(self.B, self.Hq, nq)
        ag = a_gpu.view(self.B, self.Hq, nq, W)
        if squeeze:
            o, l, ag = o[0], l[0], ag[0]
        a_list = [a_cpu[r] for r in range(BHq)] if a_cpu is not None else [
            torch.zeros((nq, 0), dtype=odt, device=self.dev) for _ in range(BHq)]
        return self._output(not isinstance(inp.q, torch.Tensor), o, l, ag, a_list,
                            np.arange(lo, nxt + nq, dtype=np.int64), store_fn=lambda: self._archive_positions(lo))

    def _archive_positions(self, lo):
        """Append-mode store_positions: every head attends the whole archive (engine.py:131)."""
        return [np.arange(lo, dtype=np.int64) for _ in range(self.B * self.Hq)]

    def _append_tc(self, ls, q, nq, squeeze, to_np=False):
        """Append step for bf16 storage on the tensor cores (hgca_append_bf16):
        archive + window attention, merge_states, and the per-head row-mean
        weights a_cpu / a_gpu feed the reference maintenance directly
        (engine.py:175-186): the window MAW EMA / init and
        StoreTier.reevaluate + re-selection. The per-row weight matrices are
        not materialised (StepOutput a_gpu / a_cpu are None; use
        keep_weights=True for them)."""
        s = self._stream()
        BHq = self.B * self.Hq
        lo, nxt = ls.lo, ls.nxt
        w_size = nxt - lo
        W, hi = w_size + nq, nxt + nq
        out = torch.empty((BHq, nq, self.D), dtype=torch.float32, device=self.dev)
        lse = torch.empty((BHq, nq), dtype=torch.float64, device=self.dev)
        mean_a = torch.empty((BHq, max(lo, 1)), dtype=torch.float32, device=self.dev)
        mean_w = torch.empty((BHq, W), dtype=torch.float32, device=self.dev)
        # hgca_append_bf16 takes <= APPEND_MAX_NQ queries per call (row groups of whole
        # heads, <= 128 rows). Longer appends run as query chunks against the same keys
        # (every kv_in row is already written, so each chunk sees the full key set, as
        # the reference's non-causal attend_dense does): the outputs are per query, and
        # the per-head row-mean weights combine as sum_c (nq_c / nq) * mean_c.
        n_ch = -(-nq // APPEND_MAX_NQ)
        step = -(-nq // n_ch)
        for c0 in range(0, nq, step):
            nc = min(step, nq - c0)
            if n_ch == 1:
                qc, oc, lc, ma, mw = q, out, lse, mean_a, mean_w
            else:
                qc = q[:, :, c0:c0 + nc].contiguous()
                oc = torch.empty((BHq, nc, self.D), dtype=torch.float32, device=self.dev)
                lc = torch.empty((BHq, nc), dtype=torch.float64, device=self.dev)
                ma, mw = torch.empty_like(mean_a), torch.empty_like(mean_w)
            nb = int(_lib.load().hgca_append_ws_bytes(self.B, self.Hq, self.Hkv, self.D, nc, lo, hi))
            ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=self.dev)
            _lib.call("hgca_append_bf16", ls.KV.data_ptr(), self.B, self.Hq, self.Hkv, self.T, self.D, qc.data_ptr(),
                      nc, float(self.shape.scale), lo, hi, oc.data_ptr(), lc.data_ptr(),
                      ma.data_ptr() if lo else None, mw.data_ptr(), ws.data_ptr(), nb, s)
            self.launches += 3
            if n_ch > 1:
                out[:, c0:c0 + nc].copy_(oc)
                lse[:, c0:c0 + nc].copy_(lc)
                wgt = nc / nq
                if c0 == 0:
                    mean_a.copy_(ma).mul_(wgt)
                    mean_w.copy_(mw).mul_(wgt)
                else:
                    mean_a.add_(ma, alpha=wgt)
                    mean_w.add_(mw, alpha=wgt)
        # maintenance (engine.py:175-186): the kernel already took the row means
        _lib.call("hgca_maw_update", mean_w.data_ptr(), BHq, 1, W, W, ls.maw.data_ptr(), self.T, lo, w_size,
                  float(self.config.cache.alpha), 0, s)
        ev_lo, ev_hi = self._evict_range(ls, nq)
        if lo:
            _lib.call("hgca_maw_update", mean_a.data_ptr(), BHq, 1, lo, lo, ls.maw.data_ptr(), self.T, 0, 0,
                      float(self.config.cache.alpha), 1, s)
            if self.config.selection == "threshold":
                _lib.call("hgca_select_threshold", ls.maw.data_ptr(), BHq, self.T, 0, lo,
                          float(self.config.cache.beta), int(lo), ls.ctx.data_ptr(), ls.ctx.shape[1], 1,
                          self._keep_ptr(ls), s)
        if ev_hi > ev_lo:
            self._ingest(ls, ev_lo, ev_hi, w_size + nq)
        elif lo:
            self._refresh_selection(ls)
        if ls.window_size + nq > self.cap:
            raise ContractError(f"append of {nq} entries overflows window capacity {self.cap}")
        ls.nxt += nq
        self.launches += 2
        o = out.view(self.B, self.Hq, nq, self.D)
        l = lse.view(self.B, self.Hq, nq)
        if squeeze:
            o, l = o[0], l[0]
        return self._output(to_np, o, l, None, None, np.arange(lo, nxt + nq, dtype=np.int64),
                            store_fn=lambda: self._archive_positions(lo))

    # ------------------------------------------------------------ inspection
    def context_indices(self, layer_idx=0):
        """Per (b*Hq + h) context-cache index lists (sparsifier.py ContextCache.indices)."""
        ls = self.layers[layer_idx]
        return mask_to_lists(ls.ctx, ls.lo)

    def store_entries(self, layer_idx=0):
        """Per (b*Hq + h) attended archive entries (context + padding) and flags."""
        ls = self.layers[layer_idx]
        return mask_to_lists(ls.ctx, ls.lo, mask_b=ls.sel, want_flags=True)

    def maw_host(self, layer_idx=0):
        ls = self.layers[layer_idx]
        return ls.maw[:, : ls.nxt].cpu().numpy()



def run_sequence(config: EngineConfig, workload, on_step=None, collect: bool = False):
    """engine.py:198-224: drive every layer through a workload's steps in order.

    `workload` yields steps with `mode` and per-layer q / keys / values stacked
    as [layers, heads, n_q, head_dim] (tierkv.Workload, workload.Workload).
    on_step(step_idx, layer_idx, inp, out, layer_state) runs after each layer
    step; layer_state.window / .store give the reference's read API. Returns
    (engine, outputs): per step, per layer StepOutputs when collect, else None.
    When the workload's length is known, max_positions is raised to hold it.
    """
    steps = workload.steps if hasattr(workload, "steps") else workload
    if hasattr(steps, "__len__"):
        total = sum(int(s.q.shape[2]) for s in steps)
        if total > config.max_positions:
            config = config.with_(max_positions=total)
    engine = HybridEngine(config)
    outputs = [] if collect else None
    for step_idx, step in enumerate(steps):
        if step.q.shape[0] < config.layers:
            raise ContractError(f"workload exhausted mid-layer at step {step_idx}: "
                                f"{step.q.shape[0]} layers provided, {config.layers} required")
        per_layer = [] if collect else None
        for li in range(config.layers):
            inp = StepInput(step.mode, step.q[li], step.keys[li], step.values[li])
            out = engine.step(li, inp)
            if on_step is not None:
                on_step(step_idx, li, inp, out, engine.layers[li])
            if collect:
                per_layer.append(out)
        if collect:
            outputs.append(per_layer)
    return engine, outputs


class DecodeGraph:
    """`steps` decode steps of `layers` replayed from ONE captured CUDA graph.

    Graph mode of hgca_decode_step (include/hgca_b200.h, desc.state): the
    window range lives in a device step state per layer that the merge
    kernel advances after every step, so one captured launch sequence --
    step-major, for every step and layer a decode and a merge kernel, each
    kernel chained to the previous one by programmatic dependent launch --
    replays token after token with no host work in between. The host only
    replays the graph and keeps its mirror of the positions; eviction /
    ingest (every blk_size steps) runs eagerly between replays, and the
    state is re-set when the window moved. A replay of `steps` tokens must
    not cross an eviction before its last step (`room()`).
    Inputs: fixed device buffers q [steps, L, B, Hq, 1, D], k / v
    [steps, L, B, Hkv, 1, D] (storage dtype) that the caller fills before a
    replay (slot [t, l] = token t of the replay, layer l); outputs out
    [steps, L, B*Hq, D] f32 and lse [steps, L, B*Hq] f64. Same kernels and
    bit-identical results as decode_device."""

    def __init__(self, eng: "HybridEngine", layers=None, steps: int = 1):
        if eng.config.keep_weights or eng._push is not None:
            raise ContractError("DecodeGraph: keep_weights and the push exchange are eager-only")
        if steps < 1:
            raise ContractError("DecodeGraph: steps must be >= 1")
        self.eng, self.steps = eng, int(steps)
        self.layers = list(range(len(eng.layers))) if layers is None else list(layers)
        B, Hq, Hkv, D, dev, tdt = eng.B, eng.Hq, eng.Hkv, eng.D, eng.dev, eng.tdtype
        n, L = self.steps, len(self.layers)
        self.q = torch.zeros((n, L, B, Hq, 1, D), dtype=tdt, device=dev)
        self.k = torch.zeros((n, L, B, Hkv, 1, D), dtype=tdt, device=dev)
        self.v = torch.zeros((n, L, B, Hkv, 1, D), dtype=tdt, device=dev)
        self.out = torch.empty((n, L, B * Hq, D), dtype=torch.float32, device=dev)
        self.lse = torch.empty((n, L, B * Hq), dtype=torch.float64, device=dev)
        if self.room() < n:
            raise ContractError(f"DecodeGraph: {n} steps cross an eviction (room {self.room()})")
        self.descs = []
        for t in range(n):
            for i, li in enumerate(self.layers):
                ls = eng.layers[li]
                if ls.state is None:
                    ls.state = torch.zeros(4, dtype=torch.int64, device=dev)
                self._sync(ls)
                d = _lib.DecodeDesc.from_buffer_copy(eng._step_desc(
                    ls, self.q[t, i].data_ptr(), self.k[t, i].data_ptr(), self.v[t, i].data_ptr(),
                    self.out[t, i].data_ptr(), self.lse[t, i].data_ptr()))
                d.state = ls.state.data_ptr()
                self.descs.append(d)
        # capture on torch's side stream (the C launchers read the current stream)
        torch.cuda.synchronize(dev)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, capture_error_mode="thread_local"):
            st = eng._stream()
            for d in self.descs:
                _lib.call("hgca_decode_step", d, st)
        torch.cuda.synchronize(dev)

    def room(self) -> int:
        """Tokens a replay may decode before an eviction must run (the last
        of them may trigger one: it is handled after the replay)."""
        cap = self.eng.cap
        return min(cap - self.eng.layers[li].window_size for li in self.layers)

    def _sync(self, ls: LayerState):
        want = (ls.lo, ls.nxt + 1)
        if ls.state_mirror != want:
            _lib.call("hgca_step_state_set", ls.state.data_ptr(), want[0], want[1], 0, self.eng._stream())
            self.eng.launches += 1
            ls.state_mirror = want

    def step(self):
        """Replay: `steps` decode steps of every captured layer -> (out, lse)."""
        eng = self.eng
        if self.room() < self.steps:
            raise ContractError(f"DecodeGraph: {self.steps} steps would cross an eviction (room {self.room()}); "
                                f"replay a graph of fewer steps or take eager steps up to the eviction")
        for li in self.layers:
            ls = eng.layers[li]
            if ls.nxt + self.steps > eng.T:
                raise ContractError("max_positions exceeded")
            self._sync(ls)
        self.graph.replay()
        for t in range(self.steps):
            for li in self.layers:
                ls = eng.layers[li]
                lo0 = ls.lo
                eng._step_done(ls)
                ls.state_mirror = (lo0, ls.nxt + 1)  # the merge kernel advanced dhi; an eviction moved lo
        return self.out, self.lse
