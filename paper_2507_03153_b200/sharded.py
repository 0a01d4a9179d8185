"""KV-sequence-sharded hybrid decode across GPUs.

The reference has one process and no collectives (engine.py:10-11); its
merge_states (attention.py:153-188) is exact and associative over disjoint key
sets, which is what makes the archive shardable:

  * archive block j (positions [j*blk, (j+1)*blk)) is owned by rank
    j % world (block-cyclic, so sinks, heavy hitters and growth stay balanced);
    threshold selection (select_salient, sparsifier.py:32-42) is per entry, so
    each rank selects only among the blocks it owns -- the threshold
    beta/divisor is a global scalar every rank already knows;
  * every rank keeps the (small) window tier and attends it densely, so the
    MAW EMA of the window (kv_cache.py:171-187) -- and therefore selection at
    eviction -- is identical on every rank without any exchange;
  * per decode step, rank 0 contributes merge_states(sparse_0, dense) and rank
    r > 0 its sparse partial over its shard; the (out f32 [B*Hq, D],
    lse f64 [B*Hq]) partials are packed into one buffer that the decode kernel
    writes in place, exchanged by ONE all_gather over NCCL (NVLink/NVSwitch),
    and folded in rank order by hgca_merge_packed on every rank.

Per-rank HBM traffic of the step is the window plus 1/world of the selected
archive rows; the collective moves (D*4 + 8) bytes per (batch, query head)
per rank.

exchange="push" replaces the all-gather with a one-shot push fused into the
merge kernel (PeerExchange): every rank owns a receive box in HBM that all
ranks map (CUDA IPC), [2 parities][world slots][packed partial] plus one
epoch flag per (parity, slot); the merge kernel stores each finished head's
row straight into its slot of every peer's box over NVLink while the rest of
the merge runs, and its last CTA publishes the step's epoch to the peers'
flags (system-scope release). hgca_merge_packed_wait then waits for the
world flags on the device and folds the box in rank order -- no NCCL call and
no host synchronisation on the step. Parity double-buffering makes slot reuse
safe: a rank can only write parity p again after it has waited for every
peer's flag of the step in between, which each peer publishes after its own
merge of parity p. Only decode steps are sharded; append steps run replicated (every
rank holds every K/V row), and their re-evaluation re-selects within the
rank's shard.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .engine import EngineConfig, HybridEngine
from .errors import ContractError


def shard_owner(block: int, world: int) -> int:
    """Rank that owns archive block `block` (block-cyclic; see
    sparsifier.ownership_words for the position mask the kernels use)."""
    return block % world


def packed_stride(rows: int, d: int) -> int:
    """Bytes of one rank's packed (out f32 [rows, d], lse f64 [rows]) partial."""
    return rows * d * 4 + rows * 8


class PeerExchange:
    """Receive boxes + epoch flags of the one-shot push (hgca_peer_alloc / hgca_peer_open)."""

    FLAG_ALIGN = 256

    def __init__(self, world: int, rank: int, stride: int, dev, timeout_ms: int = 10000):
        if not 1 <= world <= 8:
            raise ContractError("the one-shot push supports 1..8 ranks")
        self.world, self.rank, self.stride, self.timeout_ms = world, rank, stride, timeout_ms
        self.box_bytes = 2 * world * stride
        self.flags_off = -(-self.box_bytes // self.FLAG_ALIGN) * self.FLAG_ALIGN
        ptr, handle = ctypes.c_void_p(), (ctypes.c_uint8 * 64)()
        _lib.call("hgca_peer_alloc", self.flags_off + 2 * world * 8, ctypes.byref(ptr), handle)
        self.base, self.handle = ptr.value, bytes(handle)
        self.peers = None
        self._opened = []
        self.cnt = torch.zeros(1, dtype=torch.int32, device=dev)   # merge-kernel CTA counter
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)   # set by a timed-out wait
        self.epoch = 0

    def connect_ipc(self, handles):
        """Map every peer's box from its 64-byte handle (one per rank, rank order)."""
        peers = []
        for p, h in enumerate(handles):
            if p == self.rank:
                peers.append(self.base)
                continue
            ptr = ctypes.c_void_p()
            _lib.call("hgca_peer_open", (ctypes.c_uint8 * 64).from_buffer_copy(h), ctypes.byref(ptr))
            self._opened.append(ptr.value)
            peers.append(ptr.value)
        self.peers = peers

    def connect_local(self, bases):
        """Single-process ranks (tests): the peers' boxes are plain device pointers."""
        self.peers = list(bases)

    def next_step(self, sparse: bool):
        """The push descriptor of the next step (engine._push) and this rank's
        (box half, flags) for hgca_merge_packed_wait."""
        if self.peers is None:
            raise ContractError("PeerExchange is not connected")
        self.epoch += 1
        par = self.epoch & 1
        half = par * self.world * self.stride
        push = {"sparse": int(sparse), "epoch": self.epoch, "cnt": self.cnt.data_ptr(),
                "dst": [b + half + self.rank * self.stride for b in self.peers],
                "flag": [b + self.flags_off + (par * self.world + self.rank) * 8 for b in self.peers]}
        return push, self.base + half, self.base + self.flags_off + par * self.world * 8

    def close(self):
        for p in self._opened:
            _lib.call("hgca_peer_close", p)
        self._opened = []
        if self.base:
            _lib.call("hgca_peer_free", self.base)
            self.base = None


class ShardedHybridEngine(HybridEngine):
    """HybridEngine whose decode step is sequence-sharded over a process group.

    rank / world default to the process group's (torch.distributed, backend
    "nccl" on GPUs); passing them explicitly (no process group) builds one
    shard for single-process tests, which drive decode_partial() and merge()
    themselves. With world == 1 it is an ordinary HybridEngine.
    """

    def __init__(self, config: EngineConfig, group=None, dev=None, rank=None, world=None, exchange="allgather",
                 push_timeout_ms: int = 10000):
        import torch.distributed as dist

        if exchange not in ("allgather", "push"):
            raise ContractError(f"exchange must be 'allgather' or 'push', got {exchange!r}")

        self.group = group
        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        if rank is None:
            rank = self.dist.get_rank(group) if self.dist else 0
            world = self.dist.get_world_size(group) if self.dist else 1
        elif world is None:
            raise ContractError("pass world together with rank")
        super().__init__(config.with_(shard_rank=rank, shard_world=world), dev=dev)
        self.rank, self.world = rank, world
        rows, D = self.B * self.Hq, self.D
        self.rows = rows
        self.stride = packed_stride(rows, D)
        self.send = torch.empty(self.stride, dtype=torch.uint8, device=self.dev)
        self.recv = torch.empty(world * self.stride, dtype=torch.uint8, device=self.dev)
        self._send_out = self.send[: rows * D * 4].view(torch.float32).view(rows, D)
        self._send_lse = self.send[rows * D * 4:].view(torch.float64)
        self._loc_out = torch.empty((rows, D), dtype=torch.float32, device=self.dev)
        self._loc_lse = torch.empty(rows, dtype=torch.float64, device=self.dev)
        self.collectives = 0
        self.exchange = exchange
        self.xchg = None
        if exchange == "push" and world > 1:
            self.xchg = PeerExchange(world, rank, self.stride, self.dev, timeout_ms=push_timeout_ms)
            if self.dist is not None:  # exchange the IPC handles once
                handles = [None] * world
                self.dist.all_gather_object(handles, self.xchg.handle, group=group)
                self.xchg.connect_ipc(handles)

    def decode_partial(self, layer_idx, q, k, v, wts=None):
        """This rank's decode step, leaving its packed partial in self.send."""
        if self.rank == 0:
            _, _, w = super().decode_device(layer_idx, q, k, v, out=self._send_out, lse=self._send_lse, wts=wts)
        else:
            _, _, w = super().decode_device(layer_idx, q, k, v, out=self._loc_out, lse=self._loc_lse, wts=wts,
                                            out_sparse=self._send_out, lse_sparse=self._send_lse)
        return w

    def merge(self, parts, out, lse):
        """Fold `world` packed partials (rank order) into out / lse."""
        if parts.numel() != self.world * self.stride or parts.dtype != torch.uint8:
            raise ContractError("parts must be the [world * stride] uint8 allgather buffer")
        _lib.call("hgca_merge_packed", parts.data_ptr(), self.world, self.rows, self.D, self.stride,
                  out.data_ptr(), lse.data_ptr(), self._stream())
        self.launches += 1
        return out, lse

    def decode_host_packed(self, layer_idx, in_host, out_host, staging=None):
        """End-to-end decode with host buffers (as HybridEngine.decode_host_packed),
        through the sharded step: H2D, this rank's partial, all-gather, merge, D2H."""
        B, Hq, Hkv, D = self.B, self.Hq, self.Hkv, self.D
        nq, nk = B * Hq * D, B * Hkv * D
        if staging is None:
            staging = (torch.empty(nq + 2 * nk, dtype=self.tdtype, device=self.dev),
                       torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8, device=self.dev))
        dev_in, dev_out = staging
        dev_in.copy_(in_host, non_blocking=True)
        out = dev_out[: B * Hq * D * 4].view(torch.float32).view(B * Hq, D)
        lse = dev_out[B * Hq * D * 4:].view(torch.float64)
        self.decode_device(layer_idx, dev_in[:nq], dev_in[nq:nq + nk], dev_in[nq + nk:], out=out, lse=lse)
        out_host.copy_(dev_out, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        self.check_exchange()  # host sync point: a timed-out push poisoned this result
        return out_host

    def decode_device(self, layer_idx, q, k, v, out=None, lse=None, wts=None, out_sparse=None, lse_sparse=None):
        if out_sparse is not None or lse_sparse is not None:
            raise ContractError("the sharded engine owns the sparse partial buffers")
        if out is None:
            out = torch.empty((self.rows, self.D), dtype=torch.float32, device=self.dev)
        if lse is None:
            lse = torch.empty(self.rows, dtype=torch.float64, device=self.dev)
        if self.xchg is not None:
            return self._decode_push(layer_idx, q, k, v, out, lse, wts)
        w = self.decode_partial(layer_idx, q, k, v, wts=wts)
        if self.world > 1:
            if self.dist is None:
                raise ContractError("world > 1 needs an initialised process group (or call decode_partial/merge)")
            if self.dist.get_backend(self.group) == "nccl":
                self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
            else:  # gloo (CPU tests of the multi-process path): gather through host copies
                host = [torch.empty(self.stride, dtype=torch.uint8) for _ in range(self.world)]
                self.dist.all_gather(host, self.send.cpu(), group=self.group)
                self.recv.copy_(torch.cat(host))
            self.collectives += 1
            parts = self.recv
        else:
            parts = self.send
        self.merge(parts, out, lse)
        return out, lse, w

    def _decode_push(self, layer_idx, q, k, v, out, lse, wts):
        """exchange="push": the merge kernel pushes this rank's packed partial
        into every peer's box; the P-way merge waits for the peers' flags on
        the device (see the module docstring)."""
        w = self.push_partial(layer_idx, q, k, v, wts=wts)
        self.push_merge(out, lse)
        return out, lse, w

    def push_partial(self, layer_idx, q, k, v, wts=None):
        """exchange="push", first half of a step: this rank's decode step, whose
        merge kernel pushes the packed partial into every peer's box (no wait)."""
        push, self._box, self._flags = self.xchg.next_step(sparse=self.rank > 0)
        self._push = push
        try:
            _, _, w = HybridEngine.decode_device(self, layer_idx, q, k, v, out=self._loc_out, lse=self._loc_lse,
                                                 wts=wts)
        finally:
            self._push = None
        return w

    def push_merge(self, out, lse):
        """Second half: wait on the device for every peer's flag of this step,
        then the P-way merge. Ranks sharing one process (tests) enqueue every
        rank's push_partial before any push_merge, so no spinning wait sits on
        the GPU while the host still launches a peer's step."""
        _lib.call("hgca_merge_packed_wait", self._box, self.world, self.rows, self.D, self.stride, self._flags,
                  self.xchg.epoch, self.xchg.timeout_ms, self.xchg.err.data_ptr(), out.data_ptr(), lse.data_ptr(),
                  self._stream())
        self.launches += 2  # wait + merge
        self.collectives += 1
        return out, lse

    def check_exchange(self):
        """Raise if a push-exchange wait timed out (host sync)."""
        if self.xchg is not None and int(self.xchg.err.item()):
            raise RuntimeError("one-shot exchange: a peer's flag did not arrive before the timeout")

    def close(self):
        if self.xchg is not None:
            torch.cuda.synchronize(self.dev)
            self.xchg.close()
            self.xchg = None
