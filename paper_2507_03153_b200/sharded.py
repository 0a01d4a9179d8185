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
per rank. Only decode steps are sharded; append steps run replicated (every
rank holds every K/V row), and their re-evaluation re-selects within the
rank's shard.
"""

from __future__ import annotations

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


class ShardedHybridEngine(HybridEngine):
    """HybridEngine whose decode step is sequence-sharded over a process group.

    rank / world default to the process group's (torch.distributed, backend
    "nccl" on GPUs); passing them explicitly (no process group) builds one
    shard for single-process tests, which drive decode_partial() and merge()
    themselves. With world == 1 it is an ordinary HybridEngine.
    """

    def __init__(self, config: EngineConfig, group=None, dev=None, rank=None, world=None):
        import torch.distributed as dist

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
        return out_host

    def decode_device(self, layer_idx, q, k, v, out=None, lse=None, wts=None, out_sparse=None, lse_sparse=None):
        if out_sparse is not None or lse_sparse is not None:
            raise ContractError("the sharded engine owns the sparse partial buffers")
        if out is None:
            out = torch.empty((self.rows, self.D), dtype=torch.float32, device=self.dev)
        if lse is None:
            lse = torch.empty(self.rows, dtype=torch.float64, device=self.dev)
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
