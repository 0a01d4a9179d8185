"""B200-native hybrid two-tier decode attention (HGCA, arXiv 2507.03153).

Drop-in for the hot path of the reference package `tierkv`: the attention
API (attention.py), the kernel plugin slot (backends.py), store-tier
selection (sparsifier.py) and a device-resident step driver (engine.py),
all computing in libhgca_b200.so (hand-written sm_100a CUDA behind a C ABI,
include/hgca_b200.h). There is no CPU fallback.
"""

from .errors import ContractError
from .attention import AttentionResult, HeadShape, attend, attend_indexed, logsumexp, merge_states
from .backends import CUDA, install
from .kv_cache import CacheConfig, KvBlock, WindowCache, offload
from .sparsifier import (ContextCache, HeadGroupTask, StoreTier, pack_head_groups, renormalize, select_salient,
                         select_topk)
from .engine import DecodeGraph, EngineConfig, HybridEngine, LayerState, StepInput, StepOutput, run_sequence
from .sharded import ShardedHybridEngine, packed_stride, shard_owner
from .workload import Workload, WorkloadSpec, gen_workload_device, load_workload, save_workload
from . import _lib

__version__ = "0.1.0"


def library_path() -> str:
    return _lib.LIB_PATH
