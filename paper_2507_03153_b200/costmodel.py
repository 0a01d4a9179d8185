"""Analytic cost model of hybrid decode attention, recalibrated for B200.

Two layers:

1. The reference's roofline model (``perf_model.py:1-223``), same names and
   semantics: each attention pass costs ``max(flops/peak, bytes/bw)``; the
   offload baseline serialises a link transfer of the store tier with device
   attention over everything; the paper's hybrid overlaps window attention on
   the device with sparse attention on the host and pays a small merge
   transfer. ``DEFAULT_GPU/CPU/LINK`` are the reference's commodity points.

2. This framework's design on a B200, where both tiers live in HBM and one
   decode layer-step moves (``bench.partial_bytes``, DESIGN.md §(d)):
       dense window  B*Hkv*W*2D*e
     + sparse union  U*(2D*e + 4)      U = union over the G query heads of a kv head
     + q, per-item partials, scores, out, lse
   at the HBM bandwidth, plus a fixed per-launch cost (launch, pipeline fill,
   merge tail). ``predict_decode`` gives the breakdown, ``predict_sharded`` the
   sequence-sharded step (archive split P ways, one all-gather of the packed
   (out, lse) partials over NVLink), and ``fit_decode`` calibrates the fixed
   cost and effective bandwidth from measured (bytes, seconds) points, e.g.
   ``profiles/r01_configs_timing.jsonl`` (tools/costmodel_check.py).

Analytic only: nothing here launches work.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass, replace

import numpy as np

from .errors import ContractError

__all__ = [
    "DeviceSpec", "LinkSpec", "WorkloadShape", "BaselineBreakdown", "HybridBreakdown",
    "attention_cost", "kv_bytes", "merge_bytes", "time_offload_baseline", "time_hybrid",
    "speedup_heatmap", "heatmap_rows", "HEATMAP_COLUMNS", "DEFAULT_GPU", "DEFAULT_CPU", "DEFAULT_LINK",
    "B200", "B200_DECODE", "FIXED_S", "B200_DECODE_GRAPH", "FIXED_GRAPH_S", "NVLINK5", "PCIE5", "b200_spec", "DecodeShape", "DecodeBreakdown", "union_rows",
    "predict_decode", "predict_sharded", "fit_decode",
]


# ====================================================================== specs
@dataclass(frozen=True)
class DeviceSpec:
    """perf_model.py:39-47: a roofline device (ops/s, bytes/s)."""
    name: str
    peak_flops: float
    mem_bw: float

    def __post_init__(self):
        if not (self.peak_flops > 0 and self.mem_bw > 0):
            raise ContractError("device peak_flops and mem_bw must be positive")


@dataclass(frozen=True)
class LinkSpec:
    """perf_model.py:50-59: a transfer link (bytes/s, seconds per transfer)."""
    bw: float
    latency: float

    def __post_init__(self):
        if not self.bw > 0:
            raise ContractError("link bw must be positive")
        if self.latency < 0:
            raise ContractError("link latency must be >= 0")


# the reference's commodity points (perf_model.py:62-66)
DEFAULT_GPU = DeviceSpec("gpu", peak_flops=38.7e12, mem_bw=768e9)
DEFAULT_CPU = DeviceSpec("cpu", peak_flops=1.229e12, mem_bw=500e9)
DEFAULT_LINK = LinkSpec(bw=32e9, latency=10e-6)


def b200_spec(peaks_path: str | None = None) -> DeviceSpec:
    """B200 with the measured HBM copy bandwidth of this pool (MEASURED_PEAKS.json
    ``hbm_gbs``; 6,546 GB/s when absent) and the dense bf16 tensor peak."""
    bw, flops = 6546e9, 2.25e15
    path = peaks_path or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                      "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        bw = float(p.get("hbm_gbs", bw / 1e9)) * 1e9
        flops = float(p.get("bf16_tflops", flops / 1e12)) * 1e12
    except (OSError, ValueError):
        pass
    return DeviceSpec("b200", peak_flops=flops, mem_bw=bw)


B200 = b200_spec()
NVLINK5 = LinkSpec(bw=900e9, latency=12e-6)   # per direction through NVSwitch; small-message NCCL latency
PCIE5 = LinkSpec(bw=55e9, latency=10e-6)      # x16 Gen5, effective host<->device


# =============================================================== reference model
@dataclass(frozen=True)
class WorkloadShape:
    """perf_model.py:69-89: one layer-step of attention (heads = query heads = kv heads)."""
    batch: int = 1
    heads: int = 32
    head_dim: int = 128
    n_window: int = 1024
    n_store: int = 0
    n_selected: int = 0
    n_q: int = 1
    bytes_per_elem: int = 2

    def __post_init__(self):
        bad = [k for k, v in vars(self).items() if v < 0]
        if bad:
            raise ContractError(f"{bad[0]} must be >= 0")
        if self.n_selected > self.n_store:
            raise ContractError("n_selected cannot exceed n_store")

    def with_(self, **kw) -> "WorkloadShape":
        return replace(self, **kw)


def kv_bytes(n_kv: int, shape: WorkloadShape) -> float:
    """K and V bytes of n_kv entries per head (perf_model.py:92-94)."""
    return 2.0 * shape.batch * shape.heads * n_kv * shape.head_dim * shape.bytes_per_elem


def merge_bytes(shape: WorkloadShape) -> float:
    """One output row plus one lse per query row and head (perf_model.py:97-99)."""
    return shape.batch * shape.heads * shape.n_q * (shape.head_dim + 1) * shape.bytes_per_elem


def attention_cost(n_kv: int, shape: WorkloadShape, device: DeviceSpec) -> float:
    """Roofline seconds of one pass over n_kv keys per head (perf_model.py:102-117):
    4 flops per (query, key, dim); bytes = KV + q and out."""
    if n_kv < 0:
        raise ContractError("n_kv must be >= 0")
    if n_kv == 0:
        return 0.0
    rows = shape.batch * shape.heads * shape.n_q
    t_math = rows * n_kv * 4.0 * shape.head_dim / device.peak_flops
    t_mem = (kv_bytes(n_kv, shape) + 2.0 * rows * shape.head_dim * shape.bytes_per_elem) / device.mem_bw
    return max(t_math, t_mem)


@dataclass(frozen=True)
class BaselineBreakdown:
    transfer: float
    compute: float

    @property
    def total(self) -> float:
        return self.transfer + self.compute


@dataclass(frozen=True)
class HybridBreakdown:
    gpu_part: float
    cpu_part: float
    merge: float

    @property
    def total(self) -> float:
        return max(self.gpu_part, self.cpu_part) + self.merge


def time_offload_baseline(shape: WorkloadShape, gpu: DeviceSpec, link: LinkSpec) -> BaselineBreakdown:
    """Move the store tier to the device, then attend everything (perf_model.py:145-150)."""
    return BaselineBreakdown(
        transfer=link.latency + kv_bytes(shape.n_store, shape) / link.bw,
        compute=attention_cost(shape.n_window + shape.n_store + shape.n_q, shape, gpu))


def time_hybrid(shape: WorkloadShape, gpu: DeviceSpec, cpu: DeviceSpec, link: LinkSpec,
                core_efficiency: float = 0.5) -> HybridBreakdown:
    """Window on the device overlapped with the selected entries on the host,
    then the merge transfer (perf_model.py:153-166)."""
    if not 0.0 < core_efficiency <= 1.0:
        raise ContractError(f"core_efficiency must be in (0, 1], got {core_efficiency}")
    return HybridBreakdown(
        gpu_part=attention_cost(shape.n_window + shape.n_q, shape, gpu),
        cpu_part=attention_cost(shape.n_selected, shape, cpu) / core_efficiency,
        merge=link.latency + merge_bytes(shape) / link.bw)


def _cells(n_window_values, n_store_values, shape, retention_fraction, batches=None):
    for b in (batches if batches is not None else (None,)):
        for n_w in n_window_values:
            for n_s in n_store_values:
                kw = dict(n_window=int(n_w), n_store=int(n_s), n_selected=int(round(retention_fraction * n_s)))
                if b is not None:
                    kw["batch"] = int(b)
                yield shape.with_(**kw)


HEATMAP_COLUMNS = ["n_window", "n_store", "batch", "t_baseline_transfer", "t_baseline_compute",
                   "t_hybrid_gpu", "t_hybrid_cpu", "t_merge", "speedup"]


def speedup_heatmap(n_window_values, n_store_values, shape: WorkloadShape, gpu: DeviceSpec = DEFAULT_GPU,
                    cpu: DeviceSpec = DEFAULT_CPU, link: LinkSpec = DEFAULT_LINK, core_efficiency: float = 0.5,
                    retention_fraction: float = 0.2) -> np.ndarray:
    """[len(windows), len(stores)] baseline/hybrid time ratios (perf_model.py:169-191)."""
    if len(n_window_values) == 0 or len(n_store_values) == 0:
        raise ContractError("heatmap grid must be non-empty")
    vals = [time_offload_baseline(c, gpu, link).total / time_hybrid(c, gpu, cpu, link, core_efficiency).total
            for c in _cells(n_window_values, n_store_values, shape, retention_fraction)]
    return np.array(vals, dtype=np.float64).reshape(len(n_window_values), len(n_store_values))


def heatmap_rows(n_window_values, n_store_values, batch_values, shape: WorkloadShape, gpu: DeviceSpec = DEFAULT_GPU,
                 cpu: DeviceSpec = DEFAULT_CPU, link: LinkSpec = DEFAULT_LINK, core_efficiency: float = 0.5,
                 retention_fraction: float = 0.2) -> list:
    """Per-cell breakdown rows in HEATMAP_COLUMNS order (perf_model.py:199-223)."""
    out = []
    for c in _cells(n_window_values, n_store_values, shape, retention_fraction, batch_values):
        base, hyb = time_offload_baseline(c, gpu, link), time_hybrid(c, gpu, cpu, link, core_efficiency)
        out.append([c.n_window, c.n_store, c.batch, base.transfer, base.compute, hyb.gpu_part, hyb.cpu_part,
                    hyb.merge, base.total / hyb.total])
    return out


# ============================================================ B200-native model
@dataclass(frozen=True)
class DecodeShape:
    """One decode layer-step of this framework: GQA, both tiers resident in HBM."""
    batch: int = 16
    q_heads: int = 32
    kv_heads: int = 8
    head_dim: int = 128
    window: int = 512          # attended window rows per (batch, kv head), incl. the new token
    archive: int = 32256       # archive entries per (batch, kv head)
    frac: float = 0.10         # selected fraction per query head
    bytes_per_elem: int = 2
    sparse_rows: int = 256     # rows per sparse work item
    overlap: float = 0.0       # selection overlap between a group's heads: 0 independent, 1 identical

    def __post_init__(self):
        if self.q_heads % max(self.kv_heads, 1) or self.kv_heads < 1:
            raise ContractError("q_heads must be a positive multiple of kv_heads")
        if not 0.0 <= self.frac <= 1.0 or not 0.0 <= self.overlap <= 1.0:
            raise ContractError("frac and overlap must be in [0, 1]")

    @property
    def group(self) -> int:
        return self.q_heads // self.kv_heads

    def with_(self, **kw) -> "DecodeShape":
        return replace(self, **kw)


def union_rows(s: DecodeShape) -> float:
    """Expected union rows per (batch, kv head): independent selections of
    fraction f by G heads cover 1-(1-f)^G of the archive; identical ones f."""
    indep = 1.0 - (1.0 - s.frac) ** s.group
    return s.archive * (s.overlap * s.frac + (1.0 - s.overlap) * indep)


@dataclass(frozen=True)
class DecodeBreakdown:
    dense_bytes: float
    sparse_bytes: float
    other_bytes: float
    t_memory: float
    t_fixed: float
    t_exchange: float = 0.0

    @property
    def bytes(self) -> float:
        return self.dense_bytes + self.sparse_bytes + self.other_bytes

    @property
    def total(self) -> float:
        return self.t_memory + self.t_fixed + self.t_exchange


# fit_decode over the 18 bf16 round-1 points (profiles/r01_configs_timing.jsonl; C3, C4, C5):
# t = 24.5 us + bytes / 7.35 TB/s (the marginal rate is read-dominated: the pure-read probe
# reaches 7.19 TB/s, the copy peak counts reads and writes). Median |error| 6%.
FIXED_S = 24.5e-6   # per layer-step: launch, pipeline fill, merge tail
B200_DECODE = DeviceSpec("b200-decode-fit", peak_flops=2.25e15, mem_bw=7.35e12)
# Round 2, graph mode (DecodeGraph: PDL-chained replays, whole step incl. launch gaps and
# evictions), 18 bf16 points of profiles/r02_configs_timing_final.jsonl (C3, C4, C5 sweep):
# t = 13.0 us + bytes / 6.66 TB/s, median |error| 6.0% (profiles/r02_costmodel_check_graph.txt).
FIXED_GRAPH_S = 13.0e-6
B200_DECODE_GRAPH = DeviceSpec("b200-decode-graph-fit", peak_flops=2.25e15, mem_bw=6.66e12)


def _decode_bytes(s: DecodeShape, union: float):
    BK, rowpair = s.batch * s.kv_heads, 2 * s.head_dim * s.bytes_per_elem
    dense = BK * s.window * rowpair
    sparse = BK * union * (rowpair + 4)                             # rows + union entries
    items = BK * (math.ceil(s.window / 256) + math.ceil(union / s.sparse_rows) + 2)
    partials = items * s.group * (s.head_dim * 4 + 16) * 2          # written, then read by the merge
    bq = s.batch * s.q_heads
    other = (bq * s.head_dim * s.bytes_per_elem                      # q
             + bq * s.window * (4 + 8 * 2)                           # dense scores, window MAW r/w
             + bq * (s.head_dim * 4 + 8) + partials)                 # out, lse
    return dense, sparse, other


def predict_decode(s: DecodeShape, device: DeviceSpec = B200_DECODE, fixed_s: float = FIXED_S) -> DecodeBreakdown:
    """Time of one decode layer-step: algorithmic bytes at the HBM bandwidth plus a fixed cost."""
    dense, sparse, other = _decode_bytes(s, union_rows(s))
    return DecodeBreakdown(dense, sparse, other, (dense + sparse + other) / device.mem_bw, fixed_s)


def predict_sharded(s: DecodeShape, ranks: int, device: DeviceSpec = B200_DECODE, link: LinkSpec = NVLINK5,
                    fixed_s: float = FIXED_S) -> DecodeBreakdown:
    """Sequence-sharded step (DESIGN.md §(e)): every rank attends the window
    and 1/P of the archive, then one all-gather of the packed (out f32, lse
    f64) partials -- (P-1) * B*Hq*(4D+8) bytes into each rank -- and the P-way merge."""
    if ranks < 1:
        raise ContractError("ranks must be >= 1")
    part = predict_decode(s.with_(archive=int(math.ceil(s.archive / ranks))), device, fixed_s)
    if ranks == 1:
        return part
    packed = s.batch * s.q_heads * (4 * s.head_dim + 8)
    xchg = link.latency + (ranks - 1) * packed / link.bw + ranks * packed / device.mem_bw
    return replace(part, t_exchange=xchg)


def fit_decode(points) -> tuple[float, float]:
    """Least-squares (fixed seconds, bytes/s) of t = fixed + bytes/bw over
    measured (bytes, seconds) points."""
    pts = np.asarray(list(points), dtype=np.float64)
    if pts.ndim != 2 or pts.shape[0] < 2:
        raise ContractError("fit_decode needs at least two (bytes, seconds) points")
    A = np.stack([np.ones(len(pts)), pts[:, 0]], axis=1)
    (fixed, inv_bw), *_ = np.linalg.lstsq(A, pts[:, 1], rcond=None)
    if inv_bw <= 0:
        raise ContractError("measured points do not grow with bytes")
    return float(fixed), float(1.0 / inv_bw)
