"""Synthetic decode workloads on the device, and the reference's workload file format.

Two things the hot path's callers need:

* ``load_workload`` / ``save_workload`` read and write the reference's text
  format (``workload.py:185-236``: one JSON header line with ``"tierkv_workload": 1``
  and sorted keys, then per step ``mode start n_q <q> <k> <v>`` with each array
  base64 of little-endian float32 ``[layers, heads, n_q, head_dim]``), so a file
  written by ``tierkv.save_workload`` loads here bit-exactly and a file written
  here loads in ``tierkv.load_workload``. Arrays land as torch tensors, optionally
  straight on a device.
* ``gen_workload_device`` builds the reference generator's planted structure
  (``workload.py:124-182``) with batched tensor ops on the target device, so a
  128K-token, 32-head layer takes about a second (B200) instead of minutes of
  host numpy work.
  Per (layer, head) an orthonormal frame (u, w):
      q_p = lam*p*u + w;   k_j = lam*j*w + noise_j     (recency: q_p . k_j grows with j)
      sink k = u + noise;  i-th heavy hitter k = u + (i+1)*ln(boost)/scale*w + noise
  with lam = ln(1/decay)/scale and noise projected off u. The random draws come
  from a torch generator seeded with ``spec.seed`` (Philox on CUDA), so the stream
  is deterministic per (seed, device type) but NOT numpy's PCG64 stream: use
  the file format (or the test oracle's restatement) when bit-identical inputs
  to the reference's own generator are required.
"""

from __future__ import annotations

import base64
import json
import math
from dataclasses import asdict, dataclass, field

import numpy as np
import torch

from .errors import ContractError

__all__ = ["WorkloadSpec", "WorkloadStep", "Workload", "step_plan", "gen_workload_device",
           "load_workload", "save_workload"]

FORMAT_KEY = "tierkv_workload"   # workload.py:190 header marker, version 1


@dataclass(frozen=True)
class WorkloadSpec:
    """Same fields, defaults and validation as the reference's spec (workload.py:40-74)."""

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
        if not 0.0 < self.recency_decay < 1.0:
            raise ContractError(f"recency_decay must be in (0, 1), got {self.recency_decay}")
        for name in ("steps", "prefill_len", "sink_count", "heavy_hitter_count"):
            if getattr(self, name) < 0:
                raise ContractError(f"{name} must be >= 0")
        if self.heavy_hitter_boost < 0 or self.noise_scale < 0:
            raise ContractError("heavy_hitter_boost and noise_scale must be >= 0")
        events = tuple(sorted((int(s), int(n)) for s, n in self.append_events))
        seen = set()
        for s, n in events:
            if not 0 <= s < self.steps:
                raise ContractError(f"append event at step {s} outside [0, {self.steps})")
            if n < 1:
                raise ContractError(f"append event at step {s} has n_q={n} < 1")
            if s in seen:
                raise ContractError(f"two append events at step {s}")
            seen.add(s)
        object.__setattr__(self, "append_events", events)


def step_plan(spec: WorkloadSpec) -> list[tuple[str, int]]:
    """(mode, n_q) per step: the prefill append, then one decode per step
    except where an append event replaces it (workload.py:111-121)."""
    events = dict(spec.append_events)
    plan = [("append", spec.prefill_len)] if spec.prefill_len else []
    plan += [("append", events[s]) if s in events else ("decode", 1) for s in range(spec.steps)]
    return plan


@dataclass
class WorkloadStep:
    index: int
    mode: str
    start: int
    q: torch.Tensor       # [layers, heads, n_q, head_dim] float32 (views into the workload)
    keys: torch.Tensor
    values: torch.Tensor

    @property
    def n_q(self) -> int:
        return int(self.q.shape[2])


@dataclass
class Workload:
    layers: int
    heads: int
    head_dim: int
    scale: float
    spec: WorkloadSpec | None
    steps: list = field(default_factory=list)

    def __iter__(self):
        return iter(self.steps)

    def __len__(self):
        return len(self.steps)

    @property
    def total_entries(self) -> int:
        return sum(s.n_q for s in self.steps)

    def history(self, layer: int, upto: int | None = None):
        """(q, k, v) [heads, n, head_dim] of positions [0, upto) of one layer."""
        qs, ks, vs, n = [], [], [], 0
        for s in self.steps:
            if upto is not None and n >= upto:
                break
            qs.append(s.q[layer]); ks.append(s.keys[layer]); vs.append(s.values[layer])
            n += s.n_q
        q, k, v = (torch.cat(x, dim=1) for x in (qs, ks, vs))
        return (q, k, v) if upto is None else (q[:, :upto], k[:, :upto], v[:, :upto])


def _split_steps(plan, q, k, v):
    steps, cur = [], 0
    for i, (mode, n) in enumerate(plan):
        sl = slice(cur, cur + n)
        steps.append(WorkloadStep(i, mode, cur, q[:, :, sl], k[:, :, sl], v[:, :, sl]))
        cur += n
    return steps


def gen_workload_device(spec: WorkloadSpec, heads: int, head_dim: int, layers: int, scale: float | None = None,
                        device="cuda", dtype=torch.float32) -> Workload:
    """The planted-structure stream of ``spec`` generated on ``device`` (see module doc)."""
    if layers < 1 or heads < 1 or head_dim < 2:
        raise ContractError("layers, heads >= 1 and head_dim >= 2 required")
    scale = 1.0 / math.sqrt(head_dim) if scale is None else float(scale)
    dev = torch.device(device)
    gen = torch.Generator(device=dev)
    gen.manual_seed(int(spec.seed))
    plan = step_plan(spec)
    total = sum(n for _, n in plan)
    lam = math.log(1.0 / spec.recency_decay) / scale
    f64 = dict(dtype=torch.float64, device=dev)

    # token coefficients along (u, w): recency ramp, sinks, heavy hitters
    pos = torch.arange(total, **f64)
    cu = torch.zeros(total, **f64)
    cw = lam * pos
    ns = min(spec.sink_count, total)
    cu[:ns] = 1.0
    cw[:ns] = 0.0
    lo, hi = spec.sink_count, max(spec.sink_count + 1, total // 4)
    pool = min(hi, total) - lo
    if spec.heavy_hitter_count and spec.heavy_hitter_boost > 0 and pool > 0:
        cnt = min(spec.heavy_hitter_count, pool)
        hh = torch.sort(lo + torch.randperm(pool, generator=gen, device=dev)[:cnt]).values
        cu[hh] = 1.0
        cw[hh] = torch.arange(1, cnt + 1, **f64) * (math.log(spec.heavy_hitter_boost) / scale)

    # orthonormal frames [layers*heads, d]
    LH = layers * heads
    u = torch.randn((LH, head_dim), generator=gen, **f64)
    u = u / u.norm(dim=1, keepdim=True)
    w = torch.randn((LH, head_dim), generator=gen, **f64)
    w = w - (w * u).sum(dim=1, keepdim=True) * u
    w = w / w.norm(dim=1, keepdim=True)

    q = torch.empty((layers, heads, total, head_dim), dtype=dtype, device=dev)
    k = torch.empty_like(q)
    v = torch.randn((layers, heads, total, head_dim), generator=gen, dtype=torch.float32, device=dev).to(dtype)
    # keys / queries are float32 (as the reference stores them): the frame is
    # built in fp64 above, the per-token assembly and the noise in fp32
    qf, kf = q.view(LH, total, head_dim), k.view(LH, total, head_dim)
    step = max(1, (1 << 28) // max(1, total * head_dim))   # (layer, head) pairs per batch: <= 1 GB of noise
    f32 = dict(dtype=torch.float32, device=dev)
    ramp, cu32, cw32 = (lam * pos).float()[None, :, None], cu.float()[None, :, None], cw.float()[None, :, None]
    u32, w32 = u.float(), w.float()
    for i0 in range(0, LH, step):
        i1 = min(LH, i0 + step)
        U, Wf = u32[i0:i1, None, :], w32[i0:i1, None, :]                 # [n, 1, d]
        noise = torch.randn((i1 - i0, total, head_dim), generator=gen, **f32)
        noise -= (noise * U).sum(dim=2, keepdim=True) * U                 # keep q's growing u-term noise-free
        kf[i0:i1] = (cu32 * U + cw32 * Wf + spec.noise_scale * noise).to(dtype)
        qf[i0:i1] = (ramp * U + Wf).to(dtype)
        del noise
    return Workload(layers, heads, head_dim, scale, spec, _split_steps(plan, q, k, v))


# ------------------------------------------------------------------ file format
def _enc(t: torch.Tensor) -> str:
    a = t.detach().to("cpu", torch.float32).contiguous().numpy().astype("<f4", copy=False)
    return base64.b64encode(a.tobytes()).decode()


def save_workload(wl: Workload, path) -> None:
    """Write ``wl`` in the reference's text format (workload.py:189-210)."""
    header = {FORMAT_KEY: 1, "layers": wl.layers, "heads": wl.heads, "head_dim": wl.head_dim,
              "scale": wl.scale, "steps": len(wl.steps), "total_entries": wl.total_entries}
    if wl.spec is not None:
        header["spec"] = asdict(wl.spec)
    with open(path, "w") as f:
        f.write(json.dumps(header, sort_keys=True) + "\n")
        for s in wl.steps:
            f.write(f"{s.mode} {s.start} {s.n_q} {_enc(s.q)} {_enc(s.keys)} {_enc(s.values)}\n")


def load_workload(path, device=None) -> Workload:
    """Read a reference workload file (workload.py:213-236) into float32 tensors
    on ``device`` (host memory when None). Foreign or truncated files raise
    ContractError."""
    with open(path) as f:
        try:
            header = json.loads(f.readline())
        except json.JSONDecodeError as e:
            raise ContractError(f"{path}: header is not JSON ({e})") from None
        if not isinstance(header, dict) or header.get(FORMAT_KEY) != 1:
            raise ContractError(f"{path} is not a tierkv workload file")
        L, H, D = int(header["layers"]), int(header["heads"]), int(header["head_dim"])
        spec = None
        if "spec" in header:
            raw = dict(header["spec"])
            raw["append_events"] = tuple(tuple(e) for e in raw.get("append_events", ()))
            spec = WorkloadSpec(**raw)
        steps = []
        for i in range(int(header["steps"])):
            parts = f.readline().split()
            if len(parts) != 6:
                raise ContractError(f"{path}: step {i} is truncated or malformed")
            mode, start, n_q = parts[0], int(parts[1]), int(parts[2])
            arrs = []
            for blob in parts[3:]:
                a = np.frombuffer(base64.b64decode(blob), dtype="<f4")
                if a.size != L * H * n_q * D:
                    raise ContractError(f"{path}: step {i} holds {a.size} values, expected {L * H * n_q * D}")
                t = torch.from_numpy(a.astype(np.float32).reshape(L, H, n_q, D))
                arrs.append(t.to(device) if device is not None else t)
            steps.append(WorkloadStep(i, mode, start, *arrs))
    return Workload(L, H, D, float(header["scale"]), spec, steps)
