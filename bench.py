#!/usr/bin/env python
"""Hybrid decode-attention benchmark (BASELINE.json metric).

Workload (N=1): BASELINE.json configs[1] = "C2": Llama-3-8B GQA shape
(32 query / 8 KV heads, d=128), batch 16, 32K context, bf16, one attention
layer; 512-token dense window (16 blocks x 32) + per-head threshold-selected
context over the 32,256-entry archive with ~10% of entries per query head
selected (SURVEY.md §8(d) Config 2). A "step" is one decode layer-step of the
whole batch through the device engine: kv_in write, fused dense + sparse
partial kernel, merge + MAW EMA kernel, and (every 32 steps) eviction ->
ingest -> union rebuild. tokens/s = batch / step time.

value : inputs resident in HBM, CUDA events on the launching stream.
e2e   : the same step through HybridEngine.decode_host (C ABI) with pinned HOST
        q/k/v copied in and out/lse copied back + synchronized every step.
L2    : K/V (2.1 GB) >> L2 (126 MB): inputs larger than L2, no flush needed.

--impl reference: the reference's own CPU hot path (oracle/_ref compiled from
the reference's _core.pyx, else the oracle's C restatement) on every host
core, same workload/metric (bench arm for the driver's ratio).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2 = dict(batch=16, heads=32, kv_heads=8, head_dim=128, context=32768, blk_num=16, blk_size=32,
          beta=1.0, alpha=0.5, frac=0.10, dtype="bfloat16")
WORKLOAD = ("C2: Llama-3-8B GQA 32q/8kv d128, batch 16, 32K context, bf16, 512-token dense window "
            "+ threshold-selected 10%/head archive context, 1 layer")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--shard", default="seq", choices=["seq", "batch"],
                    help="N>1: 'seq' shards the KV sequence of the C2 batch over the ranks (one NCCL "
                         "all-gather of (out, lse) partials per step; strong scaling, the north star's "
                         "mode); 'batch' runs one independent C2 batch per rank (weak scaling)")
    ap.add_argument("--exchange", default="push", choices=["push", "allgather"],
                    help="--shard seq: 'push' = the merge kernel stores each rank's (out, lse) partial into "
                         "every peer's HBM box over NVLink (CUDA IPC) and the P-way merge waits on device "
                         "flags; 'allgather' = one NCCL all_gather_into_tensor per step")
    return ap.parse_args()


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU is busy."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.05)

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.perf_counter(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [r for t, r in self.rows if t0 <= t <= t1] or [r for _, r in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------- ours
def stage_engine(hg, torch, cfgd, max_positions, seed=0, sharded=False, layers=1, exchange="allgather"):
    """Build the engine and stage a 32K context: bulk-ingest the archive with
    MAW drawn so that ~frac of entries per query head pass beta/divisor, then
    decode until the window reaches its steady state. sharded: every rank
    stages the same sequence (same seed) into a ShardedHybridEngine, which
    keeps only its own archive blocks selectable."""
    B, Hq, Hkv, D = cfgd["batch"], cfgd["heads"], cfgd["kv_heads"], cfgd["head_dim"]
    cap = cfgd["blk_num"] * cfgd["blk_size"]
    cfg = hg.EngineConfig(layers=layers, heads=Hq, kv_heads=Hkv, head_dim=D, batch=B, dtype=cfgd["dtype"],
                          cache=hg.CacheConfig(blk_num=cfgd["blk_num"], blk_size=cfgd["blk_size"],
                                               alpha=cfgd["alpha"], beta=cfgd["beta"]),
                          core_count=10 ** 6, max_positions=max_positions)
    if sharded:
        try:
            eng = hg.ShardedHybridEngine(cfg, exchange=exchange)
        except RuntimeError as e:  # e.g. no CUDA IPC between these GPUs: keep the run, use NCCL
            print(f"[bench] push exchange unavailable ({e}); falling back to the NCCL all-gather", file=sys.stderr)
            eng = hg.ShardedHybridEngine(cfg, exchange="allgather")
    else:
        eng = hg.HybridEngine(cfg)
    g = torch.Generator(device="cuda").manual_seed(seed)
    tdt = eng.tdtype
    n_arch = cfgd["context"] - cap
    divisor = cap
    thr = cfgd["beta"] / divisor
    for layer in range(layers):
        k = torch.randn((B, Hkv, n_arch, D), generator=g, device="cuda").to(tdt)
        v = torch.randn((B, Hkv, n_arch, D), generator=g, device="cuda").to(tdt)
        u = torch.rand((B, Hq, n_arch), generator=g, device="cuda", dtype=torch.float64)
        maw = torch.where(u < cfgd["frac"], thr * (1.0 + u), thr * u)
        eng.bulk_ingest(layer, k, v, maw, divisor)
        del k, v, u, maw
    for _ in range(cap - 1):
        q = torch.randn((B, Hq, 1, D), generator=g, device="cuda").to(tdt)
        kk = torch.randn((B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
        for layer in range(layers):
            eng.decode_device(layer, q, kk, kk)
    torch.cuda.synchronize()
    return eng, g


def partial_bytes(eng, W_avg, U_avg, n_items):
    """Algorithmic HBM bytes of one decode kernel launch:
    dense K|V rows of the window, unique union K|V rows + their 4-byte union
    entries, the queries, the dense scores (written, re-read by the dense
    epilogue), the per-item partials (written + re-read by the fold), the MAW
    of the window (read + written, fp64) and out/lse."""
    B, Hq, Hkv, D, G = eng.B, eng.Hq, eng.Hkv, eng.D, eng.G
    e = 2 if eng.tdtype.itemsize == 2 else 4
    sc = 4 if e == 2 else 8
    dense = B * Hkv * W_avg * D * 2 * e
    sparse = U_avg * (D * 2 * e + 4)
    q = B * Hq * D * e
    dsc = B * Hq * W_avg * sc * 2
    partials = n_items * G * (D * 4 + 16) * 2
    maw = B * Hq * W_avg * 8 * 2
    out = B * Hq * (D * 4 + 8)
    return dense + sparse + q + dsc + partials + maw + out, dense, sparse


def run_ours(args, rank, world):
    import numpy as np
    import torch

    import paper_2507_03153_b200 as hg

    local = int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
        backend = os.environ.get("HGCA_DIST_BACKEND", "nccl")  # gloo: multi-rank smoke runs on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfgd = dict(C2)
    K, Wm = args.steps, args.warmup
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else min(K, 200)
    cap = cfgd["blk_num"] * cfgd["blk_size"]
    max_positions = cfgd["context"] + Wm + K + e2e_steps + 64
    seq = world > 1 and args.shard == "seq"
    clocks = ClockSampler(local)
    clocks.start()
    eng, g = stage_engine(hg, torch, cfgd, max_positions, seed=1234 if seq else 1234 + rank, sharded=seq,
                          exchange=args.exchange)
    B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
    tdt = eng.tdtype
    qs = torch.randn((Wm + K, B, Hq, 1, D), generator=g, device="cuda").to(tdt)
    ks = torch.randn((Wm + K, B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
    vs = torch.randn((Wm + K, B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
    out = torch.empty((B * Hq, D), dtype=torch.float32, device="cuda")
    lse = torch.empty(B * Hq, dtype=torch.float64, device="cuda")
    ls = eng.layers[0]
    for i in range(Wm):
        eng.decode_device(0, qs[i], ks[i], vs[i], out=out, lse=lse)
    torch.cuda.synchronize()
    exchange_note = None
    if getattr(eng, "xchg", None) is not None:  # push exchange: did every peer flag arrive in time?
        bad = torch.tensor([int(eng.xchg.err.item())])
        if world > 1:
            if dist.get_backend() == "nccl":
                bad = bad.cuda()
            dist.all_reduce(bad)
        if int(bad.item()):
            exchange_note = "push exchange timed out during warm-up; measured with the NCCL all-gather"
            print(f"[bench] {exchange_note}", file=sys.stderr)
            eng.xchg = None
    U0 = int(ls.u_cnt.sum())
    Ws = []
    eng.step_events = []
    launches0 = eng.launches
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include timed/ captures exactly these steps
    e0.record()
    for i in range(Wm, Wm + K):
        Ws.append(ls.window_size + 1)
        eng.decode_device(0, qs[i], ks[i], vs[i], out=out, lse=lse)
    e1.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    if dist:
        dist.barrier()
    launches = eng.launches - launches0
    ms = e0.elapsed_time(e1) / K
    part_ms = statistics.mean(a.elapsed_time(b) for a, b in eng.step_events)
    eng.step_events = None
    U1 = int(ls.u_cnt.sum())
    ms_max = ms
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_max = float(t)
    # ---- e2e through the public API with HOST buffers: one pinned H2D copy of
    # q|k|v in, the step, one D2H copy of out|lse back, synchronize -- every step
    nin = B * (Hq + 2 * Hkv) * D
    in_h = torch.empty(nin, dtype=tdt).pin_memory()
    in_h.copy_(torch.cat([qs[0].reshape(-1), ks[0].reshape(-1), vs[0].reshape(-1)]).cpu())
    out_h = torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8).pin_memory()
    staging = (torch.empty(nin, dtype=tdt, device="cuda"), torch.empty(out_h.numel(), dtype=torch.uint8, device="cuda"))
    for _ in range(3):
        eng.decode_host_packed(0, in_h, out_h, staging)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        eng.decode_host_packed(0, in_h, out_h, staging)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / max(e2e_steps, 1)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t)
    clocks.stop()
    if getattr(eng, "xchg", None) is not None:
        eng.check_exchange()  # a push timeout in the timed or e2e steps poisons (NaN) and raises here
    oh = out_h[: B * Hq * D * 4].view(torch.float32)
    if not np.isfinite(oh.numpy()).all() and not os.environ.get("HGCA_LIB"):  # HGCA_LIB: experimental builds
        raise RuntimeError("non-finite decode output")
    # ---- roofline of the dominant kernels: one hgca_decode_step = decode kernel + merge kernel
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")  # dram bytes per launch from the ncu --set full captures
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    W_avg = statistics.mean(Ws)
    U_avg = (U0 + U1) / 2
    BK = eng.B * eng.Hkv
    n_items = BK + int(ls.item_off[2 * BK + 1])  # dense items + sparse items of the current selection
    pbytes, dense_b, sparse_b = partial_bytes(eng, W_avg, U_avg, n_items)
    achieved = pbytes / (part_ms * 1e-3) / 1e9
    result = None
    if rank == 0:
        units = B if seq else world * B  # tokens the whole job decodes per step
        tok_s = units / (ms_max * 1e-3)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle import cpu_bench  # checker / baseline only
            cpu = cpu_bench.time_single(Hq, Hkv, D, cfgd["context"] - cap, cap, cfgd["frac"],
                                        sequences=8, reps=30)  # ~10 s of single-thread CPU work
        result = {
            "metric": "hybrid-attn decode tokens/s (1 layer, C2)",
            "value": round(tok_s, 1),
            "unit": "tokens/s",
            "n_gpus": world,
            "steps": K,
            "warmup": Wm,
            "ms_per_step": round(ms_max, 5),
            "higher_is_better": True,
            "scaling": "strong" if seq else "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "numerics": "bf16 storage; QK^T and P.V on mma.sync (fp32 accumulate, P as bf16 hi+lo), "
                        "fp32 softmax, fp64 MAW/merge",
            "data": "synthetic (torch.randn K/V/q, MAW drawn for 10% threshold selection per query head)",
            "config": {"workload": WORKLOAD, "batch": B, "q_heads": Hq, "kv_heads": Hkv, "head_dim": D,
                       "context": cfgd["context"], "window_blocks": f"{cfgd['blk_num']}x{cfgd['blk_size']}",
                       "selected_frac": cfgd["frac"],
                       "parallelism": ("1 GPU" if world == 1 else
                                       f"KV-sequence sharded x{world} (block-cyclic archive; "
                                       + ("one-shot push of packed (out, lse) partials from the merge kernel into "
                                          "the peers' HBM (CUDA IPC / NVLink) + flag-waiting P-way merge"
                                          if getattr(eng, "xchg", None) is not None else
                                          ((exchange_note + "; ") if exchange_note else "") +
                                          "NCCL all-gather of packed (out, lse) partials + P-way merge") + ")"
                                       if seq else
                                       f"batch replicas x{world} (one C2 batch per GPU, no collective)"),
                       "l2": "inputs larger than L2 (K/V 2.1 GB per GPU), no flush"},
            "hbm_gbs_step": round(pbytes / (ms_max * 1e-3) / 1e9, 1),
            "roofline": {"bound": "hbm",
                         "kernel": "hgca::decode_bf16_kernel + hgca::decode_merge_kernel (one hgca_decode_step)",
                         "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4),
                         "traffic": traffic.get("decode_step_bytes"),
                         "traffic_source": traffic.get("source"),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)",
                         "kernel_ms": round(part_ms, 5), "bytes_per_launch": int(pbytes),
                         "dense_bytes": int(dense_b), "sparse_unique_bytes": int(sparse_b),
                         "kernel_share_of_step": round(part_ms / ms, 3)},
            "e2e": {"value": round(units / (e2e_ms * 1e-3), 1), "unit": "tokens/s",
                    "ms_per_step": round(e2e_ms, 4), "steps": e2e_steps,
                    "h2d_bytes_per_step": int(in_h.numel() * in_h.element_size()),
                    "d2h_bytes_per_step": int(out_h.numel()),
                    "api": "HybridEngine.decode_host_packed (pinned host q|k|v in, out|lse back, sync)"},
            "gpu_launches": launches,
            "clocks": clocks.summary(t_wall0 - 1.0, t_wall1),
            "cpu_baseline": cpu,
        }
        if cpu:
            result["cpu_baseline"]["speedup_e2e"] = round(result["e2e"]["value"] / cpu["value"], 1)
    if dist:
        dist.destroy_process_group()
    return result


# ----------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return None
    from oracle import cpu_bench

    cfgd = dict(C2)
    cap = cfgd["blk_num"] * cfgd["blk_size"]
    steps = max(1, min(args.steps, 40))  # ~3 s of work on the box's host cores
    warm = 1
    r = cpu_bench.pool_bench(cfgd["heads"], cfgd["kv_heads"], cfgd["head_dim"], cfgd["context"] - cap, cap,
                             cfgd["frac"], batch=cfgd["batch"], steps=steps, warmup=warm)
    ms = statistics.mean(r["times"]) * 1e3
    tok = cfgd["batch"] / (ms * 1e-3)
    return {
        "impl": "reference",
        "metric": "hybrid-attn decode tokens/s (1 layer, C2)",
        "value": round(tok, 3), "unit": "tokens/s", "n_gpus": world, "steps": steps, "warmup": warm,
        "ms_per_step": round(ms, 2), "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32",
        "numerics": "fp32 (bf16-rounded values upcast), fp64 accumulation (reference _core)",
        "data": "synthetic", "config": {"workload": WORKLOAD, "batch": cfgd["batch"]},
        "cpu_baseline": {"value": round(tok, 3), "unit": "tokens/s", "cores": r["workers"], "kind": r["kind"],
                         "sample": f"{steps} step(s) x full batch of {cfgd['batch']} sequences, one process "
                                   f"per sequence over {r['workers']} host cores (reference is single-threaded "
                                   f"per engine, engine.py:10-11)"},
        "e2e": {"value": round(tok, 3), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if args.impl == "reference":
        res = run_reference(args, rank, world)
    else:
        res = run_ours(args, rank, world)
    if rank == 0 and res is not None:
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
