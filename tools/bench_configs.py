"""The other BASELINE.json configs on one B200 (manual runs; bench.py's driver line is C3, with C2 beside it).

  python tools/bench_configs.py C1      the reference's fp32 case (32 heads, 4K context, batch 1) vs its CPU path
  python tools/bench_configs.py C3      B=4, 128K context (the N=1 point of the sequence-sharded scaling run)
  python tools/bench_configs.py C4      Llama-3-70B shape (64 q / 8 kv heads), 16K context, 80 layers per
                                        decode step; the per-GPU batch shard (B=8 of 64) of the 8-GPU run
  python tools/bench_configs.py C5      sparsity sweep at 64K context: window 256..8K x selected 1..20%

Each prints one JSON line per measured point: tokens/s, ms per step, achieved GB/s of the decode step
kernels over the algorithmic bytes (bench.step_bytes) and the fraction of MEASURED_PEAKS hbm_gbs;
graph_* fields: the same steps replayed from CUDA graphs (hg.DecodeGraph), whole step time incl. evictions.
Data: synthetic randn K/V/q, MAW drawn so the threshold selects the stated fraction per query head.
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_03153_b200 as hg  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def graph_time(eng, steps):
    return bench.graph_time(hg, torch, eng, steps)


def measure(cfgd, layers=1, steps=50, warmup=5, name="", graph_steps=0):
    cap = cfgd["blk_num"] * cfgd["blk_size"]
    eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + steps + warmup + 64 + graph_steps + 16,
                                seed=7, layers=layers)
    B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
    tdt = eng.tdtype
    qs = torch.randn((warmup + steps, B, Hq, 1, D), generator=g, device="cuda").to(tdt)
    ks = torch.randn((warmup + steps, B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
    out = torch.empty((B * Hq, D), dtype=torch.float32, device="cuda")
    lse = torch.empty(B * Hq, dtype=torch.float64, device="cuda")
    for i in range(warmup):
        for layer in range(layers):
            eng.decode_device(layer, qs[i], ks[i], ks[i], out=out, lse=lse)
    torch.cuda.synchronize()
    ls = eng.layers[0]
    U = int(ls.u_cnt.sum())
    Wavg = ls.window_size + 1
    BK = B * Hkv
    n_items = BK * -(-Wavg // 256) + int(ls.item_off[2 * BK + 1])
    eng.step_events = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")
    e0.record()
    for i in range(warmup, warmup + steps):
        for layer in range(layers):
            eng.decode_device(layer, qs[i], ks[i], ks[i], out=out, lse=lse)
    e1.record()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    kern_ms = statistics.mean(a.elapsed_time(b) for a, b in eng.step_events)  # per layer-step
    eng.step_events = None
    pbytes, dense_b, sparse_b, _ = bench.step_bytes(eng, Wavg, U, n_items)
    gbs = pbytes / (kern_ms * 1e-3) / 1e9
    gr = {}
    if graph_steps:
        gms = graph_time(eng, graph_steps)
        gr = {"graph_tokens_per_s": round(B / (gms * 1e-3), 1), "graph_ms_per_step": round(gms, 5),
              "graph_achieved_gbs": round(pbytes * layers / (gms * 1e-3) / 1e9, 1),
              "graph_frac": round(pbytes * layers / (gms * 1e-3) / 1e9 / PEAK, 4)}
    return {**gr, "config": name, "batch": B, "q_heads": Hq, "kv_heads": Hkv, "context": cfgd["context"],
            "window": Wavg, "selected_frac": cfgd["frac"], "layers": layers,
            "tokens_per_s": round(B / (ms * 1e-3), 1), "ms_per_step": round(ms, 4),
            "layer_step_kernel_ms": round(kern_ms, 4), "bytes_per_layer_step": int(pbytes),
            "union_rows": U, "achieved_gbs": round(gbs, 1), "peak_gbs": PEAK, "frac": round(gbs / PEAK, 4),
            "dtype": cfgd["dtype"]}


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "C3"
    base = dict(bench.C2)
    if which == "C1":
        # the reference's own CPU-runnable case: 32 heads d=128 (MHA), batch 1, 4K context,
        # 512-token window, fp32 -- the reference-exact kernel (fp64 dot products)
        cfgd = dict(base, batch=1, heads=32, kv_heads=32, context=4096, dtype="float32")
        r = measure(cfgd, steps=200, warmup=10, name="C1 (fp32, reference-exact path)", graph_steps=400)
        from oracle import cpu_bench  # the reference's CPU path, timed beside it (baseline only)
        cpu = cpu_bench.time_single(32, 32, 128, 4096 - 512, 512, cfgd["frac"], sequences=4, reps=10)
        r["cpu_reference_tokens_per_s"] = round(cpu["value"], 2)
        r["cpu_kind"] = cpu["kind"]
        print(json.dumps(r), flush=True)
    elif which == "C3":
        cfgd = dict(base, batch=4, context=131072)
        print(json.dumps(measure(cfgd, steps=50, name="C3 (1 GPU point)", graph_steps=100)), flush=True)
    elif which == "C4":
        cfgd = dict(base, batch=8, heads=64, kv_heads=8, context=16384)
        r = measure(cfgd, layers=80, steps=10, warmup=2, name="C4 per-GPU batch shard (B=8 of 64), 80 layers",
                    graph_steps=20)
        r["projected_8gpu_tokens_per_s"] = round(8 * r["tokens_per_s"], 1)
        print(json.dumps(r), flush=True)
    elif which == "C4L":  # one layer of the C4 shape: the per-layer-step kernels in isolation
        cfgd = dict(base, batch=8, heads=64, kv_heads=8, context=16384)
        print(json.dumps(measure(cfgd, layers=1, steps=int(os.environ.get("HGCA_STEPS", "100")), warmup=5,
                                 name="C4 shape, one layer")), flush=True)
    elif which == "C5S":  # the small-step corner of C5
        for win_blocks, frac in ((8, 0.01), (8, 0.05), (256, 0.01)):
            cfgd = dict(base, batch=4, context=65536, blk_num=win_blocks, frac=frac)
            print(json.dumps(measure(cfgd, steps=30, warmup=3, name="C5 small", graph_steps=200)), flush=True)
            torch.cuda.empty_cache()
    elif which == "C5":
        for win_blocks in (8, 32, 128, 256):          # window 256 .. 8192 tokens (blocks of 32)
            for frac in (0.01, 0.05, 0.10, 0.20):
                cfgd = dict(base, batch=4, context=65536, blk_num=win_blocks, frac=frac)
                print(json.dumps(measure(cfgd, steps=30, warmup=3, name="C5 sweep", graph_steps=100)), flush=True)
                torch.cuda.empty_cache()
    else:
        raise SystemExit(f"unknown config {which}")


if __name__ == "__main__":
    main()
