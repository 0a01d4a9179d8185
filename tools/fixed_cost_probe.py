"""Where the fixed per-layer-step cost goes (small steps: C1, C5 at 1%).

For each config prints: host issue time per decode_device call (no sync),
device time per step over K back-to-back steps (CUDA events), and the
decode+merge pair time per step (events around the launches). Run under
gpurun; for per-kernel device times wrap it in tools/launch_list_cmd.sh
(the timed steps sit in NVTX range "timed").

  python tools/fixed_cost_probe.py [C1|C5S|C1B|EMPTY ...]
"""
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_03153_b200 as hg  # noqa: E402

CFGS = {
    # the reference's fp32 case: MHA 32 heads, batch 1, 4K context, window 512, ~10% selected
    "C1": dict(bench.C2, batch=1, heads=32, kv_heads=32, context=4096, dtype="float32"),
    # the same shape on bf16 storage
    "C1B": dict(bench.C2, batch=1, heads=32, kv_heads=32, context=4096, dtype="bfloat16"),
    # C5 corner: 64K, window 256, 1% selected, batch 4
    "C5S": dict(bench.C2, batch=4, context=65536, blk_num=8, frac=0.01),
    # near-empty: batch 1, 8 heads, window 64, archive 64, 1%
    "EMPTY": dict(bench.C2, batch=1, heads=8, kv_heads=8, context=128, blk_num=2, frac=0.01, dtype="float32"),
    # the north-star shape: B=4, 128K context (bench.py's line)
    "C3": dict(bench.C2, batch=4, context=131072),
    # one layer of the C4 shape (70B GQA 64q/8kv, per-GPU batch shard 8, 16K)
    "C4L": dict(bench.C2, batch=8, heads=64, kv_heads=8, context=16384),
    # the same on bf16 storage, GQA 4:1 (the tensor-core kernel)
    "EMPTYB": dict(bench.C2, batch=1, heads=32, kv_heads=8, context=128, blk_num=2, frac=0.01),
}


def run(name, steps=200, warmup=20):
    cfgd = CFGS[name]
    eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 2 * (steps + warmup) + 256, seed=7)
    B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
    tdt = eng.tdtype
    qs = torch.randn((warmup + steps, B, Hq, 1, D), generator=g, device="cuda").to(tdt)
    ks = torch.randn((warmup + steps, B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
    out = torch.empty((B * Hq, D), dtype=torch.float32, device="cuda")
    lse = torch.empty(B * Hq, dtype=torch.float64, device="cuda")
    for i in range(warmup):
        eng.decode_device(0, qs[i], ks[i], ks[i], out=out, lse=lse)
    torch.cuda.synchronize()
    # host issue rate: launches only (the GPU runs behind)
    t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed")
    e0.record()
    for i in range(warmup, warmup + steps):
        eng.decode_device(0, qs[i], ks[i], ks[i], out=out, lse=lse)
    e1.record()
    torch.cuda.nvtx.range_pop()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    host_us = (t1 - t0) * 1e6 / steps
    dev_us = e0.elapsed_time(e1) * 1e3 / steps
    # pair time with events around each launch pair (adds event overhead)
    eng.step_events = []
    for i in range(warmup, warmup + 50):
        eng.decode_device(0, qs[i % (warmup + steps)], ks[i], ks[i], out=out, lse=lse)
    torch.cuda.synchronize()
    pair_us = statistics.median(a.elapsed_time(b) for a, b in eng.step_events) * 1e3
    eng.step_events = None
    # graph mode: graphs of 16 consecutive steps (kernels chained by PDL, the
    # step state advanced on device), a 1-step graph for the tokens left
    # before each eviction; evictions run eagerly between replays
    g16 = hg.DecodeGraph(eng, layers=[0], steps=16) if eng.cap - eng.layers[0].window_size >= 16 else None
    g1 = hg.DecodeGraph(eng, layers=[0], steps=1)

    def graph_tokens(n):
        done = 0
        while done < n:
            if g16 is not None and g16.room() >= 16 and n - done >= 16:
                g16.step()
                done += 16
            else:
                g1.step()
                done += 1
        return done

    graph_tokens(warmup)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g0, g1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.nvtx.range_push("timed_graph")
    g0.record()
    graph_tokens(steps)
    g1e.record()
    torch.cuda.nvtx.range_pop()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    graph_host_us = (t1 - t0) * 1e6 / steps
    graph_us = g0.elapsed_time(g1e) * 1e3 / steps
    ls = eng.layers[0]
    print(json.dumps({"cfg": name, "dtype": cfgd["dtype"], "B": B, "Hq": Hq, "Hkv": Hkv,
                      "window": ls.window_size, "archive": ls.archive_size, "union_rows": int(ls.u_cnt.sum()),
                      "host_issue_us_per_step": round(host_us, 2), "device_us_per_step": round(dev_us, 2),
                      "pair_us_median": round(pair_us, 2), "graph_host_us_per_step": round(graph_host_us, 2),
                      "graph_device_us_per_step": round(graph_us, 2)}), flush=True)


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for n in (sys.argv[1:] or ["EMPTY", "EMPTYB", "C1", "C1B", "C5S"]):
        run(n)
