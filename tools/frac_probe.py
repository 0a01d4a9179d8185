import json, sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch, bench, bench_configs
for frac in (0.1, 0.5, 1.01):
    cfgd = dict(bench.C2, batch=4, context=32768, frac=frac)
    r = bench_configs.measure(cfgd, steps=30, warmup=3, name=f"frac {frac}", graph_steps=30)
    print(json.dumps({k: r[k] for k in ("config", "union_rows", "bytes_per_layer_step", "layer_step_kernel_ms", "achieved_gbs", "graph_ms_per_step", "graph_achieved_gbs")}), flush=True)
    torch.cuda.empty_cache()
