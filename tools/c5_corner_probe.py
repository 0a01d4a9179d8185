"""Graph-mode step time of the C5 corners (big windows with small unions) and the
headline shapes; used for the item-sizing A/B (HGCA_ITEMS_COUNT_WINDOW)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402
import bench  # noqa: E402
import bench_configs  # noqa: E402

out = []
for blk, frac in ((256, 0.01), (128, 0.01), (256, 0.05), (8, 0.01), (32, 0.01), (32, 0.05)):
    cfgd = dict(bench.C2, batch=4, context=65536, blk_num=blk, frac=frac)
    r = bench_configs.measure(cfgd, steps=20, warmup=3, name="C5", graph_steps=100)
    out.append(f"W{blk * 32}/{frac}: {r['graph_ms_per_step'] * 1e3:.1f}")
    torch.cuda.empty_cache()
print(" | ".join(out), flush=True)
