"""Predicted vs measured decode layer-steps (paper_2507_03153_b200.costmodel).

  python tools/costmodel_check.py [profiles/r01_configs_timing.jsonl] [--graph]

--graph: fit and compare the whole graph-mode step (graph_ms_per_step / layers: the
step's kernels replayed from CUDA graphs, launch gaps and evictions included) instead
of the decode + merge pair time of eager steps.

1. Fits t = fixed + bytes/bw to the measured bf16 points (tools/bench_configs.py output:
   bytes_per_layer_step, layer_step_kernel_ms).
2. For each measured config: model bytes (DecodeShape, independent selections)
   vs measured algorithmic bytes, and predicted vs measured time.
3. The paper's offload-vs-hybrid comparison (perf_model.py) recalibrated: B200
   HBM + PCIe 5 link, vs the reference's commodity points.
Analytic; runs on CPU.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2507_03153_b200 import costmodel as cm  # noqa: E402


def shape_of(r):
    return cm.DecodeShape(batch=r["batch"], q_heads=r["q_heads"], kv_heads=r["kv_heads"], head_dim=128,
                          window=r["window"], archive=r["context"] - r["window"], frac=r["selected_frac"],
                          bytes_per_elem=2 if r.get("dtype", "bfloat16") == "bfloat16" else 4)


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    graph = "--graph" in sys.argv
    path = args[0] if args else os.path.join(ROOT, "profiles", "r01_configs_timing.jsonl")
    rows = [json.loads(l) for l in open(path) if l.startswith("{")]
    if graph:
        rows = [r for r in rows if "graph_ms_per_step" in r]
        for r in rows:
            r["layer_step_kernel_ms"] = r["graph_ms_per_step"] / r.get("layers", 1)
        print("graph mode: whole-step time per layer-step (DecodeGraph replays)")
    bf = [r for r in rows if r.get("dtype") == "bfloat16"]
    fixed, bw = cm.fit_decode((r["bytes_per_layer_step"], r["layer_step_kernel_ms"] * 1e-3) for r in bf)
    print(f"fit over {len(bf)} bf16 points: fixed {fixed * 1e6:.1f} us + bytes / {bw / 1e9:.0f} GB/s "
          f"(measured copy peak {cm.B200.mem_bw / 1e9:.0f} GB/s)")
    dev = cm.DeviceSpec("b200-fit", cm.B200.peak_flops, bw)
    print(f"{'config':48s} {'U model':>9s} {'U meas':>9s} {'MB model':>9s} {'MB meas':>9s} "
          f"{'us pred':>8s} {'us meas':>8s} {'err':>6s}")
    errs = []
    for r in rows:
        if r.get("dtype") != "bfloat16":
            print(f"{r['config'][:48]:48s} (fp32 reference-exact kernel: fp64 dot products, not HBM-bound; "
                  f"{r['layer_step_kernel_ms'] * 1e3:.1f} us measured)")
            continue
        s = shape_of(r)
        p = cm.predict_decode(s, dev, fixed)
        t_meas = r["layer_step_kernel_ms"] * 1e3
        err = p.total * 1e6 / t_meas - 1
        errs.append(abs(err))
        name = f"{r['config'][:22]} B{r['batch']} {r['context'] // 1024}K W{r['window']} f{r['selected_frac']}"
        print(f"{name:48s} {cm.union_rows(s) * s.batch * s.kv_heads:9.0f} {r['union_rows']:9d} "
              f"{p.bytes / 1e6:9.1f} {r['bytes_per_layer_step'] / 1e6:9.1f} {p.total * 1e6:8.1f} {t_meas:8.1f} "
              f"{err:+6.1%}")
    print(f"median |err| {sorted(errs)[len(errs) // 2]:.1%}, max {max(errs):.1%}")
    c3 = cm.DecodeShape(batch=4, window=512, archive=131072 - 512)
    print("sequence-sharded C3 (B=4, 128K, 10%) predicted on NVLink 5:")
    for P in (1, 2, 4, 8):
        p = cm.predict_sharded(c3, P, dev, cm.NVLINK5, fixed)
        print(f"  P={P}: {p.total * 1e6:7.1f} us per layer-step ({p.t_exchange * 1e6:4.1f} us exchange) "
              f"-> {c3.batch / p.total:9.0f} tokens/s")
    shape = cm.WorkloadShape(batch=16, heads=32, head_dim=128, n_q=1, bytes_per_elem=2)
    print("paper model, offload baseline / hybrid speedup (window 512, 20% retained):")
    for label, gpu, link in (("reference commodity GPU + PCIe4", cm.DEFAULT_GPU, cm.DEFAULT_LINK),
                             ("B200 HBM + PCIe5", cm.B200, cm.PCIE5)):
        hm = cm.speedup_heatmap([512], [4096, 32768, 131072], shape, gpu=gpu, link=link)
        print(f"  {label:34s} store 4K {hm[0, 0]:6.2f}x  32K {hm[0, 1]:6.2f}x  128K {hm[0, 2]:6.2f}x")
    p = cm.predict_decode(cm.DecodeShape(), dev, fixed)
    print(f"this framework, C2 (both tiers in HBM): {p.total * 1e6:.1f} us per layer-step predicted")


if __name__ == "__main__":
    main()
