"""Time append (re-evaluation) steps at C2 scale: n_q new tokens attend the
whole archive (engine.py:127-132) and the window, merge, MAW re-evaluation +
re-selection (sparsifier.py:158-177). Reports the step (CUDA events) and the
attention kernels alone (hgca_append_bf16 under ncu: see DESIGN.md)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_03153_b200 as hg  # noqa: E402

cfgd = dict(bench.C2)
if len(sys.argv) > 1:
    cfgd["context"] = int(sys.argv[1])
eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 2048, seed=3)
B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
nqs = [int(x) for x in os.environ.get("HGCA_APPEND_NQ", "1,16,64,1,16,64").split(",")]
for i, nq in enumerate(nqs):
    q = torch.randn((B, Hq, nq, D), generator=g, device="cuda").to(eng.tdtype)
    k = torch.randn((B, Hkv, nq, D), generator=g, device="cuda").to(eng.tdtype)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    last = i == len(nqs) - 1
    if last and os.environ.get("HGCA_PROBE_PROFILE_LAST"):  # ncu --profile-from-start off: the last append only
        torch.cuda.cudart().cudaProfilerStart()
    e0.record()
    eng.step(0, hg.StepInput("append", q, k, k))
    e1.record()
    torch.cuda.synchronize()
    if last and os.environ.get("HGCA_PROBE_PROFILE_LAST"):
        torch.cuda.cudart().cudaProfilerStop()
    lo = eng.layers[0].lo
    gb = B * Hkv * (lo + eng.layers[0].window_size) * 2 * D * 2 / 1e9
    print(f"append n_q={nq}: {e0.elapsed_time(e1):.3f} ms (archive {lo}, batch {B}; K|V {gb:.2f} GB read "
          f"twice -> {2 * gb / (e0.elapsed_time(e1) * 1e-3):.0f} GB/s)", flush=True)
