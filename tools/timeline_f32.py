"""Per-warp timeline of one fp32 (reference-exact) decode step at C1 (debug
build -DHGCA_TIMELINE): where the small-step fixed cost goes.

usage (GPU box): python paper_2507_03153_b200/_build.py --timeline
                 python tools/timeline_f32.py [C1|EMPTY]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
os.environ.setdefault("HGCA_LIB", os.path.join(ROOT, "paper_2507_03153_b200", "_lib", "libhgca_b200_tl.so"))

import bench  # noqa: E402
import paper_2507_03153_b200 as hg  # noqa: E402
from fixed_cost_probe import CFGS  # noqa: E402

SLOTS = 20


def main():
    torch.cuda.set_device(0)
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    cfgd = CFGS[name]
    eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 64)
    lib = hg._lib.load()
    fn = lib.hgca_debug_timeline
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    fm = lib.hgca_debug_timeline_merge
    fm.argtypes = [ctypes.c_void_p]
    B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
    cfg = (ctypes.c_int64 * 5)()
    hg._lib.call("hgca_decode_config", eng.dcode, D, Hq // Hkv, cfg)
    nc = cfg[0]
    for it in range(3):
        q = torch.randn((B, Hq, 1, D), generator=g, device="cuda").to(eng.tdtype)
        k = torch.randn((B, Hkv, 1, D), generator=g, device="cuda").to(eng.tdtype)
        torch.cuda.synchronize()
        fn(None, 0)
        torch.cuda.synchronize()
        eng.step_events = []
        eng.decode_device(0, q, k, k)
        torch.cuda.synchronize()
        ms = eng.step_events[0][0].elapsed_time(eng.step_events[0][1])
        eng.step_events = None
        n = 148 * nc
        buf = np.zeros(n * SLOTS, np.uint64)
        fn(buf.ctypes.data, n * SLOTS)
        t = buf.reshape(n, SLOTS).astype(np.float64)
        t0 = t[:, 0].min()
        start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
        subs, items = t[:, 2], t[:, 9]
        busy = subs > 0
        first = np.where(t[:, 8] > 0, (t[:, 8] - t0) / 1e3, np.nan)
        cyc = {k: t[busy, i].sum() / max(subs[busy].sum(), 1) for k, i in
               (("wait", 3), ("score", 4), ("softmax_pv", 5), ("issue", 6), ("partial", 7))}
        print(f"--- {name} step {it}: decode+merge {ms * 1e3:.1f} us (events); warps {n} ({nc}/SM), "
              f"busy warps {int(busy.sum())}, stages {int(subs.sum())}, items {int(items.sum())}")
        print("  warp start us: p0 %.2f p50 %.2f max %.2f | end (all) p50 %.2f max %.2f | end (busy) p0 %.2f "
              "p50 %.2f max %.2f" % (start.min(), np.median(start), start.max(), np.median(end), end.max(),
                                      end[busy].min(), np.median(end[busy]), end[busy].max()))
        print("  first stage data ready us: p0 %.2f p50 %.2f max %.2f" % (
            np.nanmin(first), np.nanmedian(first), np.nanmax(first)))
        print("  cycles per stage (busy warps): " + ", ".join(f"{k} {v:.0f}" for k, v in cyc.items()))
        print("  stages per busy warp: min %d p50 %d max %d" % (subs[busy].min(), np.median(subs[busy]),
                                                                  subs[busy].max()))
        mb = np.zeros(4096 * 8, np.uint64)
        fm(mb.ctypes.data)
        tm = (mb.reshape(4096, 8)[: B * Hq, :8].astype(np.float64) - t0) / 1e3
        print("  merge CTAs (us): resident p0 %.2f max %.2f | after wait p0 %.2f max %.2f | folds done max %.2f "
              "| epilogue end p50 %.2f max %.2f" % (tm[:, 0].min(), tm[:, 0].max(), tm[:, 1].min(), tm[:, 1].max(),
                                                     tm[:, 3].max(), np.median(tm[:, 5]), tm[:, 5].max()))


if __name__ == "__main__":
    main()
