"""Per-warp timeline of one C2 decode step (debug build, -DHGCA_TIMELINE).

usage (GPU box): python paper_2507_03153_b200/_build.py --timeline
                 HGCA_LIB=paper_2507_03153_b200/_lib/libhgca_b200_tl.so python tools/timeline.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("HGCA_LIB", os.path.join(ROOT, "paper_2507_03153_b200", "_lib", "libhgca_b200_tl.so"))

import bench  # noqa: E402
import paper_2507_03153_b200 as hg  # noqa: E402

SLOTS = 16


def main():
    torch.cuda.set_device(0)
    cfgd = dict(bench.C2)
    eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 64)
    lib = hg._lib.load()
    fn = lib.hgca_debug_timeline
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
    cfg = (ctypes.c_int64 * 5)()
    hg._lib.call("hgca_decode_config", eng.dcode, D, Hq // Hkv, cfg)
    nc = cfg[0]
    tdt = eng.tdtype
    for it in range(2):
        q = torch.randn((B, Hq, 1, D), generator=g, device="cuda").to(tdt)
        k = torch.randn((B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
        torch.cuda.synchronize()
        fn(None, 0)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
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
        names = ["", "", "merge", "wait", "sub", "items", "qk", "pv", "v", "issue", "tma", "nmerge", "smma", "epi"]
        cyc = {k: t[:, i] for i, k in enumerate(names) if k}
        span = end.max()
        print(f"--- step {it}: kernel {ms*1e3:.1f} us (events), warps {n} ({nc}/SM), span {span:.1f} us")
        print("warp end us: p0 %.1f p10 %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" %
              tuple(np.percentile(end, [0, 10, 50, 90, 99, 100])))
        print("warp start us: max %.1f" % start.max())
        tot = sum(cyc[k].sum() for k in ("merge", "wait", "qk", "pv", "v", "issue"))
        clk_mhz = 1965.0
        for k in ("wait", "v", "qk", "pv", "issue", "merge"):
            print(f"  {k:6s} {cyc[k].sum()/tot:6.1%}  per sub-chunk {cyc[k].sum()/max(cyc['sub'].sum(),1):8.0f} cyc")
        sub = max(cyc['sub'].sum(), 1)
        print(f"  of which: qk-mma {cyc['smma'].sum()/sub:.0f} cyc/sub, tma-issue {cyc['tma'].sum()/sub:.0f} cyc/sub; "
              f"merges {cyc['nmerge'].sum():.0f} (max/warp {cyc['nmerge'].max():.0f}), "
              f"cyc/merge {cyc['merge'].sum()/max(cyc['nmerge'].sum(),1):.0f}, dense epilogue cyc/item "
              f"{cyc['epi'].sum()/max(len(np.nonzero(cyc['epi'])[0]),1):.0f}")
        print(f"  sub-chunks {cyc['sub'].sum():.0f} items {cyc['items'].sum():.0f} "
              f"merge cyc max/warp {cyc['merge'].max():.0f} ({cyc['merge'].max()/clk_mhz:.1f} us)")
        print(f"  busy cycles per warp mean {tot/n:.0f} = {tot/n/clk_mhz:.1f} us at {clk_mhz} MHz")


if __name__ == "__main__":
    main()
