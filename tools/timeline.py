"""Per-warp timeline of one C2 decode step (debug build, -DHGCA_TIMELINE; HGCA_TL_CFG=C4L: the C4 shape).

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

SLOTS = 20


def main():
    torch.cuda.set_device(0)
    cfgd = dict(bench.C2)
    if os.environ.get("HGCA_TL_CFG") == "C4L":  # one layer of the C4 shape
        cfgd.update(batch=8, heads=64, kv_heads=8, context=16384)
    elif os.environ.get("HGCA_TL_CFG") == "C5S":  # a small step: C5 at 64K, window 256, 1% selected
        cfgd.update(batch=4, context=65536, blk_num=8, frac=0.01)
    elif os.environ.get("HGCA_TL_CFG") == "C3":  # the north-star shape: B=4, 128K context
        cfgd.update(batch=4, context=131072)
    elif os.environ.get("HGCA_TL_CFG") == "EMPTYB":  # a near-empty bf16 step (tools/fixed_cost_probe.py)
        cfgd.update(batch=1, heads=32, kv_heads=8, context=128, blk_num=2, frac=0.01)
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
        names = ["", "", "merge", "wait", "sub", "items", "qk", "pv", "v", "issue", "tma", "mask", "smma", "epi",
                 "smax", "end", "sm"]
        cyc = {k: t[:, i] for i, k in enumerate(names) if k}
        span = end.max()
        print(f"--- step {it}: decode+merge {ms*1e3:.1f} us (events), warps {n} ({nc}/SM), decode span {span:.1f} us")
        print("warp end us: p0 %.1f p10 %.1f p50 %.1f p90 %.1f p99 %.1f max %.1f" %
              tuple(np.percentile(end, [0, 10, 50, 90, 99, 100])))
        sub = max(cyc["sub"].sum(), 1)
        parts = ["wait", "v", "smma", "mask", "smax", "qk", "pv", "end", "issue", "tma"]
        print("  cycles per sub-chunk: " + ", ".join(f"{k} {cyc[k].sum()/sub:.0f}" for k in parts))
        print("  (qk = smma + mask + smax + P^T store; issue includes tma)")
        tot = sum(cyc[k].sum() for k in ("wait", "v", "qk", "pv", "end", "issue"))
        print(f"  busy cycles per warp mean {tot/n:.0f} = {tot/n/1965:.1f} us; sub-chunks/warp "
              f"min {cyc['sub'].min():.0f} mean {cyc['sub'].mean():.1f} max {cyc['sub'].max():.0f}; "
              f"dense epilogue {cyc['epi'].sum()/max(np.count_nonzero(cyc['epi']),1):.0f} cyc/item")
        smid = cyc["sm"].astype(int)
        sm_end = np.array([end[smid == k].max() for k in range(148)])
        sm_sub = np.array([cyc["sub"][smid == k].sum() for k in range(148)])
        print(f"  per-SM: last warp end p0 {sm_end.min():.1f} p50 {np.median(sm_end):.1f} max {sm_end.max():.1f} us; "
              f"sub-chunks per SM min {sm_sub.min():.0f} max {sm_sub.max():.0f}; corr(end, sub) "
              f"{np.corrcoef(sm_end, sm_sub)[0, 1]:.2f}")
        items_end = (t[:, 17] - t0) / 1e3
        print(f"  items done: p0 {items_end.min():.1f} p50 {np.median(items_end):.1f} max {items_end.max():.1f} us; "
              f"after merge phase: p50 {np.median(end):.1f} max {end.max():.1f} us")
        fm = lib.hgca_debug_timeline_merge
        fm.argtypes = [ctypes.c_void_p]
        mb = np.zeros(4096 * 8, np.uint64)
        fm(mb.ctypes.data)
        tm = (mb.reshape(4096, 8)[: B * Hq, :8].astype(np.float64) - t0) / 1e3
        print("  merge CTAs (us): resident p0 %.1f max %.1f | after wait p0 %.1f max %.1f | sparse fold max %.1f "
              "| dense fold max %.1f | epilogue end p50 %.1f max %.1f; per CTA: sparse %.1f dense %.1f epi %.1f" % (
                  tm[:, 0].min(), tm[:, 0].max(), tm[:, 1].min(), tm[:, 1].max(), tm[:, 2].max(), tm[:, 3].max(),
                  np.median(tm[:, 5]), tm[:, 5].max(), np.median(tm[:, 2] - tm[:, 1]), np.median(tm[:, 3] - tm[:, 2]),
                  np.median(tm[:, 5] - tm[:, 4])))
        print("  merge fold detail (median per CTA, us): m/z loads + issue %.1f, bulk wait %.1f, stats+acc %.1f" % (
            np.median(tm[:, 6] - tm[:, 1]), np.median(tm[:, 7] - tm[:, 6]), np.median(tm[:, 2] - tm[:, 7])))
        # the last items: when did the finishers start them, and what were they
        BK = B * Hkv
        off = ls_off = eng.layers[0].item_off.cpu().numpy()
        NF, NS = int(off[BK]), int(off[2 * BK + 1])
        rows = int(off[2 * (BK + 1)])
        W = eng.layers[0].window_size
        dr = max(min(rows, 32), rows // 2)
        ND = BK * -(-W // dr)
        kind = lambda it: "full" if it < NF else ("dense" if it < NF + ND else "tail")  # noqa: E731
        last_start = (t[:, 18] - t0) / 1e3
        order = np.argsort(end)
        print("  last 8 finishers: end / last item start / kind: " + ", ".join(
            f"{end[i]:.1f}/{last_start[i]:.1f}/{kind(int(t[i, 19]))}" for i in order[-8:]))
        print(f"  items: {NF} full, {ND} dense (est.), {NS - NF} tail")
        # early finishers: what were they doing?
        order = np.argsort(end)
        print(f"  first 5 finishers: end {np.round(end[order[:5]], 1)} subs {cyc['sub'][order[:5]]}; "
              f"last 5: end {np.round(end[order[-5:]], 1)} subs {cyc['sub'][order[-5:]]}")


if __name__ == "__main__":
    main()
