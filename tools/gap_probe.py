"""Where a graph-mode decode step's time goes, in absolute device time
(debug build -DHGCA_TIMELINE): for the last step of a 16-step DecodeGraph
replay, every stamp relative to the END of the previous step's merge grid.

usage (GPU box): HGCA_LIB=paper_2507_03153_b200/_lib/libhgca_b200_tl.so python tools/gap_probe.py [C1 EMPTY ...]
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


def pct(x):
    return "p0 %.2f p50 %.2f max %.2f" % (np.min(x), np.median(x), np.max(x))


def run(name):
    cfgd = CFGS[name]
    eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 2048, seed=7)
    lib = hg._lib.load()
    cfg = (ctypes.c_int64 * 5)()
    hg._lib.call("hgca_decode_config", eng.dcode, eng.D, eng.Hq // eng.Hkv, cfg)
    nc = cfg[0]
    B, Hq, Hkv, D, tdt = eng.B, eng.Hq, eng.Hkv, eng.D, eng.tdtype
    S = 16 if eng.cap >= 256 else 8
    while eng.cap - eng.layers[0].window_size < 2 * S:  # decode eagerly past the next eviction
        q = torch.randn((B, Hq, 1, D), generator=g, device="cuda").to(tdt)
        k = torch.randn((B, Hkv, 1, D), generator=g, device="cuda").to(tdt)
        eng.decode_device(0, q, k, k)
    gr = hg.DecodeGraph(eng, layers=[0], steps=S)
    gr.q.copy_(torch.randn(gr.q.shape, generator=g, device="cuda").to(gr.q.dtype))
    gr.k.copy_(torch.randn(gr.k.shape, generator=g, device="cuda").to(gr.k.dtype))
    gr.v.copy_(gr.k)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gr.step()  # warm
    torch.cuda.synchronize()
    e0.record()
    gr.step()
    e1.record()
    torch.cuda.synchronize()
    per = e0.elapsed_time(e1) * 1e3 / S
    gaps = np.zeros(1024 * 4, np.uint64)
    lib.hgca_debug_gaps.argtypes = [ctypes.c_void_p]
    lib.hgca_debug_gaps(gaps.ctypes.data)
    gp = gaps.reshape(1024, 4)[:148].astype(np.float64)
    R = gp[:, 2].max()
    n = 148 * nc
    buf = np.zeros(n * SLOTS, np.uint64)
    lib.hgca_debug_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    lib.hgca_debug_timeline(buf.ctypes.data, n * SLOTS)
    t = buf.reshape(n, SLOTS).astype(np.float64)
    mb = np.zeros(4096 * 8, np.uint64)
    lib.hgca_debug_timeline_merge.argtypes = [ctypes.c_void_p]
    lib.hgca_debug_timeline_merge(mb.ctypes.data)
    tm = mb.reshape(4096, 8)[: eng.B * eng.Hq].astype(np.float64)
    us = lambda x: (x - R) / 1e3  # noqa: E731
    busy = t[:, 1] > t[:, 0]
    print(f"--- {name} ({cfgd['dtype']}): graph step {per:.2f} us (events, {S}-step replay); stamps in us after the "
          f"previous merge grid's last CTA end")
    print(f"  decode CTA entry          {pct(us(gp[:, 0]))}")
    print(f"  decode wait released      {pct(us(gp[:, 1]))}")
    print(f"  consumer warps end        {pct(us(t[busy, 1]))}")
    if cfgd["dtype"] == "float32":  # decode_f32_kernel slots: 2 stages, 3 wait, 4 score, 5 softmax+pv, 7 partial
        bz = t[busy]
        nsub = max(bz[:, 2].sum(), 1)
        print(f"  fp32 consumer cycles per stage: wait {bz[:, 3].sum() / nsub:.0f}, score {bz[:, 4].sum() / nsub:.0f}, "
              f"softmax+pv {bz[:, 5].sum() / nsub:.0f}, partial {bz[:, 7].sum() / nsub:.0f}; stages per busy warp "
              f"max {bz[:, 2].max():.0f}; first stage data {pct(us(bz[:, 8]))}")
    print(f"  merge CTA resident        {pct(us(tm[:, 0]))}")
    print(f"  merge wait released       {pct(us(tm[:, 1]))}")
    print(f"  merge CTA end (epilogue)  {pct(us(tm[:, 5]))}")
    ph = lambda i, j: np.median(tm[:, j] - tm[:, i]) / 1e3  # noqa: E731
    print(f"  merge phases (median us): issue+m/z loads {ph(1, 6):.2f} | m/z stats {ph(6, 7):.2f} | "
          f"window epilogue {ph(7, 3):.2f} | bulk wait+dot {ph(3, 2):.2f} | out/lse {ph(2, 4):.2f} | rest {ph(4, 5):.2f}")


if __name__ == "__main__":
    torch.cuda.set_device(0)
    for n in (sys.argv[1:] or ["EMPTY", "EMPTYB", "C1", "C5S"]):
        run(n)
