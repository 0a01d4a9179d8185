"""Per-stage cycle profile of the tcgen05 append pass 1 (C2 scale, n_q = 64).

  python paper_2507_03153_b200/_build.py --variant p5 HGCA_TC5_PROF   # builds libhgca_b200_p5.so
  python tools/tc/tc5_prof.py                                          # on the GPU box

Prints, per 64-key stage, a softmax warp's cycles waiting for S = Q K^T, waiting
for the P.V that frees its P buffer, and in total.
"""
import ctypes, os, sys, torch
sys.path.insert(0, ".")
os.environ["HGCA_LIB"] = "paper_2507_03153_b200/_lib/libhgca_b200_p5.so"
import bench, paper_2507_03153_b200 as hg
cfgd = dict(bench.C2)
eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 2048, seed=3)
lib = hg._lib.load()
f = lib.hgca_debug_tc5prof
f.argtypes = [ctypes.c_void_p]
for nq in (64,):
    q = torch.randn((16, 32, nq, 128), generator=g, device="cuda").to(torch.bfloat16)
    k = torch.randn((16, 8, nq, 128), generator=g, device="cuda").to(torch.bfloat16)
    eng.step(0, hg.StepInput("append", q, k, k)); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 8)()
    f(buf)
    st = buf[6]
    print("stages", st, "per stage cycles (softmax warp): wait S %.0f, wait P.V %.0f, total %.0f" % (
        buf[3]/st, buf[4]/st, buf[5]/st))
