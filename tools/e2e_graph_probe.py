import os, sys, time
import torch
sys.path.insert(0, "/root/repo")
import bench
import paper_2507_03153_b200 as hg

cfgd = dict(bench.C3)
eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 4000)
B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
tdt = eng.tdtype
nq, nk = B * Hq * D, B * Hkv * D
in_host = torch.randn(nq + 2 * nk).to(tdt).pin_memory()
out_host = torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8).pin_memory()
staging = (torch.empty(nq + 2 * nk, dtype=tdt, device="cuda"), torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8, device="cuda"))
s = torch.cuda.current_stream()
def run(fn, n=200):
    for _ in range(10): fn()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e6
t_e2e = run(lambda: eng.decode_host_packed(0, in_host, out_host, staging))
while eng.cap - eng.layers[0].window_size < 2:
    eng.decode_host_packed(0, in_host, out_host, staging)
g1 = hg.DecodeGraph(eng, steps=1)
oh_f = out_host[:B * Hq * D * 4].view(torch.float32); oh_l = out_host[B * Hq * D * 4:].view(torch.float64)
def gstep():
    g1.q.view(-1).copy_(in_host[:nq], non_blocking=True)
    g1.k.view(-1).copy_(in_host[nq:nq + nk], non_blocking=True)
    g1.v.view(-1).copy_(in_host[nq + nk:], non_blocking=True)
    o, l = g1.step()
    oh_f.copy_(o.view(-1), non_blocking=True); oh_l.copy_(l.view(-1), non_blocking=True)
    s.synchronize()
t_g = run(gstep)
def replay_only():
    g1.graph.replay(); s.synchronize()
t_r = run(replay_only, 50)
print(f"decode_host_packed {t_e2e:.1f} us; torch graph step with copies {t_g:.1f} us; bare replay+sync {t_r:.1f} us")
