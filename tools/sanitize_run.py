"""Small engine runs exercising every kernel family, for compute-sanitizer.

  compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_run.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_03153_b200 as hg  # noqa: E402


def run(dtype, steps=150, append_at=60, append_nq=8, graph=False, bn=4):
    cfg = hg.EngineConfig(layers=1, heads=8, kv_heads=2, head_dim=128, batch=2, dtype=dtype,
                          cache=hg.CacheConfig(blk_num=bn, blk_size=32, beta=1.0), core_count=4,
                          max_positions=1024)
    eng = hg.HybridEngine(cfg)
    g = torch.Generator(device="cuda").manual_seed(1)
    tdt = eng.tdtype
    n = 300
    eng.bulk_ingest(0, torch.randn((2, 2, n, 128), generator=g, device="cuda").to(tdt),
                    torch.randn((2, 2, n, 128), generator=g, device="cuda").to(tdt),
                    torch.rand((2, 8, n), generator=g, device="cuda", dtype=torch.float64) / 128, 128)
    for t in range(steps):
        if t == append_at:
            q = torch.randn((2, 8, append_nq, 128), generator=g, device="cuda").to(tdt)
            k = torch.randn((2, 2, append_nq, 128), generator=g, device="cuda").to(tdt)
            eng.step(0, hg.StepInput("append", q, k, k))
            continue
        q = torch.randn((2, 8, 1, 128), generator=g, device="cuda").to(tdt)
        k = torch.randn((2, 2, 1, 128), generator=g, device="cuda").to(tdt)
        eng.decode_device(0, q, k, k)
    if graph:  # graph mode: PDL-chained replays, first stages gathered before the launch wait
        while eng.cap - eng.layers[0].window_size < 16:
            q = torch.randn((2, 8, 1, 128), generator=g, device="cuda").to(tdt)
            k = torch.randn((2, 2, 1, 128), generator=g, device="cuda").to(tdt)
            eng.decode_device(0, q, k, k)
        gr = hg.DecodeGraph(eng, steps=8)
        for t in (gr.q, gr.k, gr.v):
            t.copy_(torch.randn(t.shape, generator=g, device="cuda").to(tdt))
        gr.step()
        gr.step()
    torch.cuda.synchronize()
    print(dtype, "ok, archive", eng.layers[0].archive_size, flush=True)


if __name__ == "__main__":
    mode = sys.argv[1] if len(sys.argv) > 1 else "all"
    if mode in ("all", "bf16-decode"):
        run("bfloat16", append_at=-1)
    if mode in ("all", "bf16-append"):
        run("bfloat16", steps=3, append_at=0)
    if mode in ("all", "bf16-append-tc5"):  # G*n_q = 64 rows: the tcgen05 append passes
        run("bfloat16", steps=3, append_at=0, append_nq=16)
    if mode in ("all", "bf16-append-tc5x2"):  # G*n_q = 256 rows: the two-tile tcgen05 passes
        run("bfloat16", steps=3, append_at=0, append_nq=64)
    if mode in ("all", "bf16-append-small"):  # G*n_q = 12 rows: split-key pass 1 with four copies
        run("bfloat16", steps=3, append_at=0, append_nq=3)
    if mode in ("all", "bf16-append-long"):  # n_q = 160 > 128: chunked tcgen05 passes
        run("bfloat16", steps=3, append_at=0, append_nq=160, bn=8)
    if mode in ("all", "f32"):
        run("float32", steps=80)
    if mode in ("all", "graph"):
        run("bfloat16", steps=40, append_at=-1, graph=True)
        run("float32", steps=40, append_at=-1, graph=True)
