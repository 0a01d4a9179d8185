"""Where the end-to-end (host buffer) decode step spends its time, C2 (run on the GPU box)."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2507_03153_b200 as hg  # noqa: E402


def wall(fn, n=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e6


def main():
    cfgd = dict(bench.C2)
    eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 4000)
    B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
    tdt = eng.tdtype
    nq, nk = B * Hq * D, B * Hkv * D
    in_host = torch.randn(nq + 2 * nk).to(tdt).pin_memory()
    out_host = torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8).pin_memory()
    dev_in = torch.empty(nq + 2 * nk, dtype=tdt, device="cuda")
    dev_out = torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8, device="cuda")
    q = dev_in[:nq].view(B, Hq, 1, D)
    k = dev_in[nq:nq + nk].view(B, Hkv, 1, D)
    v = dev_in[nq + nk:].view(B, Hkv, 1, D)
    out = torch.empty((B * Hq, D), dtype=torch.float32, device="cuda")
    lse = torch.empty(B * Hq, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream()

    t_dev = wall(lambda: eng.decode_device(0, q, k, v, out=out, lse=lse))
    t_dev_sync = wall(lambda: (eng.decode_device(0, q, k, v, out=out, lse=lse), s.synchronize()))
    t_copies = wall(lambda: (dev_in.copy_(in_host, non_blocking=True), out_host.copy_(dev_out, non_blocking=True),
                             s.synchronize()))
    t_host = wall(lambda: eng.decode_host_packed(0, in_host, out_host, staging=(dev_in, dev_out)))
    print(f"device steps back to back          {t_dev:7.1f} us/step (wall)")
    print(f"device step + stream sync          {t_dev_sync:7.1f} us/step")
    print(f"H2D {in_host.numel() * in_host.element_size() / 1e3:.0f} KB + D2H "
          f"{out_host.numel() / 1e3:.0f} KB + sync     {t_copies:7.1f} us")
    print(f"decode_host_packed (e2e)           {t_host:7.1f} us/step -> {B / t_host * 1e6:.0f} tokens/s")


if __name__ == "__main__":
    main()


def split_timing():
    """host-side split of decode_host_packed: library call (H2D, kernels, sync) vs bookkeeping."""
    cfgd = dict(bench.C2)
    eng, g = bench.stage_engine(hg, torch, cfgd, cfgd["context"] + 4000)
    B, Hq, Hkv, D = eng.B, eng.Hq, eng.Hkv, eng.D
    nq, nk = B * Hq * D, B * Hkv * D
    in_host = torch.randn(nq + 2 * nk).to(eng.tdtype).pin_memory()
    out_host = torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8).pin_memory()
    staging = (torch.empty(nq + 2 * nk, dtype=eng.tdtype, device="cuda"),
               torch.empty(B * Hq * (4 * D + 8), dtype=torch.uint8, device="cuda"))
    lib_call = hg._lib.call
    acc = {"call": 0.0, "done": 0.0, "desc": 0.0}
    orig_done, orig_desc = eng._step_done, eng._step_desc

    def timed(key, fn):
        def w(*a, **k):
            t = time.perf_counter()
            r = fn(*a, **k)
            acc[key] += time.perf_counter() - t
            return r
        return w
    hg._lib.call = timed("call", lib_call)
    eng._step_done = timed("done", orig_done)
    eng._step_desc = timed("desc", orig_desc)
    for _ in range(10):
        eng.decode_host_packed(0, in_host, out_host, staging=staging)
    for k in acc:
        acc[k] = 0.0
    n = 320
    t = time.perf_counter()
    for _ in range(n):
        eng.decode_host_packed(0, in_host, out_host, staging=staging)
    tot = (time.perf_counter() - t) / n * 1e6
    hg._lib.call = lib_call
    print(f"e2e {tot:.1f} us/step: library calls {acc['call'] / n * 1e6:.1f} (incl. ingest launches), "
          f"_step_done {acc['done'] / n * 1e6:.1f} (incl. ingest), _step_desc {acc['desc'] / n * 1e6:.1f}, "
          f"rest {tot - (acc['call'] + acc['done'] + acc['desc']) / n * 1e6:.1f}")


if __name__ == "__main__" and os.environ.get("HGCA_E2E_SPLIT"):
    split_timing()
