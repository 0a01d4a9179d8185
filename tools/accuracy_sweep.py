"""Config 5 accuracy: hybrid decode vs fp64 full attention at 64K context.

For each dense window W in {256, 1K, 4K, 8K} and top-k fraction f in
{1, 2, 5, 10, 20}% (selection="topk": per query head the f*N archive entries
of largest MAW, ties by position -- the padding order of sparsifier.py:219-226):

  1. stage a 64K-token float32 history whose keys carry attention structure
     (4 sinks + 2% heavy hitters aligned with the group's query direction,
     like the reference generator workload.py:1-22) into the archive;
  2. one append step of 16 queries: the archive is re-evaluated from the real
     attention weights (MAW := row-mean, sparsifier.py:158-177) and the top-k
     context is selected from it;
  3. decode steps fill the window to W;
  4. one measured decode step, compared with paper_2507_03153_b200.accuracy:
     err, eps (dropped oracle mass), the 2*eps*max|V| bound (harness.py:147-160).

Prints one JSON line per point. float32 storage (default): the reference-exact kernels;
HGCA_ACC_DTYPE=bfloat16: the bf16 path (tensor-core decode, tcgen05 append), the same
history rounded to bf16, so err includes the bf16 arithmetic on top of the dropped mass.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2507_03153_b200 as hg  # noqa: E402
from paper_2507_03153_b200 import accuracy  # noqa: E402

B, HQ, HKV, D, CTX = 1, 32, 8, 128, 65536


def structured(g, u, n, heavy_frac=0.02, boost=None, sinks=4):
    """keys [B, Hkv, n, D]: noise + heavy hitters / sinks along u (per kv head)."""
    boost = BOOST if boost is None else boost
    k = torch.randn((B, HKV, n, D), generator=g, device="cuda")
    heavy = torch.rand((B, HKV, n), generator=g, device="cuda") < heavy_frac
    heavy[:, :, :sinks] = True
    k += heavy[..., None].float() * boost * (D ** 0.5) * u[:, :, None, :]
    return k


def queries(g, u, nq):
    """q [B, Hq, nq, D] along the group's direction u plus noise."""
    G = HQ // HKV
    uq = u.repeat_interleave(G, dim=1)
    return (D ** 0.5) * uq[:, :, None, :] * 0.5 + torch.randn((B, HQ, nq, D), generator=g, device="cuda")


BOOST = float(os.environ.get("HGCA_ACC_BOOST", "0.5"))  # heavy-hitter key boost along u
DTYPE = os.environ.get("HGCA_ACC_DTYPE", "float32")


def point(win_blocks, frac, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    u = torch.nn.functional.normalize(torch.randn((B, HKV, D), generator=g, device="cuda"), dim=-1)
    cap = win_blocks * 32
    n_arch = CTX - cap
    cfg = hg.EngineConfig(layers=1, heads=HQ, kv_heads=HKV, head_dim=D, batch=B, dtype=DTYPE,
                          cache=hg.CacheConfig(blk_num=win_blocks, blk_size=32, alpha=0.5, beta=1.0),
                          core_count=10 ** 6, max_positions=CTX + 64, selection="topk",
                          topk=max(1, int(round(frac * n_arch))))
    eng = hg.HybridEngine(cfg)
    tdt = eng.tdtype
    k = structured(g, u, n_arch).to(tdt)
    v = torch.randn((B, HKV, n_arch, D), generator=g, device="cuda").to(tdt)
    eng.bulk_ingest(0, k, v, torch.zeros((B, HQ, n_arch), dtype=torch.float64, device="cuda"), cap)
    nq = 16
    eng.step(0, hg.StepInput("append", queries(g, u, nq).to(tdt), structured(g, u, nq, sinks=0).to(tdt),
                             torch.randn((B, HKV, nq, D), generator=g, device="cuda").to(tdt)))
    while eng.layers[0].window_size < cap - 1:
        eng.decode_device(0, queries(g, u, 1).to(tdt).contiguous(), structured(g, u, 1, sinks=0).to(tdt).contiguous(),
                          torch.randn((B, HKV, 1, D), generator=g, device="cuda").to(tdt))
    ls = eng.layers[0]
    n = ls.nxt + 1
    mask = accuracy.attended_mask(eng, 0, n)
    q = queries(g, u, 1).to(tdt).contiguous()
    out, lse, _ = eng.decode_device(0, q, structured(g, u, 1, sinks=0).to(tdt).contiguous(),
                                    torch.randn((B, HKV, 1, D), generator=g, device="cuda").to(tdt))
    m = accuracy.step_metrics(eng, 0, out, q, mask, n)
    m.update({"config": "C5 accuracy", "context": n, "window_cap": cap, "topk_frac": frac, "archive": ls.lo,
              "dtype": DTYPE, "heavy_boost": BOOST})
    return m


def main():
    for win_blocks in (8, 32, 128, 256):
        for frac in (0.01, 0.02, 0.05, 0.10, 0.20):
            print(json.dumps(point(win_blocks, frac)), flush=True)
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
