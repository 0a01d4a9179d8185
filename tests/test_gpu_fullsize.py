"""GPU parity of the bf16 decode step at the bench's full sizes (BASELINE
configs[1] = C2: batch 16, 32K context; configs[2] = C3: batch 4, 128K), on
the exact staged workload bench.py times (bench.stage_engine).

For three consecutive decode steps (the middle one crosses an eviction ->
ingest -> union rebuild), every query head of the first and the last batch
element is recomputed by the oracle (oracle/port.py: attend_indexed over the
attended archive entries (engine.py:134-149), attend_dense over window +
kv_in (engine.py:161-164), merge_states (attention.py:153-188)) on the same
bf16 values upcast to fp32. Tolerance (north star, bf16 path): per head
max|a - b| <= 1e-2 max|b|, and per element |a - b| <= 1e-2 |b| + 1e-3 max|b|;
lse within 1e-3 absolute.
"""

import math

import numpy as np
import pytest
import torch

import bench
from oracle import port

from conftest import host  # noqa: E402

pytestmark = pytest.mark.gpu

REL = 1e-2


def _rows(ls, bk, pos):
    """Logical K and V rows (fp32 numpy [n, D]) of (batch, kv-head) bk at the
    given positions: rows are stored position-rotated (16-byte chunk c of
    position p at (c & ~7) | ((c ^ p) & 7), hgca_write_rows)."""
    KV = ls.KV
    _, T, _, D = KV.shape
    epc = 16 // KV.element_size()
    ch = 2 * D // epc
    p = torch.as_tensor(np.asarray(pos, np.int64), device=KV.device)
    raw = KV[bk].view(T, ch, epc).index_select(0, p)                     # [n, ch, epc]
    c = torch.arange(ch, device=KV.device)
    phys = (c[None, :] & ~7) | ((c[None, :] ^ p[:, None]) & 7)           # [n, ch]
    log = torch.gather(raw, 1, phys[:, :, None].expand(-1, -1, epc)).view(-1, 2, D)
    log = log.float().cpu().numpy()
    return log[:, 0], log[:, 1]


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_fullsize_bf16_step_vs_oracle(cuda, name):
    cfgd = dict(bench.C2 if name == "C2" else bench.C3)
    cap = cfgd["blk_num"] * cfgd["blk_size"]
    eng, g = bench.stage_engine(cuda, torch, cfgd, cfgd["context"] + 16, seed=3, window=cap - 2)
    ls = eng.layers[0]
    B, Hq, Hkv, D, G = eng.B, eng.Hq, eng.Hkv, eng.D, eng.G
    scale = 1 / math.sqrt(D)
    arch0 = ls.archive_size
    worst_head = worst_elem = worst_lse = 0.0
    for step in range(3):
        q = torch.randn((B, Hq, 1, D), generator=g, device="cuda").to(eng.tdtype)
        kk = torch.randn((B, Hkv, 1, D), generator=g, device="cuda").to(eng.tdtype)
        vv = torch.randn((B, Hkv, 1, D), generator=g, device="cuda").to(eng.tdtype)
        lo, nxt = ls.lo, ls.nxt
        entries, _ = eng.store_entries()
        out, lse, _ = eng.decode_device(0, q, kk, vv)
        got, got_lse = host(out).reshape(B, Hq, D), host(lse).reshape(B, Hq)
        qh, kn, vn = (host(x.float()) for x in (q, kk, vv))
        for b in (0, B - 1):
            for kvh in range(Hkv):
                bk = b * Hkv + kvh
                union = np.unique(np.concatenate([entries[b * Hq + kvh * G + gi] for gi in range(G)]))
                Ku, Vu = _rows(ls, bk, union)
                Kw, Vw = _rows(ls, bk, np.arange(lo, nxt))
                dk = np.concatenate([Kw, kn[b, kvh]], 0)[None]
                dv = np.concatenate([Vw, vn[b, kvh]], 0)[None]
                for gi in range(G):
                    h = kvh * G + gi
                    ent = entries[b * Hq + h]
                    at = np.searchsorted(union, ent)
                    so, sl, _ = port.attend_indexed(qh[b, h, 0][None], Ku, Vu, at.astype(np.int64), scale, False)
                    do, dl, _ = port.attend_dense(qh[b, h, 0][None][None], dk, dv, scale, False)
                    o, l = port.merge_states(so, sl, do[0], dl[0])
                    ref, a = o[0].astype(np.float64), got[b, h].astype(np.float64)
                    mx = np.abs(ref).max()
                    err = np.abs(a - ref)
                    worst_head = max(worst_head, float(err.max() / mx))
                    worst_elem = max(worst_elem, float((err / (np.abs(ref) + 0.1 * mx)).max()))
                    worst_lse = max(worst_lse, abs(float(got_lse[b, h]) - float(l[0])))
    print(f"{name}: worst per-head rel {worst_head:.2e}, per-element (|b| + 0.1 max|b|) {worst_elem:.2e}, "
          f"lse abs {worst_lse:.2e}; archive {arch0} -> {ls.archive_size}")
    assert ls.archive_size > arch0, "no eviction inside the checked steps"
    assert worst_head <= REL, worst_head
    assert worst_elem <= REL, worst_elem
    assert worst_lse <= 1e-3, worst_lse
