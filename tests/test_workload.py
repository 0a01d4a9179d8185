"""paper_2507_03153_b200.workload: the reference's workload file format (pinned to a
file written by tierkv.save_workload, tests/golden/workload_small.tkv) and the
device generator's planted structure (the properties test_workload.py:74-130 of the
reference asserts for its own generator)."""

import math
import os

import numpy as np
import pytest
import torch

from oracle import workload as ow
from paper_2507_03153_b200 import ContractError
from paper_2507_03153_b200 import workload as wk

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "workload_small.tkv")
SPEC_KW = dict(seed=3, steps=12, prefill_len=4, append_events=((5, 3),))


def weights_last(q, k, scale, t):
    """fp64 softmax weights [heads, t+1] of query t over keys [0, t]."""
    s = np.einsum("hd,hnd->hn", q[:, t].astype(np.float64), k[:, : t + 1].astype(np.float64)) * scale
    s -= s.max(axis=1, keepdims=True)
    w = np.exp(s)
    return w / w.sum(axis=1, keepdims=True)


def spearman(x, y):
    rx = np.argsort(np.argsort(x)).astype(np.float64)
    ry = np.argsort(np.argsort(y)).astype(np.float64)
    rx -= rx.mean()
    ry -= ry.mean()
    return float((rx * ry).sum() / np.sqrt((rx * rx).sum() * (ry * ry).sum()))


class TestFileFormat:
    def test_reads_reference_file_bit_exactly(self):
        wl = wk.load_workload(GOLDEN)
        assert (wl.layers, wl.heads, wl.head_dim, wl.scale) == (2, 2, 16, 0.25)
        assert wl.spec == wk.WorkloadSpec(**SPEC_KW)
        ref = ow.gen_workload(ow.WorkloadSpec(**SPEC_KW), 2, 16, 0.25, 2)   # bit-identical restatement
        assert len(wl) == len(ref) == 13
        for a, b in zip(wl, ref):
            assert (a.mode, a.start, a.n_q) == (b.mode, b.start, b.n_q)
            np.testing.assert_array_equal(a.q.numpy(), b.q)
            np.testing.assert_array_equal(a.keys.numpy(), b.keys)
            np.testing.assert_array_equal(a.values.numpy(), b.values)

    def test_writes_reference_file_byte_identically(self, tmp_path):
        out = tmp_path / "copy.tkv"
        wk.save_workload(wk.load_workload(GOLDEN), out)
        assert out.read_bytes() == open(GOLDEN, "rb").read()

    def test_device_stream_roundtrip(self, tmp_path):
        spec = wk.WorkloadSpec(seed=5, steps=9, prefill_len=3, append_events=((2, 4),))
        wl = wk.gen_workload_device(spec, heads=3, head_dim=8, layers=2, device="cpu")
        path = tmp_path / "wl.tkv"
        wk.save_workload(wl, path)
        back = wk.load_workload(path)
        assert back.spec == spec and len(back) == len(wl) and back.total_entries == wl.total_entries
        for a, b in zip(wl, back):
            assert (a.mode, a.start, a.n_q) == (b.mode, b.start, b.n_q)
            for x, y in ((a.q, b.q), (a.keys, b.keys), (a.values, b.values)):
                assert torch.equal(x, y)

    def test_rejects_foreign_and_truncated_files(self, tmp_path):
        p = tmp_path / "bogus.json"
        p.write_text('{"something": "else"}\n')
        with pytest.raises(ContractError):
            wk.load_workload(p)
        lines = open(GOLDEN).read().splitlines(keepends=True)
        t = tmp_path / "short.tkv"
        t.write_text("".join(lines[:5]))
        with pytest.raises(ContractError):
            wk.load_workload(t)


class TestSpec:
    def test_validation_mirrors_reference(self):
        for bad in (dict(recency_decay=1.0), dict(recency_decay=0.0), dict(steps=-1),
                    dict(steps=10, append_events=((12, 4),)), dict(steps=10, append_events=((3, 0),)),
                    dict(steps=10, append_events=((3, 2), (3, 4))), dict(noise_scale=-1.0)):
            with pytest.raises(ContractError):
                wk.WorkloadSpec(**bad)
        assert wk.WorkloadSpec(steps=10, append_events=((7, 2), (3, 4))).append_events == ((3, 4), (7, 2))

    def test_step_plan(self):
        spec = wk.WorkloadSpec(seed=0, steps=5, prefill_len=3, append_events=((2, 4),))
        wl = wk.gen_workload_device(spec, heads=2, head_dim=16, layers=2, device="cpu")
        assert [(s.mode, s.n_q) for s in wl] == [("append", 3), ("decode", 1), ("decode", 1),
                                                 ("append", 4), ("decode", 1), ("decode", 1)]
        assert [s.start for s in wl] == [0, 3, 4, 5, 9, 10]
        assert wl.total_entries == 11


def _history(spec, heads=2, d=16, device="cpu"):
    wl = wk.gen_workload_device(spec, heads=heads, head_dim=d, layers=1, device=device)
    q, k, v = wl.history(0)
    return wl, q.cpu().numpy(), k.cpu().numpy()


@pytest.mark.parametrize("device", ["cpu", pytest.param("cuda", marks=pytest.mark.gpu)])
class TestPlantedStructure:
    def test_deterministic_per_seed(self, device):
        spec = wk.WorkloadSpec(seed=42, steps=20, prefill_len=4)
        _, qa, ka = _history(spec, device=device)
        _, qb, kb = _history(spec, device=device)
        np.testing.assert_array_equal(ka, kb)
        np.testing.assert_array_equal(qa, qb)
        _, _, kc = _history(wk.WorkloadSpec(seed=43, steps=20, prefill_len=4), device=device)
        assert not np.array_equal(ka, kc)

    def test_recency_rank_correlation(self, device):
        spec = wk.WorkloadSpec(seed=6, steps=256, prefill_len=0, sink_count=0, heavy_hitter_count=0,
                               heavy_hitter_boost=0.0)
        wl, q, k = _history(spec, device=device)
        t = wl.total_entries - 1
        w = weights_last(q, k, wl.scale, t)
        for h in range(q.shape[0]):
            assert spearman(w[h], np.arange(t + 1)) > 0.9

    def test_sinks_and_heavy_hitters(self, device):
        spec = wk.WorkloadSpec(seed=6, steps=384, prefill_len=64, sink_count=2, heavy_hitter_count=3,
                               heavy_hitter_boost=0.75)
        wl, q, k = _history(spec, device=device)
        total = wl.total_entries
        w = weights_last(q, k, wl.scale, total - 1)
        planted = np.sort(np.argsort(w[0, : total // 4])[-5:])
        hitters = [p for p in planted if p >= 2]
        assert len(hitters) == 3
        for t in range(total // 2, total, 64):
            wt = weights_last(q, k, wl.scale, t)
            for h in range(q.shape[0]):
                med = np.median(wt[h, : t - 64])
                assert all(wt[h, p] > med for p in hitters)
                assert wt[h, 0] > 0.25 * wt[h, t]       # a sink tracks the frontier weight
            # the i-th hitter holds ~boost^(i+1) of the newest token's weight (noise 0.05)
            for i, p in enumerate(hitters):
                ratio = wt[:, p] / wt[:, t]
                assert np.all(np.abs(np.log(ratio) - (i + 1) * math.log(0.75)) < 0.5)

    def test_boost_zero_plants_nothing(self, device):
        spec = wk.WorkloadSpec(seed=6, steps=64, prefill_len=0, sink_count=0, heavy_hitter_count=4,
                               heavy_hitter_boost=0.0)
        wl, q, k = _history(spec, device=device)
        w = weights_last(q, k, wl.scale, wl.total_entries - 1)
        assert spearman(w[0], np.arange(wl.total_entries)) > 0.9


@pytest.mark.gpu
def test_device_generation_at_128k_context():
    """One layer of the C3 shape (32 heads, d=128, 128K tokens) generated on the device."""
    spec = wk.WorkloadSpec(seed=7, steps=131072 - 128, prefill_len=128)
    wk.gen_workload_device(wk.WorkloadSpec(seed=1, steps=64), heads=2, head_dim=128, layers=1, device="cuda")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    wl = wk.gen_workload_device(spec, heads=32, head_dim=128, layers=1, device="cuda")
    e1.record()
    torch.cuda.synchronize()
    assert wl.total_entries == 131072 and wl.steps[0].q.is_cuda
    k = wl.steps[0].keys
    assert torch.isfinite(k).all()
    print(f"\n128K-token layer (32 heads, d=128) generated in {e0.elapsed_time(e1):.1f} ms")
