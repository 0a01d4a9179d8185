"""paper_2507_03153_b200.costmodel: the reference's roofline layer pinned to values
computed by tierkv.perf_model itself (tests/golden/perf_model.json), its
structural properties, and the B200 decode model against the round-1 measurements."""

import json
import os

import numpy as np
import pytest

from paper_2507_03153_b200 import ContractError
from paper_2507_03153_b200 import costmodel as cm

HERE = os.path.dirname(__file__)
GOLD = json.load(open(os.path.join(HERE, "golden", "perf_model.json")))
SHAPE = cm.WorkloadShape(batch=1, heads=32, head_dim=128, n_q=1, bytes_per_elem=2)


class TestReferenceLayer:
    def test_golden_values(self):
        assert cm.merge_bytes(SHAPE) == GOLD["merge_bytes"] == 32 * 129 * 2
        assert cm.kv_bytes(1000, SHAPE) == GOLD["kv_bytes_1000"]
        assert cm.attention_cost(1025, SHAPE.with_(n_window=1024), cm.DEFAULT_GPU) == pytest.approx(
            GOLD["cost_gpu_1025"], rel=1e-15)
        assert cm.attention_cost(8192, SHAPE.with_(n_q=64, batch=3), cm.DEFAULT_CPU) == pytest.approx(
            GOLD["cost_cpu_8192_q64"], rel=1e-15)
        cell = SHAPE.with_(n_window=256, n_store=4096, n_selected=819)
        b = cm.time_offload_baseline(cell, cm.DEFAULT_GPU, cm.DEFAULT_LINK)
        h = cm.time_hybrid(cell, cm.DEFAULT_GPU, cm.DEFAULT_CPU, cm.DEFAULT_LINK, 0.7)
        np.testing.assert_allclose([b.transfer, b.compute], GOLD["baseline"], rtol=1e-15)
        np.testing.assert_allclose([h.gpu_part, h.cpu_part, h.merge], GOLD["hybrid"], rtol=1e-15)
        np.testing.assert_allclose(cm.speedup_heatmap([256, 512, 1024], [0, 1024, 16384], SHAPE),
                                   GOLD["heatmap"], rtol=1e-14)
        rows = cm.heatmap_rows([256, 1024], [0, 4096], [1, 4], SHAPE, core_efficiency=0.25,
                               retention_fraction=0.1)
        np.testing.assert_allclose(np.array(rows, dtype=np.float64), np.array(GOLD["rows"], dtype=np.float64),
                                   rtol=1e-14)

    def test_validation(self):
        with pytest.raises(ContractError):
            cm.DeviceSpec("bad", peak_flops=0, mem_bw=1)
        with pytest.raises(ContractError):
            cm.LinkSpec(bw=-1, latency=0)
        with pytest.raises(ContractError):
            cm.WorkloadShape(n_store=4, n_selected=5)
        with pytest.raises(ContractError):
            cm.time_hybrid(SHAPE, cm.DEFAULT_GPU, cm.DEFAULT_CPU, cm.DEFAULT_LINK, core_efficiency=0.0)
        with pytest.raises(ContractError):
            cm.speedup_heatmap([], [1], SHAPE)

    def test_structure(self):
        assert cm.attention_cost(0, SHAPE, cm.DEFAULT_GPU) == 0.0
        t1, t2 = (cm.attention_cost(n, SHAPE, cm.DEFAULT_GPU) for n in (4096, 8192))
        assert t2 / t1 == pytest.approx(2.0, rel=0.01)          # memory-bound decode
        assert cm.time_offload_baseline(SHAPE, cm.DEFAULT_GPU, cm.DEFAULT_LINK).transfer == cm.DEFAULT_LINK.latency
        h = cm.time_hybrid(SHAPE.with_(n_window=64, n_store=100000, n_selected=50000), cm.DEFAULT_GPU,
                           cm.DEFAULT_CPU, cm.DEFAULT_LINK)
        assert h.total == max(h.gpu_part, h.cpu_part) + h.merge
        hm = cm.speedup_heatmap([256, 512, 1024], [0, 1024, 4096, 16384], SHAPE)
        assert np.abs(hm[:, 0] - 1.0).max() < 0.05 and (np.diff(hm, axis=1) >= -1e-12).all()


class TestB200Model:
    def test_specs(self):
        assert cm.B200.mem_bw > 5e12 and cm.NVLINK5.bw == 900e9
        assert cm.b200_spec("/nonexistent.json").mem_bw == 6546e9

    def test_union_rows(self):
        s = cm.DecodeShape(archive=10000, frac=0.1, q_heads=32, kv_heads=8)
        assert cm.union_rows(s) == pytest.approx(10000 * (1 - 0.9 ** 4))
        assert cm.union_rows(s.with_(overlap=1.0)) == pytest.approx(1000)
        assert cm.union_rows(s.with_(q_heads=8)) == pytest.approx(1000)      # MHA: G = 1
        with pytest.raises(ContractError):
            cm.DecodeShape(q_heads=30, kv_heads=8)

    def test_fit_recovers_parameters(self):
        pts = [(b, 20e-6 + b / 7e12) for b in (5e7, 2e8, 4e8, 8e8)]
        fixed, bw = cm.fit_decode(pts)
        assert fixed == pytest.approx(20e-6, rel=1e-9) and bw == pytest.approx(7e12, rel=1e-9)
        with pytest.raises(ContractError):
            cm.fit_decode([(1.0, 1.0)])

    def test_sharding_reduces_time_until_exchange_dominates(self):
        c3 = cm.DecodeShape(batch=4, window=512, archive=131072 - 512)
        t = [cm.predict_sharded(c3, p).total for p in (1, 2, 4, 8)]
        assert t[0] > t[1] > t[2] > t[3]
        assert cm.predict_sharded(c3, 1).t_exchange == 0.0 and cm.predict_sharded(c3, 8).t_exchange > 0

    def test_matches_round1_measurements(self):
        """Model bytes within 4% and predicted time within 20% of every measured bf16 point
        (median error ~6%; the worst points are the smallest steps)."""
        rows = [json.loads(l) for l in open(os.path.join(HERE, "..", "profiles", "r01_configs_timing.jsonl"))
                if l.startswith("{")]
        bf = [r for r in rows if r["dtype"] == "bfloat16"]
        assert len(bf) >= 10
        for r in bf:
            s = cm.DecodeShape(batch=r["batch"], q_heads=r["q_heads"], kv_heads=r["kv_heads"], window=r["window"],
                               archive=r["context"] - r["window"], frac=r["selected_frac"])
            p = cm.predict_decode(s)
            assert p.bytes == pytest.approx(r["bytes_per_layer_step"], rel=0.04), r["config"]
            assert p.total == pytest.approx(r["layer_step_kernel_ms"] * 1e-3, rel=0.20), r["config"]
