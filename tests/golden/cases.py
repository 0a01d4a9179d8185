"""Kernel cases shared by make_golden.py (reference outputs) and the tests
(inputs are regenerated from the per-case seed; numpy's PCG64 streams are
stable across versions)."""

import numpy as np

# key: (seed, H, nq, d, nkv, dtype, magnitude)
DENSE_CASES = {}
for _i, _nkv in enumerate((0, 1, 7, 300)):       # test_backends.py:24-39 shapes
    for _dt in ("float32", "float64"):
        DENSE_CASES[f"dense{_i}_{_dt}"] = (100 + _i, 3, 2, 16, _nkv, _dt, 1.0)
DENSE_CASES["dense_c1_float32"] = (200, 4, 1, 128, 512, "float32", 1.0)
DENSE_CASES["dense_mag_float32"] = (201, 2, 3, 64, 1000, "float32", 300.0)
DENSE_CASES["dense_mag_float64"] = (202, 2, 3, 64, 1000, "float64", 300.0)

# key: (seed, M, n, nq, d, scale)
INDEXED_CASES = {
    "idx0": (300, 12, 0, 2, 8, 0.3),
    "idx1": (301, 12, 1, 2, 8, 0.3),
    "idx2": (302, 12, 5, 2, 8, 0.3),
    "idx3": (303, 4000, 1300, 1, 128, 1.0 / np.sqrt(128)),
}


def dense_inputs(key):
    seed, H, nq, d, nkv, dt, mag = DENSE_CASES[key]
    rng = np.random.default_rng(seed)
    q = (mag * rng.standard_normal((H, nq, d))).astype(dt)
    k = (mag * rng.standard_normal((H, nkv, d))).astype(dt)
    v = rng.standard_normal((H, nkv, d)).astype(dt)
    return q, k, v, 1.0 / np.sqrt(d)


def indexed_inputs(key):
    seed, M, n, nq, d, scale = INDEXED_CASES[key]
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((nq, d)).astype(np.float32)
    k = rng.standard_normal((M, d)).astype(np.float32)
    v = rng.standard_normal((M, d)).astype(np.float32)
    idx = np.sort(rng.choice(M, size=n, replace=False)).astype(np.int64)
    return q, k, v, idx, float(scale)
