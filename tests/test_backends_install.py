"""install(): the `cuda` backend registered in a tierkv.backends-shaped module
(backends.py:65-100: `_BACKENDS` registry + module-level `active`), and the
reference's attention entry points driven through `backends.active` the way
attention.py:118/147 call it."""

import types

import numpy as np
import pytest

from cases import DENSE_CASES, INDEXED_CASES, dense_inputs, indexed_inputs


def stand_in():
    """A module with the reference's plugin-slot shape (no tierkv import needed)."""
    numpy_backend = types.SimpleNamespace(name="numpy")
    return types.SimpleNamespace(_BACKENDS={"numpy": numpy_backend}, active=numpy_backend)


def test_install_registers_and_activates():
    from paper_2507_03153_b200 import backends

    mod = stand_in()
    numpy_backend = mod.active
    ret = backends.install(mod, activate=False)
    assert ret is backends.CUDA and mod._BACKENDS["cuda"] is backends.CUDA
    assert mod.active is numpy_backend  # registered, not selected
    backends.install(mod)
    assert mod.active is backends.CUDA and mod.active.name == "cuda"
    assert callable(mod.active.attend_dense) and callable(mod.active.attend_indexed)


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(DENSE_CASES)[:4])
def test_active_attend_dense_matches_reference(cuda, key, golden):
    mod = stand_in()
    cuda.backends.install(mod)
    g = golden("kernels.npz")
    q, k, v, scale = dense_inputs(key)
    o, l, w = mod.active.attend_dense(q, k, v, scale, True)
    t = 1e-10 if q.dtype == np.float64 else 1e-6
    go, gl = g[f"{key}_out"], g[f"{key}_lse"]
    np.testing.assert_allclose(o, go, atol=t * max(1.0, np.abs(go).max()), rtol=0)
    np.testing.assert_allclose(l, gl, atol=t * max(1.0, np.abs(gl[np.isfinite(gl)]).max(initial=1)), rtol=0)
    np.testing.assert_allclose(w, g[f"{key}_w"], atol=t, rtol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(INDEXED_CASES)[:4])
def test_active_attend_indexed_matches_reference(cuda, key, golden):
    mod = stand_in()
    cuda.backends.install(mod)
    g = golden("kernels.npz")
    q, k, v, idx, scale = indexed_inputs(key)
    o, l, w = mod.active.attend_indexed(q, k, v, idx, scale, True)
    np.testing.assert_allclose(o, g[f"{key}_out"], atol=1e-6, rtol=0)
    np.testing.assert_allclose(l, g[f"{key}_lse"], atol=1e-6, rtol=0)
    np.testing.assert_allclose(w, g[f"{key}_w"], atol=1e-7, rtol=0)
