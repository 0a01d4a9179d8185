"""Shared test setup.

* `gpu` marker: tests that need a CUDA device (run with -m gpu on a B200).
* oracle/ (CPU restatement of the reference, test infrastructure only) and
  tests/golden/ (fixtures produced by the reference itself) are importable.
* reference_attention: element-by-element fp64 attention, the same test-side
  oracle the reference keeps in pkg/tests/conftest.py:10-41.
"""

import math
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests", "golden")):
    if p not in sys.path:
        sys.path.insert(0, p)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    # the C oracle is test infrastructure: build it if it is missing
    lib = os.path.join(ROOT, "oracle", "_build", "libhgca_oracle.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "all"], check=False,
                       capture_output=True)


def reference_attention(q, k, v, scale):
    """Single head: q [nq, d], k/v [n, d] -> (output, lse, weights) float64."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    nq, d = q.shape
    n = k.shape[0]
    out = np.zeros((nq, d))
    lse = np.full(nq, -np.inf)
    weights = np.zeros((nq, n))
    for i in range(nq):
        scores = []
        for j in range(n):
            s = 0.0
            for c in range(d):
                s += q[i][c] * k[j][c]
            scores.append(s * scale)
        if not scores:
            continue
        m = max(scores)
        exps = [math.exp(s - m) for s in scores]
        z = sum(exps)
        lse[i] = m + math.log(z)
        for j in range(n):
            weights[i][j] = exps[j] / z
            for c in range(d):
                out[i][c] += weights[i][j] * v[j][c]
    return out, lse, weights


def host(x):
    """numpy view of a step result (numpy already when the step got numpy inputs)."""
    return x.detach().cpu().numpy() if hasattr(x, "detach") else np.asarray(x)


@pytest.fixture
def rng():
    return np.random.default_rng(0xC0FFEE)


@pytest.fixture(scope="session")
def golden():
    def load(name):
        return np.load(os.path.join(GOLDEN, name))
    return load


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def cuda():
    if not has_cuda():
        pytest.skip("no CUDA device")
    import paper_2507_03153_b200 as pkg
    pkg._lib.load()
    return pkg


def pytest_collection_modifyitems(config, items):
    """HGCA_TEST_REVERSE=1 runs the collected tests in reverse order (a check
    that no test depends on state an earlier test left behind)."""
    if os.environ.get("HGCA_TEST_REVERSE"):
        items.reverse()
