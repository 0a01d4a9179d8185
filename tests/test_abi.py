"""CPU: the C-ABI library loads and exports exactly what include/hgca_b200.h
declares; the ctypes binding agrees with the header (no compute calls)."""

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "hgca_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(hgca_\w+)\s*\(", text, flags=re.M)))


def test_library_builds_and_loads():
    import paper_2507_03153_b200 as pkg
    from paper_2507_03153_b200 import _build

    _build.build()
    lib = pkg._lib.load()
    assert lib.hgca_version() == 1


def test_every_declared_symbol_is_exported_and_bound():
    from paper_2507_03153_b200 import _lib

    decl = declared_functions()
    assert len(decl) >= 19
    raw = ctypes.CDLL(_lib.LIB_PATH)
    for name in decl:
        assert hasattr(raw, name), f"{name} declared in hgca_b200.h but not exported"
    assert sorted(_lib.exported_symbols()) == decl


def test_nm_exports_only_the_abi():
    from paper_2507_03153_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted({l.split()[-1] for l in out.splitlines() if " T hgca_" in l})
    assert exported == declared_functions()


def test_decode_desc_layout_matches_header():
    """Compile a probe against the header and compare field offsets with ctypes."""
    from paper_2507_03153_b200._lib import DecodeDesc

    fields = [f for f, _ in DecodeDesc._fields_]
    src = "#include <stdio.h>\n#include <stddef.h>\n#include \"hgca_b200.h\"\nint main(){\n"
    src += f'printf("%zu\\n", sizeof(hgca_decode_desc));\n'
    for f in fields:
        src += f'printf("%zu\\n", offsetof(hgca_decode_desc, {f}));\n'
    src += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "p.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "p")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        vals = [int(x) for x in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(DecodeDesc)
    for f, off in zip(fields, vals[1:]):
        assert getattr(DecodeDesc, f).offset == off, f


def test_contract_errors_without_gpu():
    from paper_2507_03153_b200 import CacheConfig, ContractError, EngineConfig, HeadShape, StepInput
    import numpy as np

    with pytest.raises(ContractError):
        HeadShape(0, 4)
    with pytest.raises(ContractError):
        CacheConfig(blk_num=1, blk_size=4)
    with pytest.raises(ContractError):
        EngineConfig(heads=32, kv_heads=5)
    with pytest.raises(ContractError):
        EngineConfig(dtype="float16")
    z = np.zeros((2, 3, 4), np.float32)
    with pytest.raises(ContractError):
        StepInput("decode", z, z, z)
    with pytest.raises(ContractError):
        StepInput("prefill", z[:, :1], z[:, :1], z[:, :1])
    assert issubclass(ContractError, ValueError)


def test_product_path_fails_loudly_without_cuda():
    import torch
    from paper_2507_03153_b200 import attend, HeadShape

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    import numpy as np

    with pytest.raises(RuntimeError, match="CUDA"):
        attend(np.ones((1, 4)), np.ones((2, 4)), np.ones((2, 4)), HeadShape(1, 4))
