"""ctypes binding of the C ABI in include/hgca_b200.h (libhgca_b200.so).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ContractError

_HERE = os.path.dirname(os.path.abspath(__file__))
# HGCA_LIB: load an instrumented build of the same library (tools/ only)
LIB_PATH = os.environ.get("HGCA_LIB") or os.path.join(_HERE, "_lib", "libhgca_b200.so")

DTYPE_F32, DTYPE_F64, DTYPE_BF16 = 0, 1, 2
HGCA_OK, HGCA_EINVAL, HGCA_ECUDA = 0, 1, 2

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int
D = ctypes.c_double


class DecodeDesc(ctypes.Structure):
    """Mirror of hgca_decode_desc (include/hgca_b200.h)."""

    _fields_ = [
        ("dtype", ctypes.c_int32), ("pad0", ctypes.c_int32),
        ("B", I64), ("Hq", I64), ("Hkv", I64), ("D", I64), ("T", I64),
        ("KV", P), ("q", P), ("k_new", P), ("v_new", P),
        ("scale", D),
        ("dlo", I64), ("dhi", I64), ("w_old", I64),
        ("sparse_rows", I64),
        ("u_ent", P), ("u_cnt", P), ("item_off", P), ("item_tab", P),
        ("dsc", P), ("dsc_ld", I64),
        ("part_m", P), ("part_z", P), ("part_acc", P), ("max_items", I64),
        ("counter", P),
        ("maw", P), ("alpha", D),
        ("out", P), ("lse", P), ("wts_out", P), ("out_sparse", P), ("lse_sparse", P),
        ("push_n", ctypes.c_int32), ("push_sparse", ctypes.c_int32),
        ("push_dst", P * 8), ("push_flag", P * 8), ("epoch", ctypes.c_uint64), ("push_cnt", P),
        ("item_target", I64),
        ("state", P),
        ("merge_split", I64), ("merge_scratch", P),
    ]


# name -> argtypes (all return int unless listed in _RESTYPES)
_SIGS = {
    "hgca_version": [],
    "hgca_merge_scratch_bytes": [I64, I64, I64, I64],
    "hgca_last_error": [],
    "hgca_attend_ws_bytes": [I64, I64],
    "hgca_attend_dense": [I32, P, P, P, I64, I64, I64, I64, D, I32, P, P, P, P, P],
    "hgca_attend_indexed": [I32, P, P, P, P, I64, I64, I64, I64, D, I32, P, P, P, P, P],
    "hgca_attend_indexed_heads": [I32, P, P, P, I64, I64, P, P, P, I64, I64, I64, D, P, P, P, P, P],
    "hgca_attend_gqa": [I32, P, P, I64, I64, I64, I64, I64, I64, I64, I64, D, P, P, P, I64, P, P],
    "hgca_attend_gqa_indexed": [I32, P, P, I64, I64, I64, I64, P, P, P, I64, I64, I64, D, P, P, P, P, P],
    "hgca_merge_states": [I32, P, P, P, P, I64, I64, P, P, P, P, I64, I64, P, P],
    "hgca_merge_partials": [P, P, I64, I64, I64, P, P, P],
    "hgca_merge_packed": [P, I64, I64, I64, I64, P, P, P],
    "hgca_merge_packed_wait": [P, I64, I64, I64, I64, P, ctypes.c_uint64, I64, P, P, P, P],
    "hgca_peer_alloc": [I64, ctypes.POINTER(P), P],
    "hgca_peer_open": [P, ctypes.POINTER(P)],
    "hgca_peer_close": [P],
    "hgca_peer_free": [P],
    "hgca_select_threshold": [P, I64, I64, I64, I64, D, I64, P, I64, I32, P, P],
    "hgca_mask_to_indices": [P, P, I64, I64, I64, P, I64, P, P, P],
    "hgca_popcount_rows": [P, I64, I64, I64, P, P],
    "hgca_group_need": [P, I64, I64, I64, P, P],
    "hgca_select_topk": [P, I64, I64, I64, P, P, P, I64, P],
    "hgca_write_rows": [I32, P, I64, I64, I64, I64, P, P, I64, P],
    "hgca_decode_chunk_rows": [I32, I64],
    "hgca_decode_config": [I32, I64, I64, P],
    "hgca_item_rows": [I32, P],
    "hgca_maw_update": [P, I64, I64, I64, I64, P, I64, I64, I64, D, I32, P],
    "hgca_maw_ema": [P, I64, I64, I64, P, I64, D, P],
    "hgca_union_build": [P, I64, I64, I64, I64, I64, I64, P, P, P, P, I64, I32, P],
    "hgca_union_build_items": [P, I64, I64, I64, I64, I64, I64, P, P, P, P, I64, I64, I64, I32, P],
    "hgca_union_build_items_w": [P, I64, I64, I64, I64, I64, I64, P, P, P, P, I64, I64, I64, I64, I32, P],
    "hgca_decode_step": [ctypes.POINTER(DecodeDesc), P],
    "hgca_step_state_set": [P, I64, I64, ctypes.c_uint64, P],
    "hgca_decode_step_host": [ctypes.POINTER(DecodeDesc), P, P, I64, P, P, I64, P],
    "hgca_decode_step_host_async": [ctypes.POINTER(DecodeDesc), P, P, I64, P, P, I64, P],
    "hgca_append_ws_bytes": [I64, I64, I64, I64, I64, I64, I64],
    "hgca_append_bf16": [P, I64, I64, I64, I64, I64, P, I64, D, I64, I64, P, P, P, P, P, I64, P],
}
_RESTYPES = {"hgca_last_error": ctypes.c_char_p, "hgca_attend_ws_bytes": I64, "hgca_append_ws_bytes": I64,
             "hgca_merge_scratch_bytes": I64}

_lib = None


def load():
    """Load libhgca_b200.so; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
    return _lib


def exported_symbols():
    return sorted(_SIGS)


def call(name, *args):
    """Invoke a C-ABI entry point and map its status to exceptions."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != HGCA_OK:
        msg = lib.hgca_last_error().decode(errors="replace")
        if rc == HGCA_EINVAL:
            raise ContractError(msg)
        raise RuntimeError(f"{name}: {msg}")
    return rc
