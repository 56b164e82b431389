"""ctypes binding of the C ABI in include/ott_b200.h (libott_b200.so, sm_100a).

This is the only way the host layer reaches the GPU: there is no CPU fallback.
If the library is missing or cannot load, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

from .errors import ContractViolation, NativeError

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("OTT_LIB_PATH") or os.path.join(_PKG, "_lib", "libott_b200.so")
CSRC = os.path.join(_PKG, "csrc")

OTT_OK, OTT_ERR_CONTRACT, OTT_ERR_UNSUPPORTED, OTT_ERR_CUDA = 0, 1, 2, 3

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64


MAX_OUT_PEERS = 7  # OTT_MAX_OUT_PEERS


class OttCacheT(ctypes.Structure):
    """Mirror of ott_cache_t (include/ott_b200.h)."""

    _fields_ = [
        ("n_units", _i32), ("head_dim", _i32), ("group_size", _i32), ("residual", _i32),
        ("capacity", _i32), ("aux_capacity", _i32), ("bits", _i32), ("max_groups", _i32),
        ("blocks", _vp), ("pend_k", _vp), ("pend_v", _vp), ("pool_mask", _vp), ("subst_mask", _vp),
        ("pool_pos", _vp), ("pool_score", _vp), ("pool_k", _vp), ("pool_v", _vp),
        ("aux_pos", _vp), ("aux_score", _vp), ("aux_k", _vp), ("aux_v", _vp),
        ("pool_meta", _vp), ("params64", _vp),
        ("n_out_peers", _i32), ("out_peer", _vp * MAX_OUT_PEERS),
    ]


_lib = None


def build(verbose: bool = False) -> str:
    """Compile libott_b200.so for sm_100a with nvcc (csrc/Makefile)."""
    r = subprocess.run(["make", "-s", "-j4", "-C", CSRC], capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise NativeError(f"nvcc build failed:\n{r.stdout}\n{r.stderr}")
    return LIB_PATH


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER(OttCacheT)
        L.ott_record_bytes.argtypes = [_i32, _i32, _i32]
        L.ott_record_bytes.restype = ctypes.c_size_t
        L.ott_ring_write.argtypes = [P, _vp, _vp, _i64, _i64, _i64, _i64, _vp]
        L.ott_flush.argtypes = [P, _i64, _i32, _i64, _vp, _vp, _i64, _i64, _vp]
        L.ott_pick_splits.argtypes = [P, _i32, _i64]
        L.ott_attend_workspace_floats.argtypes = [P, _i32, _i32]
        L.ott_attend_workspace_floats.restype = ctypes.c_size_t
        L.ott_attend.argtypes = [P, _vp, _vp, _i32, _i64, _i64, _vp, _i32, _vp]
        L.ott_logits.argtypes = [P, _vp, _vp, _i32, _i64, _i64, _vp]
        L.ott_decode_step.argtypes = [P, _vp, _vp, _vp, _vp, _i32, _vp, _vp, _i32, _vp]
        L.ott_append_attend.argtypes = [P, _vp, _vp, _vp, _vp, _i32, _i64, _i64, _vp, _i32, _vp]
        L.ott_model_rmsnorm.argtypes = [_vp, _vp, _vp, _i32, _i32, ctypes.c_float, _vp]
        L.ott_model_rope_qkv.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp]
        L.ott_model_silu_mul.argtypes = [_vp, _vp, _i32, _i32, _vp]
        L.ott_attend_exact.argtypes = [_vp, _vp, _vp, _i32, _i32, _i32, _vp, _vp, _vp, _vp]
        L.ott_pool_rank.argtypes = [_vp, _vp, _i32, _vp, _vp]
        L.ott_score_rows.argtypes = [_vp, _i32, _i32, _vp, _vp]
        L.ott_num_sms.argtypes = []
        L.ott_version.restype = ctypes.c_char_p
        L.ott_last_error.restype = ctypes.c_char_p
        L.ott_cache_struct_bytes.restype = ctypes.c_size_t
        if L.ott_cache_struct_bytes() != ctypes.sizeof(OttCacheT):
            raise NativeError(f"ott_cache_t layout mismatch: library {L.ott_cache_struct_bytes()} bytes, "
                              f"binding {ctypes.sizeof(OttCacheT)}")
        _lib = L
    return _lib


EXPORTED = ("ott_record_bytes", "ott_ring_write", "ott_flush", "ott_pick_splits", "ott_attend_workspace_floats",
            "ott_attend", "ott_logits", "ott_append_attend", "ott_decode_step", "ott_num_sms", "ott_version", "ott_last_error",
            "ott_cache_struct_bytes", "ott_model_rmsnorm", "ott_model_rope_qkv", "ott_model_silu_mul",
            "ott_attend_exact", "ott_pool_rank", "ott_score_rows")


def check(status: int) -> None:
    if status == OTT_OK:
        return
    msg = lib().ott_last_error().decode()
    if status in (OTT_ERR_CONTRACT, OTT_ERR_UNSUPPORTED):
        raise ContractViolation(msg)
    raise NativeError(msg)
