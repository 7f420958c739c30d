"""ctypes loader for libm2c.so (the C ABI in include/m2c.h).  Marshalling only.

There is no fallback: if the shared library is missing this raises, and every compute call
needs a CUDA device (the library itself refuses anything but sm_100).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# (M2C_LIB: another build of the same library, for same-box A/B measurements in tools/)
LIB_PATH = os.environ.get("M2C_LIB") or os.path.join(_HERE, "libm2c.so")


class M2CError(RuntimeError):
    STATUS = {1: "INVALID_ARG", 2: "CONFIG", 3: "CAPACITY", 4: "CUDA", 5: "NCCL", 6: "STATE"}

    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"m2c error {code} ({self.STATUS.get(code, '?')}): {msg}")


class ModelDesc(C.Structure):
    _fields_ = [("d_model", C.c_int32), ("d_ff", C.c_int32), ("n_layers", C.c_int32),
                ("pred_rank", C.c_int32), ("group", C.c_int32), ("shard_index", C.c_int32),
                ("shard_count", C.c_int32), ("act", C.c_int32)]


class TierPlan(C.Structure):
    _fields_ = [("k", C.c_int32), ("k_fp16", C.c_int32), ("k_int8", C.c_int32),
                ("k_int4", C.c_int32)]

    def as_tuple(self):
        return (self.k, self.k_fp16, self.k_int8, self.k_int4)


class CacheCfg(C.Structure):
    _fields_ = [("mode", C.c_int32), ("cap_slots", C.c_int32 * 3)]


# every symbol include/m2c.h declares: (name, restype, argtypes)
_vp, _i32, _i64, _sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
_P = C.POINTER
SIGNATURES = [
    ("m2c_last_error", C.c_char_p, []),
    ("m2c_abi_version", _i32, []),
    ("m2c_record_bytes", _i64, [_i32, _i32]),
    ("m2c_tier_plan_make", C.c_int, [_i32, _i32, _i32, _i32, _i32, _P(TierPlan)]),
    ("m2c_cache_cfg_capped", C.c_int, [_P(ModelDesc), _P(TierPlan), _i32, _i32, _i32, _P(CacheCfg)]),
    ("m2c_layer_footprint", C.c_int, [_P(ModelDesc), _P(CacheCfg), _P(_sz), _P(_sz)]),
    ("m2c_create", C.c_int, [_P(ModelDesc), _i32, _vp, _vp, _P(TierPlan), _P(_vp)]),
    ("m2c_destroy", C.c_int, [_vp]),
    ("m2c_quant_pack", C.c_int, [_i32, _i32, _vp, _vp, _vp, _i64, _i64, _vp, _vp]),
    ("m2c_load_layer", C.c_int, [_vp, _i32, _vp, _vp, _vp, _vp, _vp, _P(CacheCfg), _vp, _vp]),
    ("m2c_predict_rank", C.c_int, [_vp, _i32, _vp, _P(TierPlan), _vp, _vp, _vp, _vp]),
    ("m2c_cache_lookup_fill", C.c_int,
     [_vp, _i32, _i64, _vp, _P(TierPlan), _vp, _vp, _vp, _vp, _vp, _vp]),
    ("m2c_sparse_ffn_forward", C.c_int,
     [_vp, _i32, _vp, _vp, _vp, _vp, _P(TierPlan), _vp, _vp, _vp]),
    ("m2c_nccl_unique_id", C.c_int, [C.c_char_p, _vp]),
    ("m2c_comm_init", C.c_int, [_vp, _i32, _i32, _vp, C.c_char_p]),
    ("m2c_p2p_buffer", C.c_int, [_vp, _P(C.c_uint64), _vp]),
    ("m2c_p2p_connect", C.c_int, [_vp, _i32, _vp, _vp]),
    ("m2c_set_grid", C.c_int, [_vp, _i32]),
    ("m2c_decode_step", C.c_int, [_vp, _vp, _i64]),
    ("m2c_decode_lists", C.c_int, [_vp, _i32, _vp]),
    ("m2c_set_graph", C.c_int, [_vp, _i32]),
    ("m2c_set_trace", C.c_int, [_vp, _vp, _vp]),
    ("m2c_cache_state", C.c_int, [_vp, _i32, _i32, _vp, _vp, _P(_i32)]),
    ("m2c_set_fused", C.c_int, [_vp, _i32]),
    ("m2c_stats", C.c_int, [_vp, _P(_i64), _P(_i64), _P(_i64), _i32]),
    ("m2c_profile", C.c_int, [_vp, _i32]),
    ("m2c_profile_read", C.c_int, [_vp, _P(C.c_float), _P(_i32)]),
    ("m2c_profile_fill", C.c_int, [_vp, _P(C.c_float)]),
    ("m2c_profile_events", C.c_int, [_vp, _P(C.c_float), _i64, _P(_i64)]),
    ("m2c_profile_stamps", C.c_int, [_vp, _P(C.c_uint64), _i64, _P(_i64)]),
    ("m2c_predict_candidates", C.c_int, [_vp, _i32, _vp, _i32, _vp]),
    ("m2c_select_global", C.c_int, [_vp, _vp, _i32, _P(TierPlan), _vp, _vp]),
    ("m2c_set_global_topk", C.c_int, [_vp, _P(TierPlan)]),
    ("m2c_set_lookahead", C.c_int, [_vp, _i32]),
    ("m2c_lookahead_stats", C.c_int, [_vp, _P(_i64), _i32]),
    ("m2c_set_requant", C.c_int, [_vp, _i32]),
    ("m2c_requant_stats", C.c_int, [_vp, _P(_i64), _i32]),
    ("m2c_store_frame_bytes", _sz, [_P(ModelDesc), _P(CacheCfg)]),
    ("m2c_store_write", C.c_int, [_vp, C.c_char_p]),
    ("m2c_store_attach", C.c_int, [_vp, C.c_char_p, _i32, _i32, _i32, _vp, _sz]),
    ("m2c_store_detach", C.c_int, [_vp]),
    ("m2c_store_stats", C.c_int, [_vp, _P(_i64), _P(_i64), _P(C.c_double), _P(C.c_double)]),
]

_lib = None


def lib():
    """Load libm2c.so (raises if it was not built: there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                              "(the CUDA extension is required, there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, res, args in SIGNATURES:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        raise M2CError(status, lib().m2c_last_error().decode(errors="replace"))
