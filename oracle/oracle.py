"""ctypes wrapper around the C oracle (oracle/m2c_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs; never by the product package.  numpy arrays in,
numpy arrays out; every function is a thin marshaller over one C function whose
header comment cites the paper passage it implements.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "m2c_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-fopenmp"]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _setup(_lib)
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _setup(L):
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.orc_half_to_double.restype = C.c_double
    L.orc_half_to_double.argtypes = [C.c_uint16]
    L.orc_double_to_half.restype = C.c_uint16
    L.orc_double_to_half.argtypes = [C.c_double]
    L.orc_float_to_half.restype = C.c_uint16
    L.orc_float_to_half.argtypes = [C.c_float]
    L.orc_tier_plan.argtypes = [i32, i32, i32, i32, i32, vp]
    L.orc_quant_group.argtypes = [C.c_int, vp, C.c_int, vp, vp, vp]
    L.orc_quant_group.restype = None
    L.orc_record_bytes.restype = i64
    L.orc_record_bytes.argtypes = [C.c_int, C.c_int]
    L.orc_pack.argtypes = [C.c_int, C.c_int, vp, vp, vp, i64, i64, vp]
    L.orc_dequant_record.argtypes = [C.c_int, C.c_int, vp, vp, vp, vp]
    L.orc_predict.argtypes = [C.c_int] * 3 + [vp] * 6
    L.orc_select.argtypes = [C.c_int, vp, vp, vp, vp, vp]
    L.orc_ffn.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, C.c_int, vp, vp]
    L.orc_predict_mt.argtypes = [C.c_int] * 3 + [vp] * 6 + [C.c_int]
    L.orc_ffn_mt.argtypes = [C.c_int, vp, vp, vp, vp, vp, vp, C.c_int, vp, C.c_int]
    L.orc_residual.argtypes = [C.c_int, vp, vp, vp, vp]
    L.orc_residual.restype = None
    L.orc_lru_step.argtypes = [C.c_int, C.c_int, vp, vp, vp, i32, vp, C.c_int] + [vp] * 8


def _u16(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint16) if a.dtype == np.float16 else a.astype(np.uint16)


def half_to_double(h: int) -> float:
    return lib().orc_half_to_double(int(h))


def double_to_half(v: float) -> int:
    return lib().orc_double_to_half(float(v))


def float_to_half(v: float) -> int:
    return lib().orc_float_to_half(float(v))


def tier_plan(F_r, active_pct, a16=25, a8=25, den=100):
    out = np.zeros(4, np.int32)
    rc = lib().orc_tier_plan(F_r, active_pct, a16, a8, den, _p(out))
    if rc:
        raise ValueError("invalid tier plan")
    return out


def record_bytes(bits, d):
    return lib().orc_record_bytes(bits, d)


def quant_group(bits, w_f16):
    w = _u16(w_f16)
    s = np.zeros(1, np.uint16)
    z = np.zeros(1, np.uint8)
    q = np.zeros(w.size, np.uint8)
    lib().orc_quant_group(bits, _p(w), w.size, _p(s), _p(z), _p(q))
    return int(s[0]), int(z[0]), q


def pack(bits, gate, up, down_t, n0=0, n1=None):
    gate, up, down_t = _u16(gate), _u16(up), _u16(down_t)
    F, d = gate.shape
    n1 = F if n1 is None else n1
    nb = record_bytes(bits, d)
    out = np.zeros((n1 - n0, nb), np.uint8)
    if lib().orc_pack(bits, d, _p(gate), _p(up), _p(down_t), n0, n1, _p(out)):
        raise ValueError("pack")
    return out


def dequant_record(bits, d, rec):
    rec = np.ascontiguousarray(rec, np.uint8)
    g, u, dn = (np.zeros(d) for _ in range(3))
    if lib().orc_dequant_record(bits, d, _p(rec), _p(g), _p(u), _p(dn)):
        raise ValueError("dequant")
    return g, u, dn


def predict(x, A, B):
    x = _u16(x)
    A = np.ascontiguousarray(A, np.int8)
    B = np.ascontiguousarray(B, np.int8)
    r, d = A.shape
    F_r = B.shape[0]
    h = np.zeros(r, np.int64)
    hq = np.zeros(r, np.int8)
    s = np.zeros(F_r, np.int32)
    if lib().orc_predict(d, r, F_r, _p(x), _p(A), _p(B), _p(h), _p(hq), _p(s)):
        raise ValueError("predict: non-finite x or bad shape")
    return dict(h=h, hq=hq, s=s)


def select(s, plan):
    s = np.ascontiguousarray(s, np.int32)
    plan = np.ascontiguousarray(plan, np.int32)
    F_r = s.size
    k = int(plan[0])
    rank = np.zeros(max(k, 1), np.int32)
    tier_of = np.zeros(max(F_r, 1), np.int8)
    ids = np.zeros(max(k, 1), np.int32)
    if lib().orc_select(F_r, _p(s), _p(plan), _p(rank), _p(tier_of), _p(ids)):
        raise ValueError("select: invalid plan")
    return dict(rank_list=rank[:k], tier_of=tier_of[:F_r], tier_ids=ids[:k])


def ffn(d, plan, tier_ids, rec16, rec8, rec4, x, act=0, return_a=False):
    plan = np.ascontiguousarray(plan, np.int32)
    ids = np.ascontiguousarray(tier_ids, np.int32)
    x = _u16(x)
    y = np.zeros(d)
    a = np.zeros(max(int(plan[0]), 1))
    lib().orc_ffn(d, _p(plan), _p(ids), _p(np.ascontiguousarray(rec16)),
                  _p(np.ascontiguousarray(rec8)), _p(np.ascontiguousarray(rec4)), _p(x), act,
                  _p(y), _p(a))
    return (y, a[: int(plan[0])]) if return_a else y


def predict_mt(x, A, B, threads):
    """predict() with the integer dot products split over `threads` OpenMP threads
    (bit-identical; SURVEY 8(d) multi-core oracle timing)."""
    x = _u16(x)
    A = np.ascontiguousarray(A, np.int8)
    B = np.ascontiguousarray(B, np.int8)
    r, d = A.shape
    F_r = B.shape[0]
    h = np.zeros(r, np.int64)
    hq = np.zeros(r, np.int8)
    s = np.zeros(F_r, np.int32)
    if lib().orc_predict_mt(d, r, F_r, _p(x), _p(A), _p(B), _p(h), _p(hq), _p(s), int(threads)):
        raise ValueError("predict_mt: non-finite x or bad shape")
    return dict(h=h, hq=hq, s=s)


def ffn_mt(d, plan, tier_ids, rec16, rec8, rec4, x, threads, act=0):
    """ffn() over `threads` OpenMP threads: a_n split over neurons, yhat_j split over j with
    the neuron sum in the serial order (bit-identical; SURVEY 8(d) multi-core oracle timing)."""
    plan = np.ascontiguousarray(plan, np.int32)
    ids = np.ascontiguousarray(tier_ids, np.int32)
    x = _u16(x)
    y = np.zeros(d)
    if lib().orc_ffn_mt(d, _p(plan), _p(ids), _p(np.ascontiguousarray(rec16)),
                        _p(np.ascontiguousarray(rec8)), _p(np.ascontiguousarray(rec4)), _p(x), act,
                        _p(y), int(threads)):
        raise ValueError("ffn_mt: bad threads")
    return y


def layer_forward_mt(w, recs, x, plan, threads, act=0):
    """layer_forward() on `threads` cores (timing of the oracle on all host cores)."""
    pr = predict_mt(x, w["pred_A"], w["pred_B"], threads)
    sel = select(pr["s"], plan)
    d = np.asarray(x).size
    yhat = ffn_mt(d, plan, sel["tier_ids"], recs[16], recs[8], recs[4], x, threads, act)
    return dict(pr, **sel, yhat=yhat)


def residual(x, yhat):
    x = _u16(x)
    yhat = np.ascontiguousarray(yhat, np.float64)
    d = x.size
    y16 = np.zeros(d, np.uint16)
    xn = np.zeros(d, np.uint16)
    lib().orc_residual(d, _p(x), _p(yhat), _p(y16), _p(xn))
    return y16.view(np.float16), xn.view(np.float16)


class LRUPool:
    """O7 state of one (layer, tier) pool."""

    def __init__(self, C_, F_r, resident=False):
        self.C, self.F_r = C_, F_r
        if resident:
            assert C_ == F_r
            self.occupant = np.arange(C_, dtype=np.int32)
            self.slot_of = np.arange(F_r, dtype=np.int32)
        else:
            self.occupant = np.full(C_, -1, np.int32)
            self.slot_of = np.full(F_r, -1, np.int32)
        self.last = np.full(C_, -1, np.int32)

    def step(self, t, R):
        R = np.ascontiguousarray(R, np.int32)
        n = R.size
        slots = np.zeros(max(n, 1), np.int32)
        bits = np.zeros(max((n + 31) // 32, 1), np.uint32)
        mi, ms = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
        ei, es = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
        nm, ne = np.zeros(1, np.int32), np.zeros(1, np.int32)
        rc = lib().orc_lru_step(self.C, self.F_r, _p(self.occupant), _p(self.last),
                                _p(self.slot_of), int(t), _p(R), n, _p(slots), _p(bits),
                                _p(mi), _p(ms), _p(nm), _p(ei), _p(es), _p(ne))
        if rc:
            raise ValueError("lru_step: capacity < |R| or R not ascending")
        m, e = int(nm[0]), int(ne[0])
        return dict(slots=slots[:n], hit_bits=bits[: (n + 31) // 32],
                    miss=np.stack([mi[:m], ms[:m]], 1), evict=np.stack([ei[:e], es[:e]], 1))


def layer_records(w, tiers=(16, 8, 4)):
    """Oracle-packed records of all tiers for one layer's master weights (numpy fp16)."""
    return {b: pack(b, w["w_gate"], w["w_up"], w["w_down_t"]) for b in tiers}


def records_for(w, tier_ids, plan):
    """Oracle-packed records of only the neurons ``tier_ids`` selects, each in its own tier
    (rows of other neurons are left zero): the O0 pack applied lazily, for large layers."""
    F, d = w["w_gate"].shape
    seg = [0, int(plan[1]), int(plan[1]) + int(plan[2]), int(plan[0])]
    out = {}
    for t, b in enumerate((16, 8, 4)):
        rec = np.zeros((F, record_bytes(b, d)), np.uint8)
        for n in np.asarray(tier_ids)[seg[t]:seg[t + 1]]:
            rec[n] = pack(b, w["w_gate"], w["w_up"], w["w_down_t"], int(n), int(n) + 1)[0]
        out[b] = rec
    return out


def layer_forward(w, recs, x, plan, act=0):
    """One (token, layer) of the method, O1..O6: returns every intermediate."""
    pr = predict(x, w["pred_A"], w["pred_B"])
    sel = select(pr["s"], plan)
    d = np.asarray(x).size
    yhat, a = ffn(d, plan, sel["tier_ids"], recs[16], recs[8], recs[4], x, act, return_a=True)
    return dict(pr, **sel, yhat=yhat, a=a)
