"""Pins for oracle O0 (pack / quantise / dequantise) and the fp16 conversions it rests on.

Pinned against: numpy's float16 conversion (library routine); the hand-derived worked
examples in tests/golden/quant_examples.txt; closed-form invariants of an asymmetric
min/max quantiser (q in range, deq(0) == 0 exactly, |deq - w| <= s/2 where unclipped);
the record-size arithmetic of SURVEY §8(a) (24576/12576/6432 B at d=4096).
"""
import os

import numpy as np
import pytest

from oracle import oracle as orc

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "quant_examples.txt")


def test_half_decode_matches_numpy_all_finite_codes():
    codes = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    ref = codes.view(np.float16).astype(np.float64)
    fin = np.isfinite(ref)
    got = np.array([orc.half_to_double(int(c)) for c in codes[fin][::97]])
    assert np.array_equal(got, ref[fin][::97])
    assert orc.half_to_double(0x7C00) == np.inf
    assert np.isnan(orc.half_to_double(0x7E00))


def test_half_encode_matches_numpy_rne():
    rng = np.random.default_rng(1)
    # magnitudes spanning subnormals, normals, near-overflow, plus exact ties
    v = np.concatenate([
        rng.standard_normal(4000) * 10.0 ** rng.integers(-9, 5, 4000),
        np.arange(-2048, 2048) * 2.0 ** -25,           # subnormal ties at 2^-25
        (np.arange(1024, 2048) + 0.5) * 2.0 ** -10,    # ties in [1, 2)
        [65504.0, 65519.99, 65520.0, -65520.0, 1e6, 2.0 ** -25, 2.0 ** -26, 0.0, -0.0],
    ])
    with np.errstate(over="ignore"):
        ref = v.astype(np.float16).view(np.uint16)
    got = np.array([orc.double_to_half(x) for x in v], dtype=np.uint16)
    assert np.array_equal(got, ref)


def _golden_rows():
    rows = []
    for line in open(GOLDEN):
        if line.startswith("#") or not line.strip():
            continue
        b, w, s, z, q, dq = [c.strip() for c in line.split("|")]
        rows.append((int(b), np.array(w.split(), float), float(s), int(z),
                     np.array(q.split(), int), np.array(dq.split(), float)))
    return rows


@pytest.mark.parametrize("row", _golden_rows())
def test_worked_examples(row):
    bits, w, s_ref, z_ref, q_ref, dq_ref = row
    s16, z, q = orc.quant_group(bits, w.astype(np.float16))
    assert orc.half_to_double(s16) == s_ref
    assert z == z_ref
    assert np.array_equal(q, q_ref)
    assert np.array_equal((q.astype(float) - z) * orc.half_to_double(s16), dq_ref)


def test_record_bytes_formula():
    # FP16 6d; INT8 3d + 9d/128; INT4 1.5d + 9d/128; padded to 16 B
    assert [orc.record_bytes(b, 4096) for b in (16, 8, 4)] == [24576, 12576, 6432]
    assert [orc.record_bytes(b, 8192) for b in (16, 8, 4)] == [49152, 25152, 12864]
    assert [orc.record_bytes(b, 5120) for b in (16, 8, 4)] == [30720, 15728, 8048]
    assert [orc.record_bytes(b, 256) for b in (16, 8, 4)] == [1536, 800, 416]
    assert orc.record_bytes(4, 100) == -1 and orc.record_bytes(5, 256) == -1


@pytest.mark.parametrize("bits", [8, 4])
def test_quantiser_invariants(bits):
    rng = np.random.default_rng(bits)
    maxq = (1 << bits) - 1
    for trial in range(300):
        scale = 10.0 ** rng.uniform(-6, 3)
        w = (rng.standard_normal(128) * scale + rng.choice([0, 1, -1]) * scale).astype(np.float16)
        if trial % 17 == 0:
            w[:] = np.abs(w)  # one-sided groups
        if trial % 23 == 0:
            w[::3] = 0
        s16, z, q = orc.quant_group(bits, w)
        s = orc.half_to_double(s16)
        assert 0 <= z <= maxq and q.min() >= 0 and q.max() <= maxq
        deq = (q.astype(float) - z) * s
        wf = w.astype(np.float64)
        assert np.all(deq[wf == 0] == 0.0)  # 0 is represented exactly
        err = np.abs(deq - wf)
        unclipped = (q > 0) & (q < maxq)
        # s = fp16(range/maxq) may round below range/maxq: allow one fp16 ulp of s per step
        assert np.all(err[unclipped] <= s / 2 * (1 + 2 ** -9) + 1e-300)
        if s >= 2.0 ** -14:  # normal fp16 scale: rounding of s is relative 2^-11
            assert np.all(err <= s * (1 + 2 ** -9) * 1.01 + 1e-300)


def test_all_zero_group_and_underflow():
    s16, z, q = orc.quant_group(4, np.zeros(128, np.float16))
    assert (orc.half_to_double(s16), z, int(q.max())) == (1.0, 0, 0)
    w = np.zeros(128, np.float16)
    w[5] = np.float16(2.0 ** -24)  # range/maxq underflows fp16 -> s = 2^-24
    s16, z, q = orc.quant_group(8, w)
    assert s16 == 0x0001 and q[5] == 1 and z == 0


def _rand_layer(F, d, seed):
    rng = np.random.default_rng(seed)
    mk = lambda: (rng.standard_normal((F, d)) / np.sqrt(d)).astype(np.float16)
    return mk(), mk(), mk()


def test_fp16_record_is_raw_concatenation():
    g, u, dn = _rand_layer(5, 256, 0)
    rec = orc.pack(16, g, u, dn)
    assert rec.shape == (5, 1536)
    assert np.array_equal(rec[2].view(np.float16), np.concatenate([g[2], u[2], dn[2]]))


@pytest.mark.parametrize("bits", [8, 4])
def test_packed_layout_and_roundtrip(bits):
    d = 384
    g, u, dn = _rand_layer(7, d, bits)
    # plant a group whose quantisation is known by hand: [-1, 0, ..., 0, 1] -> worked example
    g[3, :128] = 0
    g[3, 0], g[3, 1], g[3, 2] = -1, 0.5, 1
    rec = orc.pack(bits, g, u, dn)
    G = d // 128
    data = 3 * d if bits == 8 else 3 * d // 2
    r3 = rec[3]
    s16 = int(r3[data:data + 2].view(np.uint16)[0])
    z = int(r3[data + 6 * G])
    if bits == 4:
        assert (orc.half_to_double(s16), z) == (0.13330078125, 8)
        assert r3[0] == (0 | (12 << 4))          # elements 0,1 -> q 0 (low), 12 (high)
        assert r3[1] & 0x0F == 15                # element 2 -> q 15 (low nibble)
    else:
        assert (orc.half_to_double(s16), z) == (0.007843017578125, 128)
        assert list(r3[:3]) == [0, 192, 255]
    for n in range(7):
        dg, du, dd = orc.dequant_record(bits, d, rec[n])
        for deq, w in ((dg, g[n]), (du, u[n]), (dd, dn[n])):
            for gi in range(G):
                s16, z, q = orc.quant_group(bits, w[gi * 128:(gi + 1) * 128])
                s = orc.half_to_double(s16)
                assert np.array_equal(deq[gi * 128:(gi + 1) * 128], (q.astype(float) - z) * s)
                assert np.all(np.abs(deq[gi * 128:(gi + 1) * 128]
                                     - w[gi * 128:(gi + 1) * 128].astype(float)) <= s * 1.01)


def test_fifty_percent_bytes_law():
    # P:430 / S:67: 25/25/50 over (16, 8, 4) bits -> 50% of all-FP16 data bytes
    d, k = 4096, 1000
    plan = orc.tier_plan(10000, 10)
    assert list(plan) == [1000, 250, 250, 500]
    data = plan[1] * 6 * d + plan[2] * 3 * d + plan[3] * 1.5 * d
    assert data == 0.5 * k * 6 * d
    # with D4 metadata at g=128: 7B shape, k = 1100 -> 0.5088
    p7 = orc.tier_plan(11008, 10)
    nb = [orc.record_bytes(b, 4096) for b in (16, 8, 4)]
    ratio = sum(int(p7[i + 1]) * nb[i] for i in range(3)) / (int(p7[0]) * nb[0])
    assert abs(ratio - 0.5088) < 1e-4
