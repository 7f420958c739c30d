"""Pins for oracle O1-O5 (exact-integer predictor, top-k, tier split).

Pinned against: python big-integer matmul on exact rationals for O1/O2, numpy int64 matmul
(library routine) for O4; closed-form special cases (x = 0, x = c*e_j, subnormals, fp16-max
magnitudes, half-up ties) for O2/O3; python ``sorted`` brute force for O5; SPEC's
partition example 250/250/500 and the survey's per-config tier counts.
"""
from fractions import Fraction

import numpy as np
import pytest

from oracle import oracle as orc


def _exact_q127(v, M):
    # round-half-away-from-zero of 127*v/M with exact rationals (independent of the C integer trick)
    if M == 0:
        return 0
    f = Fraction(127) * Fraction(abs(int(v))) / Fraction(int(M))
    q = int(f + Fraction(1, 2))  # floor(f + 1/2) for f >= 0
    return q if v >= 0 else -q


def _rand_pred(d, r, F, seed):
    rng = np.random.default_rng(seed)
    A = rng.integers(-127, 128, (r, d)).astype(np.int8)
    B = rng.integers(-127, 128, (F, r)).astype(np.int8)
    x = (rng.standard_normal(d) * 1.3).astype(np.float16)
    return x, A, B


def _X(x):
    # x_j * 2^24 as an exact python integer (exact rationals, independent of the C conversion)
    return [int(Fraction(float(v)) * (1 << 24)) for v in np.asarray(x, np.float16).astype(np.float64)]


@pytest.mark.parametrize("seed", range(4))
def test_predictor_matches_bigint_matmul_and_exact_rounding(seed):
    d, r, F = 256, 32, 688
    x, A, B = _rand_pred(d, r, F, seed)
    out = orc.predict(x, A, B)
    X = _X(x)
    h = [sum(int(a) * xv for a, xv in zip(row, X)) for row in A.tolist()]  # python big ints
    assert [int(v) for v in out["h"]] == h
    Mh = max(abs(v) for v in h)
    assert [int(q) for q in out["hq"]] == [_exact_q127(v, Mh) for v in h]
    assert np.array_equal(out["s"], B.astype(np.int64) @ out["hq"].astype(np.int64))
    assert np.abs(out["hq"]).max() == 127


def test_predictor_extreme_magnitudes_no_overflow():
    # |x| = 65504 (fp16 max) everywhere with A = +-127: |h| ~ 2^59.9 must stay exact (int64)
    d, r, F = 8192, 4, 8
    A = np.full((r, d), 127, np.int8)
    A[1] = -127
    A[2, ::2] = -127
    A[3, :] = 0
    A[3, 5] = 1
    x = np.full(d, 65504.0, np.float16)
    B = np.eye(F, r, dtype=np.int8)
    out = orc.predict(x, A, B)
    X = _X(x)
    h = [sum(int(a) * xv for a, xv in zip(row, X)) for row in A.tolist()]
    assert [int(v) for v in out["h"]] == h
    assert h[0] == 127 * 8192 * 65504 * (1 << 24) and h[2] == 0
    # hq = Q(h): M = h[0]; h[1] = -M -> -127; h[3] = X_5 -> 127 X_5 / M rounds to 0
    assert [int(q) for q in out["hq"]] == [127, -127, 0, 0]


def test_predictor_special_cases():
    d, r, F = 128, 16, 64
    _, A, B = _rand_pred(d, r, F, 9)
    z = orc.predict(np.zeros(d, np.float16), A, B)
    assert not z["h"].any() and not z["hq"].any() and not z["s"].any()
    # x = c e_j  =>  h = c 2^24 A[:, j] exactly, hq = Q(A[:, j]) (scale-free)
    x = np.zeros(d, np.float16)
    x[7] = -3.0
    e = orc.predict(x, A, B)
    assert np.array_equal(e["h"], -3 * (1 << 24) * A[:, 7].astype(np.int64))
    col = [-int(v) for v in A[:, 7]]
    M = max(abs(v) for v in col)
    assert [int(q) for q in e["hq"]] == [_exact_q127(v, M) for v in col]
    # subnormal x: 2^-24 is X = 1
    x = np.zeros(d, np.float16)
    x[3] = np.float16(2.0 ** -24)
    assert np.array_equal(orc.predict(x, A, B)["h"], A[:, 3].astype(np.int64))
    # half-up tie in O3: h = (2, 1, -1) * c  ->  hq = (127, 64, -64)
    A2 = np.zeros((3, d), np.int8)
    A2[0, 0], A2[1, 0], A2[2, 0] = 2, 1, -1
    x = np.zeros(d, np.float16)
    x[0] = 0.5
    assert list(orc.predict(x, A2, B[:, :3])["hq"]) == [127, 64, -64]
    bad = np.zeros(d, np.float16)
    bad[3] = np.inf
    with pytest.raises(ValueError):
        orc.predict(bad, A, B)


def _brute_select(s, plan):
    k, k16, k8, _ = (int(v) for v in plan)
    order = sorted(range(len(s)), key=lambda n: (-int(s[n]), n))[:k]
    tier = {n: (0 if i < k16 else 1 if i < k16 + k8 else 2) for i, n in enumerate(order)}
    ids = [n for t in range(3) for n in sorted(m for m in order if tier[m] == t)]
    tier_of = [tier.get(n, -1) for n in range(len(s))]
    return order, tier_of, ids


@pytest.mark.parametrize("seed", range(6))
def test_select_matches_bruteforce_with_heavy_ties(seed):
    rng = np.random.default_rng(seed)
    F = int(rng.integers(1, 900))
    s = rng.integers(-4, 5, F).astype(np.int32) * int(rng.choice([1, 1000]))  # many ties
    pct = int(rng.integers(0, 101))
    plan = orc.tier_plan(F, pct, *[(25, 25, 100), (300, 0, 300), (0, 100, 300), (75, 75, 300)][seed % 4])
    got = orc.select(s, plan)
    order, tier_of, ids = _brute_select(s, plan)
    assert list(got["rank_list"]) == order
    assert list(got["tier_of"]) == tier_of
    assert list(got["tier_ids"]) == ids


def test_tier_plans_of_the_configs():
    # (0.25, 0.25, 0.5) on k = 1000 -> 250/250/500 ; SURVEY §8(a) per-config counts
    assert list(orc.tier_plan(10000, 10)) == [1000, 250, 250, 500]
    assert list(orc.tier_plan(688, 10)) == [68, 17, 17, 34]
    assert list(orc.tier_plan(11008, 10)) == [1100, 275, 275, 550]
    assert list(orc.tier_plan(13824, 10)) == [1382, 345, 345, 692]
    assert list(orc.tier_plan(28672, 10)) == [2867, 716, 716, 1435]
    assert list(orc.tier_plan(3584, 10)) == [358, 89, 89, 180]
    # sweep rule: FP16 share s%, rest INT8:INT4 = 1:2 -> weights (3s, 100-s)/300
    assert list(orc.tier_plan(3584, 50, 0, 100, 300)) == [1792, 0, 597, 1195]
    assert list(orc.tier_plan(3584, 50, 300, 0, 300)) == [1792, 1792, 0, 0]
    with pytest.raises(ValueError):
        orc.tier_plan(100, 101)


def test_tier_sizes_independent_of_scores():
    rng = np.random.default_rng(3)
    plan = orc.tier_plan(500, 20)
    for _ in range(5):
        s = rng.integers(-10 ** 6, 10 ** 6, 500).astype(np.int32)
        t = orc.select(s, plan)["tier_of"]
        assert [(t == i).sum() for i in range(3)] == list(plan[1:])


def test_zero_input_ranks_are_ids():
    # x = 0 -> all scores 0 -> ranks are ids 0..k-1 (SURVEY §8(c) pins)
    x, A, B = _rand_pred(256, 32, 688, 1)
    s = orc.predict(np.zeros_like(x), A, B)["s"]
    plan = orc.tier_plan(688, 10)
    assert list(orc.select(s, plan)["rank_list"]) == list(range(68))
