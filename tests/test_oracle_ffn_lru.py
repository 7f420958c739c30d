"""Pins for oracle O6 (sparse mixed-precision FFN), O7 (LRU) and O8 (residual).

O6 pinned against: the dense FFN y = W_d (silu(W_g x) * W_u x) in numpy float64 when 100% of
neurons are active in FP16 (the method reduces to the textbook FFN); a numpy float64
gather-matmul over the exact dequantised weights of the selected set.
O7 pinned against: an independently written move-to-front list LRU; SPEC's ATU/LRU examples
(S:263); the closed-form ATU miss ratio of SPEC's retention trace model.
O8 pinned against numpy float16 rounding.
"""
import numpy as np
import pytest

from oracle import oracle as orc


def _layer(F, d, seed, sd=0.05):
    rng = np.random.default_rng(seed)
    g = (rng.standard_normal((F, d)) / np.sqrt(d)).astype(np.float16)
    u = (rng.standard_normal((F, d)) / np.sqrt(d)).astype(np.float16)
    dn = (rng.standard_normal((F, d)) * sd).astype(np.float16)
    x = rng.standard_normal(d).astype(np.float16)
    return g, u, dn, x


@pytest.mark.parametrize("act", [0, 1])
def test_dense_equivalence_all_active_fp16(act):
    F, d = 300, 256
    g, u, dn, x = _layer(F, d, 5)
    plan = orc.tier_plan(F, 100, 100, 0, 100)
    assert list(plan) == [F, F, 0, 0]
    rec16 = orc.pack(16, g, u, dn)
    ids = np.arange(F, dtype=np.int32)
    empty = np.zeros((1, 16), np.uint8)
    y = orc.ffn(d, plan, ids, rec16, empty, empty, x, act)
    xf = x.astype(np.float64)
    gg = g.astype(np.float64) @ xf
    uu = u.astype(np.float64) @ xf
    a = (gg / (1 + np.exp(-gg)) if act == 0 else np.maximum(gg, 0)) * uu
    ref = dn.astype(np.float64).T @ a
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_mixed_tiers_equal_gather_matmul():
    F, d = 400, 384
    g, u, dn, x = _layer(F, d, 6)
    recs = {b: orc.pack(b, g, u, dn) for b in (16, 8, 4)}
    rng = np.random.default_rng(0)
    plan = orc.tier_plan(F, 20)
    s = rng.integers(-1000, 1000, F).astype(np.int32)
    sel = orc.select(s, plan)
    y, a = orc.ffn(d, plan, sel["tier_ids"], recs[16], recs[8], recs[4], x, return_a=True)
    bits = [16] * plan[1] + [8] * plan[2] + [4] * plan[3]
    Wg, Wu, Wd = [], [], []
    for n, b in zip(sel["tier_ids"], bits):
        dg, du, dd = orc.dequant_record(b, d, recs[b][n])
        Wg.append(dg), Wu.append(du), Wd.append(dd)
    Wg, Wu, Wd = map(np.array, (Wg, Wu, Wd))
    xf = x.astype(np.float64)
    gg, uu = Wg @ xf, Wu @ xf
    a_ref = gg / (1 + np.exp(-gg)) * uu
    assert np.allclose(a, a_ref, rtol=1e-12, atol=0)
    ref = Wd.T @ a_ref
    assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref))
    # quantised tiers stay close to the FP16 weights (sanity: dequant is not garbage)
    y16 = orc.ffn(d, orc.tier_plan(F, 20, 100, 0, 100), np.sort(sel["rank_list"]), recs[16],
                  recs[8], recs[4], x)
    assert np.max(np.abs(y - y16)) < 0.2 * np.max(np.abs(y16))


@pytest.mark.parametrize("threads", [1, 3, 8])
def test_multicore_oracle_is_bit_identical(threads):
    """SURVEY 8(d)'s multi-core oracle timing variant computes exactly what the serial oracle
    does (same per-output operation order); its timing is therefore of the same program."""
    F, d, r = 400, 384, 32
    g, u, dn, x = _layer(F, d, 7)
    recs = {b: orc.pack(b, g, u, dn) for b in (16, 8, 4)}
    rng = np.random.default_rng(1)
    A = rng.integers(-127, 128, (r, d)).astype(np.int8)
    B = rng.integers(-127, 128, (F, r)).astype(np.int8)
    w = {"pred_A": A, "pred_B": B}
    plan = orc.tier_plan(F, 20)
    for act in (0, 1):
        ref = orc.layer_forward(w, recs, x, plan, act)
        got = orc.layer_forward_mt(w, recs, x, plan, threads, act)
        for key in ("h", "hq", "s", "tier_ids"):
            assert np.array_equal(ref[key], got[key]), key
        assert np.array_equal(ref["yhat"], got["yhat"])


def test_residual_rounding():
    rng = np.random.default_rng(2)
    x = rng.standard_normal(4096).astype(np.float16)
    yhat = rng.standard_normal(4096) * 10.0 ** rng.integers(-6, 2, 4096)
    y16, xn = orc.residual(x, yhat)
    assert np.array_equal(y16, yhat.astype(np.float16))
    assert np.array_equal(xn, (x.astype(np.float64) + y16.astype(np.float64)).astype(np.float16))


# ---------------------------------------------------------------- O7: LRU
class ListLRU:
    """Independent move-to-front model of reading R7: a recency list of slots, front = most
    recent.  Slots touched in the same step are ordered among themselves by slot id, larger
    ids nearer the front (so the back-most, i.e. first victim, is the smallest slot)."""

    def __init__(self, C):
        self.order = list(range(C - 1, -1, -1))  # back of list = end = slot 0 first victim
        self.occ = [None] * C

    def step(self, R):
        where = {n: s for s, n in enumerate(self.occ) if n is not None}
        hits = [n for n in R if n in where]
        misses = [n for n in R if n not in where]
        touched = [where[n] for n in hits]
        stale = [s for s in self.order if s not in set(touched)]
        victims = stale[::-1][: len(misses)]  # from the back
        ev, placed = [], {}
        for n, s in zip(misses, victims):
            if self.occ[s] is not None:
                ev.append((self.occ[s], s))
            self.occ[s] = n
            placed[n] = s
        touched_all = sorted(touched + victims, reverse=True)
        self.order = touched_all + [s for s in stale if s not in set(victims)]
        slots = [where.get(n, placed.get(n)) for n in R]
        return slots, [n in where for n in R], list(zip(misses, victims)), ev


@pytest.mark.parametrize("C", [16, 24, 64])
def test_lru_matches_list_model(C):
    F, k = 64, 16
    rng = np.random.default_rng(C)
    pool, ref = orc.LRUPool(C, F), ListLRU(C)
    A = set(rng.choice(F, k, replace=False).tolist())
    for t in range(200):
        keep = {n for n in A if rng.random() < 0.7}
        rest = [n for n in range(F) if n not in keep]
        A = keep | set(rng.choice(rest, k - len(keep), replace=False).tolist())
        R = np.array(sorted(A), np.int32)
        out = pool.step(t, R)
        slots, hit, miss, ev = ref.step(list(R))
        assert list(out["slots"]) == slots
        bits = [(int(out["hit_bits"][i // 32]) >> (i % 32)) & 1 for i in range(k)]
        assert bits == [int(h) for h in hit]
        assert [tuple(m) for m in out["miss"]] == miss
        assert [tuple(e) for e in out["evict"]] == ev
        # invariants: hits and misses partition R; a hit never moves slot
        assert sum(bits) + len(miss) == k
        assert all(pool.occupant[s] == n for n, s in zip(R, out["slots"]))
        if C == k:  # ATU: resident set == required set, |evictions| == |misses| once full
            assert set(pool.occupant.tolist()) == set(R.tolist())
            if t > 0:
                assert len(ev) == len(miss)


def test_spec_examples():
    # S:263 ATU: resident {1,2,3,4}, required {1,2,3,5} -> 3 hits, miss {5}, evict {4}
    p = orc.LRUPool(4, 8)
    p.step(0, [1, 2, 3, 4])
    out = p.step(1, [1, 2, 3, 5])
    assert out["hit_bits"][0] == 0b0111 and out["miss"][:, 0].tolist() == [5]
    assert out["evict"][:, 0].tolist() == [4]
    # S:264 cold unit -> 0 hits, k misses, 0 evictions
    out = orc.LRUPool(4, 8).step(0, [0, 3, 5, 7])
    assert out["hit_bits"][0] == 0 and len(out["miss"]) == 4 and len(out["evict"]) == 0
    # S:274 3-slot unit, accesses 1, 2, 3 then require {4} -> evict 1
    p = orc.LRUPool(3, 8)
    for t, n in enumerate([1, 2, 3]):
        p.step(t, [n])
    assert p.step(3, [4])["evict"][:, 0].tolist() == [1]
    # S:273 slack >= F - k -> no evictions after warm-up
    p = orc.LRUPool(8, 8)
    rng = np.random.default_rng(0)
    evs = [len(p.step(t, np.sort(rng.choice(8, 3, replace=False)))["evict"]) for t in range(50)]
    assert sum(evs) == 0
    # resident mode: identity, always hits
    p = orc.LRUPool(8, 8, resident=True)
    out = p.step(0, [2, 5])
    assert out["slots"].tolist() == [2, 5] and out["hit_bits"][0] == 0b11
    with pytest.raises(ValueError):
        orc.LRUPool(2, 8).step(0, [1, 2, 3])


def test_slack_zero_lru_misses_equal_atu_set_difference():
    # with capacity k the miss set at every step is R_t minus R_{t-1}
    F, k = 200, 20
    rng = np.random.default_rng(4)
    p = orc.LRUPool(k, F)
    prev = set()
    for t in range(100):
        R = np.sort(rng.choice(F, k, replace=False) if t % 3 else
                    np.array(sorted(prev))[:k] if prev else rng.choice(F, k, replace=False))
        out = p.step(t, R)
        assert set(out["miss"][:, 0].tolist()) == set(R.tolist()) - prev
        prev = set(R.tolist())


def test_atu_miss_ratio_closed_form():
    # SPEC trace model: retain each active neuron w.p. p, refill uniformly.
    # E[miss ratio] = 1 - p - (1-p)^2 k / (F - p k)  (= 0.196 at p=0.8, k=1000, F=11008)
    F, k, p = 11008, 1000, 0.8
    rng = np.random.default_rng(11)
    pool = orc.LRUPool(k, F)
    A = rng.choice(F, k, replace=False)
    misses = []
    for t in range(160):
        keep = A[rng.random(k) < p]
        mask = np.ones(F, bool)
        mask[keep] = False
        A = np.concatenate([keep, rng.choice(np.flatnonzero(mask), k - keep.size, replace=False)])
        out = pool.step(t, np.sort(A))
        if t >= 10:
            misses.append(len(out["miss"]) / k)
    expect = 1 - p - (1 - p) ** 2 * k / (F - p * k)
    assert abs(expect - 0.1961) < 1e-3
    assert abs(np.mean(misses) - expect) < 0.006
