"""GPU <-> oracle parity through the C ABI (libm2c.so), on the same seeded synthetic inputs.

Bar (R12): integers (packed bytes, scores, ranks, tiers, slots, hit bits, miss and
eviction logs) bit-exact; activations within D10 = max_i |y_i - yhat_i| /
max(|yhat_i|, 2^-6 rms(yhat)) <= 2e-3, yhat the oracle's unrounded double.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from synth import get_config, layer_input_stream, layer_weights, token_stream

pytestmark = pytest.mark.gpu
TOL = 2e-3


def d10(y, yhat):
    y = np.asarray(y, np.float64)
    yhat = np.asarray(yhat, np.float64)
    floor = 2.0 ** -6 * np.sqrt(np.mean(yhat ** 2))
    return float(np.max(np.abs(y - yhat) / np.maximum(np.abs(yhat), floor)))


@pytest.fixture(scope="module")
def m2c():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2410_14740_b200.build import build
    build()
    import paper_2410_14740_b200 as pkg
    return pkg


def _np(w):
    return {k: v.cpu().numpy() for k, v in w.items()}


def _plan_np(plan):
    return np.array(plan.as_tuple(), np.int32)


def _ctx(m2c, cfg, plan, n_layers=1, shard=(0, 1)):
    return m2c.M2CContext(cfg.d_model, cfg.d_ff, n_layers, cfg.pred_rank, plan, shard=shard,
                          act=0 if cfg.act == "silu" else 1)


# ------------------------------------------------------------------ a0: pack
@pytest.mark.parametrize("shape", [(256, 688, 688), (4096, 11008, 300), (5120, 13824, 200),
                                   (8192, 3584, 130)])
def test_quant_pack_bit_exact(m2c, shape):
    d, F, n = shape
    cfg = get_config("T").with_(d_model=d, d_ff=F)
    w = layer_weights(cfg, 3, device="cuda", parts=("gate", "up", "down"))
    g, u, dn = w["w_gate"], w["w_up"], w["w_down_t"]
    # edge rows: all zero, tiny (scale underflow), huge, one-sided, constant
    g[0] = 0
    u[1] = 2.0 ** -24
    dn[2] = 60000.0
    g[3] = g[3].abs()
    u[4] = -0.5
    gn, un, dnn = g.cpu().numpy(), u.cpu().numpy(), dn.cpu().numpy()
    n0, n1 = 0, n  # ragged: n is not a multiple of any tile
    for bits in (16, 8, 4):
        rec = m2c.quant_pack(d, bits, g, u, dn, n0, n1).cpu().numpy()
        ref = orc.pack(bits, gn, un, dnn, n0, n1)
        assert rec.shape == ref.shape
        bad = np.argwhere(rec != ref)
        assert bad.size == 0, f"bits={bits}: {len(bad)} bytes differ, first {bad[:4]}"
    # offset range
    rec = m2c.quant_pack(d, 4, g, u, dn, 5, 9).cpu().numpy()
    assert np.array_equal(rec, orc.pack(4, gn, un, dnn, 5, 9))


def test_quant_pack_rejects_bad_args(m2c):
    x = torch.zeros(4, 256, dtype=torch.float16, device="cuda")
    with pytest.raises(m2c.M2CError):
        m2c.quant_pack(256, 5, x, x, x)
    with pytest.raises(m2c.M2CError):
        m2c.quant_pack(200, 8, x, x, x)


# ------------------------------------------------------------------ a1-a3: predict + select
def _check_predict(got, ref, plan):
    k = plan.k
    assert np.array_equal(got["scores"].cpu().numpy(), ref["s"])
    assert np.array_equal(got["tier_ids"].cpu().numpy()[:k], ref["tier_ids"])
    assert np.array_equal(got["rank_list"].cpu().numpy()[:k], ref["rank_list"])
    assert np.array_equal(got["tier_of"].cpu().numpy(), ref["tier_of"])


def test_predict_rank_T_32_tokens(m2c):
    cfg = get_config("T")
    plan = m2c.plan_of(cfg)
    w = layer_weights(cfg, 0, device="cuda")
    wn = _np(w)
    ctx = _ctx(m2c, cfg, plan)
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    xs = token_stream(cfg, 32, device="cuda")
    for t in range(32):
        got = ctx.predict_rank(0, xs[t].contiguous())
        pr = orc.predict(xs[t].cpu().numpy(), wn["pred_A"], wn["pred_B"])
        sel = orc.select(pr["s"], _plan_np(plan))
        _check_predict(got, dict(pr, **sel), plan)
    ctx.close()


@pytest.mark.parametrize("name,shard", [("S7", (0, 1)), ("S13", (0, 1)), ("S70", (3, 8)),
                                        ("S70", (0, 1))])
def test_predict_rank_full_shapes(m2c, name, shard):
    cfg = get_config(name)
    P = shard[1]
    plan = m2c.plan_of(cfg, P)
    w = layer_weights(cfg, 1, device="cuda", shard=shard, parts=("A", "B"))
    F_r = cfg.d_ff // P
    dummy = torch.zeros(F_r, cfg.d_model, dtype=torch.float16, device="cuda")
    ctx = _ctx(m2c, cfg, plan, shard=shard)
    ctx.load_layer(0, dummy, dummy, dummy, w["pred_A"], w["pred_B"])
    xs = layer_input_stream(cfg, 1, 3, device="cuda")
    An, Bn = w["pred_A"].cpu().numpy(), w["pred_B"].cpu().numpy()
    for t in range(3):
        got = ctx.predict_rank(0, xs[t].contiguous())
        pr = orc.predict(xs[t].cpu().numpy(), An, Bn)
        sel = orc.select(pr["s"], _plan_np(plan))
        _check_predict(got, dict(pr, **sel), plan)
    ctx.close()


@pytest.mark.parametrize("pct,a16,a8,den", [(0, 25, 25, 100), (100, 25, 25, 100),
                                            (50, 100, 0, 100), (37, 0, 0, 100),
                                            (10, 0, 100, 300), (5, 75, 75, 300)])
def test_predict_rank_plans_and_degenerate_inputs(m2c, pct, a16, a8, den):
    cfg = get_config("T")
    plan = m2c.tier_plan_make(cfg.d_ff, pct, a16, a8, den)
    w = layer_weights(cfg, 0, device="cuda")
    wn = _np(w)
    ctx = _ctx(m2c, cfg, plan)
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    xs = [torch.zeros(cfg.d_model, dtype=torch.float16, device="cuda"),  # all scores tie
          token_stream(cfg, 1, device="cuda")[0].contiguous()]
    e = torch.zeros(cfg.d_model, dtype=torch.float16, device="cuda")
    e[17] = -3.0
    xs.append(e)
    for x in xs:
        got = ctx.predict_rank(0, x, plan)
        pr = orc.predict(x.cpu().numpy(), wn["pred_A"], wn["pred_B"])
        sel = orc.select(pr["s"], _plan_np(plan))
        _check_predict(got, dict(pr, **sel), plan)
    ctx.close()


def test_predict_rank_rejects_bad_plan(m2c):
    cfg = get_config("T")
    plan = m2c.plan_of(cfg)
    w = layer_weights(cfg, 0, device="cuda")
    ctx = _ctx(m2c, cfg, plan)
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    bad = m2c.tier_plan_make(cfg.d_ff, 10)
    bad.k_int4 += 1
    with pytest.raises(m2c.M2CError):
        ctx.predict_rank(0, token_stream(cfg, 1, device="cuda")[0].contiguous(), bad)
    ctx.close()


# ------------------------------------------------------------------ a6-a7: FFN (resident)
def _ffn_case(m2c, cfg, layer, n_tokens, shard=(0, 1)):
    P = shard[1]
    plan = m2c.plan_of(cfg, P)
    w = layer_weights(cfg, layer, device="cuda", shard=shard)
    wn = _np(w)
    ctx = _ctx(m2c, cfg, plan, shard=shard)
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    xs = layer_input_stream(cfg, layer, n_tokens, device="cuda")
    worst, worst_p = 0.0, 0.0
    pn = _plan_np(plan)
    for t in range(n_tokens):
        x = xs[t].contiguous()
        sel = ctx.predict_rank(0, x)
        yp, y = ctx.sparse_ffn_forward(0, x, sel["tier_ids"])
        xn = x.cpu().numpy()
        ref = orc.select(orc.predict(xn, wn["pred_A"], wn["pred_B"])["s"], pn)
        assert np.array_equal(sel["tier_ids"].cpu().numpy(), ref["tier_ids"])
        recs = orc.records_for(wn, ref["tier_ids"], pn)
        yhat = orc.ffn(cfg.d_model, pn, ref["tier_ids"], recs[16], recs[8], recs[4], xn,
                       act=0 if cfg.act == "silu" else 1)
        worst = max(worst, d10(y.cpu().numpy(), yhat))
        worst_p = max(worst_p, d10(yp.cpu().numpy(), yhat))
    ctx.close()
    return worst, worst_p


def test_ffn_T_32_tokens(m2c):
    e16, e32 = _ffn_case(m2c, get_config("T"), 0, 32)
    assert e16 <= TOL and e32 <= 1e-4, (e16, e32)


def test_ffn_relu_flag(m2c):
    e16, e32 = _ffn_case(m2c, get_config("T").with_(act="relu"), 0, 8)
    assert e16 <= TOL and e32 <= 1e-4, (e16, e32)


@pytest.mark.parametrize("name,shard,layer", [("S7", (0, 1), 5), ("S13", (0, 1), 7),
                                              ("S70", (5, 8), 11), ("S70", (1, 2), 3),
                                              ("S70H", (0, 1), 20)])
def test_ffn_full_shapes(m2c, name, shard, layer):
    e16, e32 = _ffn_case(m2c, get_config(name), layer, 2, shard)
    assert e16 <= TOL and e32 <= 1e-4, (e16, e32)


def test_ffn_dense_equivalence_all_fp16(m2c):
    """100% active, all FP16: the method reduces to the dense FFN."""
    cfg = get_config("T")
    plan = m2c.tier_plan_make(cfg.d_ff, 100, 100, 0, 100)
    w = layer_weights(cfg, 0, device="cuda")
    ctx = _ctx(m2c, cfg, plan)
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    x = token_stream(cfg, 1, device="cuda")[0].contiguous()
    sel = ctx.predict_rank(0, x, plan)
    yp, y = ctx.sparse_ffn_forward(0, x, sel["tier_ids"], plan=plan)
    xd = x.double().cpu().numpy()
    g = w["w_gate"].double().cpu().numpy() @ xd
    u = w["w_up"].double().cpu().numpy() @ xd
    dense = w["w_down_t"].double().cpu().numpy().T @ (g / (1 + np.exp(-g)) * u)
    assert d10(y.cpu().numpy(), dense) <= TOL
    assert d10(yp.cpu().numpy(), dense) <= 1e-4
    # cuBLAS fp32 as a library cross-check of the same dense FFN
    xf = x.float()
    gf, uf = w["w_gate"].float() @ xf, w["w_up"].float() @ xf
    dense32 = (w["w_down_t"].float().t() @ (torch.nn.functional.silu(gf) * uf)).cpu().numpy()
    assert d10(dense32, dense) <= 1e-4
    ctx.close()


def test_ffn_empty_active_set(m2c):
    cfg = get_config("T")
    plan = m2c.tier_plan_make(cfg.d_ff, 0)
    w = layer_weights(cfg, 0, device="cuda")
    ctx = _ctx(m2c, cfg, plan)
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    x = token_stream(cfg, 1, device="cuda")[0].contiguous()
    sel = ctx.predict_rank(0, x, plan)
    yp, y = ctx.sparse_ffn_forward(0, x, sel["tier_ids"], plan=plan)
    assert float(yp.abs().max()) == 0.0 and float(y.float().abs().max()) == 0.0
    ctx.close()


# ------------------------------------------------------------------ a4-a5: LRU cache
def _bits(bm, k):
    bm = bm.cpu().numpy().view(np.uint32)
    return np.array([(bm[i // 32] >> (i % 32)) & 1 for i in range(k)], np.uint32)


@pytest.mark.parametrize("mode,mult", [("lru", None), ("atu", None), ("lru", (3, 2))])
def test_lru_cache_sequence_bit_exact(m2c, mode, mult):
    """Cache state over 40 tokens vs oracle O7 per tier pool; y after the fills vs O6."""
    cfg = get_config("T").with_(d_ff=688)
    plan = m2c.plan_of(cfg)
    w = layer_weights(cfg, 0, device="cuda")
    wn = _np(w)
    recs = orc.layer_records(wn)
    ctx = _ctx(m2c, cfg, plan)
    if mult is None:
        cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, mode)
    else:
        cc = m2c.api.CacheCfg()
        cc.mode = 1
        kt = plan.as_tuple()[1:]
        for t in range(3):
            cc.cap_slots[t] = kt[t] * mult[0] // mult[1]
    ctx.reserve_host_tier(ctx.layer_footprint(cc)[1])
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
    pools = [orc.LRUPool(int(cc.cap_slots[t]), cfg.d_ff) for t in range(3)]
    seg = [0, plan.k_fp16, plan.k_fp16 + plan.k_int8, plan.k]
    xs = token_stream(cfg, 40, device="cuda")
    ev = torch.cuda.Event()
    total_miss = 0
    for t in range(40):
        x = xs[t].contiguous()
        sel = ctx.predict_rank(0, x)
        ids = sel["tier_ids"]
        lk = ctx.cache_lookup_fill(0, 100 + t, ids, fill_done=ev)
        yp, y = ctx.sparse_ffn_forward(0, x, ids, lk["slots"], lk["hit_bitmap"], fill_done=ev)
        idn = ids.cpu().numpy()
        slots = lk["slots"].cpu().numpy()
        bits = _bits(lk["hit_bitmap"], plan.k)
        ml, el = lk["miss_log"].cpu().numpy(), lk["evict_log"].cpu().numpy()
        cnt = lk["counts"].cpu().numpy()
        for tau in range(3):
            ref = pools[tau].step(100 + t, idn[seg[tau]:seg[tau + 1]])
            assert np.array_equal(slots[seg[tau]:seg[tau + 1]], ref["slots"])
            rb = np.array([(ref["hit_bits"][i // 32] >> (i % 32)) & 1
                           for i in range(seg[tau + 1] - seg[tau])], np.uint32)
            assert np.array_equal(bits[seg[tau]:seg[tau + 1]], rb)
            nm, ne = len(ref["miss"]), len(ref["evict"])
            assert cnt[tau] == nm and cnt[3 + tau] == ne
            assert np.array_equal(ml[seg[tau]:seg[tau] + nm], ref["miss"])
            assert np.array_equal(el[seg[tau]:seg[tau] + ne], ref["evict"])
            total_miss += nm
        yhat = orc.ffn(cfg.d_model, _plan_np(plan), idn, recs[16], recs[8], recs[4],
                       x.cpu().numpy())
        assert d10(y.cpu().numpy(), yhat) <= TOL
        assert d10(yp.cpu().numpy(), yhat) <= 1e-4
    assert total_miss > 0
    st = ctx.stats()
    assert sum(st["misses"]) == total_miss
    with pytest.raises(m2c.M2CError):  # step must strictly increase
        ctx.cache_lookup_fill(0, 100, ids)
    ctx.close()


# ------------------------------------------------------------------ whole token
# (engine-vs-oracle replay tests: tests/test_gpu_engines.py)
def test_decode_step_lru_matches_api_chain(m2c):
    cfg = get_config("T")
    L = 2
    plan = m2c.plan_of(cfg)
    ws = [layer_weights(cfg, l, device="cuda") for l in range(L)]
    ctxs = []
    for _ in range(2):
        ctx = _ctx(m2c, cfg, plan, n_layers=L)
        cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, "lru")
        ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
        for l, w in enumerate(ws):
            ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
        ctxs.append(ctx)
    a, b = ctxs
    xs = token_stream(cfg, 12, device="cuda")
    ev = torch.cuda.Event()
    for t in range(12):
        x = xs[t].contiguous().clone()
        a.decode_step(x, t + 1)
        xc = xs[t].contiguous().clone()
        for l in range(L):
            sel = b.predict_rank(l, xc, rank_list=False, tier_of=False, scores=False)
            lk = b.cache_lookup_fill(l, t + 1, sel["tier_ids"], logs=False, fill_done=ev)
            _, y = b.sparse_ffn_forward(l, xc, sel["tier_ids"], lk["slots"], lk["hit_bitmap"],
                                        fill_done=ev, want_partial=False)
            xc = xc + y
        torch.cuda.synchronize()
        assert torch.equal(x, xc), t
    sa, sb = a.stats(), b.stats()
    assert sa["hits"] == sb["hits"] and sa["misses"] == sb["misses"]
    assert sum(sa["misses"]) > 0 and sum(sa["hits"]) > 0
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("P,pct,a16,a8,den", [(2, 10, 25, 25, 100), (4, 10, 25, 25, 100),
                                              (4, 30, 0, 100, 300), (8, 5, 100, 0, 100)])
def test_global_topk_under_sharding_equals_unsharded(m2c, P, pct, a16, a8, den):
    """NEXT-3: every rank's local top-min(F_r, k) candidates, all-gathered, give each rank
    its part of the GLOBAL selection; the union over ranks equals the unsharded oracle's tier
    lists bit-exactly (the shard-local default, R13, does not)."""
    cfg = get_config("T")
    F = cfg.d_ff
    F_r = F // P
    gplan = m2c.tier_plan_make(F, pct, a16, a8, den)
    n = min(F_r, gplan.k)
    full = layer_weights(cfg, 0, device="cuda", parts=("A", "B"))  # (the CUDA generator's draws)
    An, Bn = full["pred_A"].cpu().numpy(), full["pred_B"].cpu().numpy()
    ctxs = []
    for r in range(P):
        w = layer_weights(cfg, 0, device="cuda", shard=(r, P), parts=("A", "B"))
        dummy = torch.zeros(F_r, cfg.d_model, dtype=torch.float16, device="cuda")
        ctx = _ctx(m2c, cfg, m2c.tier_plan_make(F_r, pct, a16, a8, den), shard=(r, P))
        ctx.load_layer(0, dummy, dummy, dummy, w["pred_A"], w["pred_B"])
        ctxs.append(ctx)
    xs = layer_input_stream(cfg, 0, 4, device="cuda")
    gp = np.array(gplan.as_tuple(), np.int32)
    for t in range(4):
        x = xs[t].contiguous()
        keys = torch.cat([c.predict_candidates(0, x, n) for c in ctxs])
        got = [[], [], []]
        for r, c in enumerate(ctxs):
            ids, cnt = c.select_global(keys, n, gplan)
            ids, cnt = ids.cpu().numpy(), cnt.cpu().numpy()
            off = [0, gplan.k_fp16, gplan.k_fp16 + gplan.k_int8]
            for tier in range(3):
                seg = ids[off[tier]:off[tier] + cnt[tier]]
                assert np.all(np.diff(seg) > 0)  # ascending local ids
                got[tier].extend((r * F_r + seg).tolist())
        ref = orc.select(orc.predict(xs[t].cpu().numpy(), An, Bn)["s"], gp)["tier_ids"]
        off = [0, gplan.k_fp16, gplan.k_fp16 + gplan.k_int8, gplan.k]
        for tier in range(3):
            assert sorted(got[tier]) == ref[off[tier]:off[tier + 1]].tolist(), (t, tier)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("name,layers", [("T", 3), ("S7", 3), ("S70H", 2)])
def test_decode_layer_split_equals_fused(m2c, name, layers):
    """The layer-split engine (k_decode one layer per launch, the partial y handed to the next
    launch through the all-reduce buffer -- the d_ff-sharded decode) is bit-identical to the
    whole-token k_decode (same shares, same reduction order, same selection)."""
    cfg = get_config(name)
    plan = m2c.plan_of(cfg)
    ctxs = []
    for mode in (1, 2):
        ctx = _ctx(m2c, cfg, plan, n_layers=layers)
        for l in range(layers):
            w = layer_weights(cfg, l, device="cuda")
            ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
        ctx.set_fused(mode)
        ctxs.append(ctx)
    xs = token_stream(cfg, 5, device="cuda")
    for t in range(5):
        outs = []
        for ctx in ctxs:
            x = xs[t].contiguous().clone()
            ctx.decode_step(x, t + 1)
            outs.append(x)
        torch.cuda.synchronize()
        for l in range(layers):
            assert torch.equal(ctxs[0].decode_lists(l), ctxs[1].decode_lists(l)), (t, l)
        assert torch.equal(outs[0], outs[1]), t
    assert ctxs[0].stats()["kernels_per_token"] == 1
    assert ctxs[1].stats()["kernels_per_token"] == layers + 1  # L launches + the final residual
    for c in ctxs:
        c.close()


def test_lru_full_s13_layer_against_oracle(m2c):
    """BASELINE configs[2] at full size (one 5120 x 13824 layer, pools capped at 25% of the
    layer's FP16 bytes, C = (1696, 1696, 3402)): 32 tokens of predict -> LRU lookup + fill ->
    FFN through the C ABI; every token's slots, hit bits, miss and eviction logs equal oracle
    O7 per tier pool bit-exactly (through the cold start into the eviction regime), and at
    sampled tokens y equals O6 within the tolerance."""
    cfg = get_config("S13")
    plan = m2c.plan_of(cfg)
    w = layer_weights(cfg, 0, device="cuda")
    wn = _np(w)
    ctx = _ctx(m2c, cfg, plan)
    cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, "lru")
    # R8: M = 0.25 * 6dF / sum_t k_t nb_t with 16-B padded records = 4.9166 -> (1696, 1696, 3402)
    # (SURVEY's 3403 rounds M to 4.918 first)
    assert [int(cc.cap_slots[t]) for t in range(3)] == [1696, 1696, 3402]
    ctx.reserve_host_tier(ctx.layer_footprint(cc)[1])
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
    pools = [orc.LRUPool(int(cc.cap_slots[t]), cfg.d_ff) for t in range(3)]
    seg = [0, plan.k_fp16, plan.k_fp16 + plan.k_int8, plan.k]
    xs = layer_input_stream(cfg, 0, 32, device="cuda")
    ev = torch.cuda.Event()
    recs = None
    n_evict = 0
    for t in range(32):
        x = xs[t].contiguous()
        sel = ctx.predict_rank(0, x, rank_list=False, tier_of=False, scores=False)
        ids = sel["tier_ids"]
        lk = ctx.cache_lookup_fill(0, 10 + t, ids, fill_done=ev)
        _, y = ctx.sparse_ffn_forward(0, x, ids, lk["slots"], lk["hit_bitmap"], fill_done=ev,
                                      want_partial=False)
        idn = ids.cpu().numpy()
        slots = lk["slots"].cpu().numpy()
        bits = _bits(lk["hit_bitmap"], plan.k)
        ml, el = lk["miss_log"].cpu().numpy(), lk["evict_log"].cpu().numpy()
        cnt = lk["counts"].cpu().numpy()
        for tau in range(3):
            ref = pools[tau].step(10 + t, idn[seg[tau]:seg[tau + 1]])
            assert np.array_equal(slots[seg[tau]:seg[tau + 1]], ref["slots"]), (t, tau)
            rb = np.array([(ref["hit_bits"][i // 32] >> (i % 32)) & 1
                           for i in range(seg[tau + 1] - seg[tau])], np.uint32)
            assert np.array_equal(bits[seg[tau]:seg[tau + 1]], rb), (t, tau)
            nm, ne = len(ref["miss"]), len(ref["evict"])
            assert cnt[tau] == nm and cnt[3 + tau] == ne, (t, tau)
            assert np.array_equal(ml[seg[tau]:seg[tau] + nm], ref["miss"])
            assert np.array_equal(el[seg[tau]:seg[tau] + ne], ref["evict"])
            n_evict += ne
        if t in (0, 17, 31):
            if recs is None:
                recs = orc.layer_records(wn)
            ref = orc.select(orc.predict(x.cpu().numpy(), wn["pred_A"], wn["pred_B"])["s"],
                             _plan_np(plan))
            assert np.array_equal(idn, ref["tier_ids"]), t
            yhat = orc.ffn(cfg.d_model, _plan_np(plan), idn, recs[16], recs[8], recs[4],
                           x.cpu().numpy())
            assert d10(y.cpu().numpy(), yhat) <= TOL, t
    assert n_evict > 0  # the pools filled up and evicted
    ctx.close()


def test_decode_step_lru_s13_shape_matches_api_chain(m2c):
    """The LRU decode engine bench.py times at configs[2] (graph-captured select-only k_decode
    at d = 5120 -> k_lru -> copy-stream k_fill || hit FFN -> miss FFN -> reduce) equals the
    per-call C-ABI chain bit-exactly over 10 tokens of a 3-layer full-width S13 stack."""
    cfg = get_config("S13")
    L = 3
    plan = m2c.plan_of(cfg)
    ctxs = []
    for _ in range(2):
        ctx = _ctx(m2c, cfg, plan, n_layers=L)
        cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, "lru")
        ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
        for l in range(L):
            w = layer_weights(cfg, l, device="cuda")
            ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
            del w
        ctxs.append(ctx)
    a, b = ctxs
    xs = token_stream(cfg, 10, device="cuda")
    ev = torch.cuda.Event()
    for t in range(10):
        x = xs[t].contiguous().clone()
        a.decode_step(x, t + 1)
        xc = xs[t].contiguous().clone()
        for l in range(L):
            sel = b.predict_rank(l, xc, rank_list=False, tier_of=False, scores=False)
            lk = b.cache_lookup_fill(l, t + 1, sel["tier_ids"], logs=False, fill_done=ev)
            _, y = b.sparse_ffn_forward(l, xc, sel["tier_ids"], lk["slots"], lk["hit_bitmap"],
                                        fill_done=ev, want_partial=False)
            xc = xc + y
        torch.cuda.synchronize()
        assert torch.equal(x, xc), t
    sa, sb = a.stats(), b.stats()
    assert sa["hits"] == sb["hits"] and sa["misses"] == sb["misses"]
    assert sa["kernels_per_token"] > 1
    for c in ctxs:
        c.close()


def test_profile_fill_reports_lru_fills(m2c):
    """m2c_profile_fill (the S13 roofline's denominator): positive fill durations for LRU
    layers of a profiled decode step; a resident whole-token step has none (M2C_ERR_STATE)."""
    cfg = get_config("T")
    L = 2
    plan = m2c.plan_of(cfg)
    ctx = _ctx(m2c, cfg, plan, n_layers=L)
    cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, "lru")
    ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
    for l in range(L):
        w = layer_weights(cfg, l, device="cuda")
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
    ctx.profile(True)
    x = token_stream(cfg, 1, device="cuda")[0].contiguous()
    ctx.decode_step(x, 1)  # cold pools: every selected record is a miss
    ms = ctx.profile_fill()
    assert len(ms) == L and all(v > 0 for v in ms)
    ctx.close()
    res = _ctx(m2c, cfg, plan, n_layers=1)
    w = layer_weights(cfg, 0, device="cuda")
    res.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    res.profile(True)
    res.decode_step(x.clone(), 1)
    with pytest.raises(m2c.M2CError):
        res.profile_fill()
    res.close()
