"""The decode ENGINES bench.py times, checked against the oracle by replay.

Every engine of m2c_decode_step records, through the parity trace (m2c_set_trace), each
layer's input x_l and output y_l (before the fp16 rounding; after the all-reduce when
sharded).  The oracle recomputes each (token, layer) from the recorded x_l:
  * the tier lists (m2c_decode_lists) equal O1..O5 bit-exactly;
  * LRU/ATU engines: every (layer, tier) pool's occupant / last-use state (m2c_cache_state)
    equals O7 stepped with those lists bit-exactly, after every token;
  * y_l equals O6 within D10 <= 2e-3 (north_star), d_ff-sharded: Sigma_r yhat^(r).
No oracle input comes from anything but the trace and the seeded generators; no expected value
comes from the CUDA path.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as orc
from synth import get_config, layer_weights, token_stream

pytestmark = pytest.mark.gpu
TOL = 2e-3


def d10(y, yhat):
    y = np.asarray(y, np.float64)
    yhat = np.asarray(yhat, np.float64)
    if not np.any(yhat):
        return float(np.max(np.abs(y)))
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


def oracle_layer(wn, plan, x, act=0):
    """O1..O6 for one (token, layer): tier lists and the unrounded yhat.  The records of the
    selected neurons are packed by the oracle (O0) one by one into compact per-tier arrays."""
    pn = np.array(plan.as_tuple() if hasattr(plan, "as_tuple") else plan, np.int32)
    sel = orc.select(orc.predict(x, wn["pred_A"], wn["pred_B"])["s"], pn)
    ids = sel["tier_ids"]
    seg = [0, int(pn[1]), int(pn[1]) + int(pn[2]), int(pn[0])]
    d = x.size
    recs, cids = [], np.zeros_like(ids)
    for t, b in enumerate((16, 8, 4)):
        part = ids[seg[t]:seg[t + 1]]
        r = np.zeros((max(len(part), 1), orc.record_bytes(b, d)), np.uint8)
        for i, n in enumerate(part):
            r[i] = orc.pack(b, wn["w_gate"], wn["w_up"], wn["w_down_t"], int(n), int(n) + 1)[0]
        recs.append(r)
        cids[seg[t]:seg[t + 1]] = np.arange(len(part), dtype=np.int32)
    yhat = orc.ffn(d, pn, cids, recs[0], recs[1], recs[2], x, act)
    return ids, yhat


def _stack(m2c, cfg, plan, L, shard=(0, 1), cc_mode=None, B_hook=None, full=None):
    # full: the layers whose FFN weights are kept on the host for the oracle (None = all; the
    # others keep only the predictor, enough for the tier-list check)
    ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan, shard=shard,
                         act=0 if cfg.act == "silu" else 1)
    cc = None
    if cc_mode:
        cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, cc_mode)
        ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
    ws = []
    for l in range(L):
        w = layer_weights(cfg, l, device="cuda", shard=shard)
        if B_hook:
            w["pred_B"] = B_hook(w["pred_B"])
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
        if full is not None and l not in full:
            w = {k: w[k] for k in ("pred_A", "pred_B")}
        ws.append(_np(w))
        del w
    return ctx, ws, cc


def _check_token(ctx, ws, plan, layers, act=0, y_layers=None, check_lists=True):
    """Replay one decoded token's trace through the oracle; returns the worst D10."""
    tx, ty = ctx.trace_x.cpu().numpy(), ctx.trace_y.cpu().numpy()
    worst = 0.0
    lists = []
    for l in range(layers):
        if not check_lists:  # (the global-top-k chain keeps no per-layer lists: y only)
            ids, yhat = oracle_layer(ws[l], plan, tx[l], act)
            assert d10(ty[l], yhat) <= TOL, l
            continue
        got = ctx.decode_lists(l).cpu().numpy()
        if y_layers is None or l in y_layers:
            ids, yhat = oracle_layer(ws[l], plan, tx[l], act)
            assert np.array_equal(got, ids), f"layer {l}: tier lists differ from the oracle"
            e = d10(ty[l], yhat)
            assert e <= TOL, (l, e)
            worst = max(worst, e)
        else:
            pn = np.array(plan.as_tuple(), np.int32)
            ids = orc.select(orc.predict(tx[l], ws[l]["pred_A"], ws[l]["pred_B"])["s"], pn)["tier_ids"]
            assert np.array_equal(got, ids), f"layer {l}: tier lists differ from the oracle"
        lists.append(got)
    return worst, lists


# ------------------------------------------------------------------ resident engines
@pytest.mark.parametrize("name,layers,tokens,engine", [
    ("T", 3, 8, 1), ("T", 3, 4, 2), ("T", 3, 4, 0),
    ("S7", 3, 3, 1), ("S7", 2, 2, 2), ("S70H", 2, 2, 1), ("S13", 2, 2, 1)])
def test_resident_engine_replay_against_oracle(m2c, name, layers, tokens, engine):
    """Whole-token k_decode (engine 1), layer-split k_decode (2, the d_ff-sharded engine's
    kernel) and the per-phase chain (0): per-layer lists bit-exact, y within D10."""
    cfg = get_config(name)
    plan = m2c.plan_of(cfg)
    ctx, ws, _ = _stack(m2c, cfg, plan, layers)
    ctx.set_fused(engine)
    ctx.set_trace(True)
    xs = token_stream(cfg, tokens, device="cuda")
    for t in range(tokens):
        x = xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
        torch.cuda.synchronize()
        assert torch.equal(ctx.trace_x[layers], x)  # the trace's x_L is the output
        _check_token(ctx, ws, plan, layers, act=0 if cfg.act == "silu" else 1)
    kpt = ctx.stats()["kernels_per_token"]
    assert kpt == {1: 1, 2: layers + 1}.get(engine, kpt)
    ctx.close()


def test_full_s7_stack_decode_replay_against_oracle(m2c):
    """BASELINE configs[1] at full size in the launch configuration bench.py times (32 layers,
    k_decode, CUDA graph): every layer's lists equal the oracle's on the traced input; y at
    sampled layers within the tolerance."""
    cfg = get_config("S7")
    plan = m2c.plan_of(cfg)
    ctx, ws, _ = _stack(m2c, cfg, plan, cfg.n_layers)
    ctx.set_trace(True)
    xs = token_stream(cfg, 3, device="cuda")
    for t in range(3):
        x = xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
        torch.cuda.synchronize()
        _check_token(ctx, ws, plan, cfg.n_layers, y_layers={0, 13, cfg.n_layers - 1} if t == 0 else {31})
    assert ctx.stats()["kernels_per_token"] == 1
    ctx.close()


def test_full_s70h_stack_decode_replay_against_oracle(m2c):
    """The bench default (the 1-GPU point of configs[3]) at full size in the launch
    configuration bench.py times: 40 layers of 8192 x 28672, one k_decode launch per token
    (streaming FFN shares, 1024 threads); every layer's lists equal the oracle's on the traced
    input, y at sampled layers within the tolerance."""
    cfg = get_config("S70H")
    plan = m2c.plan_of(cfg)
    ys = {0, 20, cfg.n_layers - 1}
    ctx, ws, _ = _stack(m2c, cfg, plan, cfg.n_layers, full=ys)
    ctx.set_trace(True)
    xs = token_stream(cfg, 2, device="cuda")
    for t in range(2):
        x = xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
        torch.cuda.synchronize()
        _check_token(ctx, ws, plan, cfg.n_layers, y_layers=ys if t == 0 else {cfg.n_layers - 1})
    assert ctx.stats()["kernels_per_token"] == 1
    ctx.close()


@pytest.mark.parametrize("kind", ["zero_x", "tied_B"])
def test_decode_degenerate_ties_against_oracle(m2c, kind):
    """Massive score ties: x = 0 (every score 0: one bucket holds every neuron, the exact
    block-wide fallback) and a predictor whose B rows repeat in runs of 7 (partial ties at
    every cut, ranked by id)."""
    cfg = get_config("S7")
    plan = m2c.plan_of(cfg)
    hook = (lambda B: B[torch.arange(B.shape[0], device=B.device) // 7 * 7].contiguous()) \
        if kind == "tied_B" else None
    ctx, ws, _ = _stack(m2c, cfg, plan, 2, B_hook=hook)
    ctx.set_trace(True)
    xs = token_stream(cfg, 3, device="cuda")
    for t in range(3):
        x = torch.zeros_like(xs[t]) if kind == "zero_x" else xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
        torch.cuda.synchronize()
        _check_token(ctx, ws, plan, 2)
    ctx.stats()  # raises if the device flagged an error (barrier timeout, count mismatch)
    ctx.close()


# configs[4] tier mixes: FP16 share 0 / 100 % and 50 % active, on the S70 shard 0 of 8 and on
# the 40-layer 1-GPU shape (empty tiers, the all-FP16 streaming share)
@pytest.mark.parametrize("shape,pct,share", [
    ("S70/8", 10, 0), ("S70/8", 10, 100), ("S70/8", 50, 25),
    ("S70H", 10, 0), ("S70H", 10, 100), ("S70H", 50, 25)])
def test_sweep_tier_mixes_against_oracle(m2c, shape, pct, share):
    name, P = (shape.split("/")[0], int(shape.split("/")[1])) if "/" in shape else (shape, 1)
    cfg = get_config(name).with_(active_pct=pct, a16=3 * share, a8=100 - share, den=300)
    plan = m2c.tier_plan_make(cfg.d_ff // P, pct, 3 * share, 100 - share, 300)
    ctx, ws, _ = _stack(m2c, cfg, plan, 2, shard=(0, P))
    ctx.set_trace(True)
    xs = token_stream(cfg, 2, device="cuda")
    for t in range(2):
        x = xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
        torch.cuda.synchronize()
        _check_token(ctx, ws, plan, 2)
    assert ctx.stats()["kernels_per_token"] == 1
    ctx.close()


# ------------------------------------------------------------------ LRU / ATU engines
def _lru_engine_case(m2c, cfg, L, tokens, mode, attach=None, lookahead=False, y_every=4):
    plan = m2c.plan_of(cfg)
    ctx, ws, cc = _stack(m2c, cfg, plan, L, cc_mode=mode)
    if lookahead:
        ctx.set_lookahead(True)
    if attach:
        attach(ctx)
    ctx.set_trace(True)
    pools = [[orc.LRUPool(int(cc.cap_slots[t]), cfg.d_ff) for t in range(3)] for _ in range(L)]
    seg = [0, plan.k_fp16, plan.k_fp16 + plan.k_int8, plan.k]
    xs = token_stream(cfg, tokens, device="cuda")
    worst = 0.0
    for t in range(tokens):
        x = xs[t].contiguous().clone()
        step = 5 + 3 * t
        ctx.decode_step(x, step)
        torch.cuda.synchronize()
        w, lists = _check_token(ctx, ws, plan, L, y_layers=set(range(L)) if t % y_every == 0 else set())
        worst = max(worst, w)
        for l in range(L):
            for tau in range(3):
                pools[l][tau].step(step, lists[l][seg[tau]:seg[tau + 1]])
                occ, last = ctx.cache_state(l, tau)
                assert np.array_equal(occ.cpu().numpy(), pools[l][tau].occupant), (t, l, tau)
                assert np.array_equal(last.cpu().numpy(), pools[l][tau].last), (t, l, tau)
    st = ctx.stats()
    return ctx, st, worst


@pytest.mark.parametrize("mode", ["lru", "atu"])
def test_lru_engine_T_against_oracle(m2c, mode):
    ctx, st, _ = _lru_engine_case(m2c, get_config("T"), 3, 24, mode, y_every=1)
    assert sum(st["misses"]) > 0 and sum(st["hits"]) > 0
    ctx.close()


def test_lru_engine_s13_full_width_against_oracle(m2c):
    """The engine bench.py times at configs[2] (select-only k_decode -> per-tier sort ->
    k_missq -> copy-stream early fill into staging || k_lru -> hit FFN -> miss FFN from
    staging -> scatter), full S13 width, 3 layers x 32 tokens through the cold start into the
    eviction regime: lists and every pool's state bit-exact against O7 after every token, y
    against O6 every 4th token."""
    ctx, st, worst = _lru_engine_case(m2c, get_config("S13"), 3, 32, "lru")
    assert sum(st["misses"]) > 0
    assert st["kernels_per_token"] > 3
    ctx.close()


@pytest.mark.parametrize("n_fixed,n_dyn,ahead", [(1, 2, 1), (0, 1, 0), (4, 0, 0)])
def test_store_backed_engine_against_oracle(m2c, tmp_path, n_fixed, n_dyn, ahead):
    """NEXT-1: miss fills served from the file-backed two-level DRAM cache (fixed area + FIFO
    frames filled by the I/O thread): lists, pool states and y against the oracle."""
    path = str(tmp_path / "m2c_store.bin")

    def attach(ctx):
        ctx.store_write(path)
        ctx.store_attach(path, n_fixed, n_dyn, ahead)

    ctx, st, _ = _lru_engine_case(m2c, get_config("T"), 4, 10, "lru", attach=attach, y_every=2)
    ss = ctx.store_stats()
    assert ss["bytes_read"] > 0
    ctx.close()


@pytest.mark.parametrize("mode", ["lru", "atu"])
def test_lookahead_engine_against_oracle(m2c, mode):
    """NEXT-2: staging layer l+1's predicted misses during layer l: lists, pool states and y
    against the oracle, and a share of the misses served from staging."""
    ctx, st, _ = _lru_engine_case(m2c, get_config("T"), 4, 12, mode, lookahead=True, y_every=2)
    staged = ctx.lookahead_stats()
    assert 0 < staged <= sum(st["misses"])
    ctx.close()


# ------------------------------------------------------------------ d_ff-sharded engines
@pytest.mark.parametrize("name,layers", [("T", 3), ("S7", 3)])
def test_p2p_fused_allreduce_two_ranks_against_oracle(m2c, name, layers):
    """§8(e): two d_ff shards (ranks 0/1 of P = 2) share one GPU, 74 CTAs each, and run the
    whole-token k_decode CONCURRENTLY with the all-reduce fused into its reduction phase over
    peer memory.  Both ranks trace the same x_l (bit-identical); each rank's lists equal the
    oracle's shard-local selection (R13) on x_l; the traced y_l (after the exchange) equals
    Sigma_r yhat^(r) of the oracle within D10."""
    from paper_2410_14740_b200._lib import lib
    from paper_2410_14740_b200.api import check
    cfg = get_config(name)
    P = 2
    plan = m2c.plan_of(cfg, P)
    ctxs, wss = [], []
    for r in range(P):
        ctx, ws, _ = _stack(m2c, cfg, plan, layers, shard=(r, P))
        ctx.set_grid(74)
        ctx.set_trace(True)
        ctxs.append(ctx)
        wss.append(ws)
    ptrs = [c.p2p_buffer()[0] for c in ctxs]
    for c in ctxs:
        c.p2p_connect(dev_ptrs=ptrs)
    xs = token_stream(cfg, 4, device="cuda")
    for t in range(4):
        xr = [xs[t].contiguous().clone() for _ in range(P)]
        torch.cuda.synchronize()
        for c, x in zip(ctxs, xr):  # both ranks in flight at once (no stream dependency)
            check(lib().m2c_decode_step(c._h, x.data_ptr(), t + 1))
        torch.cuda.synchronize()
        for c in ctxs:
            assert c.stats()["kernels_per_token"] == 1  # raises on a p2p / barrier timeout
        assert torch.equal(xr[0], xr[1])
        assert torch.equal(ctxs[0].trace_x, ctxs[1].trace_x)
        tx = ctxs[0].trace_x.cpu().numpy()
        ty = ctxs[0].trace_y.cpu().numpy()
        for l in range(layers):
            ysum = np.zeros(cfg.d_model)
            for r in range(P):
                ids, yhat = oracle_layer(wss[r][l], plan, tx[l])
                assert np.array_equal(ctxs[r].decode_lists(l).cpu().numpy(), ids), (t, l, r)
                ysum += yhat
            assert d10(ty[l], ysum) <= TOL, (t, l)
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("engine", ["split", "chain", "global"])
def test_nccl_wiring_single_rank(m2c, engine):
    """The collectives of the sharded engines (ncclAllReduce between layer launches / in the
    chain, ncclAllGather of the global-top-k keys), captured in the decode graph, run for real
    with a one-rank communicator (identity collectives): every token bit-identical to the same
    engine without a communicator, and the traced layers equal the oracle."""
    cfg = get_config("T")
    L = 3
    plan = m2c.plan_of(cfg)
    ctxs = []
    for with_comm in (False, True):
        ctx, ws, _ = _stack(m2c, cfg, plan, L)
        ctx.set_fused(2 if engine == "split" else 0)
        if with_comm:
            ctx.comm_init(1, 0, m2c.nccl_unique_id())
            if engine == "global":
                ctx.set_global_topk(plan)  # one rank: the global plan is the plan
            ctx.set_trace(True)
        ctxs.append(ctx)
    xs = token_stream(cfg, 4, device="cuda")
    for t in range(4):
        outs = []
        for ctx in ctxs:
            x = xs[t].contiguous().clone()
            ctx.decode_step(x, t + 1)
            outs.append(x)
        torch.cuda.synchronize()
        assert torch.equal(outs[0], outs[1]), t
        _check_token(ctxs[1], ws, plan, L, check_lists=engine != "global")
    kpt = ctxs[1].stats()["kernels_per_token"]
    assert kpt == (L + 1 if engine == "split" else kpt) and kpt > 1
    for c in ctxs:
        c.close()


def _ipc_worker(rank, world, port, out):
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist

    import paper_2410_14740_b200 as m2c
    from paper_2410_14740_b200 import dist as m2c_dist
    from synth import get_config, layer_weights, token_stream
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = get_config("T")
        L = 3
        ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, m2c.plan_of(cfg, world),
                             shard=(rank, world))
        for l in range(L):
            w = layer_weights(cfg, l, device="cuda", shard=(rank, world))
            ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
        ctx.set_grid(32)
        ctx.set_trace(True)
        m2c_dist.p2p_init(ctx)  # CUDA IPC handles over the process group
        xs = token_stream(cfg, 2, device="cuda")
        res = []
        for t in range(2):
            x = xs[t].contiguous().clone()
            dist.barrier()
            ctx.decode_step(x, t + 1)
            torch.cuda.synchronize()
            assert ctx.stats()["kernels_per_token"] == 1  # the whole-token kernel ran
            res.append((ctx.trace_x.cpu().numpy().tobytes(), ctx.trace_y.cpu().numpy().tobytes(),
                        [ctx.decode_lists(l).cpu().numpy().tobytes() for l in range(L)]))
        out[rank] = res
        dist.barrier()
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_p2p_ipc_two_processes_against_oracle(m2c):
    """§8(e) across processes: two ranks in two processes (one GPU here; on a node, one GPU
    each) exchange their buffers' CUDA IPC handles over the process group (dist.p2p_init) and
    decode with the in-kernel exchange; both trace the same x_l, and every layer replays
    through the oracle (shard-local lists, Sigma_r yhat^(r))."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_ipc_worker, args=(2, port, out), nprocs=2, join=True)
        res = dict(out)
    cfg = get_config("T")
    L, P = 3, 2
    plan = m2c.plan_of(cfg, P)
    wss = [[_np(layer_weights(cfg, l, device="cuda", shard=(r, P))) for l in range(L)] for r in range(P)]
    for t in range(2):
        assert res[0][t][0] == res[1][t][0] and res[0][t][1] == res[1][t][1], t
        tx = np.frombuffer(res[0][t][0], np.float16).reshape(L + 1, cfg.d_model)
        ty = np.frombuffer(res[0][t][1], np.float32).reshape(L, cfg.d_model)
        for l in range(L):
            ysum = np.zeros(cfg.d_model)
            for r in range(P):
                ids, yhat = oracle_layer(wss[r][l], plan, tx[l])
                assert np.frombuffer(res[r][t][2][l], np.int32).tolist() == ids.tolist(), (t, l, r)
                ysum += yhat
            assert d10(ty[l], ysum) <= TOL, (t, l)


def test_requant_fills_equal_host_fills(m2c):
    """a5 fill source (include/m2c.h m2c_set_requant): an INT8 / INT4 miss whose neuron is resident
    in the FP16 pool is filled by quantising that record on the GPU (the offline pack's function,
    bit-identical to O0) instead of copying the host tier's record.  At full S13 width, 3 layers
    x 24 tokens: the same token stream with the requantised fills on and off gives bit-identical
    layer inputs / outputs and cache state, the same miss counts, and requantised fills > 0."""
    cfg = get_config("S13")
    plan = m2c.plan_of(cfg)
    L, T = 3, 24
    runs = []
    for rq in (True, False):
        ctx, ws, cc = _stack(m2c, cfg, plan, L, cc_mode="lru")
        ctx.set_requant(rq)
        ctx.set_trace(True)
        xs = token_stream(cfg, T, device="cuda")
        tr = []
        for t in range(T):
            x = xs[t].contiguous().clone()
            ctx.decode_step(x, 5 + 3 * t)
            torch.cuda.synchronize()
            tr.append((ctx.trace_x.clone(), ctx.trace_y.clone()))
        state = [[tuple(v.cpu() for v in ctx.cache_state(l, tau)) for tau in range(3)] for l in range(L)]
        runs.append((tr, state, ctx.stats()["misses"], ctx.requant_stats()))
        ctx.close()
    (tr1, s1, m1, q1), (tr0, s0, m0, q0) = runs
    assert q1[0] == 0 and q1[1] + q1[2] > 0, q1
    assert q0 == [0, 0, 0]
    assert m1 == m0
    for (x1, y1), (x0, y0) in zip(tr1, tr0):
        assert torch.equal(x1, x0) and torch.equal(y1, y0)
    for l in range(L):
        for tau in range(3):
            assert all(torch.equal(a, b) for a, b in zip(s1[l][tau], s0[l][tau]))
