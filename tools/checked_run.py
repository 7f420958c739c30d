"""Workload for the bounds-checked build (tests/test_gpu_checked.py): every decode engine at
the shapes the bench times, with M2C_LIB pointing at a libm2c.so built with -DM2C_CHECKS=1
(index / capacity invariants trap instead of corrupting memory).  A few tokens each:
  T      whole-token k_decode, layer-split k_decode, per-phase chain, per-call API
  S7     whole-token k_decode (whole FFN shares), and x = 0 (the exact tie fallback)
  S70H   whole-token k_decode (streaming FFN shares, 1024 threads)
  S13    early-fill LRU engine (select-only k_decode, k_missq, k_fill, k_requant, k_lru, k_ffn)
  T      ATU engine, LRU engine with the NEXT-2 lookahead
usage: M2C_LIB=build/checked/libm2c.so python tools/checked_run.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2410_14740_b200 as m2c  # noqa: E402
from synth import get_config, layer_weights, token_stream  # noqa: E402


def run(name, L, mode="resident", fused=1, tokens=3, zero_x=False, lookahead=False, api=False):
    cfg = get_config(name)
    plan = m2c.plan_of(cfg)
    ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan, act=0 if cfg.act == "silu" else 1)
    cc = None
    if mode != "resident":
        cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, mode)
        ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
    for l in range(L):
        w = layer_weights(cfg, l, device="cuda")
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
        del w
    ctx.set_fused(fused)
    if lookahead:
        ctx.set_lookahead(True)
    xs = token_stream(cfg, tokens + 1, device="cuda")
    for t in range(tokens):
        x = torch.zeros_like(xs[t]) if zero_x else xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
    torch.cuda.synchronize()
    if api:
        sel = ctx.predict_rank(0, xs[tokens].contiguous())
        ctx.sparse_ffn_forward(0, xs[tokens].contiguous(), sel["tier_ids"])
        torch.cuda.synchronize()
    ctx.stats()  # raises if a kernel flagged an invariant violation
    ctx.close()
    print(f"  {name} L={L} {mode} fused={fused} zero_x={zero_x} lookahead={lookahead}: ok", flush=True)


run("T", 3, fused=1, tokens=4, api=True)
run("T", 3, fused=2, tokens=4)
run("T", 3, fused=0, tokens=4)
run("S7", 2)
run("S7", 2, zero_x=True)
run("S70H", 2, tokens=2)
run("S13", 2, mode="lru", tokens=6)
run("T", 3, mode="atu", tokens=6)
run("T", 3, mode="lru", tokens=6, lookahead=True)
print("checked run done")
