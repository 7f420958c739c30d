"""A small workload for compute-sanitizer (tests/test_gpu_sanitizer.py): the T-config
whole-token k_decode, the layer-split engine, the LRU/ATU engine and the per-call API, a few
tokens each.  usage: compute-sanitizer --tool {memcheck,racecheck,synccheck} python
tools/sanitize_case.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

cfg = get_config("T")
plan = m2c.plan_of(cfg)
L = 2
xs = token_stream(cfg, 3, device="cuda")
for mode, fused in (("resident", 1), ("resident", 2), ("lru", 1)):
    ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan)
    cc = None
    if mode != "resident":
        cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, mode)
        ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
    for l in range(L):
        w = layer_weights(cfg, l, device="cuda")
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
    ctx.set_fused(fused)
    ctx.set_graph(False)  # (sanitizers instrument eager launches)
    for t in range(2):
        x = xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
    torch.cuda.synchronize()
    ctx.stats()
    if mode == "resident" and fused == 1:
        sel = ctx.predict_rank(0, xs[2].contiguous())
        ctx.sparse_ffn_forward(0, xs[2].contiguous(), sel["tier_ids"])
        torch.cuda.synchronize()
    ctx.close()
print("sanitize case done")
