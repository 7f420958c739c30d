"""Per-call API fill/FFN ordering check at S13 size: the LRU layer run through predict ->
lookup+fill -> FFN with the fill_done event vs. with a full device sync between them; every
token must be bit-identical (caught torch.cuda.Event's lazy creation: an unrecorded event has
handle 0 and the C ABI skipped the wait).  usage: python tools/race_s13.py   (GPU)"""
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, layer_input_stream
cfg = get_config("S13"); plan = m2c.plan_of(cfg)
w = layer_weights(cfg, 0, device="cuda")
def run(sync):
    ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, 1, cfg.pred_rank, plan)
    cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, "lru")
    ctx.reserve_host_tier(ctx.layer_footprint(cc)[1])
    ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
    xs = layer_input_stream(cfg, 0, 32, device="cuda")
    ev = torch.cuda.Event()
    ys = []
    for t in range(32):
        x = xs[t].contiguous()
        sel = ctx.predict_rank(0, x, rank_list=False, tier_of=False, scores=False)
        lk = ctx.cache_lookup_fill(0, 10 + t, sel["tier_ids"], fill_done=ev)
        if sync: torch.cuda.synchronize()
        _, y = ctx.sparse_ffn_forward(0, x, sel["tier_ids"], lk["slots"], lk["hit_bitmap"], fill_done=ev, want_partial=False)
        ys.append(y.clone())
    torch.cuda.synchronize()
    ctx.close()
    return torch.stack(ys)
ref = run(True)
for rep in range(4):
    got = run(False)
    bad = (got != ref).any(dim=1).nonzero().flatten().tolist()
    print("rep", rep, "tokens differing from synced run:", bad, flush=True)
