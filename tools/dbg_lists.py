"""Debug: decode lists of k_decode vs predict_rank on the same layer input.
usage: python tools/dbg_lists.py CONFIG [TOKENS]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

cfg = get_config(sys.argv[1])
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3
plan = m2c.plan_of(cfg)
ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, 1, cfg.pred_rank, plan, act=0 if cfg.act == "silu" else 1)
w = layer_weights(cfg, 0, device="cuda")
ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
xs = token_stream(cfg, T, device="cuda")
print("plan", plan.k, plan.k_fp16, plan.k_int8, plan.k_int4)
for t in range(T):
    x0 = xs[t].contiguous()
    x = x0.clone()
    ctx.decode_step(x, t + 1)
    lists = ctx.decode_lists(0).cpu()
    sel = ctx.predict_rank(0, x0)
    ref = sel["tier_ids"].cpu()
    _, y = ctx.sparse_ffn_forward(0, x0, sel["tier_ids"], want_partial=False)
    torch.cuda.synchronize()
    xc = x0 + y
    bad = (lists != ref).nonzero().flatten().tolist()
    print(f"token {t}: lists equal {len(bad) == 0} (first bad {bad[:8]}), x equal {torch.equal(x, xc)}, "
          f"max|dx| {float((x.float() - xc.float()).abs().max()):.3g}")
    if bad:
        print(" got", lists[bad[:8]].tolist(), " want", ref[bad[:8]].tolist())
try:
    print(ctx.stats())
except Exception as e:
    print("stats:", e)
