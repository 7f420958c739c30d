"""Debug helper: one context, N layers, decode a few tokens fused or unfused, report errors.
usage: python tools/dbg_decode.py CONFIG PARTS FUSED(0/1) [LAYERS] [TOKENS]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

name, parts, fused = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
L = int(sys.argv[4]) if len(sys.argv) > 4 else 1
T = int(sys.argv[5]) if len(sys.argv) > 5 else 2
cfg = get_config(name)
plan = m2c.plan_of(cfg, parts)
ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan, shard=(0, parts),
                     act=0 if cfg.act == "silu" else 1)
for l in range(L):
    w = layer_weights(cfg, l, device="cuda", shard=(0, parts))
    ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
torch.cuda.synchronize()
print("loaded", flush=True)
ctx.set_fused(bool(fused))
xs = token_stream(cfg, T, device="cuda")
for t in range(T):
    x = xs[t].contiguous().clone()
    ctx.decode_step(x, t + 1)
    torch.cuda.synchronize()
    print("token", t, "ok", float(x.float().abs().max()), flush=True)
print(ctx.stats())
