"""Raw k_decode stamp deltas (ns) for one token: distribution per phase (resolution check).
usage: python tools/stamp_dump.py [CONFIG]   (GPU)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

name = sys.argv[1] if len(sys.argv) > 1 else "S7"
cfg = get_config(name)
L = 4
plan = m2c.plan_of(cfg, 1)
ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan)
for l in range(L):
    w = layer_weights(cfg, l, device="cuda")
    ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
xs = token_stream(cfg, 12, device="cuda")
x = torch.empty(cfg.d_model, dtype=torch.float16, device="cuda")
for t in range(8):
    x.copy_(xs[t]); ctx.decode_step(x, t + 1)
ctx.profile(True)
x.copy_(xs[9]); ctx.decode_step(x, 100)
s = ctx.profile_stamps().astype(np.int64)
ctx.profile(False)
a = s[2]
for nm, i, j in [("load", 4, 2), ("cutbins", 2, 3), ("cand", 3, 10), ("lists", 10, 11), ("ffn", 5, 6)]:
    dd = a[:, j] - a[:, i]
    print(nm, "min", dd.min(), "med", int(np.median(dd)), "max", dd.max(), "uniq mod 32:", sorted(set((dd % 32).tolist()))[:8],
          "sample", dd[:12].tolist())
print(ctx.stats())
