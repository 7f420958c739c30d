"""Phase timeline of the select-only k_decode launches of an LRU stack (S13 engine): per-CTA
stamps of each layer's launch.  usage: python tools/selonly_timeline.py [CONFIG] [LAYERS]  (GPU)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

name = sys.argv[1] if len(sys.argv) > 1 else "S13"
cfg = get_config(name)
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
plan = m2c.plan_of(cfg)
ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan)
cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, "lru")
ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
for l in range(L):
    w = layer_weights(cfg, l, device="cuda")
    ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
    del w
xs = token_stream(cfg, 24, device="cuda")
x = torch.empty(cfg.d_model, dtype=torch.float16, device="cuda")
for t in range(16):
    x.copy_(xs[t]); ctx.decode_step(x, t + 1)
ctx.profile(True)
acc = []
for t in range(16, 24):
    x.copy_(xs[t]); ctx.decode_step(x, t + 1)
    acc.append(ctx.profile_stamps().astype(np.int64))
ctx.profile(False)
spans = {"start->prologue done (13)": (12, 13), "P2 (0->1)": (0, 1), "Bs (1->4)": (1, 4),
         "P3 (4->5)": (4, 5), "tail sync+clear (5->9)": (5, 9)}
print(f"{name}: {L} layers, select-only k_decode per layer (us; mean over CTAs / max-min crit)")
for k, (i, j) in spans.items():
    mean = np.mean([(s[:, :, j] - s[:, :, i]).mean() for s in acc]) / 1e3
    crit = np.mean([(s[l, :, j].max() - s[l, :, i].min()) for s in acc for l in range(L)]) / 1e3
    print(f"  {k:28s} mean {mean:6.2f}  crit {crit:6.2f}")
tot = np.mean([(s[l, :, 9].max() - s[l, :, 12].min()) for s in acc for l in range(L)]) / 1e3
print(f"  first stamp -> last stamp: {tot:.2f} us per launch")
