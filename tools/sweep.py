"""configs[4] (SW): the active-ratio x FP16-share sweep on the 70B FFN shape at P = 8, as the
per-rank work of one rank measured on ONE GPU (this environment has one): rank 0's shard
(F_r = 3584) of an L-layer 8192 x 28672 stack through the layer-split k_decode (the sharded
engine), without the all-reduce.  Per point: tokens/s of the rank's stack, achieved GB/s of
its algorithmic bytes and the fraction of the HBM peak.  Active in {5, 10, 20, 30, 40, 50}%,
FP16 share in {0, 25, 50, 75, 100}%, the rest INT8:INT4 = 1:2 (R3).
usage: python tools/sweep.py [LAYERS] [TOKENS]   (GPU; JSON lines)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_14740_b200 as m2c
from bench import _peaks, algorithmic_bytes
from synth import layer_weights, token_stream
from synth.configs import sweep_points

L = int(sys.argv[1]) if len(sys.argv) > 1 else 16
T = int(sys.argv[2]) if len(sys.argv) > 2 else 32
P = 8
peak, peak_src = _peaks()
pts = sweep_points()
base = pts[0].with_(n_layers=L)
weights = []  # one shard's weights, shared by every point (only the plan changes)
for l in range(L):
    weights.append(layer_weights(base, l, device="cuda", shard=(0, P)))
xs = token_stream(base, 8 + T, device="cuda")
for pt in pts:
    cfg = pt.with_(n_layers=L)
    plan = m2c.plan_of(cfg, P)
    ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan, shard=(0, P))
    for l, w in enumerate(weights):
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    ctx.set_fused(2)  # the layer-split engine a sharded rank runs
    x = torch.empty(cfg.d_model, dtype=torch.float16, device="cuda")
    for t in range(8):
        x.copy_(xs[t])
        ctx.decode_step(x, t + 1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(T):
        x.copy_(xs[8 + t])
        ctx.decode_step(x, 100 + t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / T
    ab = algorithmic_bytes(cfg, plan, P)
    gbs = ab["token"] / (ms * 1e-3) / 1e9
    print(json.dumps({"point": cfg.name, "active_pct": cfg.active_pct, "fp16_share": cfg.a16 // 3,
                      "plan": list(plan.as_tuple()), "layers": L, "rank_ms_per_token": ms,
                      "us_per_layer": ms * 1e3 / L, "GB_s": gbs, "hbm_frac": gbs / peak,
                      "peak": peak, "peak_src": peak_src}), flush=True)
    ctx.close()
