"""Per-rank decode cost of the d_ff-sharded S70 stack, measured on ONE GPU (no all-reduce):
rank 0's shard of an 80 x (8192 x 28672) stack at P ways, through the layer-split k_decode
(the sharded engine) and through the per-phase kernel chain.  Each rank of a real P-GPU run
does this work plus one 32 KB all-reduce per layer.
usage: python tools/shard_cost.py [P ...]   (GPU; JSON lines)"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

cfg = get_config("S70")
Ps = [int(a) for a in sys.argv[1:]] or [8, 4]
for P in Ps:
    plan = m2c.plan_of(cfg, P)
    ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, cfg.n_layers, cfg.pred_rank, plan, shard=(0, P))
    for l in range(cfg.n_layers):
        w = layer_weights(cfg, l, device="cuda", shard=(0, P))
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
        del w
    xs = token_stream(cfg, 40, device="cuda")
    x = torch.empty(cfg.d_model, dtype=torch.float16, device="cuda")
    for mode, name in ((1, "whole-token k_decode"), (2, "layer-split k_decode"), (0, "kernel chain")):
        ctx.set_fused(mode)
        for t in range(8):
            x.copy_(xs[t])
            ctx.decode_step(x, t + 1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(32):
            x.copy_(xs[8 + t])
            ctx.decode_step(x, 100 + t)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 32
        print(json.dumps({"P": P, "engine": name, "layers": cfg.n_layers, "F_r": cfg.d_ff // P,
                          "ms_per_token_per_rank": ms, "us_per_layer": ms * 1e3 / cfg.n_layers,
                          "kernels_per_token": ctx.stats()["kernels_per_token"]}), flush=True)
    ctx.close()
    torch.cuda.empty_cache()
