"""Bit-identity check across builds: sha256 of the decoded tokens of a few stacks (the
streaming-FFN configs included), printed as one line per config.
usage: python tools/hash_out.py   (GPU)"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

for name, L, P, fused in (("S70H", 4, 1, 1), ("S70", 3, 2, 1), ("S7", 3, 1, 1), ("S70H", 3, 1, 0)):
    cfg = get_config(name)
    plan = m2c.plan_of(cfg, P)
    ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan, shard=(0, P))
    for l in range(L):
        w = layer_weights(cfg, l, device="cuda", shard=(0, P))
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
        del w
    ctx.set_fused(fused)
    xs = token_stream(cfg, 6, device="cuda")
    h = hashlib.sha256()
    for t in range(6):
        x = xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
        torch.cuda.synchronize()
        h.update(x.cpu().numpy().tobytes())
    print(name, L, P, "fused" if fused else "chain", h.hexdigest()[:16], ctx.stats()["kernels_per_token"], flush=True)
    ctx.close()
