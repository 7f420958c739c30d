"""§8(e) cost of the all-reduce fused into k_decode, measured on ONE GPU: P d_ff shards of an
L-layer stack share the GPU (148 / P CTAs each) and decode concurrently on their own streams.
  alone     rank 0's shard decoded by itself at 148 / P CTAs, no exchange (the compute floor)
  all-none  all shards concurrently, no exchange (P independent kernels)
  all-p2p   all shards concurrently with the in-kernel exchange (flagged peer stores)
all-p2p - all-none is what the exchange adds per token (on one GPU the 'peer' is the same
HBM; across NVLink add the link latency, ~1-2 us per layer-chunk round trip).
usage: python tools/p2p_cost.py [CONFIG] [LAYERS] [TOKENS] [P]   (GPU; JSON lines)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_14740_b200 as m2c
from paper_2410_14740_b200._lib import lib
from paper_2410_14740_b200.api import check
from synth import get_config, layer_weights, token_stream

name = sys.argv[1] if len(sys.argv) > 1 else "S7"
cfg = get_config(name)
L = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_layers
T = int(sys.argv[3]) if len(sys.argv) > 3 else 32
P = int(sys.argv[4]) if len(sys.argv) > 4 else 2
G = 148 // P
plan = m2c.plan_of(cfg, P)


def make(p2p):
    ctxs = []
    for r in range(P):
        ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan, shard=(r, P))
        for l in range(L):
            w = layer_weights(cfg, l, device="cuda", shard=(r, P))
            ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
            del w
        ctx.set_grid(G)
        ctxs.append(ctx)
    if p2p:
        ptrs = [c.p2p_buffer()[0] for c in ctxs]
        for c in ctxs:
            c.p2p_connect(dev_ptrs=ptrs)
    return ctxs


xs = token_stream(cfg, 8 + T, device="cuda")


def run(ctxs, who):
    xr = [torch.empty(cfg.d_model, dtype=torch.float16, device="cuda") for _ in ctxs]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for t in range(8 + T):
        if t == 8:
            torch.cuda.synchronize()
            e0.record()
        for x in xr:
            x.copy_(xs[t])
        torch.cuda.synchronize()  # (inputs in place; both ranks launch with no dependency)
        for i in who:
            check(lib().m2c_decode_step(ctxs[i]._h, xr[i].data_ptr(), t + 1))
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    for i in who:
        ctxs[i].stats()
    return e0.elapsed_time(e1) / T


for label, p2p, who in (("alone", False, [0]), ("all-none", False, list(range(P))),
                        ("all-p2p", True, list(range(P)))):
    ctxs = make(p2p)
    ms = run(ctxs, who)
    print(json.dumps({"config": name, "layers": L, "P": P, "ctas_per_rank": G, "mode": label, "ms_per_token": ms,
                      "us_per_layer": ms * 1e3 / L, "note": "per-token wall incl. host sync"}),
          flush=True)
    for c in ctxs:
        c.close()
