"""Debug helper: one token through k_decode at several grid sizes, y against the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream
from test_gpu_engines import oracle_layer, d10

name = sys.argv[1] if len(sys.argv) > 1 else "T"
cfg = get_config(name)
plan = m2c.plan_of(cfg)
w = layer_weights(cfg, 0, device="cuda")
wn = {k: v.cpu().numpy() for k, v in w.items()}
xs = token_stream(cfg, 3, device="cuda")
for G in [int(g) for g in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "8", "148"])]:
    for spec in (0, 1):
        ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, 1, cfg.pred_rank, plan)
        ctx.load_layer(0, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
        ctx.set_grid(G)
        ctx.set_fused(1)
        ctx.set_trace(True)
        errs = []
        for t in range(3):
            x = xs[t].contiguous().clone()
            ctx.decode_step(x, t + 1)
            torch.cuda.synchronize()
            tx, ty = ctx.trace_x.cpu().numpy(), ctx.trace_y.cpu().numpy()
            ids, yhat = oracle_layer(wn, plan, tx[0])
            errs.append(d10(ty[0], yhat))
            if t == 0:
                r = ty[0] / np.where(yhat == 0, 1, yhat)
        print(f"G={G}: errs {['%.3g' % e for e in errs]}  y/yhat median {np.median(r):.4g}", flush=True)
        ctx.close()
        break
