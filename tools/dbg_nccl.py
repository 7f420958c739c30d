import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream
cfg = get_config("T"); L = 3; plan = m2c.plan_of(cfg)
ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan)
for l in range(L):
    w = layer_weights(cfg, l, device="cuda")
    ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
ctx.comm_init(1, 0, m2c.nccl_unique_id())
x = token_stream(cfg, 1, device="cuda")[0].contiguous().clone()
ctx.decode_step(x, 1); torch.cuda.synchronize()
print("graph kpt", ctx.stats())
ctx.set_graph(False)
x = token_stream(cfg, 1, device="cuda")[0].contiguous().clone()
ctx.decode_step(x, 2); torch.cuda.synchronize()
print("eager kpt", ctx.stats())
