"""Copy-versus-compute timeline of the LRU decode engine (S13, configs[2]): per layer, the
compute stream's marks (select done, FFN done, reduce done) and the copy stream's miss fill
(start, end) from CUDA events (m2c_profile_events), averaged over tokens; the fill's overlap
with compute and the per-(layer, tier) hit ratios.
usage: python tools/lru_timeline.py [CONFIG] [TOKENS]   (GPU)"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

name = sys.argv[1] if len(sys.argv) > 1 else "S13"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 8
cfg = get_config(name)
plan = m2c.plan_of(cfg)
L = cfg.n_layers
ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan)
cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, "lru")
ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
for l in range(L):
    w = layer_weights(cfg, l, device="cuda")
    ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
    del w
W = 64
xs = token_stream(cfg, W + 3 * T, device="cuda")  # fresh tokens for each pass
x = torch.empty(cfg.d_model, dtype=torch.float16, device="cuda")
for t in range(W):  # cache warm-up (as bench.py)
    x.copy_(xs[t])
    ctx.decode_step(x, t + 1)
torch.cuda.synchronize()
# per-(layer, tier) hit ratios over the timed tokens, from the pools' occupants before each step
# and the step's tier lists (m2c_cache_state, m2c_decode_lists)
seg = [0, plan.k_fp16, plan.k_fp16 + plan.k_int8, plan.k]
hit = np.zeros((L, 3))
req = np.zeros((L, 3))
for t in range(T):
    occ = [[set(ctx.cache_state(l, tau)[0].cpu().numpy().tolist()) for tau in range(3)] for l in range(L)]
    x.copy_(xs[W + t])
    ctx.decode_step(x, W + t + 1)
    torch.cuda.synchronize()
    for l in range(L):
        ids = ctx.decode_lists(l).cpu().numpy()
        for tau in range(3):
            part = ids[seg[tau]:seg[tau + 1]]
            hit[l, tau] += sum(1 for n in part if int(n) in occ[l][tau])
            req[l, tau] += len(part)
hr = hit / np.maximum(req, 1)
print("per-(layer, tier) hit ratio, FP16 / INT8 / INT4 (mean over %d tokens):" % T)
for l in range(L):
    print("  layer %2d: %.3f %.3f %.3f" % (l, hr[l, 0], hr[l, 1], hr[l, 2]))
print("  all layers: %.3f %.3f %.3f" % tuple(hit.sum(0) / np.maximum(req.sum(0), 1)))
# uninstrumented token time (graph replays, CUDA events) and miss bytes per token
ctx.stats(reset=True)
ctx.requant_stats(reset=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for t in range(T):
    x.copy_(xs[W + T + t])
    ctx.decode_step(x, 500 + t)
e1.record()
torch.cuda.synchronize()
st, rq = ctx.stats(), ctx.requant_stats()
miss_b = sum((m - q) * m2c.record_bytes(b, cfg.d_model) for m, q, b in zip(st["misses"], rq, (16, 8, 4))) / T
print("uninstrumented: %.3f ms/token, %.1f MB/token over PCIe (requantised fills %s), misses %s"
      % (e0.elapsed_time(e1) / T, miss_b / 1e6, rq, st["misses"]))
ctx.profile(True)
ev = []
for t in range(T):
    x.copy_(xs[W + 2 * T + t])
    ctx.decode_step(x, 1000 + t)
    ev.append(ctx.profile_events())
ctx.profile(False)
ev = np.array(ev)  # [T, L, 7]
tok = np.mean(ev[:, -1, 4] - ev[:, 0, 0])
print(f"{name}: {L} layers, token {tok:.3f} ms (instrumented, eager events)")
print(f"{'layer':>5} {'start':>8} {'sel':>7} {'fill0':>7} {'lru':>7} {'hitffn':>7} {'fill1':>7} {'ffn':>7} {'red':>7}  (ms from the layer start)")
ovl = []
for l in range(L):
    e = np.mean(ev[:, l, :] - ev[:, l, 0:1], axis=0)
    if l < 4 or l == L - 1:
        print(f"{l:5d} {np.mean(ev[:, l, 0]):8.3f} {e[2]:7.3f} {e[5]:7.3f} {e[7]:7.3f} {e[8]:7.3f} {e[6]:7.3f} {e[3]:7.3f} {e[4]:7.3f}")
print("per-layer means (ms): layer %.4f | select %.4f | fill start->end %.4f | after the fill: FFN done %.4f, reduce %.4f"
      % (np.mean(np.diff(ev[:, :, 0], axis=1)), np.mean(ev[:, :, 2] - ev[:, :, 0]),
         np.mean(ev[:, :, 6] - ev[:, :, 5]), np.mean(ev[:, :, 3] - ev[:, :, 6]), np.mean(ev[:, :, 4] - ev[:, :, 3])))
lay = np.mean(np.diff(ev[:, :, 0], axis=1))
fill = np.mean(ev[:, :, 6] - ev[:, :, 5])
print("compute stream: select -> miss queue %.4f -> requant %.4f" % (np.mean(ev[:, :, 9] - ev[:, :, 2]), np.mean(ev[:, :, 10] - ev[:, :, 9])))
print("compute stream: select -> LRU update %.4f, -> hit FFN done %.4f ms; miss FFN after max(fill, hit FFN) %.4f"
      % (np.mean(ev[:, :, 7] - ev[:, :, 2]), np.mean(ev[:, :, 8] - ev[:, :, 2]),
         np.mean(ev[:, :, 3] - np.maximum(ev[:, :, 6], ev[:, :, 8]))))
print("fill share of the layer time: %.3f; layer time not covered by its fill: %.4f ms" % (fill / lay, lay - fill))
