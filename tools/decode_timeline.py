"""Per-phase critical-path timeline of the persistent decode kernel from its per-CTA stamps.
usage: python tools/decode_timeline.py [CONFIG] [LAYERS] [TOKENS]   (GPU; prints a table)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

name = sys.argv[1] if len(sys.argv) > 1 else "S7"
cfg = get_config(name)
L = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_layers
T = int(sys.argv[3]) if len(sys.argv) > 3 else 8
plan = m2c.plan_of(cfg, 1)
ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan, act=0 if cfg.act == "silu" else 1)
for l in range(L):
    w = layer_weights(cfg, l, device="cuda")
    ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"])
    del w
xs = token_stream(cfg, 8 + T, device="cuda")
x = torch.empty(cfg.d_model, dtype=torch.float16, device="cuda")
for t in range(8):
    x.copy_(xs[t]); ctx.decode_step(x, t + 1)
ctx.profile(True)
rows = []
for t in range(T):
    x.copy_(xs[8 + t]); ctx.decode_step(x, 100 + t)
    s = ctx.profile_stamps().astype(np.int64)  # [L, G, 10]
    rows.append(s)
ctx.profile(False)
names = ["P1 h", "B1", "P2 s+hist", "B2", "P3 select", "P4 ffn", "B4", "P5 reduce", "B5"]
acc = {k: [] for k in names}
accm = {k: [] for k in names}
tot = []
for s in rows:
    tot.append((s[-1, :, 9].max() - s[0, :, 0].min()) / 1e3)
    for l in range(L):
        a = s[l]
        nxt0 = s[l + 1, :, 0] if l + 1 < L else a[:, 9]
        # phase = (last CTA done) - (first CTA released); barrier = (last release) - (last arrival)
        spans = {
            "P1 h": (a[:, 1].max() - a[:, 0].min(), (a[:, 1] - a[:, 0]).mean()),
            "B1": (a[:, 2].max() - a[:, 1].max(), (a[:, 2] - a[:, 1].max()).mean()),
            "P2 s+hist": (a[:, 3].max() - a[:, 2].min(), (a[:, 3] - a[:, 2]).mean()),
            "B2": (a[:, 4].max() - a[:, 3].max(), (a[:, 4] - a[:, 3].max()).mean()),
            "P3 select": (a[:, 5].max() - a[:, 4].min(), (a[:, 5] - a[:, 4]).mean()),
            "P4 ffn": (a[:, 6].max() - a[:, 5].min(), (a[:, 6] - a[:, 5]).mean()),
            "B4": (a[:, 7].max() - a[:, 6].max(), (a[:, 7] - a[:, 6].max()).mean()),
            "P5 reduce": (a[:, 8].max() - a[:, 7].min(), (a[:, 8] - a[:, 7]).mean()),
            "B5": (nxt0.max() - a[:, 8].max(), (nxt0 - a[:, 8].max()).mean()),
        }
        for k, (mx, mn) in spans.items():
            acc[k].append(mx / 1e3)
            accm[k].append(mn / 1e3)
print(f"{name}: {L} layers, token {np.mean(tot):.1f} us ({np.mean(tot) / L:.2f} us/layer)")
print(f"{'phase':12s} {'crit us':>8s} {'mean-CTA us':>12s}")
for k in names:
    print(f"{k:12s} {np.mean(acc[k]):8.2f} {np.mean(accm[k]):12.2f}")
s = rows[-1][L // 2]
print("P4 per-CTA us (mid layer): min %.2f median %.2f max %.2f argmax %d" % (
    ((s[:, 6] - s[:, 5]) / 1e3).min(), np.median((s[:, 6] - s[:, 5]) / 1e3),
    ((s[:, 6] - s[:, 5]) / 1e3).max(), int(np.argmax(s[:, 6] - s[:, 5]))))
print("P3 per-CTA us (mid layer): min %.2f median %.2f max %.2f" % (
    ((s[:, 5] - s[:, 4]) / 1e3).min(), np.median((s[:, 5] - s[:, 4]) / 1e3), ((s[:, 5] - s[:, 4]) / 1e3).max()))
G = rows[-1].shape[1]
p4 = np.mean([(s[:, :, 6] - s[:, :, 5]) / 1e3 for s in rows], axis=(0, 1))  # per CTA
print("P4 mean per CTA by sixths of the grid:", " ".join(f"{p4[i * G // 6:(i + 1) * G // 6].mean():.2f}" for i in range(6)))
sub = {"P3a cuts": (4, 10), "P3a classify": (10, 11), "B3": (11, 12), "P3b gather": (12, 13),
       "P3b tail": (13, 5), "P4 setup": (5, 14), "P4 gate/up": (14, 15), "P4 down": (15, 6)}
for k, (i, j) in sub.items():
    v = np.mean([((s[:, :, j] - s[:, :, i]) / 1e3).mean() for s in rows])
    print(f"{k:12s} mean-CTA {v:.2f} us")
print(ctx.stats())
