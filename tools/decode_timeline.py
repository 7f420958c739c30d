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
L = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] else cfg.n_layers
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
names = ["P2 hq+s+hist", "Bs", "P3 select", "P3 tail", "P4 ffn", "By", "R red+h", "Bx"]
acc = {k: [] for k in names}
accm = {k: [] for k in names}
tot = []
pro = []
for s in rows:
    tot.append((s[-1, :, 9].max() - s[0, :, 12].min()) / 1e3)
    pro.append((s[0, :, 13].max() - s[0, :, 12].min()) / 1e3)
    for l in range(L):
        a = s[l]
        nxt0 = s[l + 1, :, 0] if l + 1 < L else a[:, 9]
        # phase = (last CTA done) - (first CTA started); barrier = (last release) - (last arrival)
        def ph(i, j):
            return (a[:, j].max() - a[:, i].min(), (a[:, j] - a[:, i]).mean())
        def br(i, nxt):
            return (nxt.max() - a[:, i].max(), (nxt - a[:, i].max()).mean())
        spans = {
            "P2 hq+s+hist": ph(0, 1),
            "Bs": br(1, a[:, 4]),
            "P3 select": ph(4, 10),
            "P3 tail": ph(10, 5),
            "P4 ffn": ph(5, 6),
            "By": br(6, a[:, 7]),
            "R red+h": ph(7, 8),
            "Bx": br(8, nxt0),
        }
        for k, (mx, mn) in spans.items():
            acc[k].append(mx / 1e3)
            accm[k].append(mn / 1e3)
print(f"{name}: {L} layers, token {np.mean(tot):.1f} us ({np.mean(tot) / L:.2f} us/layer), prologue {np.mean(pro):.2f} us")
print(f"{'phase':14s} {'crit us':>8s} {'mean-CTA us':>12s}")
for k in names:
    print(f"{k:14s} {np.mean(acc[k]):8.2f} {np.mean(accm[k]):12.2f}")
s = rows[-1][L // 2]
print("P4 per-CTA us (mid layer): min %.2f median %.2f max %.2f argmax %d" % (
    ((s[:, 6] - s[:, 5]) / 1e3).min(), np.median((s[:, 6] - s[:, 5]) / 1e3),
    ((s[:, 6] - s[:, 5]) / 1e3).max(), int(np.argmax(s[:, 6] - s[:, 5]))))
G = rows[-1].shape[1]
p4 = np.mean([(s[:, :, 6] - s[:, :, 5]) / 1e3 for s in rows], axis=(0, 1))  # per CTA
print("P4 mean per CTA by sixths of the grid:", " ".join(f"{p4[i * G // 6:(i + 1) * G // 6].mean():.2f}" for i in range(6)))
for nm, (i, j) in {"gate/up": (14, 15), "down": (15, 6), "P2+Bs": (0, 4), "P3": (4, 5)}.items():
    v = np.mean([(s[:, :, j] - s[:, :, i]) / 1e3 for s in rows], axis=(0, 1))
    print(f"{nm:8s} by sixths:", " ".join(f"{v[q * G // 6:(q + 1) * G // 6].mean():.2f}" for q in range(6)))
sub = {"P2 h+max": (0, 20), "P2 hq+B": (20, 21), "P2 dots": (21, 22), "P2 atomics": (22, 1), "P3 hist load": (4, 2), "P3 scan": (2, 3), "P3 rank": (3, 10), "P3 tail": (10, 5), "P4 issue": (5, 14), "P4 gate/up": (14, 15), "P4 down": (15, 6)}
for k, (i, j) in sub.items():
    v = np.mean([((s[:, :, j] - s[:, :, i]) / 1e3).mean() for s in rows])
    print(f"{k:12s} mean-CTA {v:.2f} us")
print(ctx.stats())
