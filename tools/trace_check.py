"""Round-2 quick check of the decode engine against the oracle via the parity trace (D9).
usage: python tools/trace_check.py [CONFIG LAYERS TOKENS] ..."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2410_14740_b200 as m2c
from oracle import oracle as orc
from synth import get_config, layer_weights, token_stream


def d10(y, yhat):
    y = np.asarray(y, np.float64); yhat = np.asarray(yhat, np.float64)
    floor = 2.0 ** -6 * np.sqrt(np.mean(yhat ** 2))
    return float(np.max(np.abs(y - yhat) / np.maximum(np.abs(yhat), floor)))


def run(name, L, T, kind=""):
    cfg = get_config(name)
    plan = m2c.plan_of(cfg)
    pn = np.array(plan.as_tuple(), np.int32)
    ctx = m2c.M2CContext(cfg.d_model, cfg.d_ff, L, cfg.pred_rank, plan)
    ws = []
    for l in range(L):
        w = layer_weights(cfg, l, device="cuda")
        B = w["pred_B"]
        if kind == "tied_B":
            B = B[torch.arange(B.shape[0], device=B.device) // 7 * 7].contiguous()
            w["pred_B"] = B
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], B)
        ws.append({k: v.cpu().numpy() for k, v in w.items()})
        del w
    ctx.set_trace(True)
    xs = token_stream(cfg, T, device="cuda")
    worst = 0.0
    for t in range(T):
        x = torch.zeros_like(xs[t]) if kind == "zero_x" else xs[t].contiguous().clone()
        ctx.decode_step(x, t + 1)
        torch.cuda.synchronize()
        ctx.stats()
        tx, ty = ctx.trace_x.cpu().numpy(), ctx.trace_y.cpu().numpy()
        assert np.array_equal(tx[L], x.cpu().numpy()), "trace x_L != output"
        for l in range(L):
            wn = ws[l]
            ref = orc.select(orc.predict(tx[l], wn["pred_A"], wn["pred_B"])["s"], pn)
            got = ctx.decode_lists(l).cpu().numpy()
            assert np.array_equal(got, ref["tier_ids"]), (name, t, l, "lists differ")
            recs = orc.records_for(wn, ref["tier_ids"], pn)
            yhat = orc.ffn(cfg.d_model, pn, ref["tier_ids"], recs[16], recs[8], recs[4], tx[l])
            e = d10(ty[l], yhat) if np.any(yhat) else float(np.max(np.abs(ty[l])))
            worst = max(worst, e)
            assert e <= 2e-3, (name, t, l, e)
    print(f"{name}{'/' + kind if kind else ''} L={L} T={T}: lists bit-exact, worst D10 {worst:.2e}", flush=True)
    ctx.close()


if __name__ == "__main__":
    args = sys.argv[1:] or ["T", "3", "4"]
    for i in range(0, len(args), 3):
        nm = args[i]
        kind = ""
        if "/" in nm:
            nm, kind = nm.split("/")
        run(nm, int(args[i + 1]), int(args[i + 2]), kind)
