"""NEXT-4: the paper's ablation in structure (`fig:ablation` P:461-483: +MP inference -> +LRU
cache -> +SSDs) and its media latency / copy-size figures (`fig: ete-gpu-dram-ssd`
P:268-276, `fig: bandwidth_time_tensor` P:311-320), on synthetic LLaMA-2-7B FFN shapes.

Points (all an L-layer 4096 x 11008 stack, batch-1 decode through m2c_decode_step):
  dense   every neuron active, all FP16, resident in HBM (the dense FFN)
  mp      10% active, FP16/INT8/INT4 = 1:1:2, resident in HBM          (+MP inference)
  lru     mp + HBM neuron cache capped at 25% of the FP16 FFN bytes, misses from pinned DRAM
  ssd     lru + the DRAM tier backed by a layer-major file: fixed area of 2 layers, FIFO of 2
          frames, I/O thread 1 layer ahead (+SSDs; the file is in the page cache after it is
          written, so this measures the DRAM-frame path, not the drive)
Plus a copy-size sweep: cudaMemcpyAsync H2D (pinned) and D2D GB/s by size.
usage: python tools/ablation.py [LAYERS] [TOKENS]   (GPU; prints JSON lines)"""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2410_14740_b200 as m2c
from synth import get_config, layer_weights, token_stream

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = int(sys.argv[2]) if len(sys.argv) > 2 else 16


def run(point):
    cfg = get_config("S7")
    F = cfg.d_ff
    if point == "dense":
        plan = m2c.tier_plan_make(F, 100, 100, 0, 100)
    else:
        plan = m2c.plan_of(cfg)
    ctx = m2c.M2CContext(cfg.d_model, F, L, cfg.pred_rank, plan)
    cc = None
    if point in ("lru", "ssd"):
        cc = m2c.cache_cfg_capped(ctx.desc, plan, 1, 4, "lru")
        ctx.reserve_host_tier(L * ctx.layer_footprint(cc)[1])
    for l in range(L):
        w = layer_weights(cfg, l, device="cuda")
        ctx.load_layer(l, w["w_gate"], w["w_up"], w["w_down_t"], w["pred_A"], w["pred_B"], cc)
        del w
    path = None
    if point == "ssd":
        path = os.path.join(tempfile.gettempdir(), "m2c_ablation_store.bin")
        ctx.store_write(path)
        ctx.store_attach(path, 2, 2, 1)
    xs = token_stream(cfg, 8 + T, device="cuda")
    x = torch.empty(cfg.d_model, dtype=torch.float16, device="cuda")
    for t in range(8):  # warm-up (and the LRU cache)
        x.copy_(xs[t])
        ctx.decode_step(x, t + 1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in range(T):
        x.copy_(xs[8 + t])
        ctx.decode_step(x, 9 + t)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / T
    out = {"point": point, "layers": L, "tokens": T, "ms_per_token": dt * 1e3,
           "tokens_per_s": 1.0 / dt, "plan": list(plan.as_tuple())}
    st = ctx.stats()
    if cc is not None:
        out["hits"], out["misses"] = st["hits"], st["misses"]
    if path:
        out["store"] = ctx.store_stats()
    ctx.close()
    if path:
        os.remove(path)
    return out


def copy_sweep():
    res = []
    for mb in (0.0625, 0.25, 1, 4, 16, 64, 256):
        n = int(mb * 2 ** 20)
        h = torch.empty(n, dtype=torch.uint8).pin_memory()
        d0 = torch.empty(n, dtype=torch.uint8, device="cuda")
        d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for name, fn in (("h2d", lambda: d0.copy_(h, non_blocking=True)), ("d2d", lambda: d1.copy_(d0))):
            fn()
            reps = max(3, int(64 / max(mb, 0.0625)))
            e0.record()
            for _ in range(reps):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            res.append({"copy": name, "MiB": mb, "us": ms * 1e3, "GB/s": n / (ms * 1e-3) / 1e9})
    return res


if __name__ == "__main__":
    for p in ("dense", "mp", "lru", "ssd"):
        print(json.dumps(run(p)), flush=True)
    for r in copy_sweep():
        print(json.dumps(r), flush=True)
