"""Seeded synthetic weights and token streams (SURVEY.md §8(d) "Synthetic inputs").

Recipe (restated in DESIGN.md "Input recipe"):
  * W_gate, W_up  ~ N(0, 1/d)            -> fp16, neuron-major [F, d]
  * W_down^T      ~ N(0, sigma_d^2)      -> fp16, neuron-major [F, d] (row n = down column n)
    with sigma_d chosen so rms(y) ~= 0.1 rms(x) at the config's k (stable residual stack)
  * predictor A [r, d], B [F, r]: uniform int8 in [-127, 127]
  * tokens: AR(1) stream x^{t+1} = fp16(rho x^t + sqrt(1-rho^2) eps_t), eps ~ N(0, I)

Every tensor is drawn from its own ``torch.Generator`` seeded by
``seed_for(master, layer, matrix)`` so a tensor does not depend on the order in
which others were drawn, and the same call on the same device is
bit-reproducible.  Parity tests draw once and hand the SAME tensors to both the
oracle (host copy) and the CUDA path.
"""
from __future__ import annotations

import math

import torch

MASTER_SEED = 241014740
_MASK64 = (1 << 64) - 1

# E[silu(g)^2] for g ~ N(0, 1) (Monte-Carlo, 4e6 samples: 0.3557); a generator constant
_E_SILU2 = 0.3557

_MATRIX_IDS = {"gate": 1, "up": 2, "down": 3, "A": 4, "B": 5, "tok": 6, "xin": 7}


def _splitmix64(z: int) -> int:
    z = (z + 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def seed_for(*keys: int) -> int:
    """Counter-style seed derivation: fold the keys through splitmix64 (63-bit result)."""
    z = 0
    for k in keys:
        z = _splitmix64(z ^ (int(k) & _MASK64))
    return z & ((1 << 63) - 1)


def _gen(device, *keys) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed_for(*keys))
    return g


def sigma_down(cfg) -> float:
    k = cfg.d_ff * cfg.active_pct // 100
    return 0.1 / math.sqrt(max(k, 1) * _E_SILU2)


def layer_weights(cfg, layer: int, device="cpu", master: int = MASTER_SEED, shard=(0, 1),
                  parts=("gate", "up", "down", "A", "B")) -> dict:
    """Weights of FFN layer ``layer``.  ``shard=(rank, P)`` returns rows [rank*F/P, (rank+1)*F/P)
    of the neuron-major matrices (the full matrix is drawn first, so slices of different P agree).
    """
    d, F, r = cfg.d_model, cfg.d_ff, cfg.pred_rank
    rank, P = shard
    assert F % P == 0
    lo, hi = rank * F // P, (rank + 1) * F // P
    out = {}
    std = {"gate": 1.0 / math.sqrt(d), "up": 1.0 / math.sqrt(d), "down": sigma_down(cfg)}
    for name in ("gate", "up", "down"):
        if name not in parts:
            continue
        g = _gen(device, master, layer, _MATRIX_IDS[name])
        w = torch.randn(F, d, generator=g, device=device, dtype=torch.float32)
        w = (w[lo:hi] * std[name]).to(torch.float16).contiguous()
        out["w_" + name if name != "down" else "w_down_t"] = w
    if "A" in parts:
        g = _gen(device, master, layer, _MATRIX_IDS["A"])
        out["pred_A"] = torch.randint(-127, 128, (r, d), generator=g, device=device,
                                      dtype=torch.int8)
    if "B" in parts:
        g = _gen(device, master, layer, _MATRIX_IDS["B"])
        B = torch.randint(-127, 128, (F, r), generator=g, device=device, dtype=torch.int8)
        out["pred_B"] = B[lo:hi].contiguous()
    return out


def _ar1(d, n, rho, g, device, scale=1.0):
    xs = torch.empty(n, d, dtype=torch.float16, device=device)
    x = torch.randn(d, generator=g, device=device, dtype=torch.float32) * scale
    xs[0] = x.to(torch.float16)
    c = math.sqrt(max(0.0, 1.0 - rho * rho))
    for t in range(1, n):
        eps = torch.randn(d, generator=g, device=device, dtype=torch.float32) * scale
        x = rho * xs[t - 1].float() + c * eps
        xs[t] = x.to(torch.float16)
    return xs


def token_stream(cfg, n_tokens: int, device="cpu", master: int = MASTER_SEED, rho=None):
    """Layer-0 inputs x_0^t, t = 0..n_tokens-1, fp16 [n_tokens, d] (AR(1))."""
    g = _gen(device, master, 0xFFFF, _MATRIX_IDS["tok"])
    return _ar1(cfg.d_model, n_tokens, cfg.rho if rho is None else rho, g, device)


def layer_input_stream(cfg, layer: int, n_tokens: int, device="cpu", master: int = MASTER_SEED,
                       rho=None, scale=1.0):
    """Stand-alone inputs for layer ``layer`` (per-layer parity at any depth without replaying
    a GPU-produced residual stream): an AR(1) stream of its own seed."""
    g = _gen(device, master, layer, _MATRIX_IDS["xin"])
    return _ar1(cfg.d_model, n_tokens, cfg.rho if rho is None else rho, g, device, scale)
