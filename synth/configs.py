"""Workload shapes from BASELINE.json ``configs`` (SURVEY.md §8(a) shorthand T/S7/S13/S70/SW).

Plain data only.  The tier-plan rule (k, k16, k8, k4) is NOT computed here: the
product computes it in ``m2c_tier_plan_make`` and the oracle in
``orc_tier_plan`` (reading R3), independently.
"""
from __future__ import annotations

from dataclasses import dataclass, replace


@dataclass(frozen=True)
class ModelConfig:
    name: str
    d_model: int          # d
    d_ff: int             # F (neurons per layer, whole model, before sharding)
    n_layers: int         # L
    pred_rank: int        # r (SURVEY Q1 proposal: 32 for T, 256 otherwise)
    active_pct: int       # active ratio in percent of F_r
    # tier weights: k16 = floor(k*a16/den), k8 = floor(k*a8/den), k4 = k-k16-k8
    a16: int = 25
    a8: int = 25
    den: int = 100
    cache_mode: str = "resident"   # resident | lru | atu
    cap_frac_fp16: float = 0.0     # LRU budget as a fraction of the layer's FP16 FFN bytes
    group: int = 128
    act: str = "silu"              # silu (LLaMA-2) | relu (ReGLU flag)
    rho: float = 0.955             # AR(1) token correlation: layer-0 top-k overlap 0.80
    shards: tuple = (1,)           # P values this config is run at
    warmup_tokens: int = 16
    timed_tokens: int = 256

    def with_(self, **kw) -> "ModelConfig":
        return replace(self, **kw)


CONFIGS = {
    # configs[0]: single synthetic FFN layer, 10% active, 1:1:2, 32 tokens, resident
    "T": ModelConfig("T", 256, 688, 1, 32, 10, timed_tokens=32, warmup_tokens=4),
    # configs[1]: LLaMA-2-7B-shaped FFN stack, whole model resident in HBM, 1 GPU
    "S7": ModelConfig("S7", 4096, 11008, 32, 256, 10),
    # configs[2]: LLaMA-2-13B-shaped stack, HBM neuron cache capped at 25% of FFN weights
    "S13": ModelConfig("S13", 5120, 13824, 40, 256, 10, cache_mode="lru",
                       cap_frac_fp16=0.25, warmup_tokens=64),
    # configs[3]: LLaMA-2-70B-shaped stack, d_ff sharded over 2/4/8 GPUs
    "S70": ModelConfig("S70", 8192, 28672, 80, 256, 10, shards=(1, 2, 4, 8)),
    # 1-GPU point of S70: half-depth stack (SURVEY §7 hard part 7; all 3 tiers of 80 layers
    # exceed one B200's HBM)
    "S70H": ModelConfig("S70H", 8192, 28672, 40, 256, 10),
}


def get_config(name: str) -> ModelConfig:
    return CONFIGS[name]


def sweep_points():
    """configs[4]: active in {5..50}% x FP16 share in {0..100}%, rest INT8:INT4 = 1:2."""
    pts = []
    for act in (5, 10, 20, 30, 40, 50):
        for share in (0, 25, 50, 75, 100):
            pts.append(CONFIGS["S70"].with_(name=f"SW-a{act}-f{share}", active_pct=act,
                                            a16=3 * share, a8=100 - share, den=300,
                                            timed_tokens=128))
    return pts
