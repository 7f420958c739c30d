"""CPU-side checks of the boundary: libm2c.so loads without a GPU, exports every symbol
include/m2c.h declares, its pure-host helpers agree with the oracle's host logic and with
the survey's per-config numbers, and compute entry points fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest
import torch

from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "m2c.h")


@pytest.fixture(scope="module")
def m2c():
    from paper_2410_14740_b200.build import build
    build()
    import paper_2410_14740_b200 as pkg
    return pkg


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(m2c_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(m2c):
    syms = declared_symbols()
    assert len(syms) >= 15
    L = m2c.lib()
    for s in syms:
        assert hasattr(L, s), s
    from paper_2410_14740_b200._lib import SIGNATURES
    assert sorted(n for n, _, _ in SIGNATURES) == syms


def test_record_bytes_and_plans_match_oracle(m2c):
    from paper_2410_14740_b200 import record_bytes, tier_plan_make
    for d in (256, 4096, 5120, 8192):
        for b in (16, 8, 4):
            assert record_bytes(b, d) == orc.record_bytes(b, d)
    assert record_bytes(5, 256) == -1
    rng = np.random.default_rng(0)
    for _ in range(200):
        F = int(rng.integers(0, 40000))
        pct = int(rng.integers(0, 101))
        a16 = int(rng.integers(0, 301))
        a8 = int(rng.integers(0, 301 - a16))
        p = tier_plan_make(F, pct, a16, a8, 300)
        assert list(p.as_tuple()) == list(orc.tier_plan(F, pct, a16, a8, 300))


def test_capped_cache_sizing_s13(m2c):
    # S13 at 25% of the FP16 FFN bytes -> C = (1696, 1696, 3403) with unpadded
    # record sizes; with the 16-B padded INT8/INT4 records (15728 / 8048 B) M = 4.9166 -> 3402
    from paper_2410_14740_b200 import cache_cfg_capped, tier_plan_make
    from paper_2410_14740_b200._lib import ModelDesc
    desc = ModelDesc(5120, 13824, 40, 256, 128, 0, 1, 0)
    plan = tier_plan_make(13824, 10)
    cfg = cache_cfg_capped(desc, plan, 1, 4, "lru")
    assert list(cfg.cap_slots) == [1696, 1696, 3402]
    atu = cache_cfg_capped(desc, plan, 1, 4, "atu")
    assert list(atu.cap_slots) == [345, 345, 692]


def test_footprint(m2c):
    from paper_2410_14740_b200._lib import CacheCfg, ModelDesc, check, lib
    desc = ModelDesc(4096, 11008, 32, 256, 128, 0, 1, 0)
    cfg = CacheCfg()
    hb, hh = C.c_size_t(), C.c_size_t()
    check(lib().m2c_layer_footprint(C.byref(desc), C.byref(cfg), C.byref(hb), C.byref(hh)))
    assert hh.value == 0
    pools = 11008 * (24576 + 12576 + 6432)
    assert pools <= hb.value <= pools + 256 * 4 * 8 + 256 * 4096 + 11008 * 256
    # S7 all three tiers resident: 15.35 GB for 32 layers
    assert abs(32 * hb.value / 1e9 - 15.47) < 0.2
    bad = ModelDesc(4000, 11008, 32, 256, 128, 0, 1, 0)
    assert lib().m2c_layer_footprint(C.byref(bad), C.byref(cfg), C.byref(hb), C.byref(hh)) == 2


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_compute_calls_fail_loudly_without_gpu(m2c):
    from paper_2410_14740_b200 import M2CError, tier_plan_make
    with pytest.raises((M2CError, RuntimeError, AssertionError)):
        m2c.M2CContext(256, 688, 1, 32, tier_plan_make(688, 10))
