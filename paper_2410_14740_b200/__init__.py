"""m2c: B200-native (sm_100a) dynamic sparse mixed-precision FFN decode of M2Cache
(arXiv 2410.14740).  The compute lives in libm2c.so (C ABI: include/m2c.h); this package is
the ctypes binding (``api``) plus the build recipe (``build``).  No CPU fallback."""
from ._lib import M2CError, lib  # noqa: F401
from .api import (  # noqa: F401
    M2CContext,
    cache_cfg_capped,
    cache_cfg_resident,
    nccl_unique_id,
    plan_of,
    quant_pack,
    record_bytes,
    tier_plan_make,
)
