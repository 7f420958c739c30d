"""The roofline accounting bench.py reports against SURVEY §8(d)'s computed
algorithmic bytes: record sizes (§8(a) "Record bytes nb_τ"), per-layer and per-token bytes
(§8(d) "Algorithmic bytes per token" table).  CPU only (host functions of libm2c)."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


@pytest.fixture(scope="module")
def bench():
    import bench as b
    return b


def test_record_bytes_match_survey():
    from paper_2410_14740_b200 import record_bytes
    # 24576/12576/6432 (d=4096), 30720/15720/8040 (d=5120) and
    # 49152/25152/12864 (d=8192), before 16-B padding
    for d, want in ((4096, (24576, 12576, 6432)), (5120, (30720, 15720, 8040)),
                    (8192, (49152, 25152, 12864))):
        got = [record_bytes(b, d) for b in (16, 8, 4)]
        assert got == [(w + 15) // 16 * 16 for w in want], d


@pytest.mark.parametrize("name,P,layer_mb,token_mb", [
    ("S7", 1, 17.62, 564.0),     # 13.75 FFN + 3.87 predictor per layer
    ("S13", 1, 26.4, 1057.0),
    ("S70", 8, 11.9, None),      # per rank
    ("S70", 1, 81.1, 6490.0),
])
def test_algorithmic_bytes_match_survey(bench, name, P, layer_mb, token_mb):
    from paper_2410_14740_b200 import plan_of
    from synth import get_config
    cfg = get_config(name)
    ab = bench.algorithmic_bytes(cfg, plan_of(cfg, P), P)
    assert abs(ab["layer"] / 1e6 - layer_mb) <= 0.06 * max(1.0, layer_mb / 10), ab
    if token_mb is not None:
        assert abs(ab["token"] / 1e6 - token_mb) / token_mb <= 0.01, ab
    assert ab["token"] == cfg.n_layers * ab["layer"]
