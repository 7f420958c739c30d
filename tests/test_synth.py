"""The seeded input generator: determinism, shard slicing, and the adjacent-token overlap
target of SURVEY §8(d) ("Almost 80% of the neurons overlap between tokens")."""
import numpy as np
import torch

from oracle import oracle as orc
from synth import get_config, layer_weights, token_stream
from synth.configs import sweep_points


def test_deterministic_and_order_independent():
    cfg = get_config("T")
    a = layer_weights(cfg, 0)
    b = layer_weights(cfg, 0, parts=("B", "gate"))
    assert torch.equal(a["w_gate"], b["w_gate"]) and torch.equal(a["pred_B"], b["pred_B"])
    c = layer_weights(cfg, 1)
    assert not torch.equal(a["w_gate"], c["w_gate"])
    assert torch.equal(token_stream(cfg, 5), token_stream(cfg, 5))


def test_shards_are_slices_of_the_full_matrix():
    cfg = get_config("T").with_(d_ff=688)
    full = layer_weights(cfg, 0)
    for P in (2, 4):
        for r in range(P):
            s = layer_weights(cfg, 0, shard=(r, P))
            lo, hi = r * 688 // P, (r + 1) * 688 // P
            assert torch.equal(s["w_up"], full["w_up"][lo:hi])
            assert torch.equal(s["pred_B"], full["pred_B"][lo:hi])
            assert torch.equal(s["pred_A"], full["pred_A"])


def test_shapes_dtypes_ranges():
    cfg = get_config("T")
    w = layer_weights(cfg, 0)
    assert w["w_gate"].shape == (688, 256) and w["w_gate"].dtype == torch.float16
    assert w["pred_A"].dtype == torch.int8 and int(w["pred_A"].min()) >= -127
    assert abs(float(w["w_gate"].float().std()) - 1 / 16) < 0.01
    assert len(sweep_points()) == 30


def test_adjacent_token_overlap_near_80pct():
    cfg = get_config("S7")
    w = layer_weights(cfg, 0, parts=("A", "B"))
    A, B = w["pred_A"].numpy(), w["pred_B"].numpy()
    plan = orc.tier_plan(cfg.d_ff, cfg.active_pct)
    xs = token_stream(cfg, 12).numpy()
    sets = [set(orc.select(orc.predict(x, A, B)["s"], plan)["rank_list"].tolist()) for x in xs]
    ov = [len(a & b) / len(a) for a, b in zip(sets, sets[1:])]
    assert 0.76 < np.mean(ov) < 0.84
