"""World-size-2 CPU (gloo) checks of the sharded path's host logic (R13):
NCCL-id bootstrap broadcast, the §8(e) IPC-handle exchange, shard slicing, max-over-ranks timing, and the exchange step's
semantics -- the all-reduced sum of the ranks' oracle partials equals the oracle run on the
union of the shard-local selections (the FFN output is a sum over independent neurons).
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch

    from oracle import oracle as orc
    from paper_2410_14740_b200 import dist as m2c_dist
    from synth import get_config, layer_weights, token_stream

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # bootstrap: rank 0's random 128-byte id reaches every rank unchanged
        uid = m2c_dist.broadcast_unique_id(lambda: os.urandom(128))
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert all(i == uid for i in ids)
        # timing: max over ranks
        assert m2c_dist.max_over_ranks(float(rank + 1)) == float(world)
        # §8(e) bootstrap: every rank connects to all exchange-buffer handles in rank order

        class _Ctx:
            def p2p_buffer(self):
                return 0, bytes([rank + 1]) * 64

            def p2p_connect(self, dev_ptrs=None, ipc_handles=None):
                self.got = ipc_handles

        fc = _Ctx()
        m2c_dist.p2p_init(fc)
        assert fc.got == [bytes([q + 1]) * 64 for q in range(world)]
        # the sharded layer through the oracle, partial sums all-reduced over gloo
        cfg = get_config("T")
        lo, hi = m2c_dist.shard_range(cfg.d_ff, world, rank)
        w = {k: v.numpy() for k, v in layer_weights(cfg, 0, shard=(rank, world)).items()}
        full = {k: v.numpy() for k, v in layer_weights(cfg, 0).items()}
        assert np.array_equal(w["w_up"], full["w_up"][lo:hi])
        plan = orc.tier_plan(cfg.d_ff // world, cfg.active_pct)
        x = token_stream(cfg, 1).numpy()[0]
        recs = orc.layer_records(w)
        r = orc.layer_forward(w, recs, x, plan)
        y = torch.from_numpy(r["yhat"].copy())
        dist.all_reduce(y)
        gids = (r["tier_ids"] + lo).astype(np.int64)
        all_ids = [None] * world
        dist.all_gather_object(all_ids, gids.tolist())
        if rank == 0:
            # union selection, tiers as each rank assigned them, on the unsharded weights
            frecs = orc.layer_records(full)
            tiers = [[], [], []]
            for rr, lst in enumerate(all_ids):
                pr = orc.tier_plan(cfg.d_ff // world, cfg.active_pct)
                seg = [0, pr[1], pr[1] + pr[2], pr[0]]
                for t in range(3):
                    tiers[t] += lst[seg[t]:seg[t + 1]]
            uplan = np.array([sum(map(len, tiers)), len(tiers[0]), len(tiers[1]), len(tiers[2])],
                             np.int32)
            uids = np.array(tiers[0] + tiers[1] + tiers[2], np.int32)
            yu = orc.ffn(cfg.d_model, uplan, uids, frecs[16], frecs[8], frecs[4], x)
            out["err"] = float(np.max(np.abs(y.numpy() - yu)) / np.max(np.abs(yu)))
            out["k"] = int(uplan[0])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_host_logic_gloo(world):
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        assert out["err"] < 1e-12
        assert out["k"] == world * (688 // world * 10 // 100)


def test_shard_range_errors():
    from paper_2410_14740_b200.dist import shard_range
    assert shard_range(28672, 8, 7) == (25088, 28672)
    with pytest.raises(ValueError):
        shard_range(100, 3, 0)


def _worker_global_topk(rank, world, port, out):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

    from oracle import oracle as orc
    from paper_2410_14740_b200 import dist as m2c_dist
    from synth import get_config, layer_input_stream, layer_weights

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # NEXT-3's exchange: every rank's top-min(F_r, k) candidates by (score desc, global id
        # asc), all-gathered, contain the global top-k -- the union of the ranks' parts of the
        # global selection equals the unsharded selection (scores from the oracle's predictor)
        cfg = get_config("T")
        F = cfg.d_ff
        lo, hi = m2c_dist.shard_range(F, world, rank)
        w = {k: v.numpy() for k, v in layer_weights(cfg, 0, shard=(rank, world), parts=("A", "B")).items()}
        gplan = orc.tier_plan(F, 30)
        n = min(hi - lo, int(gplan[0]))
        x = layer_input_stream(cfg, 0, 1).numpy()[0]
        s = orc.predict(x, w["pred_A"], w["pred_B"])["s"]
        cand = sorted(((int(s[i]), lo + i) for i in range(hi - lo)), key=lambda c: (-c[0], c[1]))[:n]
        allc = [None] * world
        dist.all_gather_object(allc, cand)
        merged = sorted((c for lst in allc for c in lst), key=lambda c: (-c[0], c[1]))
        k, k16, k8 = int(gplan[0]), int(gplan[1]), int(gplan[2])
        mine = [[g for (_, g) in merged[a:b] if lo <= g < hi] for a, b in ((0, k16), (k16, k16 + k8), (k16 + k8, k))]
        parts = [None] * world
        dist.all_gather_object(parts, mine)
        if rank == 0:
            full = {kk: v.numpy() for kk, v in layer_weights(cfg, 0, parts=("A", "B")).items()}
            ref = orc.select(orc.predict(x, full["pred_A"], full["pred_B"])["s"], gplan)["tier_ids"]
            got = []
            for t in range(3):
                got += sorted(g for pr in parts for g in pr[t])
            out["equal"] = got == ref.tolist()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_global_topk_exchange_gloo(world):
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker_global_topk, args=(world, port, out), nprocs=world, join=True)
        assert out["equal"]
