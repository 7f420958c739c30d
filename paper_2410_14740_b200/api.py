"""Python binding of libm2c with the C ABI's names (argument marshalling only).

Every step of the path runs in libm2c's sm_100a kernels; this module only allocates memory
with PyTorch (device regions, the pinned host tier, outputs), passes raw pointers and the
current torch streams, and raises ``M2CError`` on a non-zero status.  Names follow
include/m2c.h; see that header for argument meaning, layout and error behaviour.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from ._lib import CacheCfg, M2CError, ModelDesc, TierPlan, check, lib  # noqa: F401

MODE = {"resident": 0, "lru": 1, "atu": 2}
DECODE_STAMPS = 24  # M2C_DECODE_STAMPS (include/m2c.h)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libm2c compute calls take CUDA tensors (no CPU fallback)")


def _event_handle(ev, stream):
    """cudaEvent_t of a torch.cuda.Event.  torch creates the CUDA event lazily at its first
    record(): an event never recorded has handle 0, which the C ABI would read as 'no event'
    (no wait -- the miss FFN would race the fills).  Force its creation on `stream` first."""
    if ev is None:
        return None
    if not ev.cuda_event:
        ev.record(stream)
    h = ev.cuda_event
    if not h:
        raise M2CError(1, "fill_done: could not create the CUDA event")
    return h


def record_bytes(tier_bits: int, d_model: int) -> int:
    return int(lib().m2c_record_bytes(tier_bits, d_model))


def tier_plan_make(F_r: int, active_pct: int, a16: int = 25, a8: int = 25, den: int = 100) -> TierPlan:
    p = TierPlan()
    check(lib().m2c_tier_plan_make(F_r, active_pct, a16, a8, den, C.byref(p)))
    return p


def plan_of(cfg, shard_count: int = 1) -> TierPlan:
    return tier_plan_make(cfg.d_ff // shard_count, cfg.active_pct, cfg.a16, cfg.a8, cfg.den)


def cache_cfg_resident() -> CacheCfg:
    c = CacheCfg()
    c.mode = 0
    return c


def cache_cfg_capped(desc: ModelDesc, plan: TierPlan, budget_num: int, budget_den: int,
                     mode: str = "lru") -> CacheCfg:
    c = CacheCfg()
    check(lib().m2c_cache_cfg_capped(C.byref(desc), C.byref(plan), budget_num, budget_den,
                                     MODE[mode], C.byref(c)))
    return c


def quant_pack(d_model: int, tier_bits: int, w_gate, w_up, w_down_t, n_begin=0, n_end=None,
               stream=None):
    """m2c_quant_pack: records [n_end-n_begin, record_bytes] uint8 on the inputs' device."""
    _require_cuda(w_gate, w_up, w_down_t)
    n_end = w_gate.shape[0] if n_end is None else n_end
    nb = max(record_bytes(tier_bits, d_model), 16)  # bad bits/d: the C ABI reports the error
    out = torch.empty((max(n_end - n_begin, 0), nb), dtype=torch.uint8, device=w_gate.device)
    st = stream if stream is not None else torch.cuda.current_stream(w_gate.device)
    check(lib().m2c_quant_pack(d_model, tier_bits, _ptr(w_gate), _ptr(w_up), _ptr(w_down_t),
                               n_begin, n_end, _ptr(out), C.c_void_p(st.cuda_stream)))
    return out


def nccl_lib_path():
    try:
        import nvidia.nccl  # type: ignore
        p = os.path.join(list(nvidia.nccl.__path__)[0], "lib", "libnccl.so.2")
        if os.path.exists(p):
            return p
    except Exception:
        pass
    return None


class M2CContext:
    """One m2c_ctx: a rank's FFN stack (its neuron slice of every layer) on one device."""

    def __init__(self, d_model, d_ff, n_layers, pred_rank, plan: TierPlan, shard=(0, 1),
                 act=0, device=None, compute_stream=None, copy_stream=None):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.desc = ModelDesc(d_model, d_ff, n_layers, pred_rank, 128, shard[0], shard[1], act)
        self.F_r = d_ff // shard[1]
        self.plan = plan
        # a dedicated (non-default) stream: the decode step is CUDA-graph captured on it; calls
        # are ordered with the caller's current stream by event waits both ways (_call)
        # the compute stream outranks the copy stream: the miss fill's long-running CTAs must
        # not delay the per-layer compute chain's CTAs (LRU engine, P:396 overlap)
        prio = -1 if os.environ.get("M2C_PRIO", "1") != "0" else 0
        self.compute = compute_stream or torch.cuda.Stream(self.device, priority=prio)
        self.copy = copy_stream or torch.cuda.Stream(self.device)
        h = C.c_void_p()
        check(lib().m2c_create(C.byref(self.desc), self.device.index,
                               C.c_void_p(self.compute.cuda_stream),
                               C.c_void_p(self.copy.cuda_stream), C.byref(plan), C.byref(h)))
        self._h = h
        self.regions = {}   # layer -> (hbm tensor, host tensor or None)
        self._host_pool = None

    def _call(self, fn, *args):
        cur = torch.cuda.current_stream(self.device)
        if cur.cuda_stream == self.compute.cuda_stream:
            return check(fn(*args))
        self.compute.wait_stream(cur)
        try:
            check(fn(*args))
        finally:
            cur.wait_stream(self.compute)

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: modules may already be torn down
            pass

    def close(self):
        if getattr(self, "_h", None):
            torch.cuda.synchronize(self.device)
            lib().m2c_destroy(self._h)
            self._h = None

    # ---- sizes / memory ----
    def layer_footprint(self, cfg: CacheCfg):
        hb, hh = C.c_size_t(), C.c_size_t()
        check(lib().m2c_layer_footprint(C.byref(self.desc), C.byref(cfg), C.byref(hb), C.byref(hh)))
        return hb.value, hh.value

    def reserve_host_tier(self, nbytes: int):
        """One pinned host buffer for every layer's host tier (sliced 256-B aligned)."""
        self._host_pool = torch.empty(nbytes + 256, dtype=torch.uint8, pin_memory=True)
        self._host_off = (-self._host_pool.data_ptr()) % 256

    def _host_slice(self, nbytes):
        if self._host_pool is None:
            self.reserve_host_tier(nbytes)
        t = self._host_pool[self._host_off:self._host_off + nbytes]
        if t.numel() != nbytes:
            raise M2CError(3, "pinned host tier exhausted; call reserve_host_tier with the total")
        self._host_off += (nbytes + 255) // 256 * 256
        return t

    # ---- NEXT-3: exact global top-k under sharding (include/m2c.h) ----
    def predict_candidates(self, layer, x, n_cand):
        _require_cuda(x)
        keys = torch.empty(max(n_cand, 1), dtype=torch.int64, device=self.device)
        self._call(lib().m2c_predict_candidates, self._h, layer, _ptr(x), n_cand, _ptr(keys))
        return keys[:n_cand]

    def select_global(self, keys_all, n_cand, global_plan: TierPlan):
        """keys_all: [P * n_cand] int64 (every rank's candidates, rank order) -> this rank's
        (tier_ids [global k] in segments at the global plan's offsets, counts [3])."""
        _require_cuda(keys_all)
        ids = torch.full((max(global_plan.k, 1),), -1, dtype=torch.int32, device=self.device)
        cnt = torch.zeros(3, dtype=torch.int32, device=self.device)
        self._call(lib().m2c_select_global, self._h, _ptr(keys_all.contiguous()), n_cand,
                   C.byref(global_plan), _ptr(ids), _ptr(cnt))
        return ids[:global_plan.k], cnt

    def set_global_topk(self, global_plan: TierPlan = None):
        """Sharded decode with the exact global selection (NEXT-3); None: shard-local (R13)."""
        check(lib().m2c_set_global_topk(self._h, C.byref(global_plan) if global_plan else None))

    # ---- NEXT-2: cross-layer lookahead staging (include/m2c.h) ----
    def set_lookahead(self, enable: bool):
        self._call(lib().m2c_set_lookahead, self._h, 1 if enable else 0)

    def set_requant(self, enable: bool = True):
        """GPU requantisation of INT misses from resident FP16 records (include/m2c.h)."""
        self._call(lib().m2c_set_requant, self._h, 1 if enable else 0)

    def requant_stats(self, reset=False):
        v = (C.c_int64 * 3)()
        check(lib().m2c_requant_stats(self._h, v, 1 if reset else 0))
        return [int(x) for x in v]

    def lookahead_stats(self, reset=False):
        v = C.c_int64()
        check(lib().m2c_lookahead_stats(self._h, C.byref(v), 1 if reset else 0))
        return v.value

    # ---- NEXT-1: SSD -> DRAM store (include/m2c.h) ----
    def store_write(self, path: str):
        """Write every layer's host tier to a layer-major file (the paper's SSD copy)."""
        self._call(lib().m2c_store_write, self._h, path.encode())

    def store_attach(self, path: str, n_fixed: int, n_dynamic: int, lookahead: int = 2,
                     drop_host_tier: bool = True):
        """Serve the miss fills from DRAM frames of the file: layers [0, n_fixed) fixed, a FIFO
        of n_dynamic frames filled `lookahead` layers ahead by an I/O thread."""
        cfg = next(c for (_, _, c) in self.regions.values())
        fb = lib().m2c_store_frame_bytes(C.byref(self.desc), C.byref(cfg))
        nbytes = (n_fixed + n_dynamic) * fb
        self._frames = torch.empty(nbytes + 4096, dtype=torch.uint8, pin_memory=True)
        off = (-self._frames.data_ptr()) % 4096
        self._call(lib().m2c_store_attach, self._h, path.encode(), n_fixed, n_dynamic, lookahead,
                   C.c_void_p(self._frames.data_ptr() + off), nbytes)
        self._host_dropped = drop_host_tier
        if drop_host_tier:  # the fills no longer read it
            self._host_pool = None
            self.regions = {l: (hb, None, c) for l, (hb, _, c) in self.regions.items()}

    def store_stats(self):
        b, n = C.c_int64(), C.c_int64()
        io, st = C.c_double(), C.c_double()
        check(lib().m2c_store_stats(self._h, C.byref(b), C.byref(n), C.byref(io), C.byref(st)))
        return {"bytes_read": b.value, "layer_loads": n.value, "io_s": io.value, "stall_s": st.value}

    def store_detach(self):
        if getattr(self, "_host_dropped", False):
            raise M2CError(6, "store_detach: the in-memory host tier was dropped at attach")
        self._call(lib().m2c_store_detach, self._h)

    # ---- a0 + load ----
    def load_layer(self, layer, w_gate, w_up, w_down_t, pred_A, pred_B, cfg: CacheCfg = None):
        cfg = cfg or cache_cfg_resident()
        _require_cuda(w_gate, w_up, w_down_t, pred_A, pred_B)
        hb, hh = self.layer_footprint(cfg)
        hbm = torch.empty(hb + 256, dtype=torch.uint8, device=self.device)
        off = (-hbm.data_ptr()) % 256
        hbm = hbm[off:off + hb]
        host = self._host_slice(hh) if hh else None
        self._call(lib().m2c_load_layer, self._h, layer, _ptr(w_gate), _ptr(w_up), _ptr(w_down_t),
                                   _ptr(pred_A), _ptr(pred_B), C.byref(cfg), _ptr(hbm),
                                   _ptr(host))
        self.regions[layer] = (hbm, host, cfg)

    # ---- a1-a3 ----
    def predict_rank(self, layer, x, plan: TierPlan = None, rank_list=True, tier_of=True,
                     scores=True):
        plan = plan or self.plan
        _require_cuda(x)
        dev = self.device
        out = {"tier_ids": torch.empty(max(plan.k, 1), dtype=torch.int32, device=dev)}
        if rank_list:
            out["rank_list"] = torch.empty(max(plan.k, 1), dtype=torch.int32, device=dev)
        if tier_of:
            out["tier_of"] = torch.empty(self.F_r, dtype=torch.int8, device=dev)
        if scores:
            out["scores"] = torch.empty(self.F_r, dtype=torch.int32, device=dev)
        self._call(lib().m2c_predict_rank, self._h, layer, _ptr(x), C.byref(plan),
                                     _ptr(out.get("rank_list")), _ptr(out.get("tier_of")),
                                     _ptr(out["tier_ids"]), _ptr(out.get("scores")))
        for key in ("tier_ids", "rank_list"):
            if key in out:
                out[key] = out[key][:plan.k]
        return out

    # ---- a4-a5 ----
    def cache_lookup_fill(self, layer, step, tier_ids, plan: TierPlan = None, logs=True,
                          fill_done=None):
        plan = plan or self.plan
        dev = self.device
        k = plan.k
        out = {"slots": torch.empty(max(k, 1), dtype=torch.int32, device=dev),
               "hit_bitmap": torch.zeros((k + 31) // 32 + 1, dtype=torch.int32, device=dev)}
        if logs:
            out["miss_log"] = torch.full((max(k, 1), 2), -1, dtype=torch.int32, device=dev)
            out["evict_log"] = torch.full((max(k, 1), 2), -1, dtype=torch.int32, device=dev)
            out["counts"] = torch.zeros(6, dtype=torch.int32, device=dev)
        ev = _event_handle(fill_done, self.copy)
        self._call(lib().m2c_cache_lookup_fill, self._h, layer, step, _ptr(tier_ids), C.byref(plan),
                                          _ptr(out["slots"]), _ptr(out["hit_bitmap"]),
                                          _ptr(out.get("miss_log")), _ptr(out.get("evict_log")),
                                          _ptr(out.get("counts")),
                                          C.c_void_p(ev) if ev else None)
        out["slots"] = out["slots"][:k]
        return out

    # ---- a6-a7 ----
    def sparse_ffn_forward(self, layer, x, tier_ids, slots=None, hit_bitmap=None,
                           plan: TierPlan = None, fill_done=None, want_partial=True, want_y=True):
        plan = plan or self.plan
        d = self.desc.d_model
        yp = torch.empty(d, dtype=torch.float32, device=self.device) if want_partial else None
        y = torch.empty(d, dtype=torch.float16, device=self.device) if want_y else None
        ev = _event_handle(fill_done, self.copy)
        self._call(lib().m2c_sparse_ffn_forward, self._h, layer, _ptr(x), _ptr(tier_ids), _ptr(slots),
                                           _ptr(hit_bitmap), C.byref(plan),
                                           C.c_void_p(ev) if ev else None, _ptr(yp), _ptr(y))
        return yp, y

    # ---- whole token ----
    def decode_step(self, x_inout, step: int):
        self._call(lib().m2c_decode_step, self._h, _ptr(x_inout), int(step))

    def decode_lists(self, layer):
        """Tier lists [k] (k16 | k8 | k4 ascending segments) of the last decode step's layer."""
        out = torch.empty(max(self.plan.k, 1), dtype=torch.int32, device=self.device)
        self._call(lib().m2c_decode_lists, self._h, layer, _ptr(out))
        return out[:self.plan.k]

    def set_trace(self, enable: bool = True):
        """Parity trace (D9): afterwards every decode_step records x_l [L+1, d] fp16 and y_l
        [L, d] f32 into ``self.trace_x`` / ``self.trace_y`` (device tensors owned here)."""
        L, d = self.desc.n_layers, self.desc.d_model
        if enable:
            self.trace_x = torch.zeros(L + 1, d, dtype=torch.float16, device=self.device)
            self.trace_y = torch.zeros(L, d, dtype=torch.float32, device=self.device)
            check(lib().m2c_set_trace(self._h, _ptr(self.trace_x), _ptr(self.trace_y)))
        else:
            check(lib().m2c_set_trace(self._h, None, None))
            self.trace_x = self.trace_y = None

    def cache_state(self, layer, tier):
        """LRU/ATU pool state of (layer, tier): (occupant int32 [cap], last_use int32 [cap])."""
        cap = C.c_int32()
        check(lib().m2c_cache_state(self._h, layer, tier, None, None, C.byref(cap)))
        occ = torch.empty(max(cap.value, 1), dtype=torch.int32, device=self.device)
        last = torch.empty(max(cap.value, 1), dtype=torch.int32, device=self.device)
        # (the copies run on the compute stream: _call orders the caller's stream after them --
        # reading the tensors unordered returned stale blocks of the caching allocator)
        self._call(lib().m2c_cache_state, self._h, layer, tier, _ptr(occ), _ptr(last), C.byref(cap))
        return occ[:cap.value], last[:cap.value]

    def set_graph(self, enable: bool):
        check(lib().m2c_set_graph(self._h, 1 if enable else 0))

    def set_fused(self, enable):
        """True/1: the persistent decode kernel when eligible; 2: the layer-split k_decode (one
        launch per layer, the sharded engine) even unsharded; False/0: the per-phase chain."""
        check(lib().m2c_set_fused(self._h, int(enable)))

    def profile(self, enable: bool):
        check(lib().m2c_profile(self._h, 1 if enable else 0))

    def profile_read(self):
        """Per-layer phase times (ms) of the last decode step: [L, 4] = predict, select,
        cache+FFN, reduce; plus the FFN launches per layer."""
        L = self.desc.n_layers
        ms = (C.c_float * (4 * L))()
        n = C.c_int32()
        check(lib().m2c_profile_read(self._h, ms, C.byref(n)))
        return [list(ms[4 * l:4 * l + 4]) for l in range(L)], n.value

    def profile_fill(self):
        """Miss-fill duration (ms) per layer of the last profiled decode step (0: resident)."""
        ms = (C.c_float * self.desc.n_layers)()
        check(lib().m2c_profile_fill(self._h, ms))
        return list(ms)

    def profile_events(self):
        """Per-layer CUDA-event timeline of the last (kernel-chain) decode step, ms since the
        first mark: numpy float32 [n_layers, 9] (include/m2c.h m2c_profile_events)."""
        import numpy as np
        n = C.c_int64()
        check(lib().m2c_profile_events(self._h, None, 0, C.byref(n)))
        buf = (C.c_float * n.value)()
        check(lib().m2c_profile_events(self._h, buf, n.value, C.byref(n)))
        return np.frombuffer(buf, dtype=np.float32).copy().reshape(self.desc.n_layers, -1)

    def profile_stamps(self):
        """Raw k_decode stamps of the last decode step (profiling on): numpy uint64
        [n_layers, G, DECODE_STAMPS] in ns (include/m2c.h documents the stamp points)."""
        import numpy as np
        n = C.c_int64()
        check(lib().m2c_profile_stamps(self._h, None, 0, C.byref(n)))
        buf = (C.c_uint64 * n.value)()
        check(lib().m2c_profile_stamps(self._h, buf, n.value, C.byref(n)))
        a = np.frombuffer(buf, dtype=np.uint64).copy()
        return a.reshape(self.desc.n_layers, -1, DECODE_STAMPS)

    def stats(self, reset=False):
        kpt = C.c_int64()
        hits = (C.c_int64 * 3)()
        miss = (C.c_int64 * 3)()
        check(lib().m2c_stats(self._h, C.byref(kpt), hits, miss, 1 if reset else 0))
        return {"kernels_per_token": kpt.value, "hits": list(hits), "misses": list(miss)}

    # ---- multi-GPU ----
    def comm_init(self, nranks, rank, unique_id: bytes, nccl_lib=None):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        path = nccl_lib or nccl_lib_path()
        check(lib().m2c_comm_init(self._h, nranks, rank, buf,
                                  path.encode() if path else None))

    def set_grid(self, ctas: int):
        """CTAs of this context's kernels (1..SM count)."""
        check(lib().m2c_set_grid(self._h, int(ctas)))

    def p2p_buffer(self):
        """§8(e) exchange buffer: (device address, 64-byte cudaIpcMemHandle)."""
        ptr = C.c_uint64()
        h = C.create_string_buffer(64)
        check(lib().m2c_p2p_buffer(self._h, C.byref(ptr), h))
        return ptr.value, h.raw

    def p2p_connect(self, dev_ptrs=None, ipc_handles=None):
        """Connect the in-kernel all-reduce: every rank's buffer address (same process) or
        IPC handle (one per process, this rank's own entry is ignored)."""
        P = self.desc.shard_count
        ptrs = (C.c_uint64 * P)(*dev_ptrs) if dev_ptrs is not None else None
        hs = C.create_string_buffer(b"".join(ipc_handles), 64 * P) if ipc_handles is not None else None
        check(lib().m2c_p2p_connect(self._h, P, ptrs, hs))


def nccl_unique_id(nccl_lib=None) -> bytes:
    buf = C.create_string_buffer(128)
    path = nccl_lib or nccl_lib_path()
    check(lib().m2c_nccl_unique_id(path.encode() if path else None, buf))
    return buf.raw
