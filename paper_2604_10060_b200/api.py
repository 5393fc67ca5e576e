"""Python host mirror of the reference's hot-path interface over the C-ABI (include/kvc.h).

`ClusterKVCache` is the GPU-backed counterpart of the reference's `StreamEngine`
(core/include/kvclust/engine.hpp:62-100) together with the views its tests use on
`HierIndex` / `TieredStore` / `Maintainer` / `RetrievalResult`. Method names follow the
reference (process_frame ~ StreamEngine::process(Frame), query ~ StreamEngine::process(Query),
flat_topk ~ oracle_flat_topk, ...). Errors raise the reference's exception names
(error.hpp:9-82) as Python classes.

There is no CPU fallback: constructing a cache without a CUDA device raises NoDevice, and
importing without the built library raises ImportError.
"""
from __future__ import annotations

import atexit
import ctypes as C
import os
import weakref
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libkvc.so")

f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
vp = C.c_void_p

MEM_HOST, MEM_DEVICE = 0, 1
DTYPE_F32, DTYPE_BF16 = 0, 1
CAUSES = ("retrieval", "maintenance", "prefetch", "completion", "offload")


# ----------------------------------------------------------------------------- errors
class KvcError(RuntimeError):
    code = -1


class DegenerateVector(KvcError): code = -2
class DimMismatch(KvcError): code = -3
class EmptyInput(KvcError): code = -4
class EmptyCluster(KvcError): code = -5
class TooFewPoints(KvcError): code = -6
class BadLayer(KvcError): code = -7
class UnknownCluster(KvcError): code = -8
class EmptyIndex(KvcError): code = -9
class ConfigError(KvcError): code = -10
class InvariantViolation(KvcError): code = -11
class CudaError(KvcError): code = -20
class CapacityError(KvcError): code = -21
class NoDevice(KvcError): code = -22


_BY_CODE = {c.code: c for c in (DegenerateVector, DimMismatch, EmptyInput, EmptyCluster,
                                 TooFewPoints, BadLayer, UnknownCluster, EmptyIndex, ConfigError,
                                 InvariantViolation, CudaError, CapacityError, NoDevice)}


# ----------------------------------------------------------------------------- config
class Config(C.Structure):
    """kvc_cfg: EngineConfig flattened (engine.hpp:21-33) + device data-plane sizing."""

    _fields_ = [
        ("k_v", C.c_int32), ("k_s", C.c_int32), ("window_frames", C.c_int32),
        ("prefetch_k", C.c_int32), ("prefetch_enabled", C.c_int32), ("token_mode", C.c_int32),
        ("token_budget", C.c_int64),
        ("lookup_cost_per_candidate_us", C.c_double), ("compute_cost_per_token_us", C.c_double),
        ("tau_min", C.c_double), ("tau_max", C.c_double), ("n0", C.c_double),
        ("defer_host_splits", C.c_int32), ("max_split_depth", C.c_int32),
        ("visual_floor", C.c_double),
        ("target_visual_cluster_size", C.c_int32), ("target_semantic_cluster_size", C.c_int32),
        ("kmeans_max_iters", C.c_int32), ("kmeans_tol", C.c_double),
        ("alpha_us", C.c_double), ("beta_us_per_byte", C.c_double),
        ("bytes_per_entry", C.c_int64), ("device_capacity_entries", C.c_int64),
        ("build_batch_frames", C.c_int32), ("batched_ingest", C.c_int32),
        ("ingest_overhead_us", C.c_double), ("offload_horizon_frames", C.c_int32),
        ("seed", C.c_uint64),
        ("kv_dtype", C.c_int32), ("page_tokens", C.c_int32), ("max_pages", C.c_int64),
        ("pool_bytes", C.c_int64), ("max_slots", C.c_int32), ("max_cluster_pages", C.c_int32),
        ("max_buffer_pages", C.c_int32), ("max_partitions", C.c_int32),
        ("max_candidates", C.c_int32), ("max_tokens", C.c_int32), ("parity_mode", C.c_int32),
        ("check_invariants", C.c_int32), ("tier_stage_pages", C.c_int32),
        ("host_pool_bytes", C.c_int64),
    ]

    @classmethod
    def make(cls, **kw) -> "Config":
        c = cls()
        lib().kvc_cfg_default(C.byref(c))
        for k, v in kw.items():
            if not hasattr(c, k):
                raise ConfigError(f"unknown config key: {k}")  # harness.cpp:162-237 rejects unknown keys
            setattr(c, k, v)
        return c


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2604_10060_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        L.kvc_cfg_default.argtypes = [vp]
        L.kvc_last_error.restype = C.c_char_p
        L.kvc_create.argtypes = [vp, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.kvc_destroy.argtypes = [vp]
        L.kvc_stream.argtypes = [vp]
        L.kvc_stream.restype = vp
        L.kvc_ingest_frame.argtypes = [vp, C.c_int64, f32p, vp, vp, C.c_int32, C.c_int32, i64p, i64p]
        L.kvc_decode_step.argtypes = [vp, C.c_int64, vp, C.c_int32, vp, C.c_int32, i64p, C.c_int32]
        L.kvc_last_ranked.argtypes = [vp, C.c_int32, i64p, i32p, C.c_int32]
        L.kvc_last_selected.argtypes = [vp, C.c_int32, i64p, C.c_int32]
        L.kvc_last_attended.argtypes = [vp, C.c_int32, i64p, i32p, C.c_int32]
        L.kvc_last_layer_meta.argtypes = [vp, C.c_int32, f64p, i64p]
        L.kvc_last_query_meta.argtypes = [vp, f64p]
        L.kvc_last_digest.argtypes = [vp]
        L.kvc_last_digest.restype = C.c_uint64
        L.kvc_flat_topk.argtypes = [vp, f32p, C.c_int32, C.c_int32, i64p, i32p]
        L.kvc_build_now.argtypes = [vp]
        L.kvc_bulk_load.argtypes = [vp, f32p, vp, vp, C.c_int32, C.c_int32, i32p, i64p, i32p,
                                    C.c_int32, i64p]
        L.kvc_n_clusters.argtypes = [vp]
        L.kvc_cluster_ids.argtypes = [vp, i64p, C.c_int32]
        L.kvc_cluster.argtypes = [vp, C.c_int64, i64p, f64p, f64p, f64p]
        L.kvc_cluster_entries.argtypes = [vp, C.c_int64, C.c_int32, i64p, i32p, C.c_int32]
        L.kvc_cluster_payload.argtypes = [vp, C.c_int64, C.c_int32, f32p, f32p, C.c_int32]
        L.kvc_n_partitions.argtypes = [vp]
        L.kvc_partition.argtypes = [vp, C.c_int32, f64p, i64p, C.c_int32]
        L.kvc_partition_layer.argtypes = [vp, C.c_int32, C.c_int32, i64p, C.c_int32]
        L.kvc_maint_stats.argtypes = [vp, i64p]
        L.kvc_ledger.argtypes = [vp, i64p, i64p, f64p]
        L.kvc_ledger.restype = C.c_int64
        L.kvc_ledger_log_size.argtypes = [vp]
        L.kvc_ledger_op.argtypes = [vp, C.c_int32, i64p]
        L.kvc_check.argtypes = [vp]
        L.kvc_offload.argtypes = [vp, C.c_int64, f64p]
        L.kvc_fetch.argtypes = [vp, C.c_int64, C.c_int32, f64p]
        L.kvc_tier_sync.argtypes = [vp]
        L.kvc_tier_stats.argtypes = [vp, i64p]
        L.kvc_cluster_tier.argtypes = [vp, C.c_int64, i64p]
        L.kvc_debug_tier_check.argtypes = [vp, i64p]
        L.kvc_debug_split_two.argtypes = [vp, f32p, C.c_int32, C.c_uint64, i32p, i32p, f64p]
        L.kvc_debug_kmeans.argtypes = [vp, f32p, C.c_int32, i32p, i32p, C.c_int32, C.c_double,
                                       C.POINTER(C.c_uint64), i32p, i32p, f64p]
        L.kvc_exchange_bytes.restype = C.c_size_t
        L.kvc_exchange_bytes.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        L.kvc_ipc_alloc.argtypes = [C.c_size_t, C.POINTER(vp), C.c_void_p]
        L.kvc_ipc_open.argtypes = [C.c_void_p, C.POINTER(vp)]
        L.kvc_ipc_close.argtypes = [vp]
        L.kvc_ipc_free.argtypes = [vp]
        L.kvc_set_peers.argtypes = [vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.kvc_peer_output.argtypes = [vp, vp, C.c_int32]
        L.kvc_launch_count.argtypes = [vp]
        L.kvc_launch_count.restype = C.c_int64
        L.kvc_last_step_timing.argtypes = [vp, f64p]
        L.kvc_set_timing.argtypes = [vp, C.c_int32]
        L.kvc_set_head_dim.argtypes = [vp, C.c_int32]
        L.kvc_last_ingest_timing.argtypes = [vp, f64p]
        L.kvc_debug_resolve_profile.argtypes = [vp, f64p]
        L.kvc_debug_event_profile.argtypes = [vp, f64p, C.c_int32]
        L.kvc_debug_wave_profile.argtypes = [vp, f64p, C.c_int32]
        L.kvc_debug_assign_check.argtypes = [vp, vp, C.c_int32, C.c_int64, C.c_int32, f64p]
        L.kvc_debug_div_check.argtypes = [C.c_uint64, C.c_uint64, C.c_int32, C.POINTER(C.c_uint64)]
        L.kvc_host_split_two.argtypes = [f32p, C.c_int32, C.c_int32, C.c_uint64, i32p, i32p]
        L.kvc_host_kmeans.argtypes = [f32p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double,
                                      C.c_uint64, i32p, f64p, i32p]
        L.kvc_host_tau.restype = C.c_double
        L.kvc_host_tau.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double]
        L.kvc_host_mix_seed.restype = C.c_uint64
        L.kvc_host_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.kvc_host_rng_first2.argtypes = [C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.kvc_host_rng_first2.restype = None
        _lib = L
    return _lib


EXPORTED = [
    "kvc_cfg_default", "kvc_create", "kvc_destroy", "kvc_last_error", "kvc_stream",
    "kvc_ingest_frame", "kvc_decode_step", "kvc_last_ranked", "kvc_last_selected",
    "kvc_last_attended", "kvc_last_layer_meta", "kvc_last_query_meta", "kvc_last_digest",
    "kvc_flat_topk", "kvc_build_now", "kvc_bulk_load", "kvc_n_clusters", "kvc_cluster_ids",
    "kvc_cluster", "kvc_cluster_entries", "kvc_cluster_payload", "kvc_n_partitions",
    "kvc_partition", "kvc_partition_layer", "kvc_maint_stats", "kvc_ledger",
    "kvc_ledger_log_size", "kvc_ledger_op", "kvc_check", "kvc_offload", "kvc_fetch",
    "kvc_launch_count", "kvc_last_step_timing", "kvc_set_timing", "kvc_set_head_dim", "kvc_last_ingest_timing",
    "kvc_debug_resolve_profile", "kvc_host_split_two", "kvc_host_kmeans", "kvc_host_tau",
    "kvc_host_mix_seed", "kvc_host_rng_first2", "kvc_debug_div_check", "kvc_debug_assign_check", "kvc_tier_sync",
    "kvc_tier_stats", "kvc_cluster_tier", "kvc_debug_tier_check", "kvc_debug_split_two", "kvc_debug_kmeans", "kvc_exchange_bytes", "kvc_ipc_alloc",
    "kvc_ipc_open", "kvc_ipc_close", "kvc_ipc_free", "kvc_set_peers", "kvc_peer_output",
    "kvc_debug_event_profile", "kvc_debug_wave_profile", "kvc_add_partition", "kvc_append_frame", "kvc_add_cluster", "kvc_adopt",
    "kvc_reset_window", "kvc_set_retrieval", "kvc_place_frame", "kvc_insert", "kvc_materialize", "kvc_touch",
    "kvc_pin", "kvc_enforce_capacity", "kvc_visual_topk", "kvc_semantic_topk", "kvc_last_frames",
    "kvc_last_predicted", "kvc_reconfigure", "kvc_add_partition_ex", "kvc_add_cluster_ex",
]


def _check(rc: int):
    if rc < 0:
        msg = lib().kvc_last_error().decode(errors="replace")
        raise _BY_CODE.get(rc, KvcError)(f"[{rc}] {msg}")
    return rc


def _p(a, t):
    return a.ctypes.data_as(t)


def _ptr(x):
    """Host numpy array -> (pointer, MEM_HOST); torch CUDA tensor -> (data_ptr, MEM_DEVICE)."""
    if isinstance(x, np.ndarray):
        return C.c_void_p(x.ctypes.data), MEM_HOST
    if hasattr(x, "data_ptr"):
        if getattr(x, "is_cuda", False):
            return C.c_void_p(x.data_ptr()), MEM_DEVICE
        return C.c_void_p(x.data_ptr()), MEM_HOST
    raise TypeError(type(x))


@dataclass
class LayerMeta:
    lookup_us: float
    transfer_us: float
    stall_us: float
    completion_us: float
    compute_us: float
    verified_clusters: int
    prefetch_hits: int
    rep_count: int
    n_predicted: int
    attended_count: int


_LIVE = weakref.WeakSet()


@atexit.register
def _close_all():
    """Destroys every live context at interpreter exit (device memory is released explicitly, so
    compute-sanitizer's leak check reports only real leaks)."""
    for kv in list(_LIVE):
        try:
            kv.close()
        except Exception:
            pass


class ClusterKVCache:
    """One stream's cluster-level KV cache on the current CUDA device (kvc_create)."""

    def __init__(self, cfg: Config, d: int, L: int):
        self.cfg, self.d, self.L = cfg, d, L
        self.h = vp()
        _check(lib().kvc_create(C.byref(cfg), d, L, C.byref(self.h)))
        self.es = 2 if cfg.kv_dtype == DTYPE_BF16 else 4
        _LIVE.add(self)

    def close(self):
        if self.h:
            lib().kvc_destroy(self.h)
            self.h = vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return lib().kvc_stream(self.h) or 0

    # ------------------------------------------------------------------ hot path
    def process_frame(self, frame_id: int, visual, keys, values, want_assigned: bool = True):
        """StreamEngine::process(Frame). keys/values [L, T, d] (numpy host or torch CUDA)."""
        T = int(keys.shape[1])
        kp, mem = _ptr(keys)
        vp_, mem2 = _ptr(values)
        assert mem == mem2
        vis = np.ascontiguousarray(visual, np.float32)
        assigned = np.full(self.L * T, -1, np.int64) if want_assigned else None
        pid = C.c_int64(-1)
        _check(lib().kvc_ingest_frame(self.h, frame_id, _p(vis, f32p), kp, vp_, T, mem,
                                      _p(assigned, i64p) if assigned is not None else None,
                                      C.byref(pid)))
        return pid.value, (assigned.reshape(self.L, T) if assigned is not None else None)

    def query(self, query_id: int, q, out=None, gt=None):
        """StreamEngine::process(Query) + attention. Returns out [L, d] (numpy if host)."""
        qp, qm = _ptr(q)
        if out is None:
            out = np.zeros((self.L, self.d), np.float32)
        op, om = _ptr(out)
        g = None if gt is None else np.ascontiguousarray(gt, np.int64)
        _check(lib().kvc_decode_step(self.h, query_id, qp, qm, op, om,
                                     _p(g, i64p) if g is not None else None,
                                     0 if g is None else len(g)))
        return out

    def build_now(self):
        _check(lib().kvc_build_now(self.h))

    def bulk_load(self, visual, keys, values, assign, frame_ids, token_ids, n_clusters):
        """HierIndex::add_partition + add_cluster per cluster (see kvc.h). keys [L, N, d]."""
        N = int(keys.shape[1])
        kp, mem = _ptr(keys)
        vp_, _ = _ptr(values)
        a = np.ascontiguousarray(assign, np.int32)
        f = np.ascontiguousarray(frame_ids, np.int64)
        t = np.ascontiguousarray(token_ids, np.int32)
        vis = np.ascontiguousarray(visual, np.float32)
        pid = C.c_int64(-1)
        _check(lib().kvc_bulk_load(self.h, _p(vis, f32p), kp, vp_, N, n_clusters, _p(a, i32p),
                                   _p(f, i64p), _p(t, i32p), mem, C.byref(pid)))
        return pid.value

    # ------------------------------------------------------------------ last query views
    def ranked(self, l: int, cap: int = 4096):
        ids = np.zeros(cap, np.int64)
        buf = np.zeros(cap, np.int32)
        n = _check(lib().kvc_last_ranked(self.h, l, _p(ids, i64p), _p(buf, i32p), cap))
        return [(int(ids[i]), int(buf[i])) for i in range(n)]

    def selected(self, l: int, cap: int = 1 << 16):
        ids = np.zeros(cap, np.int64)
        n = _check(lib().kvc_last_selected(self.h, l, _p(ids, i64p), cap))
        return ids[:n].tolist()

    def attended(self, l: int, cap: int = 1 << 20):
        fr = np.zeros(cap, np.int64)
        tk = np.zeros(cap, np.int32)
        n = _check(lib().kvc_last_attended(self.h, l, _p(fr, i64p), _p(tk, i32p), cap))
        return fr[:n].copy(), tk[:n].copy()

    def layer_meta(self, l: int) -> LayerMeta:
        lat = np.zeros(5)
        ints = np.zeros(5, np.int64)
        _check(lib().kvc_last_layer_meta(self.h, l, _p(lat, f64p), _p(ints, i64p)))
        return LayerMeta(*lat.tolist(), *[int(x) for x in ints])

    def query_meta(self):
        dd = np.zeros(2)
        lib().kvc_last_query_meta(self.h, _p(dd, f64p))
        return float(dd[0]), float(dd[1])

    def digest(self) -> int:
        return int(lib().kvc_last_digest(self.h))

    def flat_topk(self, q, layer: int, k: int):
        ids = np.zeros(max(k, 1), np.int64)
        buf = np.zeros(max(k, 1), np.int32)
        qq = np.ascontiguousarray(q, np.float32)
        n = _check(lib().kvc_flat_topk(self.h, _p(qq, f32p), layer, k, _p(ids, i64p), _p(buf, i32p)))
        return [(int(ids[i]), int(buf[i])) for i in range(n)]

    # ------------------------------------------------------------------ index / store views
    def cluster_ids(self):
        n = lib().kvc_n_clusters(self.h)
        ids = np.zeros(max(n, 1), np.int64)
        lib().kvc_cluster_ids(self.h, _p(ids, i64p), n)
        return ids[:n].tolist()

    def cluster(self, cid: int):
        """(info[10], variance, rep[d], buffer_rep[d]) -- see kvc_cluster."""
        info = np.zeros(10, np.int64)
        var = C.c_double()
        rep = np.zeros(self.d)
        brep = np.zeros(self.d)
        _check(lib().kvc_cluster(self.h, cid, _p(info, i64p), C.byref(var), _p(rep, f64p), _p(brep, f64p)))
        return info, var.value, rep, brep

    def cluster_entries(self, cid: int, which: int = 0, cap: int = 1 << 20):
        fr = np.zeros(cap, np.int64)
        tk = np.zeros(cap, np.int32)
        n = _check(lib().kvc_cluster_entries(self.h, cid, which, _p(fr, i64p), _p(tk, i32p), cap))
        return fr[:n].copy(), tk[:n].copy()

    def cluster_payload(self, cid: int, which: int = 0, cap: int = 1 << 16):
        k = np.zeros((cap, self.d), np.float32)
        v = np.zeros((cap, self.d), np.float32)
        n = _check(lib().kvc_cluster_payload(self.h, cid, which, _p(k, f32p), _p(v, f32p), cap))
        return k[:n].copy(), v[:n].copy()

    def n_partitions(self) -> int:
        return lib().kvc_n_partitions(self.h)

    def partition(self, p: int, cap: int = 1 << 16):
        rep = np.zeros(self.d)
        fr = np.zeros(cap, np.int64)
        n = _check(lib().kvc_partition(self.h, p, _p(rep, f64p), _p(fr, i64p), cap))
        return rep, fr[:n].copy()

    def partition_layer(self, p: int, layer: int, cap: int = 1 << 16):
        ids = np.zeros(cap, np.int64)
        n = _check(lib().kvc_partition_layer(self.h, p, layer, _p(ids, i64p), cap))
        return ids[:n].tolist()

    def maint_stats(self):
        o = np.zeros(9, np.int64)
        lib().kvc_maint_stats(self.h, _p(o, i64p))
        return o

    def ledger(self):
        ops = np.zeros(5, np.int64)
        by = np.zeros(5, np.int64)
        co = np.zeros(5)
        dev = lib().kvc_ledger(self.h, _p(ops, i64p), _p(by, i64p), _p(co, f64p))
        return ops, by, co, int(dev)

    def ledger_log(self):
        n = lib().kvc_ledger_log_size(self.h)
        out = np.zeros((n, 4), np.int64)
        for i in range(n):
            lib().kvc_ledger_op(self.h, i, _p(out[i], i64p))
        return out

    def check(self):
        _check(lib().kvc_check(self.h))

    def set_retrieval(self, **fields):
        """Per-call RetrievalConfig (kvc_set_retrieval): k_v, k_s, prefetch_k, prefetch_enabled,
        lookup / compute cost constants; other fields keep the context's configuration."""
        import copy

        c = copy.copy(self.cfg)
        for k, v in fields.items():
            setattr(c, k, v)
        _check(lib().kvc_set_retrieval(self.h, C.byref(c)))
        self.cfg = c

    def offload(self, cid: int) -> float:
        c = C.c_double()
        _check(lib().kvc_offload(self.h, cid, C.byref(c)))
        return c.value

    def fetch(self, cid: int, cause: int = 0) -> float:
        c = C.c_double()
        _check(lib().kvc_fetch(self.h, cid, cause, C.byref(c)))
        return c.value

    # ------------------------------------------------------------------ physical host tier
    TIER_KEYS = ("host_pages", "host_capacity_pages", "host_clusters", "offloads", "fetches",
                 "bytes_d2h", "bytes_h2d", "queued", "in_flight", "stage_pages", "batches", "copies",
                 "read_fetches", "read_fetch_bytes")

    def tier_sync(self):
        """Completes every queued / in-flight host-tier migration (kvc_tier_sync)."""
        _check(lib().kvc_tier_sync(self.h))

    def tier_stats(self) -> dict:
        out = np.zeros(len(self.TIER_KEYS), np.int64)
        _check(lib().kvc_tier_stats(self.h, _p(out, i64p)))
        return dict(zip(self.TIER_KEYS, (int(x) for x in out)))

    def cluster_tier(self, cid: int):
        """(first host page, host pages, migration busy) of a cluster's host-tier extent."""
        out = np.zeros(3, np.int64)
        _check(lib().kvc_cluster_tier(self.h, cid, _p(out, i64p)))
        return int(out[0]), int(out[1]), bool(out[2])

    def tier_check(self):
        """(host ids outside extents, Device clusters with host pages, Host clusters fully in
        HBM, fill / tail mismatches) -- all zero once tier_sync() returned."""
        out = np.zeros(4, np.int64)
        _check(lib().kvc_debug_tier_check(self.h, _p(out, i64p)))
        return tuple(int(x) for x in out)

    def debug_split_two(self, pts, seed: int):
        """split_two of host points [n, d] through the device split kernel (split.cu):
        (assign, k_live, iterations, degenerate, objective)."""
        pts = np.ascontiguousarray(pts, np.float32)
        n = pts.shape[0]
        assign = np.zeros(n, np.int32)
        meta = np.zeros(3, np.int32)
        obj = np.zeros(1, np.float64)
        _check(lib().kvc_debug_split_two(self.h, _p(pts, f32p), n, seed, _p(assign, i32p), _p(meta, i32p),
                                         _p(obj, f64p)))
        return assign, int(meta[0]), int(meta[1]), bool(meta[2]), float(obj[0])

    def debug_kmeans(self, sets, ks, seeds, max_iters: int = 50, tol: float = 1e-6):
        """spherical_kmeans of several point sets [n_i, d] in one batch-build launch
        (kmeans_dev.cu): [(assign, k_live, iterations, objective)] per set."""
        sets = [np.ascontiguousarray(x, np.float32) for x in sets]
        pts = np.ascontiguousarray(np.concatenate(sets, 0))
        n = np.array([x.shape[0] for x in sets], np.int32)
        k = np.array(ks, np.int32)
        sd = np.array(seeds, np.uint64)
        assign = np.zeros(int(n.sum()), np.int32)
        meta = np.zeros(2 * len(sets), np.int32)
        obj = np.zeros(len(sets), np.float64)
        _check(lib().kvc_debug_kmeans(self.h, _p(pts, f32p), len(sets), _p(n, i32p), _p(k, i32p), max_iters, tol,
                                      sd.ctypes.data_as(C.POINTER(C.c_uint64)), _p(assign, i32p), _p(meta, i32p),
                                      _p(obj, f64p)))
        out, o = [], 0
        for i, x in enumerate(sets):
            out.append((assign[o:o + len(x)].copy(), int(meta[2 * i]), int(meta[2 * i + 1]), float(obj[i])))
            o += len(x)
        return out

    # ------------------------------------------------------------------ fused output exchange
    def set_peers(self, n_ranks: int, rank: int, dom_offset: int, total_domains: int, bufs):
        """kvc_set_peers: bufs = every rank's mapped exchange buffer (device pointers, rank order)."""
        arr = (C.c_void_p * len(bufs))(*[C.c_void_p(int(b)) for b in bufs])
        _check(lib().kvc_set_peers(self.h, n_ranks, rank, dom_offset, total_domains, arr))

    def peer_output(self, out):
        """The last step's gathered outputs [total_domains, d] (torch CUDA tensor or numpy)."""
        p, mem = _ptr(out)
        _check(lib().kvc_peer_output(self.h, p, mem))
        return out

    # ------------------------------------------------------------------ instrumentation
    def launch_count(self) -> int:
        return int(lib().kvc_launch_count(self.h))

    def set_timing(self, on: bool):
        lib().kvc_set_timing(self.h, 1 if on else 0)

    def resolve_profile(self, decode=False):
        t = np.zeros(16)
        if decode:
            t[0] = -1.0
        lib().kvc_debug_resolve_profile(self.h, _p(t, f64p))
        return t

    EVENT_KEYS = ("events_us", "stage_us", "kmeans_us", "host_stats_us", "upload_us", "relaunch_us", "events",
                  "split_two_calls", "spec_splits", "spec_hits")

    def event_profile(self, reset: bool = False) -> dict:
        """Host-event slow-path profile (kvc_debug_event_profile), cumulative."""
        t = np.zeros(10)
        _check(lib().kvc_debug_event_profile(self.h, _p(t, f64p), 1 if reset else 0))
        return dict(zip(self.EVENT_KEYS, t.round(1).tolist()))

    WAVE_KEYS = ("frames_with_events", "waves", "passes", "rolled_back_domains", "verify_kmeans", "events",
                 "stage_us", "kmeans_jobs", "kmeans_us", "install_us", "relaunch_us", "verify_commit_us",
                 "verified_swapped")

    def wave_profile(self, reset: bool = False) -> dict:
        """Wave-engine profile (kvc_debug_wave_profile), cumulative."""
        t = np.zeros(13)
        _check(lib().kvc_debug_wave_profile(self.h, _p(t, f64p), 1 if reset else 0))
        return dict(zip(self.WAVE_KEYS, t.round(1).tolist()))

    def assign_check(self, keys, partition: int = 0):
        """Distance-tile self-check on a frame keys [L, T, d] (see kvc_debug_assign_check):
        (max |approx - exact|, top-M violations, top-M exact mismatches, certified margin)."""
        kp, mem = _ptr(keys)
        out = np.zeros(4)
        _check(lib().kvc_debug_assign_check(self.h, kp, int(keys.shape[1]), partition, mem, _p(out, f64p)))
        return float(out[0]), int(out[1]), int(out[2]), float(out[3])

    def ingest_timing(self):
        t = np.zeros(10)
        lib().kvc_last_ingest_timing(self.h, _p(t, f64p))
        return t

    def step_timing(self):
        t = np.zeros(10)
        lib().kvc_last_step_timing(self.h, _p(t, f64p))
        return t


# ----------------------------------------------------------------------------- device self-checks
def debug_div_check(n: int, seed: int = 1, max_den: int = 1 << 20) -> int:
    """Mismatches of the resolve chains' reciprocal division against __ddiv_rn (device)."""
    m = C.c_uint64()
    _check(lib().kvc_debug_div_check(n, seed, max_den, C.byref(m)))
    return int(m.value)


# ----------------------------------------------------------------------------- host slow path
def host_split_two(pts: np.ndarray, seed: int):
    """split_two (clustering.cpp:180-208) as run by the split slow path: (assign, degenerate)."""
    p = np.ascontiguousarray(pts, np.float32)
    n, d = p.shape
    a = np.zeros(n, np.int32)
    deg = C.c_int32()
    _check(lib().kvc_host_split_two(_p(p, f32p), n, d, seed, _p(a, i32p), C.byref(deg)))
    return a, bool(deg.value)


def host_kmeans(pts: np.ndarray, k: int, max_iters: int = 50, tol: float = 1e-6, seed: int = 0):
    """spherical_kmeans (clustering.cpp:80-178): (assign, k_live, objective, iterations)."""
    p = np.ascontiguousarray(pts, np.float32)
    n, d = p.shape
    a = np.zeros(n, np.int32)
    obj = C.c_double()
    it = C.c_int32()
    live = _check(lib().kvc_host_kmeans(_p(p, f32p), n, d, k, max_iters, tol, seed, _p(a, i32p),
                                        C.byref(obj), C.byref(it)))
    return a, live, obj.value, it.value


def ipc_alloc(nbytes: int):
    """cudaMalloc + cudaIpcGetMemHandle: (device pointer, 64-byte handle)."""
    ptr = C.c_void_p()
    h = (C.c_uint8 * 64)()
    _check(lib().kvc_ipc_alloc(nbytes, C.byref(ptr), h))
    return ptr.value, bytes(h)


def ipc_open(handle: bytes) -> int:
    ptr = C.c_void_p()
    hb = (C.c_uint8 * 64).from_buffer_copy(handle)
    _check(lib().kvc_ipc_open(hb, C.byref(ptr)))
    return ptr.value
