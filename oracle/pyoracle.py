"""ctypes front-end to the parity checker -- TEST INFRASTRUCTURE ONLY.

Loads
  * oracle/_ref/kvc_oracle.so     -- our plain-C restatement (kvc_oracle.c), always buildable;
  * oracle/_ref/libkvclust_ref.so -- the unmodified reference library + ref_shim.cpp driver
                                     (present when oracle/Makefile ran where /root/reference
                                     exists; the prebuilt .so travels with the repo snapshot).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module. The product (paper_2604_10060_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field, fields

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

f32p = C.POINTER(C.c_float)
f64p = C.POINTER(C.c_double)
i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
u64p = C.POINTER(C.c_uint64)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def build():
    """Compile the checker (restatement always; reference when /root/reference exists)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "-j8"], check=True)


_restate = None
_ref = None


def restatement():
    global _restate
    if _restate is None:
        path = os.path.join(REF_DIR, "kvc_oracle.so")
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.kvo_gen_stream.argtypes = [C.c_void_p, i32p, f32p, f32p, f32p, f32p, i64p, i32p]
        lib.kvo_cosine_fd.restype = C.c_double
        lib.kvo_cosine_fd.argtypes = [f32p, f64p, C.c_int, C.POINTER(C.c_int)]
        lib.kvo_tau.restype = C.c_double
        lib.kvo_tau.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double]
        lib.kvo_updated_stats.argtypes = [f64p, C.c_double, C.c_int64, f32p, C.c_int, f64p, f64p]
        lib.kvo_mix_seed.restype = C.c_uint64
        lib.kvo_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.kvo_rng_init.argtypes = [C.c_void_p, C.c_uint64]
        lib.kvo_rng_u64.restype = C.c_uint64
        lib.kvo_rng_u64.argtypes = [C.c_void_p]
        lib.kvo_rng_uniform.restype = C.c_double
        lib.kvo_rng_uniform.argtypes = [C.c_void_p]
        lib.kvo_rng_gaussian.restype = C.c_double
        lib.kvo_rng_gaussian.argtypes = [C.c_void_p]
        lib.kvo_rank.restype = C.c_int
        lib.kvo_rank.argtypes = [f64p, i64p, C.c_int, C.c_int, i32p]
        lib.kvo_attend_f32.argtypes = [f32p, f32p, f32p, C.c_int, C.c_int, C.c_double, f64p]
        lib.kvo_token_rank.restype = C.c_int
        lib.kvo_token_rank.argtypes = [f32p, f32p, i64p, i32p, C.c_int, C.c_int, C.c_int, i32p]
        _restate = lib
    return _restate


def reference():
    """The compiled reference (oracle/_ref/libkvclust_ref.so) or None when absent."""
    global _ref
    if _ref is None:
        path = os.path.join(REF_DIR, "libkvclust_ref.so")
        if not os.path.exists(path):
            return None
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        vp = C.c_void_p
        lib.ref_stream_gen.argtypes = [vp, C.POINTER(vp)]
        lib.ref_stream_free.argtypes = [vp]
        lib.ref_stream_n_events.argtypes = [vp]
        lib.ref_stream_kind.argtypes = [vp, C.c_int]
        lib.ref_stream_frame.argtypes = [vp, C.c_int, i64p, f32p, f32p, f32p]
        lib.ref_stream_query.argtypes = [vp, C.c_int, i64p, f32p, i64p, C.c_int]
        lib.ref_drv_create.argtypes = [vp, C.c_int, C.c_int, C.POINTER(vp)]
        lib.ref_drv_free.argtypes = [vp]
        lib.ref_drv_set_checks.argtypes = [vp, C.c_int]
        lib.ref_drv_frame.argtypes = [vp, C.c_int64, f32p, f32p, f32p, C.c_int, i64p, i64p]
        lib.ref_drv_build_now.argtypes = [vp]
        lib.ref_drv_bulk_load.argtypes = [vp, f32p, f32p, f32p, C.c_int, C.c_int, i32p, i64p, i32p, i64p]
        lib.ref_drv_query.argtypes = [vp, C.c_int64, f32p, i64p, C.c_int]
        lib.ref_drv_q_ranked.argtypes = [vp, C.c_int, i64p, i32p, C.c_int]
        lib.ref_drv_q_selected.argtypes = [vp, C.c_int, i64p, C.c_int]
        lib.ref_drv_q_attended.argtypes = [vp, C.c_int, i64p, i32p, C.c_int]
        lib.ref_drv_q_layer_meta.argtypes = [vp, C.c_int, f64p, i64p]
        lib.ref_drv_q_meta.argtypes = [vp, f64p]
        lib.ref_drv_q_digest.restype = C.c_uint64
        lib.ref_drv_q_digest.argtypes = [vp]
        lib.ref_drv_maint_stats.argtypes = [vp, i64p]
        lib.ref_drv_ledger.restype = C.c_int64
        lib.ref_drv_ledger.argtypes = [vp, i64p, i64p, f64p]
        lib.ref_drv_ledger_log_size.argtypes = [vp]
        lib.ref_drv_ledger_op.argtypes = [vp, C.c_int, i64p]
        lib.ref_drv_n_partitions.argtypes = [vp]
        lib.ref_drv_partition.argtypes = [vp, C.c_int, f64p, i64p, C.c_int]
        lib.ref_drv_n_clusters.argtypes = [vp]
        lib.ref_drv_cluster_ids.argtypes = [vp, i64p, C.c_int]
        lib.ref_drv_cluster.argtypes = [vp, C.c_int64, i64p, f64p, f64p, f64p]
        lib.ref_drv_cluster_entries.argtypes = [vp, C.c_int64, C.c_int, i64p, i32p, C.c_int]
        lib.ref_drv_partition_layer.argtypes = [vp, C.c_int, C.c_int, i64p, C.c_int]
        lib.ref_drv_flat_topk.argtypes = [vp, f32p, C.c_int, C.c_int, i64p, i32p]
        lib.ref_eng_create.argtypes = [vp, C.c_int, C.c_int, C.POINTER(vp)]
        lib.ref_eng_free.argtypes = [vp]
        lib.ref_eng_frame.argtypes = [vp, C.c_int64, f32p, f32p, f32p, C.c_int]
        lib.ref_eng_query.argtypes = [vp, C.c_int64, f32p, i64p, C.c_int]
        lib.ref_eng_finish.argtypes = [vp]
        lib.ref_eng_n_rows.argtypes = [vp]
        lib.ref_eng_row.restype = C.c_uint64
        lib.ref_eng_row.argtypes = [vp, C.c_int, i64p, f64p]
        lib.ref_eng_maint_stats.argtypes = [vp, i64p]
        lib.ref_prim_cosine_fd.restype = C.c_double
        lib.ref_prim_cosine_fd.argtypes = [f32p, f64p, C.c_int]
        lib.ref_prim_dot_fd.restype = C.c_double
        lib.ref_prim_dot_fd.argtypes = [f32p, f64p, C.c_int]
        lib.ref_prim_norm_d.restype = C.c_double
        lib.ref_prim_norm_d.argtypes = [f64p, C.c_int]
        lib.ref_prim_tau.restype = C.c_double
        lib.ref_prim_tau.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_double]
        lib.ref_prim_updated_stats.argtypes = [f64p, C.c_double, C.c_int64, f32p, C.c_int, f64p, f64p]
        lib.ref_prim_mix_seed.restype = C.c_uint64
        lib.ref_prim_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.ref_prim_rng.argtypes = [C.c_uint64, C.c_int, u64p, f64p, f64p]
        lib.ref_prim_split_two.argtypes = [f32p, C.c_int, C.c_int, C.c_uint64, i32p]
        lib.ref_prim_kmeans.argtypes = [f32p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
                                        C.c_uint64, i32p, f64p, C.POINTER(C.c_int)]
        lib.ref_time_decode.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, f32p, f32p, i32p, f32p,
                                        C.c_int, C.c_int, C.c_int, f64p]
        lib.ref_time_mt.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, f32p, f32p,
                                    i32p, f32p, C.c_int, C.c_int, C.c_int, C.c_int, f32p, f32p,
                                    f32p, C.c_int, f64p]
        _ref = lib
    return _ref


# --------------------------------------------------------------------------- configs

class _Struct(C.Structure):
    def asdict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class StreamCfg(_Struct):
    """workload.hpp:16-39 StreamConfig."""

    _fields_ = [
        ("n_scenes", C.c_int), ("frames_per_scene", C.c_int), ("tokens_per_frame", C.c_int),
        ("d", C.c_int), ("L", C.c_int),
        ("visual_noise", C.c_double), ("semantic_noise", C.c_double), ("drift_rate", C.c_double),
        ("cross_layer_eps", C.c_double), ("n_queries", C.c_int), ("cross_modal_mix", C.c_double),
        ("gt_top_m", C.c_int), ("scene_cycle", C.c_int), ("queries_at_end", C.c_int),
        ("seed", C.c_uint64),
    ]

    @classmethod
    def make(cls, **kw):
        # reference defaults (workload.hpp:16-39)
        base = dict(n_scenes=6, frames_per_scene=32, tokens_per_frame=4, d=32, L=4,
                    visual_noise=0.05, semantic_noise=0.1, drift_rate=0.01, cross_layer_eps=0.02,
                    n_queries=24, cross_modal_mix=0.6, gt_top_m=16, scene_cycle=0,
                    queries_at_end=0, seed=42)
        base.update(kw)
        return cls(**base)


def config1_stream(**kw) -> StreamCfg:
    """BASELINE.md §3 / SURVEY.md §8(d) config 1."""
    base = dict(n_scenes=4, frames_per_scene=16, tokens_per_frame=196, d=128, L=8, n_queries=32,
                queries_at_end=1, semantic_noise=0.02, seed=42)
    base.update(kw)
    return StreamCfg.make(**base)


class EngineCfg(_Struct):
    """engine.hpp:21-33 EngineConfig, flattened (same layout as kvc.h's kvc_engine_cfg)."""

    _fields_ = [
        ("k_v", C.c_int), ("k_s", C.c_int), ("window_frames", C.c_int), ("prefetch_k", C.c_int),
        ("prefetch_enabled", C.c_int), ("token_mode", C.c_int), ("token_budget", C.c_int64),
        ("lookup_cost_per_candidate_us", C.c_double), ("compute_cost_per_token_us", C.c_double),
        ("tau_min", C.c_double), ("tau_max", C.c_double), ("n0", C.c_double),
        ("defer_host_splits", C.c_int), ("max_split_depth", C.c_int), ("visual_floor", C.c_double),
        ("target_visual_cluster_size", C.c_int), ("target_semantic_cluster_size", C.c_int),
        ("kmeans_max_iters", C.c_int), ("kmeans_tol", C.c_double),
        ("alpha_us", C.c_double), ("beta_us_per_byte", C.c_double),
        ("bytes_per_entry", C.c_int64), ("device_capacity_entries", C.c_int64),
        ("build_batch_frames", C.c_int), ("batched_ingest", C.c_int),
        ("ingest_overhead_us", C.c_double), ("offload_horizon_frames", C.c_int),
        ("seed", C.c_uint64),
    ]

    @classmethod
    def make(cls, **kw):
        base = dict(k_v=4, k_s=4, window_frames=4, prefetch_k=4, prefetch_enabled=0, token_mode=0,
                    token_budget=256, lookup_cost_per_candidate_us=0.02,
                    compute_cost_per_token_us=0.6, tau_min=0.05, tau_max=0.3, n0=32.0,
                    defer_host_splits=1, max_split_depth=4, visual_floor=0.75,
                    target_visual_cluster_size=8, target_semantic_cluster_size=32,
                    kmeans_max_iters=50, kmeans_tol=1e-6, alpha_us=10.0, beta_us_per_byte=0.001,
                    bytes_per_entry=0, device_capacity_entries=1 << 20, build_batch_frames=32,
                    batched_ingest=0, ingest_overhead_us=10.0, offload_horizon_frames=16, seed=0)
        base.update(kw)
        return cls(**base)


def config1_engine(**kw) -> EngineCfg:
    """BASELINE.md §3 config-1 engine: 16 clusters/layer at build, top-4."""
    base = dict(build_batch_frames=16, target_visual_cluster_size=16,
                target_semantic_cluster_size=196, k_v=1, k_s=4, window_frames=4, seed=0)
    base.update(kw)
    return EngineCfg.make(**base)


# --------------------------------------------------------------------------- streams

@dataclass
class Stream:
    """A generated stream as flat arrays (event order preserved in `kinds`)."""

    d: int
    L: int
    T: int
    kinds: np.ndarray          # [E] 0 frame / 1 query
    visual: np.ndarray         # [F, d] f32
    keys: np.ndarray           # [F, L, T, d] f32
    values: np.ndarray         # [F, L, T, d] f32
    q: np.ndarray              # [Q, L, d] f32
    gt: list = field(default_factory=list)   # per query: sorted frame ids

    def events(self):
        """Yields ('frame', idx) / ('query', idx) in stream order."""
        fi = qi = 0
        for k in self.kinds:
            if k == 0:
                yield "frame", fi
                fi += 1
            else:
                yield "query", qi
                qi += 1


def gen_stream_restated(cfg: StreamCfg) -> Stream:
    lib = restatement()
    F = cfg.n_scenes * cfg.frames_per_scene
    Q = cfg.n_queries
    d, L, T = cfg.d, cfg.L, cfg.tokens_per_frame
    kinds = np.zeros(F + Q, np.int32)
    visual = np.zeros((F, d), np.float32)
    keys = np.zeros((F, L, T, d), np.float32)
    values = np.zeros((F, L, T, d), np.float32)
    q = np.zeros((max(Q, 1), L, d), np.float32)
    gt = np.zeros((max(Q, 1), cfg.gt_top_m), np.int64)
    ngt = np.zeros(max(Q, 1), np.int32)
    rc = lib.kvo_gen_stream(C.byref(cfg), _p(kinds, i32p), _p(visual, f32p), _p(keys, f32p),
                            _p(values, f32p), _p(q, f32p), _p(gt, i64p), _p(ngt, i32p))
    if rc != 0:
        raise ValueError(f"kvo_gen_stream failed: {rc}")
    return Stream(d, L, T, kinds, visual, keys, values, q[:Q],
                  [gt[i, : ngt[i]].copy() for i in range(Q)])


def gen_stream_reference(cfg: StreamCfg) -> Stream:
    lib = reference()
    assert lib is not None, "oracle/_ref/libkvclust_ref.so not built"
    h = C.c_void_p()
    rc = lib.ref_stream_gen(C.byref(cfg), C.byref(h))
    if rc != 0:
        raise ValueError(lib.ref_last_error().decode())
    try:
        n = lib.ref_stream_n_events(h)
        d, L, T = cfg.d, cfg.L, cfg.tokens_per_frame
        kinds = np.array([lib.ref_stream_kind(h, i) for i in range(n)], np.int32)
        F = int((kinds == 0).sum())
        Q = n - F
        visual = np.zeros((F, d), np.float32)
        keys = np.zeros((F, L, T, d), np.float32)
        values = np.zeros((F, L, T, d), np.float32)
        q = np.zeros((Q, L, d), np.float32)
        gts = []
        fi = qi = 0
        fid = C.c_int64()
        gtbuf = np.zeros(max(cfg.gt_top_m, 1), np.int64)
        for i in range(n):
            if kinds[i] == 0:
                lib.ref_stream_frame(h, i, C.byref(fid), _p(visual[fi], f32p), _p(keys[fi], f32p),
                                     _p(values[fi], f32p))
                fi += 1
            else:
                m = lib.ref_stream_query(h, i, C.byref(fid), _p(q[qi], f32p), _p(gtbuf, i64p),
                                         len(gtbuf))
                gts.append(gtbuf[:m].copy())
                qi += 1
        return Stream(d, L, T, kinds, visual, keys, values, q, gts)
    finally:
        lib.ref_stream_free(h)


# --------------------------------------------------------------------------- driver

class RefDriver:
    """StreamEngine-faithful driver over the compiled reference (ref_shim.cpp)."""

    def __init__(self, ecfg: EngineCfg, d: int, L: int, checks: bool = True):
        self.lib = reference()
        assert self.lib is not None
        self.h = C.c_void_p()
        self.d, self.L = d, L
        self.ecfg = ecfg
        rc = self.lib.ref_drv_create(C.byref(ecfg), d, L, C.byref(self.h))
        if rc != 0:
            raise ValueError(self.lib.ref_last_error().decode())
        self.lib.ref_drv_set_checks(self.h, 1 if checks else 0)

    def close(self):
        if self.h:
            self.lib.ref_drv_free(self.h)
            self.h = C.c_void_p()

    __del__ = close

    def _chk(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.lib.ref_last_error().decode()}")

    def frame(self, frame_id, visual, keys, values):
        """keys/values [L, T, d]; returns (pid, assigned[L, T])."""
        T = keys.shape[1]
        out = np.full(self.L * T, -1, np.int64)
        pid = C.c_int64(-1)
        self._chk(self.lib.ref_drv_frame(self.h, frame_id, _p(np.ascontiguousarray(visual), f32p),
                                         _p(np.ascontiguousarray(keys), f32p),
                                         _p(np.ascontiguousarray(values), f32p), T,
                                         _p(out, i64p), C.byref(pid)))
        return pid.value, out.reshape(self.L, T)

    def build_now(self):
        self._chk(self.lib.ref_drv_build_now(self.h))

    def bulk_load(self, visual, keys, values, assign, frame_ids, token_ids, n_clusters):
        """The checker side of kvc_bulk_load (ref_shim.cpp ref_drv_bulk_load): keys/values
        [L, N, d] f32, assign [L, N]; returns the partition id."""
        k = np.ascontiguousarray(keys, np.float32)
        v = np.ascontiguousarray(values, np.float32)
        a = np.ascontiguousarray(assign, np.int32)
        fr = np.ascontiguousarray(frame_ids, np.int64)
        tk = np.ascontiguousarray(token_ids, np.int32)
        pid = C.c_int64(-1)
        self._chk(self.lib.ref_drv_bulk_load(self.h, _p(np.ascontiguousarray(visual, np.float32), f32p),
                                             _p(k, f32p), _p(v, f32p), k.shape[1], n_clusters, _p(a, i32p),
                                             _p(fr, i64p), _p(tk, i32p), C.byref(pid)))
        return pid.value

    def query(self, qid, q, gt=None):
        gt = np.zeros(0, np.int64) if gt is None else np.ascontiguousarray(gt, np.int64)
        self._chk(self.lib.ref_drv_query(self.h, qid, _p(np.ascontiguousarray(q), f32p),
                                         _p(gt, i64p), len(gt)))

    def ranked(self, l, cap=4096):
        ids = np.zeros(cap, np.int64)
        buf = np.zeros(cap, np.int32)
        n = self.lib.ref_drv_q_ranked(self.h, l, _p(ids, i64p), _p(buf, i32p), cap)
        return [(int(ids[i]), int(buf[i])) for i in range(n)]

    def selected(self, l, cap=1 << 16):
        ids = np.zeros(cap, np.int64)
        n = self.lib.ref_drv_q_selected(self.h, l, _p(ids, i64p), cap)
        return ids[:n].tolist()

    def attended(self, l, cap=1 << 20):
        fr = np.zeros(cap, np.int64)
        tk = np.zeros(cap, np.int32)
        n = self.lib.ref_drv_q_attended(self.h, l, _p(fr, i64p), _p(tk, i32p), cap)
        return fr[:n].copy(), tk[:n].copy()

    def layer_meta(self, l):
        lat = np.zeros(5)
        ints = np.zeros(4, np.int64)
        self.lib.ref_drv_q_layer_meta(self.h, l, _p(lat, f64p), _p(ints, i64p))
        return lat, ints

    def query_meta(self):
        dd = np.zeros(2)
        self.lib.ref_drv_q_meta(self.h, _p(dd, f64p))
        return float(dd[0]), float(dd[1])

    def digest(self):
        return int(self.lib.ref_drv_q_digest(self.h))

    def maint_stats(self):
        o = np.zeros(9, np.int64)
        self.lib.ref_drv_maint_stats(self.h, _p(o, i64p))
        return o

    def ledger(self):
        ops = np.zeros(5, np.int64)
        by = np.zeros(5, np.int64)
        co = np.zeros(5)
        dev = self.lib.ref_drv_ledger(self.h, _p(ops, i64p), _p(by, i64p), _p(co, f64p))
        return ops, by, co, int(dev)

    def ledger_log(self):
        n = self.lib.ref_drv_ledger_log_size(self.h)
        out = np.zeros((n, 4), np.int64)
        for i in range(n):
            self.lib.ref_drv_ledger_op(self.h, i, _p(out[i], i64p))
        return out

    def n_partitions(self):
        return self.lib.ref_drv_n_partitions(self.h)

    def partition(self, p, cap=1 << 16):
        rep = np.zeros(self.d)
        fr = np.zeros(cap, np.int64)
        n = self.lib.ref_drv_partition(self.h, p, _p(rep, f64p), _p(fr, i64p), cap)
        return rep, fr[:n].copy()

    def partition_layer(self, p, layer, cap=1 << 16):
        ids = np.zeros(cap, np.int64)
        n = self.lib.ref_drv_partition_layer(self.h, p, layer, _p(ids, i64p), cap)
        return ids[:n].tolist()

    def cluster_ids(self):
        n = self.lib.ref_drv_n_clusters(self.h)
        ids = np.zeros(max(n, 1), np.int64)
        self.lib.ref_drv_cluster_ids(self.h, _p(ids, i64p), n)
        return ids[:n].tolist()

    def cluster(self, cid):
        info = np.zeros(10, np.int64)
        var = C.c_double()
        rep = np.zeros(self.d)
        brep = np.zeros(self.d)
        self._chk(self.lib.ref_drv_cluster(self.h, cid, _p(info, i64p), C.byref(var), _p(rep, f64p),
                                           _p(brep, f64p)))
        return info, var.value, rep, brep

    def cluster_entries(self, cid, which=0, cap=1 << 20):
        fr = np.zeros(cap, np.int64)
        tk = np.zeros(cap, np.int32)
        n = self.lib.ref_drv_cluster_entries(self.h, cid, which, _p(fr, i64p), _p(tk, i32p), cap)
        return fr[:n].copy(), tk[:n].copy()

    def flat_topk(self, q, layer, k):
        ids = np.zeros(max(k, 1), np.int64)
        buf = np.zeros(max(k, 1), np.int32)
        n = self.lib.ref_drv_flat_topk(self.h, _p(np.ascontiguousarray(q, np.float32), f32p),
                                       layer, k, _p(ids, i64p), _p(buf, i32p))
        if n < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return [(int(ids[i]), int(buf[i])) for i in range(n)]


def attended_digest(per_layer):
    """FNV-1a digest of attended (frame, token) lists per layer (engine.cpp:18-35)."""
    h = 1469598103934665603
    M = (1 << 64) - 1

    def fnv(h, x):
        x &= M
        for i in range(8):
            h ^= (x >> (8 * i)) & 0xFF
            h = (h * 1099511628211) & M
        return h

    for l, (frames, tokens) in enumerate(per_layer):
        for f, t in zip(frames.tolist(), tokens.tolist()):
            h = fnv(h, l)
            h = fnv(h, f)
            h = fnv(h, t)
    return h


def time_reference(mode: int, threads: int, keys: np.ndarray, values: np.ndarray, assign: np.ndarray,
                   C_: int, warmup: int, steps: int, k_s: int = 16, window_tokens: int = 784,
                   queries: np.ndarray | None = None, fvis=None, fkeys=None, fvals=None):
    """CPU timing of the reference hot path (ref_shim.cpp ref_time_mt). keys/values [L, N, d] f32.
    Returns (max-over-threads us/step, mean us/step)."""
    lib = reference()
    assert lib is not None
    L, N, d = keys.shape
    k = np.ascontiguousarray(keys, np.float32)
    v = np.ascontiguousarray(values, np.float32)
    a = np.ascontiguousarray(assign, np.int32)
    q = np.ascontiguousarray(queries if queries is not None else np.zeros((warmup + steps, L, d)), np.float32)
    T = 0 if fkeys is None else fkeys.shape[2]
    fv_ = np.ascontiguousarray(fvis, np.float32) if fvis is not None else None
    fk = np.ascontiguousarray(fkeys if fkeys is not None else np.zeros((1, d)), np.float32)
    fvv = np.ascontiguousarray(fvals if fvals is not None else np.zeros((1, d)), np.float32)
    out = np.zeros(2)
    rc = lib.ref_time_mt(mode, threads, d, L, N, C_, _p(k, f32p), _p(v, f32p), _p(a, i32p), _p(q, f32p),
                         warmup, steps, k_s, window_tokens, _p(fv_, f32p) if fv_ is not None else None, _p(fk, f32p), _p(fvv, f32p), T,
                         _p(out, f64p))
    if rc != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return float(out[0]), float(out[1])
