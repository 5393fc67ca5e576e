"""CPU tests of the checker itself (no GPU): the C restatement (oracle/kvc_oracle.c) is pinned
bit-for-bit against the compiled reference (oracle/_ref) and against the reference tests' known
answers (tests/golden/kats.json); the shim driver is pinned against the real StreamEngine."""
import ctypes as C
import json
import math
import os

import numpy as np
import pytest

from oracle import pyoracle as po

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def kats():
    with open(os.path.join(GOLDEN, "kats.json")) as f:
        return json.load(f)


# ------------------------------------------------------------------ known answers (no reference needed)

def test_tau_kats():
    """maintainer.cpp:11-14; test_maintainer.cpp:64-81."""
    lib = po.restatement()
    k = kats()["tau"]
    assert lib.kvo_tau(0, 0.05, 0.3, 32.0) == 0.3
    prev = lib.kvo_tau(0, 0.05, 0.3, 32.0)
    for n in range(1, 1000):  # strictly decreasing over the operating range
        cur = lib.kvo_tau(n, 0.05, 0.3, 32.0)
        assert cur < prev and 0.05 <= cur <= 0.3
        prev = cur
    assert abs(lib.kvo_tau(16, 0.1, 0.5, 16.0) - k["tau16_named"]) < 1e-4
    assert abs(lib.kvo_tau(16, 0.1, 0.5, 16.0) - (0.1 + 0.4 * math.exp(-1.0))) < 1e-12


def test_updated_stats_hand_example():
    """Eq. 3/4 hand example (test_maintainer.cpp:83-94)."""
    lib = po.restatement()
    k = kats()["updated_stats"]
    rep = np.array(k["rep"], np.float64)
    key = np.array(k["key"], np.float32)
    out = np.zeros(2)
    var = C.c_double()
    lib.kvo_updated_stats(po._p(rep, po.f64p), k["var"], k["n"], po._p(key, po.f32p), 2, po._p(out, po.f64p),
                          C.byref(var))
    assert np.allclose(out, k["rep_out"]) and abs(var.value - k["var_out"]) < 1e-15


def test_updated_stats_long_replay_exact():
    """500-insert recursion replays bit-for-bit against a literal restatement in numpy order
    (test_maintainer.cpp:116-134 style)."""
    lib = po.restatement()
    rng = np.random.default_rng(62)
    d = 8
    first = rng.standard_normal(d).astype(np.float32)
    r = first.astype(np.float64)
    var = 0.0
    rr, vv = r.copy(), 0.0
    for i in range(1, 500):
        k = rng.standard_normal(d).astype(np.float32)
        out = np.zeros(d)
        v = C.c_double()
        lib.kvo_updated_stats(po._p(np.ascontiguousarray(r), po.f64p), var, i, po._p(k, po.f32p), d,
                              po._p(out, po.f64p), C.byref(v))
        r, var = out, v.value
        dn = float(i)
        rr = np.array([(dn * rr[j] + float(k[j])) / (dn + 1.0) for j in range(d)])
        sq = 0.0
        for j in range(d):
            diff = float(k[j]) - rr[j]
            sq += diff * diff
        vv = (dn * vv + sq) / (dn + 1.0)
        assert np.array_equal(r, rr) and var == vv


def test_mix_seed_and_rng_kats():
    lib = po.restatement()
    k = kats()
    for (a, b, z) in k["mix_seed"]:
        assert lib.kvo_mix_seed(a, b) == z
    st = (C.c_uint8 * 4096)()
    lib.kvo_rng_init(st, 5489)
    assert lib.kvo_rng_u64(st) == k["mt19937_64_first_5489"]
    for _ in range(9998):
        lib.kvo_rng_u64(st)
    assert lib.kvo_rng_u64(st) == k["mt19937_64_10000th_default"]  # the C++ standard's check value


def test_attention_restatement_matches_numpy():
    lib = po.restatement()
    rng = np.random.default_rng(3)
    n, d = 37, 16
    q = rng.standard_normal(d).astype(np.float32)
    K = rng.standard_normal((n, d)).astype(np.float32)
    V = rng.standard_normal((n, d)).astype(np.float32)
    out = np.zeros(d)
    lib.kvo_attend_f32(po._p(q, po.f32p), po._p(K, po.f32p), po._p(V, po.f32p), n, d, 0.25, po._p(out, po.f64p))
    s = (K.astype(np.float64) @ q.astype(np.float64)) * 0.25
    p = np.exp(s - s.max())
    ref = (p[:, None] * V.astype(np.float64)).sum(0) / p.sum()
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-12)


def test_stream_hash_pinned():
    """The restated generator reproduces the config-1 stream the golden fixtures were made from."""
    s = po.gen_stream_restated(po.config1_stream())
    g = kats()["config1_stream_sha256"]
    import hashlib

    h = hashlib.sha256()
    for a in (s.visual, s.keys, s.values, s.q):
        h.update(np.ascontiguousarray(a).tobytes())
    assert h.hexdigest() == g


# ------------------------------------------------------------------ against the compiled reference

def test_gen_stream_bit_exact_vs_reference(ref_lib):
    for cfg in (po.StreamCfg.make(), po.StreamCfg.make(scene_cycle=2, n_scenes=5, queries_at_end=1, seed=7),
                po.StreamCfg.make(n_scenes=2, frames_per_scene=3, tokens_per_frame=9, d=24, L=3, seed=99)):
        a, b = po.gen_stream_restated(cfg), po.gen_stream_reference(cfg)
        for name in ("kinds", "visual", "keys", "values", "q"):
            assert np.array_equal(getattr(a, name), getattr(b, name)), name
        assert all(np.array_equal(x, y) for x, y in zip(a.gt, b.gt))


def test_primitives_bit_exact_vs_reference(ref_lib):
    lib = po.restatement()
    rng = np.random.default_rng(11)
    for _ in range(200):
        d = int(rng.integers(2, 130))
        a = rng.standard_normal(d).astype(np.float32)
        b = rng.standard_normal(d)
        err = C.c_int()
        assert lib.kvo_cosine_fd(po._p(a, po.f32p), po._p(b, po.f64p), d, C.byref(err)) == \
            ref_lib.ref_prim_cosine_fd(po._p(a, po.f32p), po._p(b, po.f64p), d)
        n = int(rng.integers(0, 5000))
        assert lib.kvo_tau(n, 0.05, 0.3, 32.0) == ref_lib.ref_prim_tau(n, 0.05, 0.3, 32.0)
        r1, r2 = np.zeros(d), np.zeros(d)
        v1, v2 = C.c_double(), C.c_double()
        lib.kvo_updated_stats(po._p(b, po.f64p), 0.125, n, po._p(a, po.f32p), d, po._p(r1, po.f64p), C.byref(v1))
        ref_lib.ref_prim_updated_stats(po._p(b, po.f64p), 0.125, n, po._p(a, po.f32p), d, po._p(r2, po.f64p),
                                       C.byref(v2))
        assert np.array_equal(r1, r2) and v1.value == v2.value
    u64 = np.zeros(64, np.uint64)
    uni = np.zeros(64)
    gau = np.zeros(64)
    ref_lib.ref_prim_rng(2024, 64, u64.ctypes.data_as(po.u64p), po._p(uni, po.f64p), po._p(gau, po.f64p))
    st = (C.c_uint8 * 4096)()
    lib.kvo_rng_init(st, 2024)
    assert [lib.kvo_rng_u64(st) for _ in range(64)] == u64.tolist()
    lib.kvo_rng_init(st, 2024)
    assert [lib.kvo_rng_gaussian(st) for _ in range(64)] == gau.tolist()


def test_driver_matches_stream_engine(ref_lib):
    """ref_shim's StreamEngine-following driver == the real StreamEngine (attended digests)."""
    s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=3, frames_per_scene=10, tokens_per_frame=12, d=24, L=3,
                                                 n_queries=9, semantic_noise=0.05, seed=17))
    ecfg = po.EngineCfg.make(build_batch_frames=6, offload_horizon_frames=3, device_capacity_entries=300,
                             prefetch_enabled=1)
    drv = po.RefDriver(ecfg, s.d, s.L)
    eng = C.c_void_p()
    assert ref_lib.ref_eng_create(C.byref(ecfg), s.d, s.L, C.byref(eng)) == 0
    digs = []
    for kind, i in s.events():
        if kind == "frame":
            drv.frame(i, s.visual[i], s.keys[i], s.values[i])
            ref_lib.ref_eng_frame(eng, i, po._p(s.visual[i], po.f32p), po._p(s.keys[i], po.f32p),
                                  po._p(s.values[i], po.f32p), s.T)
        else:
            drv.query(i, s.q[i], s.gt[i])
            digs.append(drv.digest())
            ref_lib.ref_eng_query(eng, i, po._p(s.q[i], po.f32p), po._p(s.gt[i], po.i64p), len(s.gt[i]))
    ref_lib.ref_eng_finish(eng)
    ints = np.zeros(4, np.int64)
    dd = np.zeros(2)
    rows = [ref_lib.ref_eng_row(eng, i, po._p(ints, po.i64p), po._p(dd, po.f64p)) for i in range(ref_lib.ref_eng_n_rows(eng))]
    st = np.zeros(9, np.int64)
    ref_lib.ref_eng_maint_stats(eng, po._p(st, po.i64p))
    ref_lib.ref_eng_free(eng)
    assert rows == digs
    assert np.array_equal(st, drv.maint_stats())


def test_golden_config1_matches_reference(ref_lib):
    """The committed fixture equals what the reference produces now (fixture freshness)."""
    path = os.path.join(GOLDEN, "config1_expect.json")
    with open(path) as f:
        g = json.load(f)
    s = po.gen_stream_restated(po.config1_stream())
    drv = po.RefDriver(po.config1_engine(), s.d, s.L, checks=False)
    qi = 0
    for kind, i in s.events():
        if kind == "frame":
            drv.frame(i, s.visual[i], s.keys[i], s.values[i])
        else:
            drv.query(i, s.q[i], s.gt[i])
            assert drv.digest() == int(g["queries"][qi]["digest"])
            assert [drv.selected(l) for l in range(s.L)] == g["queries"][qi]["selected"]
            qi += 1
    assert drv.maint_stats().tolist() == g["maint_stats"]
