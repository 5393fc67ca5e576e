"""Edge cases the fast paths must not fail on:

* K4 v3's boundary set S (clusters whose fp32-mirror score is within the error margin of the
  top-k_s boundary) holds 256 entries in shared memory; a near-tie-heavy query (many identical
  representatives) overflows it. The reference ranks any number of ties by id
  (index.cpp:210-240), so the kernel runs an exact chunked tournament instead of failing.
* The general scoring kernel (K4 v1 `k_score_select`) is the live path for d > 128 or page sizes
  that are not a multiple of 32; it is parity-tested here both by shape (d = 256) and forced
  (KVC_K4=v1) on the config-1 stream.
* A K6 shape whose shared-memory ring cannot fit (fp32, d = 256, 64-token pages) is rejected at
  construction with ConfigError; 32-token pages work.
* oracle_flat_topk over more candidates than shared memory holds uses global scratch.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.harness import Replay, product_config

pytestmark = pytest.mark.gpu


def _tie_state(n_clusters, n_tied, d=128, per=4, seed=3):
    """One domain: n_tied clusters whose members are all the same unit vector u (identical
    representatives -> exact score ties), the rest random directions."""
    rng = np.random.default_rng(seed)
    u = rng.standard_normal(d).astype(np.float32)
    u /= np.linalg.norm(u)
    N = n_clusters * per
    keys = np.empty((1, N, d), np.float32)
    for c in range(n_clusters):
        if c < n_tied:
            keys[0, c * per:(c + 1) * per] = u
        else:
            v = rng.standard_normal(d).astype(np.float32)
            keys[0, c * per:(c + 1) * per] = v / np.linalg.norm(v)
    vals = rng.standard_normal((1, N, d)).astype(np.float32)
    assign = np.repeat(np.arange(n_clusters, dtype=np.int32), per)[None, :]
    frames = (np.arange(N) // 196).astype(np.int64)
    tokens = (np.arange(N) % 196).astype(np.int32)
    return u, keys, vals, assign, frames, tokens


@pytest.mark.parametrize("n_clusters,n_tied", [(400, 400), (700, 300), (300, 20)])
def test_k4_boundary_overflow_is_exact(ref_lib, n_clusters, n_tied):
    from paper_2604_10060_b200 import ClusterKVCache

    u, keys, vals, assign, frames, tokens = _tie_state(n_clusters, n_tied)
    ecfg = po.EngineCfg.make(k_v=1, k_s=16, build_batch_frames=1, offload_horizon_frames=1 << 30,
                             device_capacity_entries=1 << 40)
    kv = ClusterKVCache(product_config(ecfg, max_candidates=1024), 128, 1)
    ref = po.RefDriver(ecfg, 128, 1, checks=False)
    vis = np.zeros(128, np.float32)
    vis[0] = 1
    kv.bulk_load(vis, keys, vals, assign, frames, tokens, n_clusters)
    ref.bulk_load(vis, keys, vals, assign, frames, tokens, n_clusters)
    rng = np.random.default_rng(1)
    for i in range(6):
        q = u + (0.0 if i == 0 else 0.01) * rng.standard_normal(128).astype(np.float32)
        q = (q / np.linalg.norm(q)).astype(np.float32)[None, :]
        kv.query(i, q)
        ref.query(i, q)
        assert kv.ranked(0) == ref.ranked(0), i
        assert kv.selected(0) == ref.selected(0), i
        assert kv.digest() == ref.digest(), i


def test_config1_forced_general_scoring_kernel(ref_lib, monkeypatch):
    """K4 v1 (`k_score_select`) on the whole config-1 stream, bit-exact with the reference."""
    monkeypatch.setenv("KVC_K4", "v1")
    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine()
    r = Replay(s, ecfg, po.RefDriver(ecfg, s.d, s.L, checks=False)).run()
    r.final_compare()
    assert r.mismatches == [], r.mismatches[:5]
    assert r.att_err < 1e-3


def test_wide_rows_d256_fp32(ref_lib):
    """d = 256 (K4 v1 by shape, K6 <256, f32>) on a drifting stream with 32-token pages."""
    from paper_2604_10060_b200 import ClusterKVCache
    from paper_2604_10060_b200.api import ConfigError

    s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=3, frames_per_scene=8, tokens_per_frame=24, d=256,
                                                 L=2, n_queries=8, semantic_noise=0.03, seed=11))
    ecfg = po.EngineCfg.make(build_batch_frames=6, k_v=2, k_s=4)
    with pytest.raises(ConfigError):
        ClusterKVCache(product_config(ecfg, page_tokens=64), s.d, s.L)
    r = Replay(s, ecfg, po.RefDriver(ecfg, s.d, s.L, checks=False), dev_kw=dict(page_tokens=32)).run()
    r.final_compare()
    assert r.mismatches == [], r.mismatches[:5]
    assert r.att_err < 1e-3


def test_flat_topk_beyond_shared_memory(ref_lib):
    """oracle_flat_topk (retrieval.cpp:145-164) over 16,000 candidates (> 227 KB of rank state)."""
    from paper_2604_10060_b200 import ClusterKVCache

    n = 16000
    _, keys, vals, assign, frames, tokens = _tie_state(n, 50, per=1, seed=9)
    ecfg = po.EngineCfg.make(build_batch_frames=1, offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40)
    kv = ClusterKVCache(product_config(ecfg, max_slots=20000), 128, 1)
    ref = po.RefDriver(ecfg, 128, 1, checks=False)
    vis = np.zeros(128, np.float32)
    vis[0] = 1
    kv.bulk_load(vis, keys, vals, assign, frames, tokens, n)
    ref.bulk_load(vis, keys, vals, assign, frames, tokens, n)
    rng = np.random.default_rng(4)
    for k in (1, 16, 100):
        q = rng.standard_normal(128).astype(np.float32)
        assert kv.flat_topk(q, 0, k) == ref.flat_topk(q, 0, k)
    q = keys[0, 0].copy()  # the tied direction: 50 exact ties broken by id
    assert kv.flat_topk(q, 0, 60) == ref.flat_topk(q, 0, 60)


@pytest.mark.parametrize("d", [8, 16, 48])
def test_head_widths_without_a_k6_instantiation(ref_lib, d):
    """d outside {32, 64, 128, 256} (the reference's own unit tests use d = 8 / 16): selection and
    bookkeeping bit-exact, attention through the generic kernel within 1e-3 of the fp64 oracle."""
    s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=3, frames_per_scene=8, tokens_per_frame=12, d=d,
                                                 L=3, n_queries=8, semantic_noise=0.05, seed=13))
    ecfg = po.EngineCfg.make(build_batch_frames=6, k_v=2, k_s=3)
    r = Replay(s, ecfg, po.RefDriver(ecfg, s.d, s.L, checks=False)).run()
    r.final_compare()
    assert r.mismatches == [], r.mismatches[:5]
    assert r.att_err < 1e-3
