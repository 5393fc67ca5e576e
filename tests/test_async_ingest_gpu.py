"""Pipelined ingest (a frame's host replay deferred until the next frame's kernels are in flight)
must leave exactly the state of the synchronous path: same clusters, statistics, ledger and
decode results, on streams with seeds, deferred / immediate splits, cadence offloads and capacity
evictions (which exercise the re-resolve of a token decided before the previous frame's cadence)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.harness import product_config

pytestmark = pytest.mark.gpu


def _state(kv):
    ids = kv.cluster_ids()
    rows = []
    for c in ids:
        info, var, rep, brep = kv.cluster(c)
        rows.append((c, info.tolist(), var, rep.tobytes(), brep.tobytes(), kv.cluster_entries(c)[0].tobytes()))
    return ids, kv.maint_stats().tolist(), [x.tolist() if hasattr(x, "tolist") else x for x in kv.ledger()], rows


@pytest.mark.parametrize("cfg", [
    dict(stream=dict(n_scenes=6, frames_per_scene=16, tokens_per_frame=16, d=32, L=4, scene_cycle=2, drift_rate=0.06,
                     semantic_noise=0.05, n_queries=12, queries_at_end=0, seed=7),
         engine=dict(build_batch_frames=8, offload_horizon_frames=2, prefetch_enabled=1, device_capacity_entries=900)),
    dict(stream=dict(n_scenes=4, frames_per_scene=12, tokens_per_frame=48, d=64, L=3, n_queries=8, queries_at_end=0,
                     semantic_noise=0.08, seed=19),
         engine=dict(build_batch_frames=6, offload_horizon_frames=3, device_capacity_entries=1200)),
])
def test_async_ingest_equals_sync(cfg):
    from paper_2604_10060_b200 import ClusterKVCache

    s = po.gen_stream_restated(po.StreamCfg.make(**cfg["stream"]))
    ecfg = po.EngineCfg.make(**cfg["engine"])
    kv_s = ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, s.L)
    kv_a = ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, s.L)
    outs_s, outs_a = [], []
    for kind, i in s.events():
        if kind == "frame":
            kv_s.process_frame(i, s.visual[i], s.keys[i], s.values[i], want_assigned=True)   # synchronous
            kv_a.process_frame(i, s.visual[i], s.keys[i], s.values[i], want_assigned=False)  # pipelined
        else:
            outs_s.append(kv_s.query(i, s.q[i]).copy())
            outs_a.append(kv_a.query(i, s.q[i]).copy())
    for a, b in zip(outs_s, outs_a):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-6)  # page layouts may differ (migration timing)
    st_s, st_a = _state(kv_s), _state(kv_a)
    assert st_s[0] == st_a[0]
    assert st_s[1] == st_a[1]
    assert st_s[2] == st_a[2]
    assert st_s[3] == st_a[3]
    st = kv_s.maint_stats()
    assert st[2] + st[3] > 0, "stream must exercise splits"


def test_async_ingest_gpu_splits_equal_sync_host_splits(monkeypatch):
    """Every split of >= 2 rows on the GPU (split.cu) in the pipelined, speculative path leaves the
    state of the synchronous path with host splits."""
    from paper_2604_10060_b200 import ClusterKVCache

    s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=4, frames_per_scene=12, tokens_per_frame=48, d=64, L=3,
                                                 n_queries=8, queries_at_end=0, semantic_noise=0.08, seed=23))
    ecfg = po.EngineCfg.make(build_batch_frames=6, offload_horizon_frames=3, device_capacity_entries=1200)
    monkeypatch.setenv("KVC_SPLIT_DEV_MIN", "0")
    kv_s = ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, s.L)
    monkeypatch.setenv("KVC_SPLIT_DEV_MIN", "2")
    kv_a = ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, s.L)
    for kind, i in s.events():
        if kind == "frame":
            kv_s.process_frame(i, s.visual[i], s.keys[i], s.values[i], want_assigned=True)
            kv_a.process_frame(i, s.visual[i], s.keys[i], s.values[i], want_assigned=False)
        else:
            np.testing.assert_allclose(kv_s.query(i, s.q[i]), kv_a.query(i, s.q[i]), rtol=0, atol=1e-6)
    st_s, st_a = _state(kv_s), _state(kv_a)
    assert st_s == st_a
    assert kv_s.maint_stats()[5] > 0, "stream must exercise split_two"
