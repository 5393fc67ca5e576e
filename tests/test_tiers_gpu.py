"""Physical host tier (K5): the TieredStore residence (store.cpp:95-130) is a real placement.

A Host cluster's member pages live in one contiguous pinned host extent; residence changes are
migrated asynchronously (one copy per cluster on the transfer stream). These tests check that
(i) after kvc_tier_sync the page tables agree with the logical residence everywhere,
(ii) payloads survive offload -> fetch round trips bit for bit, and
(iii) parity with the reference is unchanged whether migrations are forced after every event or
left to run asynchronously (attention reads pages wherever they physically are).
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.harness import Replay, attention_oracle, product_config, rel_err

pytestmark = pytest.mark.gpu

DRIFT = dict(n_scenes=6, frames_per_scene=16, tokens_per_frame=16, d=32, L=4, scene_cycle=2,
             drift_rate=0.06, semantic_noise=0.05, n_queries=12, seed=7)


def _drift_engine():
    return po.EngineCfg.make(build_batch_frames=8, offload_horizon_frames=4, prefetch_enabled=1,
                             device_capacity_entries=1500)


def test_offload_fetch_roundtrip_payload():
    from paper_2604_10060_b200 import ClusterKVCache

    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine(offload_horizon_frames=1 << 20)
    kv = ClusterKVCache(product_config(ecfg, check_invariants=0), s.d, s.L)
    n = 0
    for kind, i in s.events():
        if kind == "frame":
            kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
            n += 1
            if n == 24:
                break
    kv.tier_sync()
    ids = [c for c in kv.cluster_ids() if kv.cluster(c)[0][6] == 0][:12]
    assert len(ids) >= 4
    before = {c: kv.cluster_payload(c) for c in ids}
    for c in ids:
        kv.offload(c)
    kv.tier_sync()
    st = kv.tier_stats()
    assert st["offloads"] >= len(ids) and st["host_pages"] > 0, st
    for c in ids:
        start, npg, busy = kv.cluster_tier(c)
        assert start >= 0 and npg > 0 and not busy
        k, v = kv.cluster_payload(c)  # read through the host mapping
        assert np.array_equal(k, before[c][0]) and np.array_equal(v, before[c][1])
    assert kv.tier_check() == (0, 0, 0, 0)
    # a decode step attends host-resident clusters in place (before any fetch migrates them)
    q = s.q[0]
    out = kv.query(0, q)
    for l in range(s.L):
        fr, tk = kv.attended(l)
        assert rel_err(out[l], attention_oracle(s, fr, tk, l, q[l])) < 1e-3
    for c in ids:
        if kv.cluster(c)[0][6] == 1:
            kv.fetch(c)
    kv.tier_sync()
    for c in ids:
        assert kv.cluster_tier(c)[1] == 0
        k, v = kv.cluster_payload(c)
        assert np.array_equal(k, before[c][0]) and np.array_equal(v, before[c][1])
    assert kv.tier_check() == (0, 0, 0, 0)
    assert kv.tier_stats()["host_pages"] == 0


def _replay(sync_each: bool):
    s = po.gen_stream_restated(po.StreamCfg.make(**DRIFT))
    ecfg = _drift_engine()
    ref = po.RefDriver(ecfg, s.d, s.L, checks=False) if po.reference() is not None else None
    r = Replay(s, ecfg, ref)
    for kind, i in s.events():
        if kind == "frame":
            r.frame(i)
        else:
            r.query(i)
        if sync_each:
            r.kv.tier_sync()
            assert r.kv.tier_check() == (0, 0, 0, 0), (kind, i)
    r.final_compare()
    return r


@pytest.mark.parametrize("sync_each", [True, False])
def test_drift_parity_with_physical_tier(ref_lib, sync_each):
    """Deferred splits, prefetch and a 1500-entry capacity: many offloads and fetches."""
    r = _replay(sync_each)
    assert r.mismatches == [], r.mismatches[:5]
    assert r.att_err < 1e-3
    r.kv.tier_sync()
    st = r.kv.tier_stats()
    assert st["offloads"] > 0 and st["fetches"] > 0, st
    assert st["queued"] == 0 and st["in_flight"] == 0 and st["stage_pages"] == 0
    assert r.kv.tier_check() == (0, 0, 0, 0)


def test_host_tier_full_fails_loudly():
    from paper_2604_10060_b200.api import CapacityError, ClusterKVCache

    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine(offload_horizon_frames=1 << 20)
    kv = ClusterKVCache(product_config(ecfg, check_invariants=0, host_pool_bytes=2 * 64 * 128 * 4 * 2), s.d, s.L)
    for kind, i in s.events():
        if kind == "frame":
            kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
            if i >= 20:
                break
    with pytest.raises(CapacityError):
        for c in kv.cluster_ids():
            if kv.cluster(c)[0][6] == 0:
                kv.offload(c)
        kv.tier_sync()


def _offloaded_engine(monkeypatch, fr: bool):
    """config-1 stream, 40 frames ingested, every Device cluster offloaded and synced."""
    from paper_2604_10060_b200 import ClusterKVCache

    monkeypatch.setenv("KVC_FETCH_ON_READ", "1" if fr else "0")
    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine(offload_horizon_frames=1 << 20)
    kv = ClusterKVCache(product_config(ecfg, check_invariants=0), s.d, s.L)
    monkeypatch.delenv("KVC_FETCH_ON_READ")
    n = 0
    for kind, i in s.events():
        if kind == "frame":
            kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
            n += 1
            if n == 40:
                break
    kv.tier_sync()
    for c in kv.cluster_ids():
        if kv.cluster(c)[0][6] == 0:
            kv.offload(c)
    kv.tier_sync()
    return s, kv


def test_fetch_on_read(monkeypatch):
    """A decode step copies its selected Host clusters into HBM between K4 and K6 (select.cu R6,
    tiers.cu k_fetch_read): same outputs and the same logical ledger as the queued-fetch path,
    extents released, page tables consistent, payloads bit for bit, nothing left to migrate."""
    runs = [_offloaded_engine(monkeypatch, fr) for fr in (False, True)]
    s = runs[0][0]
    payload = {c: runs[0][1].cluster_payload(c) for c in runs[0][1].cluster_ids()}
    outs = [[], []]
    for j, (_, kv) in enumerate(runs):
        for qi in range(6):
            outs[j].append(kv.query(qi, s.q[qi % len(s.q)]).copy())
    for a, b in zip(*outs):
        np.testing.assert_array_equal(a, b)
    (_, off), (_, on) = runs
    lo, ln = off.ledger(), on.ledger()
    assert np.array_equal(lo[0], ln[0]) and np.array_equal(lo[1], ln[1])
    st = on.tier_stats()
    assert st["read_fetches"] > 0 and st["read_fetch_bytes"] > 0, st
    assert off.tier_stats()["read_fetches"] == 0
    for kv in (off, on):
        kv.tier_sync()
        assert kv.tier_check() == (0, 0, 0, 0)
    for c in on.cluster_ids():
        k, v = on.cluster_payload(c)
        assert np.array_equal(k, payload[c][0]) and np.array_equal(v, payload[c][1])
        if on.cluster(c)[0][6] == 0:  # Device: no extent left behind
            assert on.cluster_tier(c)[1] == 0
    # the copies replaced the queued fetches' host-link traffic
    st_on, st_off = on.tier_stats(), off.tier_stats()
    assert st_on["bytes_h2d"] == st_off["bytes_h2d"], (st_on, st_off)
    assert st_on["copies"] < st_off["copies"]
