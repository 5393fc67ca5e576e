"""The wave engine (context_waves.cpp: a frame's host events settled for all domains at once with
predicted split counters, verified afterwards, rolled back per domain on a misprediction) must
leave exactly the state of the one-domain-at-a-time path (KVC_WAVES=0), which the reference
parity tests pin: same cluster ids, fp64 statistics bitwise, member lists, maintainer counters,
ledger and decode outputs.

Covered: the drift regime at config-2 geometry (d = 128, bf16; clusters crossing the Eq. 5
threshold about once per domain per frame), the reference's own streams (seeds, recursive
splits, deferred splits), and KVC_WAVES_PERTURB=1, which makes every first-pass prediction wrong
so that the verification and the snapshot / restore rollback run on every domain with events."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.harness import compare_state, product_config

pytestmark = pytest.mark.gpu


def _drift_pair(monkeypatch, perturb: bool, D=8, N=24_000, C=48, frames=6, pre=0):
    import torch

    from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload

    T, HD = 196, 128
    cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=16, window_frames=4, build_batch_frames=1,
                      offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                      pool_bytes=int(1.6 * D * (N + 64 * C + 400 * T) * HD * 4), max_slots=max(4096, 8 * D * C),
                      max_cluster_pages=512, max_tokens=T)
    st = workload.clustered_state(D, N, C, HD, T, seed=42)
    kvs = []
    for waves in (False, True):
        monkeypatch.setenv("KVC_WAVES", "1" if waves else "0")
        monkeypatch.setenv("KVC_WAVES_PERTURB", "1" if (waves and perturb) else "0")
        kv = ClusterKVCache(cfg, HD, D)
        kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
        kvs.append(kv)
    monkeypatch.delenv("KVC_WAVES_PERTURB", raising=False)
    fk, fv, fvis, fids = workload.frames_drift(st, frames, N // T + 1 + 100000, seed=7)
    q = torch.randn(4, D, HD, generator=torch.Generator().manual_seed(3)).numpy().astype(np.float32)
    outs = [[], []]
    for i in range(frames):
        for j, kv in enumerate(kvs):
            kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=(i % 2 == 0))
        if i % 2 == 1:
            for j, kv in enumerate(kvs):
                outs[j].append(kv.query(10_000_000 + i, q[i % 4]).copy())
    return kvs, outs


@pytest.mark.parametrize("perturb,D,frames,relaunch", [(False, 8, 6, "spec"), (True, 8, 6, "spec"), (False, 32, 14, "spec"),
                                                        (False, 8, 6, "seq"), (True, 8, 6, "seq")],
                         ids=["8dom", "8dom-perturbed", "32dom-14frames", "8dom-seq-relaunch", "8dom-perturbed-seq-relaunch"])
def test_waves_equal_sequential_drift(monkeypatch, perturb, D, frames, relaunch):
    """relaunch: the resolve kernel of the rounds after a split -- the speculative one seeded by
    the fp32 routing simulation (default) or the sequential one (KVC_RELAUNCH=seq); ties are
    reported by both, so the label exchange is exercised with either."""
    monkeypatch.setenv("KVC_RELAUNCH", relaunch)
    (seq, wav), outs = _drift_pair(monkeypatch, perturb, D=D, frames=frames)
    ms, mw = seq.maint_stats(), wav.maint_stats()
    assert ms.tolist() == mw.tolist()
    assert ms[2] >= 8, "the drift frames must split"
    mism = compare_state(wav, seq)
    assert not mism, mism[:5]
    for a, b in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b)
    prof = wav.wave_profile()
    assert prof["events"] >= ms[2]
    if D >= 32:  # enough domains that predictions go wrong and domains are rolled back on their own
        assert prof["rolled_back_domains"] > 0
    if perturb:
        assert prof["rolled_back_domains"] > 0 and prof["passes"] > prof["frames_with_events"]


@pytest.mark.parametrize("perturb", [False, True])
def test_waves_reference_stream(monkeypatch, perturb):
    """The config-1-like reference stream (seeds on new partitions, immediate and recursive splits,
    deferred splits settled by queries) through both paths, every frame with per-entry outputs."""
    from paper_2604_10060_b200 import ClusterKVCache

    s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=5, frames_per_scene=14, tokens_per_frame=40, d=32, L=6,
                                                 scene_cycle=2, drift_rate=0.05, semantic_noise=0.06,
                                                 n_queries=10, queries_at_end=0, seed=11))
    ecfg = po.EngineCfg.make(build_batch_frames=6, offload_horizon_frames=3, device_capacity_entries=1500,
                             tau_min=0.02, tau_max=0.3)
    kvs = []
    for waves in (False, True):
        monkeypatch.setenv("KVC_WAVES", "1" if waves else "0")
        monkeypatch.setenv("KVC_WAVES_PERTURB", "1" if (waves and perturb) else "0")
        kvs.append(ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, s.L))
    monkeypatch.delenv("KVC_WAVES_PERTURB", raising=False)
    outs = [[], []]
    for kind, i in s.events():
        for j, kv in enumerate(kvs):
            if kind == "frame":
                a = kv.process_frame(i, s.visual[i], s.keys[i], s.values[i], want_assigned=True)
                if j == 0:
                    a0 = a
                else:
                    np.testing.assert_array_equal(a0[1], a[1])  # per-entry cluster ids
            else:
                outs[j].append(kv.query(i, s.q[i]).copy())
    seq, wav = kvs
    assert seq.maint_stats().tolist() == wav.maint_stats().tolist()
    assert seq.maint_stats()[2] > 0, "stream must exercise immediate splits"
    mism = compare_state(wav, seq)
    assert not mism, mism[:5]
    ko, kb, kc, kd = wav.ledger()
    ro, rb, rc, rd = seq.ledger()
    assert np.array_equal(ko, ro) and np.array_equal(kb, rb) and kd == rd
    for a, b in zip(outs[0], outs[1]):
        np.testing.assert_array_equal(a, b)
