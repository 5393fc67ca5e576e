"""Token-level top-k retrieval baseline (retrieve_token_baseline, retrieval.cpp:166-254) on the GPU
against the compiled reference driven in RetrievalMode::TokenBaseline (engine.cpp:153-158,179-203).

Bar: attended (frame, token) sets and their digest bit-exact (the selection is exact: fp32 scan +
fp64 re-score of the boundary rows with the reference's tie-break), latency model / ledger totals
equal (floating sums to 1e-9 relative), attention within 1e-3 of the fp64 restatement.
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.harness import attention_oracle, product_config, rel_err

pytestmark = pytest.mark.gpu


def _run(stream, ecfg, kv_dtype=0, check_attention=True):
    from paper_2604_10060_b200 import ClusterKVCache

    ref = po.RefDriver(ecfg, stream.d, stream.L, checks=False)
    kv = ClusterKVCache(product_config(ecfg, kv_dtype=kv_dtype, check_invariants=0), stream.d, stream.L)
    mism, att_err, nq = [], 0.0, 0
    keys, values = stream.keys, stream.values
    if kv_dtype == 1:
        import torch

        kb = torch.from_numpy(stream.keys).bfloat16()
        vb = torch.from_numpy(stream.values).bfloat16()
        keys, values = kb.float().numpy(), vb.float().numpy()
        kraw, vraw = kb.view(torch.int16).numpy(), vb.view(torch.int16).numpy()
    for kind, i in stream.events():
        if kind == "frame":
            if kv_dtype == 1:
                kv.process_frame(i, stream.visual[i], kraw[i], vraw[i])
            else:
                kv.process_frame(i, stream.visual[i], keys[i], values[i])
            ref.frame(i, stream.visual[i], keys[i], values[i])
            continue
        out = kv.query(i, stream.q[i], gt=stream.gt[i])
        ref.query(i, stream.q[i], stream.gt[i])
        nq += 1
        for l in range(stream.L):
            a_fr, a_tk = kv.attended(l)
            r_fr, r_tk = ref.attended(l)
            if not (np.array_equal(a_fr, r_fr) and np.array_equal(a_tk, r_tk)):
                mism.append(("attended", i, l, len(a_fr), len(r_fr)))
            m = kv.layer_meta(l)
            klat = [m.lookup_us, m.transfer_us, m.stall_us, m.completion_us, m.compute_us]
            rlat, _ = ref.layer_meta(l)
            if not np.allclose(klat, rlat, rtol=1e-9, atol=1e-9):
                mism.append(("latency", i, l, list(klat), list(rlat)))
            if check_attention and len(a_fr):
                s2 = po.Stream(stream.d, stream.L, stream.T, stream.kinds, stream.visual, keys, values,
                               stream.q, stream.gt)
                att_err = max(att_err, rel_err(out[l], attention_oracle(s2, a_fr, a_tk, l, stream.q[i, l])))
        if kv.digest() != ref.digest():
            mism.append(("digest", i))
        kt, kr = kv.query_meta()
        rt, rr = ref.query_meta()
        if not (abs(kt - rt) <= 1e-9 * max(1.0, abs(rt)) and kr == rr):
            mism.append(("query_meta", i, kt, rt, kr, rr))
    ko, kb_, kc, _ = kv.ledger()
    ro, rb, rc, _ = ref.ledger()
    if not (np.array_equal(ko, ro) and np.array_equal(kb_, rb) and np.allclose(kc, rc, rtol=1e-9)):
        mism.append(("ledger", ko.tolist(), ro.tolist(), kb_.tolist(), rb.tolist()))
    return mism, att_err, nq


SMALL = dict(n_scenes=3, frames_per_scene=8, tokens_per_frame=24, d=64, L=3, n_queries=6, semantic_noise=0.05,
             seed=5, queries_at_end=0)


@pytest.mark.parametrize("budget", [1, 37, 200, 100000])
def test_token_baseline_matches_reference(ref_lib, budget):
    s = po.gen_stream_restated(po.StreamCfg.make(**SMALL))
    ecfg = po.EngineCfg.make(token_mode=1, token_budget=budget, window_frames=2)
    mism, att_err, nq = _run(s, ecfg)
    assert nq > 0
    assert mism == [], mism[:5]
    assert att_err < 1e-3, att_err


def test_token_baseline_config1_shape(ref_lib):
    """Config-1 stream (64 frames x 196 tokens, 8 domains, d = 128), budget = the cluster run's
    selection scale (4 clusters x ~196 tokens)."""
    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine(token_mode=1, token_budget=784)
    mism, att_err, nq = _run(s, ecfg)
    assert nq == 32
    assert mism == [], mism[:5]
    assert att_err < 1e-3, att_err


def test_token_baseline_bf16(ref_lib):
    s = po.gen_stream_restated(po.StreamCfg.make(**SMALL))
    ecfg = po.EngineCfg.make(token_mode=1, token_budget=50, window_frames=2)
    mism, att_err, _ = _run(s, ecfg, kv_dtype=1)
    assert mism == [], mism[:5]
    assert att_err < 1e-3, att_err


def test_token_mode_rejects_cluster_views():
    from paper_2604_10060_b200 import ClusterKVCache
    from paper_2604_10060_b200.api import ConfigError

    s = po.gen_stream_restated(po.StreamCfg.make(**SMALL))
    kv = ClusterKVCache(product_config(po.EngineCfg.make(token_mode=1, token_budget=8)), s.d, s.L)
    kv.process_frame(0, s.visual[0], s.keys[0], s.values[0])
    assert kv.cluster_ids() == []
    with pytest.raises(ConfigError):
        kv.check()


@pytest.mark.parametrize("budget", [3000, 7000])
def test_token_baseline_large_exact_tie_group(ref_lib, budget):
    """Static frames: every row of a domain holds the same key, so all 7,840 rows tie at the exact
    boundary value (a boundary set above 4,096 rows takes the radix path, and the tie group is far
    above the 1,024 rows ranked in shared memory): the reference ranks them by (frame, token)
    (retrieval.cpp:198-204); the kernel's second radix select over the packed (frame, token) keys
    must pick the same rows."""
    rng = np.random.default_rng(3)
    d, L, T, F = 64, 2, 196, 40
    key = rng.standard_normal((L, d)).astype(np.float32)
    keys = np.broadcast_to(key[None, :, None, :], (F, L, T, d)).copy()
    values = rng.standard_normal((F, L, T, d)).astype(np.float32)
    visual = np.broadcast_to(rng.standard_normal(d).astype(np.float32), (F, d)).copy()
    q = rng.standard_normal((3, L, d)).astype(np.float32)
    kinds = np.array([0] * F + [1] * 3, np.int32)
    s = po.Stream(d, L, T, kinds, visual, keys, values, q, [[0, 1]] * 3)
    ecfg = po.EngineCfg.make(token_mode=1, token_budget=budget, window_frames=2)
    mism, att_err, nq = _run(s, ecfg)
    assert nq == 3
    assert mism == [], mism[:5]
    assert att_err < 1e-3, att_err
