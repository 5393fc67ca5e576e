"""GPU parity against the compiled reference (or golden fixtures) on the config-1 stream.

Bar (BASELINE.json north_star): routed cluster ids, ranked / selected cluster-id lists and the
attended-set digest bit-exact; attention within 1e-3 max relative error (normwise: max|out-ref|
/ max|ref|, fp32 vs the fp64 restatement over the reference's attended set).
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.harness import Replay, attention_oracle, compare_state, rel_err

pytestmark = pytest.mark.gpu

ATT_TOL = 1e-3


@pytest.fixture(params=["spec", "seq"])
def resolve_mode(request, monkeypatch):
    """Both device resolve kernels: speculate-and-verify (default) and the sequential one."""
    if request.param == "seq":
        monkeypatch.setenv("KVC_RESOLVE", "seq")
    else:
        monkeypatch.delenv("KVC_RESOLVE", raising=False)
    return request.param


@pytest.fixture(scope="module")
def stream1():
    return po.gen_stream_restated(po.config1_stream())


def _run(stream, ecfg, ref_lib_present=True, dev_kw=None, check_attention=True, max_events=None):
    ref = po.RefDriver(ecfg, stream.d, stream.L, checks=False) if po.reference() is not None else None
    r = Replay(stream, ecfg, ref, dev_kw).run(check_attention=check_attention, max_events=max_events)
    r.final_compare()
    return r


def test_config1_full_stream(stream1, ref_lib, resolve_mode):
    """64 frames (16 build + 48 online with ~360 splits) and 32 queries, top-4."""
    r = _run(stream1, po.config1_engine())
    assert r.mismatches == [], r.mismatches[:5]
    assert r.att_err < ATT_TOL, r.att_err


def test_config1_bf16(stream1, ref_lib):
    """Keys/values rounded to bf16 before either side sees them (SURVEY §7 hard part 5)."""
    import torch

    s = po.Stream(stream1.d, stream1.L, stream1.T, stream1.kinds, stream1.visual,
                  torch.from_numpy(stream1.keys).bfloat16().float().numpy(),
                  torch.from_numpy(stream1.values).bfloat16().float().numpy(), stream1.q, stream1.gt)
    from paper_2604_10060_b200 import ClusterKVCache  # noqa: F401

    ecfg = po.config1_engine()
    ref = po.RefDriver(ecfg, s.d, s.L, checks=False)
    from tests.harness import product_config
    from paper_2604_10060_b200 import ClusterKVCache as KV

    kv = KV(product_config(ecfg, kv_dtype=1), s.d, s.L)
    kbf = torch.from_numpy(s.keys).bfloat16()
    vbf = torch.from_numpy(s.values).bfloat16()
    mism = []
    att_err = 0.0
    for kind, i in s.events():
        if kind == "frame":
            kk = kbf[i].contiguous().view(torch.int16).numpy()
            vv = vbf[i].contiguous().view(torch.int16).numpy()
            pid, asg = kv.process_frame(i, s.visual[i], kk, vv)
            rpid, rasg = ref.frame(i, s.visual[i], s.keys[i], s.values[i])
            if pid != rpid or not np.array_equal(asg, rasg):
                mism.append(("frame", i))
        else:
            out = kv.query(i, s.q[i], gt=s.gt[i])
            ref.query(i, s.q[i], s.gt[i])
            for l in range(s.L):
                if kv.ranked(l) != ref.ranked(l) or kv.selected(l) != ref.selected(l):
                    mism.append(("query", i, l))
                # K6's bf16 instantiation against the fp64 restatement over the reference's set
                fr, tk = ref.attended(l)
                att_err = max(att_err, rel_err(out[l], attention_oracle(s, fr, tk, l, s.q[i, l])))
            if kv.digest() != ref.digest():
                mism.append(("digest", i))
    assert mism == [], mism[:5]
    assert att_err < ATT_TOL, att_err
    mism = compare_state(kv, ref)
    assert mism == [], mism[:5]


def test_decode_only_config1b(ref_lib):
    """Config 1b: build over all 64 frames (4 partitions x 4 clusters), k_v = 4, k_s = 4."""
    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine(build_batch_frames=64, target_semantic_cluster_size=784, k_v=4, k_s=4)
    r = _run(s, ecfg)
    assert r.mismatches == [], r.mismatches[:5]
    assert r.att_err < ATT_TOL


def test_flat_topk_matches_reference(stream1, ref_lib):
    ecfg = po.config1_engine()
    ref = po.RefDriver(ecfg, stream1.d, stream1.L, checks=False)
    r = Replay(stream1, ecfg, ref)
    n = 0
    for kind, i in stream1.events():
        if kind != "frame":
            continue
        r.frame(i)
        n += 1
        if n in (16, 30, 64):
            for l in range(stream1.L):
                for k in (1, 4, 1000):
                    q = stream1.q[(n + l) % len(stream1.q), l]
                    assert r.kv.flat_topk(q, l, k) == ref.flat_topk(q, l, k)
    assert r.mismatches == []


def test_eager_policy(ref_lib, resolve_mode):
    """defer_host_splits = false: eager fetch + split, domains resolved one at a time."""
    s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=3, frames_per_scene=12, tokens_per_frame=32,
                                                 d=32, L=3, n_queries=6, semantic_noise=0.05, seed=5))
    ecfg = po.EngineCfg.make(build_batch_frames=8, defer_host_splits=0, offload_horizon_frames=2)
    r = _run(s, ecfg)
    assert r.mismatches == [], r.mismatches[:5]
    assert r.att_err < ATT_TOL


def test_deferred_and_prefetch_drift(ref_lib, resolve_mode):
    """Drift preset (workload.cpp:337-346) scaled down: deferred splits, buffers, settles, prefetch."""
    s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=6, frames_per_scene=16, tokens_per_frame=16,
                                                 d=32, L=4, scene_cycle=2, drift_rate=0.06,
                                                 semantic_noise=0.05, n_queries=12, seed=7))
    ecfg = po.EngineCfg.make(build_batch_frames=8, offload_horizon_frames=4, prefetch_enabled=1,
                             device_capacity_entries=1500)
    r = _run(s, ecfg)
    assert r.mismatches == [], r.mismatches[:5]
    st = r.kv.maint_stats()
    assert st[3] > 0, "stream must exercise the deferred path"
    assert r.att_err < ATT_TOL


def test_config1_against_golden_fixture(stream1):
    """Same stream, no reference library needed: the committed fixture (tests/golden, made by
    tests/golden/make_golden.py from the reference) pins assignments, rankings and digests."""
    import hashlib
    import json
    import os

    from paper_2604_10060_b200 import ClusterKVCache
    from tests.harness import product_config

    with open(os.path.join(os.path.dirname(__file__), "golden", "config1_expect.json")) as f:
        g = json.load(f)
    s = stream1
    kv = ClusterKVCache(product_config(po.config1_engine()), s.d, s.L)
    fi = qi = 0
    for kind, i in s.events():
        if kind == "frame":
            pid, asg = kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
            exp = g["frames"][fi]
            assert pid == exp["partition"]
            assert hashlib.sha256(asg.astype(np.int64).tobytes()).hexdigest() == exp["assigned_sha256"], i
            fi += 1
        else:
            kv.query(i, s.q[i], gt=s.gt[i])
            exp = g["queries"][qi]
            assert [kv.ranked(l) for l in range(s.L)] == [[tuple(x) for x in r] for r in exp["ranked"]]
            assert [kv.selected(l) for l in range(s.L)] == exp["selected"]
            assert str(kv.digest()) == exp["digest"]
            assert kv.query_meta()[1] == exp["recall"]
            qi += 1
    assert kv.maint_stats().tolist() == g["maint_stats"]
    ops, by, co, dev = kv.ledger()
    assert ops.tolist() == g["ledger"]["ops"] and by.tolist() == g["ledger"]["bytes"]
    assert dev == g["ledger"]["device_entries"]


def test_async_decode_pipeline_matches_sync():
    """Without parity / recall / host outputs a query returns before its step completes: step i+1
    is launched before step i's bookkeeping is replayed and relaunched when that bookkeeping
    settles a split. Outputs and bookkeeping must equal the synchronous (parity-mode) run."""
    import torch

    from paper_2604_10060_b200 import ClusterKVCache
    from tests.harness import product_config

    s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=6, frames_per_scene=16, tokens_per_frame=16,
                                                 d=32, L=4, scene_cycle=2, drift_rate=0.06,
                                                 semantic_noise=0.05, n_queries=24, queries_at_end=0,
                                                 seed=7))
    ecfg = po.EngineCfg.make(build_batch_frames=8, offload_horizon_frames=4, prefetch_enabled=1,
                             device_capacity_entries=1500)
    kv_s = ClusterKVCache(product_config(ecfg), s.d, s.L)
    kv_a = ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, s.L)
    outs_s, outs_a = [], []
    for kind, i in s.events():
        if kind == "frame":
            kv_s.process_frame(i, s.visual[i], s.keys[i], s.values[i])
            kv_a.process_frame(i, s.visual[i], s.keys[i], s.values[i])
        else:
            outs_s.append(kv_s.query(i, s.q[i]).copy())
            o = torch.zeros(s.L, s.d, device="cuda")
            qd = torch.from_numpy(np.ascontiguousarray(s.q[i])).cuda()
            torch.cuda.synchronize()  # inputs are produced on torch's stream, consumed on kv.stream
            kv_a.query(i, qd, out=o)
            outs_a.append((o, qd))  # device inputs stay alive until the step completes
    torch.cuda.synchronize()
    assert len(outs_a) > 0
    for (a, _), b in zip(outs_a, outs_s):
        assert np.array_equal(a.cpu().numpy(), b)
    assert kv_a.maint_stats().tolist() == kv_s.maint_stats().tolist()
    la, ls = kv_a.ledger(), kv_s.ledger()
    assert la[0].tolist() == ls[0].tolist() and la[1].tolist() == ls[1].tolist() and la[3] == ls[3]
    st = kv_a.maint_stats()
    print("deferred marks", st[3], "settled splits", st[4])
    assert st[3] > 0 and st[4] > 0  # deferred splits were settled on the async path


def test_pinned_host_buffers_zero_copy(stream1):
    """A query and output in pinned host memory are used in place (K4 reads the query over the
    link, K6 writes the rows to the host): outputs equal the pageable (copied) path bitwise, and
    the pinned output is complete when query() returns."""
    import torch

    from paper_2604_10060_b200 import ClusterKVCache
    from tests.harness import product_config

    s = stream1
    ecfg = po.config1_engine()
    kv_p = ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, s.L)
    kv_c = ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, s.L)
    q_pin = torch.zeros(s.L, s.d).pin_memory()
    o_pin = torch.zeros(s.L, s.d).pin_memory()
    n = 0
    for kind, i in s.events():
        if kind == "frame":
            kv_p.process_frame(i, s.visual[i], s.keys[i], s.values[i])
            kv_c.process_frame(i, s.visual[i], s.keys[i], s.values[i])
            continue
        q_pin.copy_(torch.from_numpy(np.ascontiguousarray(s.q[i], np.float32)))
        o_pin.fill_(float("nan"))
        kv_p.query(i, q_pin.numpy(), out=o_pin.numpy())
        ref = kv_c.query(i, np.ascontiguousarray(s.q[i], np.float32).copy())
        assert np.array_equal(o_pin.numpy(), ref), i
        assert kv_p.digest() == kv_c.digest()
        n += 1
    assert n > 0
