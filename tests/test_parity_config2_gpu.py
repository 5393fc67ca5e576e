"""Parity at the HEADLINE shape (config 2) on a 4-domain slice: one layer's four
KV heads of LLaVA-OV-7B, each domain at full size (N = 131,124 tokens = 669 frames x 196, C = 256
clusters, top-16 retrieval + 4-frame window, bf16 K/V, d = 128) -- the exact kernel
instantiations the bench times (K4 `k_select3`, K6 `k_attend<128, bf16>`, the tensor-core ingest
tile and the speculate-and-verify resolve).

Both sides get the same state: the product through kvc_bulk_load, the compiled reference through
ref_drv_bulk_load (add_partition + add_cluster + TieredStore adoption, ref_shim.cpp), on the bf16
values rounded to f32. Then an event stream of absorb-regime frames (`frames_near`), drift-regime
frames with gen_stream's dynamics (`frames_drift`: noise 0.02, drift 0.01/frame -> splits) and
decode steps. Compared:
  * per frame: placed partition and every routed cluster id (Maintainer::on_insert's return);
  * per step: ranked / selected lists per domain, the attended-set digest (engine.cpp:18-35),
    ttft / recall, and K6's outputs against the fp64 restatement over the reference's attended
    set -- normwise max|out - ref| / max|ref| < 1e-3 (BASELINE.json north_star);
  * at the end: maintainer stats, ledger, and every cluster's integer fields, fp64 rep /
    variance / buffer_rep BITWISE and member lists (tests/harness.py compare_state).
The `tiered` variant uses the reference cadence (horizon 16): the first new frame offloads every
stale cluster to the physical pinned host tier and the decode steps fetch them back.

The same slice runs at the two other per-domain shapes the bench times: config 3 (1-hour stream,
705,600 tokens and C = 1,378 clusters per domain, tiered: the bench's `offload` phase) and config 5
(one stream of 65,464 tokens and C = 128 per domain: the bench's `streams` phase).
"""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.harness import compare_state, rel_err

pytestmark = pytest.mark.gpu

ATT_TOL = 1e-3
D, T, HD, TOPK, W = 4, 196, 128, 16, 4
SHAPES = {  # per-domain stream length (tokens) and clusters
    "config2": (669 * 196, 256),
    "config3": (3600 * 196, 1378),
    "config5": (334 * 196, 128),
}


def _attend_oracle(q, K, V):
    import ctypes as Cc

    lib = po.restatement()
    out = np.zeros(K.shape[1], np.float64)
    lib.kvo_attend_f32(po._p(np.ascontiguousarray(q, np.float32), po.f32p),
                       po._p(np.ascontiguousarray(K, np.float32), po.f32p),
                       po._p(np.ascontiguousarray(V, np.float32), po.f32p), K.shape[0], K.shape[1],
                       1.0 / np.sqrt(K.shape[1]), po._p(out, po.f64p))
    del Cc
    return out


@pytest.mark.parametrize("shape,tiered", [("config2", False), ("config2", True), ("config3", True),
                                          ("config5", False)],
                         ids=["resident", "tiered", "config3-tiered", "config5"])
def test_config2_slice_matches_reference(ref_lib, shape, tiered):
    import torch

    N, C = SHAPES[shape]

    from paper_2604_10060_b200 import ClusterKVCache, workload
    from tests.harness import product_config

    st = workload.clustered_state(D, N, C, HD, T, seed=42)
    keys_f = st.keys.float().cpu().numpy()
    vals_f = st.values.float().cpu().numpy()
    horizon = 16 if tiered else 1 << 30
    ecfg = po.EngineCfg.make(k_v=1, k_s=TOPK, window_frames=W, build_batch_frames=1,
                             offload_horizon_frames=horizon, device_capacity_entries=1 << 40)
    kv_bytes = D * (N + 64 * C + 64 * T) * HD * 2 * 2
    kv = ClusterKVCache(product_config(ecfg, kv_dtype=1, check_invariants=0, pool_bytes=int(1.6 * kv_bytes),
                                       max_slots=8 * D * C, max_cluster_pages=512, max_tokens=T,
                                       max_candidates=2048 if C > 1024 else 1024,
                                       host_pool_bytes=int(1.3 * kv_bytes) if tiered else 1 << 20,
                                       tier_stage_pages=8192),
                        HD, D)
    ref = po.RefDriver(ecfg, HD, D, checks=False)
    pid = kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
    rpid = ref.bulk_load(st.visual, keys_f, vals_f, st.assign, st.frame_ids, st.token_ids, C)
    assert pid == rpid
    mism = compare_state(kv, ref, members=False)
    assert mism == [], mism[:3]

    # event stream: 10 absorb frames, 12 drift frames, a decode step after every second frame and
    # 8 at the end (26 steps)
    first = N // T + 1
    nk, nv, nvis, nids = workload.frames_near(st, 10, first, seed=5)
    dk, dv, dvis, dids = workload.frames_drift(st, 12, first + 10, seed=6)
    fk = torch.cat([nk, dk]); fv = torch.cat([nv, dv])
    fvis = np.concatenate([nvis, dvis]); fids = np.concatenate([nids, dids])
    fk_f, fv_f = fk.float().cpu().numpy(), fv.float().cpu().numpy()
    nq = 11 + 8
    qs = workload.queries_near(st, nq + 7, seed=9).cpu().numpy()
    # queries that target the drifted tail too: the last drift frame's keys' mean per domain
    tail = fk_f[-1].mean(axis=1)
    qs[nq:] = tail / np.linalg.norm(tail, axis=-1, keepdims=True)
    events = []
    for i in range(len(fids)):
        events.append(("frame", i))
        if i % 2 == 1:
            events.append(("query", len([e for e in events if e[0] == "query"])))
    while len([e for e in events if e[0] == "query"]) < len(qs):
        events.append(("query", len([e for e in events if e[0] == "query"])))

    # row lookup for the attention oracle: bulk rows by (frame, token), new frames by index
    def rows(l, fr, tk):
        K = np.empty((len(fr), HD), np.float32)
        V = np.empty((len(fr), HD), np.float32)
        old = fr < first
        idx = fr[old] * T + tk[old]
        K[old], V[old] = keys_f[l, idx], vals_f[l, idx]
        new = ~old
        fi = fr[new] - first
        K[new], V[new] = fk_f[fi, l, tk[new]], fv_f[fi, l, tk[new]]
        return K, V

    mism, att_err, n_att = [], 0.0, 0
    for kind, i in events:
        if kind == "frame":
            kk = fk[i].contiguous()
            vv = fv[i].contiguous()
            p, asg = kv.process_frame(int(fids[i]), fvis[i], kk.view(torch.int16).cpu().numpy(),
                                      vv.view(torch.int16).cpu().numpy())
            rp, rasg = ref.frame(int(fids[i]), fvis[i], fk_f[i], fv_f[i])
            if p != rp or not np.array_equal(asg, rasg):
                bad = np.argwhere(asg != rasg)
                mism.append(("frame", i, p, rp, bad[:3].tolist()))
                break
        else:
            q = np.ascontiguousarray(qs[i])
            out = kv.query(i, q)
            ref.query(i, q)
            for l in range(D):
                if kv.ranked(l) != ref.ranked(l):
                    mism.append(("ranked", i, l))
                if kv.selected(l) != ref.selected(l):
                    mism.append(("selected", i, l))
                fr, tk = ref.attended(l)
                kfr, ktk = kv.attended(l)
                if not (np.array_equal(fr, kfr) and np.array_equal(tk, ktk)):
                    mism.append(("attended", i, l, len(fr), len(kfr)))
                    continue
                K, V = rows(l, fr, tk)
                att_err = max(att_err, rel_err(out[l], _attend_oracle(q[l], K, V)))
                n_att += len(fr)
            if kv.digest() != ref.digest():
                mism.append(("digest", i))
            if kv.query_meta() != ref.query_meta():
                mism.append(("query_meta", i, kv.query_meta(), ref.query_meta()))
            if mism:
                break
    assert mism == [], mism[:5]
    st_k, st_r = kv.maint_stats(), ref.maint_stats()
    print("maint", st_k.tolist(), "attended tokens/domain/step", n_att / (len(qs) * D), "att_err", att_err)
    assert np.array_equal(st_k, st_r), (st_k.tolist(), st_r.tolist())
    assert st_k[2] + st_k[3] > 0, "the drift frames must exercise the split / defer branches"
    ko, kb, kc, kd = kv.ledger()
    ro, rb, rc, rd = ref.ledger()
    assert np.array_equal(ko, ro) and np.array_equal(kb, rb) and kd == rd
    if tiered:
        assert ko[4] > 0 and ko[0] > 0, "cadence offloads and retrieval fetches expected"
        kv.tier_sync()
    assert att_err < ATT_TOL, att_err
    assert n_att / (len(qs) * D) > 7000  # ~16 clusters x ~490 + window: the headline's attended size
    mism = compare_state(kv, ref)
    assert mism == [], mism[:5]
