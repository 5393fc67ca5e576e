"""Parity harness: replays one synthetic stream through the product (ClusterKVCache over
libkvc.so) and through the checker (the compiled reference via oracle/pyoracle.RefDriver, or the
committed golden fixtures when the reference library is absent), comparing event by event.

Test infrastructure only (imports oracle/).
"""
from __future__ import annotations

import numpy as np

from oracle import pyoracle as po


def product_config(ecfg: "po.EngineCfg", **dev):
    """Same EngineConfig fields as the checker's, plus data-plane sizing."""
    from paper_2604_10060_b200 import Config

    kw = {name: getattr(ecfg, name) for name, _ in ecfg._fields_}
    kw.update(dict(parity_mode=1, check_invariants=1))
    kw.update(dev)
    return Config.make(**kw)


def attention_oracle(stream: "po.Stream", frames, tokens, layer: int, q: np.ndarray):
    """fp64 restatement over an attended (frame, token) set (kvc_oracle.c kvo_attend_f32)."""
    import ctypes as C

    lib = po.restatement()
    K = np.ascontiguousarray(stream.keys[frames, layer, tokens], np.float32)
    V = np.ascontiguousarray(stream.values[frames, layer, tokens], np.float32)
    out = np.zeros(stream.d, np.float64)
    lib.kvo_attend_f32(po._p(np.ascontiguousarray(q, np.float32), po.f32p), po._p(K, po.f32p),
                       po._p(V, po.f32p), len(frames), stream.d, 1.0 / np.sqrt(stream.d),
                       po._p(out, po.f64p))
    return out


def rel_err(a, b):
    """max |a - b| / max |b| (normwise relative, fp32 vs fp64)."""
    den = max(np.abs(b).max(), 1e-30)
    return float(np.abs(np.asarray(a, np.float64) - b).max() / den)


class Replay:
    """Drives both sides in lock-step and records the first divergence."""

    def __init__(self, stream, ecfg, ref: "po.RefDriver | None", dev_kw=None):
        from paper_2604_10060_b200 import ClusterKVCache

        self.s = stream
        self.ref = ref
        self.kv = ClusterKVCache(product_config(ecfg, **(dev_kw or {})), stream.d, stream.L)
        self.mismatches = []
        self.att_err = 0.0
        self.frames = 0
        self.queries = 0

    def frame(self, i):
        s = self.s
        pid, asg = self.kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
        if self.ref is not None:
            rpid, rasg = self.ref.frame(i, s.visual[i], s.keys[i], s.values[i])
            if pid != rpid:
                self.mismatches.append(("partition", i, pid, rpid))
            if not np.array_equal(asg, rasg):
                bad = np.argwhere(asg != rasg)
                self.mismatches.append(("assign", i, bad[:5].tolist(), asg[tuple(bad[0])], rasg[tuple(bad[0])]))
        self.frames += 1
        return pid, asg

    def query(self, i, check_attention=True):
        s = self.s
        out = self.kv.query(i, s.q[i], gt=s.gt[i] if len(s.gt) > i else None)
        self.queries += 1
        if self.ref is not None:
            self.ref.query(i, s.q[i], s.gt[i] if len(s.gt) > i else None)
            for l in range(s.L):
                if self.kv.ranked(l) != self.ref.ranked(l):
                    self.mismatches.append(("ranked", i, l, self.kv.ranked(l), self.ref.ranked(l)))
                if self.kv.selected(l) != self.ref.selected(l):
                    self.mismatches.append(("selected", i, l))
            if self.kv.digest() != self.ref.digest():
                self.mismatches.append(("digest", i))
            if self.kv.query_meta() != self.ref.query_meta():
                self.mismatches.append(("query_meta", i, self.kv.query_meta(), self.ref.query_meta()))
        if check_attention:
            for l in range(s.L):
                fr, tk = self.kv.attended(l)
                ref = attention_oracle(s, fr, tk, l, s.q[i, l])
                self.att_err = max(self.att_err, rel_err(out[l], ref))
        return out

    def run(self, check_attention=True, max_events=None):
        n = 0
        for kind, i in self.s.events():
            if max_events is not None and n >= max_events:
                break
            if kind == "frame":
                self.frame(i)
            else:
                self.query(i, check_attention)
            n += 1
        return self

    def final_compare(self):
        if self.ref is None:
            return
        if not np.array_equal(self.kv.maint_stats(), self.ref.maint_stats()):
            self.mismatches.append(("maint_stats", self.kv.maint_stats().tolist(), self.ref.maint_stats().tolist()))
        ko, kb, kc, kd = self.kv.ledger()
        ro, rb, rc, rd = self.ref.ledger()
        if not (np.array_equal(ko, ro) and np.array_equal(kb, rb) and np.allclose(kc, rc, rtol=0, atol=1e-6) and kd == rd):
            self.mismatches.append(("ledger", ko.tolist(), ro.tolist(), kd, rd))
        self.mismatches.extend(compare_state(self.kv, self.ref))


def compare_state(kv, ref, members=True, limit=20):
    """Every cluster of the product against the checker (index.hpp:29-50 ClusterRecord): the ten
    integer fields, the fp64 Eq. 3/4 state (`variance`, `rep`, and `buffer_rep` while a buffer is
    held) BITWISE, and the member / buffer (frame, token) lists in stored order."""
    out = []
    ids = kv.cluster_ids()
    if ids != ref.cluster_ids():
        return [("cluster_ids", len(ids), len(ref.cluster_ids()))]
    for cid in ids:
        ki, kvar, krep, kbrep = kv.cluster(cid)
        ri, rvar, rrep, rbrep = ref.cluster(cid)
        if not np.array_equal(ki, ri):
            out.append(("cluster_info", cid, ki.tolist(), ri.tolist()))
        elif np.float64(kvar).tobytes() != np.float64(rvar).tobytes():
            out.append(("cluster_variance", cid, kvar, rvar))
        elif krep.tobytes() != rrep.tobytes():
            out.append(("cluster_rep", cid, int(np.argmax(krep != rrep))))
        elif ri[3] > 0 and kbrep.tobytes() != rbrep.tobytes():
            out.append(("cluster_buffer_rep", cid))
        elif members:
            for which in (0, 1):
                kf, kt = kv.cluster_entries(cid, which)
                rf, rt = ref.cluster_entries(cid, which)
                if not (np.array_equal(kf, rf) and np.array_equal(kt, rt)):
                    out.append(("cluster_entries", cid, which))
        if len(out) >= limit:
            break
    return out
