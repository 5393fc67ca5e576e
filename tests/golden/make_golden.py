"""Regenerates the committed golden fixtures from the compiled reference (oracle/_ref).

Run where /root/reference exists (the reference library is built by oracle/Makefile):
    python tests/golden/make_golden.py
Outputs (small, committed): kats.json, config1_expect.json.
"""
import ctypes as C
import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import pyoracle as po  # noqa: E402


def kats():
    ref = po.reference()
    assert ref is not None, "build oracle/_ref first (make -C oracle)"
    u64 = np.zeros(1, np.uint64)
    uni = np.zeros(1)
    gau = np.zeros(1)
    ref.ref_prim_rng(5489, 1, u64.ctypes.data_as(po.u64p), po._p(uni, po.f64p), po._p(gau, po.f64p))
    rep = np.array([1.0, 0.0])
    key = np.array([0.0, 1.0], np.float32)
    out = np.zeros(2)
    var = C.c_double()
    ref.ref_prim_updated_stats(po._p(rep, po.f64p), 0.0, 1, po._p(key, po.f32p), 2, po._p(out, po.f64p),
                               C.byref(var))
    s = po.gen_stream_restated(po.config1_stream())
    h = hashlib.sha256()
    for a in (s.visual, s.keys, s.values, s.q):
        h.update(np.ascontiguousarray(a).tobytes())
    return {
        "source": "compiled reference (oracle/_ref) + reference tests test_maintainer.cpp:64-94",
        "tau": {"tau16_named": ref.ref_prim_tau(16, 0.1, 0.5, 16.0), "expected_approx": 0.24715,
                "closed_form": 0.1 + 0.4 * math.exp(-1.0)},
        "updated_stats": {"rep": [1.0, 0.0], "var": 0.0, "n": 1, "key": [0.0, 1.0], "rep_out": out.tolist(),
                          "var_out": var.value},
        "mix_seed": [[a, b, int(ref.ref_prim_mix_seed(a, b))] for a, b in ((0, 1), (0, 2), (42, 7), (2**63, 5))],
        "mt19937_64_first_5489": int(u64[0]),
        "mt19937_64_10000th_default": 9981545732273789042,
        "config1_stream_sha256": h.hexdigest(),
    }


def config1():
    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine()
    drv = po.RefDriver(ecfg, s.d, s.L, checks=False)
    frames, queries = [], []
    for kind, i in s.events():
        if kind == "frame":
            pid, asg = drv.frame(i, s.visual[i], s.keys[i], s.values[i])
            frames.append({"frame": i, "partition": int(pid),
                           "assigned_sha256": hashlib.sha256(asg.astype(np.int64).tobytes()).hexdigest()})
        else:
            drv.query(i, s.q[i], s.gt[i])
            ttft, recall = drv.query_meta()
            queries.append({"query": i, "digest": str(drv.digest()), "ttft_us": ttft, "recall": recall,
                            "ranked": [drv.ranked(l) for l in range(s.L)],
                            "selected": [drv.selected(l) for l in range(s.L)]})
    ops, by, co, dev = drv.ledger()
    return {"stream": po.config1_stream().asdict(), "engine": ecfg.asdict(), "frames": frames,
            "queries": queries, "maint_stats": drv.maint_stats().tolist(),
            "ledger": {"ops": ops.tolist(), "bytes": by.tolist(), "cost_us": co.tolist(), "device_entries": dev}}


if __name__ == "__main__":
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats(), f, indent=1)
    with open(os.path.join(HERE, "config1_expect.json"), "w") as f:
        json.dump(config1(), f)
    print("wrote", HERE)
