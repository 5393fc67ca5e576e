"""Quick end-to-end check on a GPU box: config-1 replay vs the reference, with timings."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import pyoracle as po
from tests.harness import Replay

s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=3, frames_per_scene=8, tokens_per_frame=16, d=32, L=3,
                                             n_queries=6, semantic_noise=0.05, seed=5))
ecfg = po.EngineCfg.make(build_batch_frames=8)
ref = po.RefDriver(ecfg, s.d, s.L, checks=False)
t = time.time()
r = Replay(s, ecfg, ref).run()
r.final_compare()
print("small:", time.time() - t, "mismatches", r.mismatches[:5], "att", r.att_err, flush=True)

s = po.gen_stream_restated(po.config1_stream())
ecfg = po.config1_engine()
ref = po.RefDriver(ecfg, s.d, s.L, checks=False)
t = time.time()
r = Replay(s, ecfg, ref)
tf = tq = 0.0
for kind, i in s.events():
    t0 = time.time()
    if kind == "frame":
        r.frame(i); tf += time.time() - t0
    else:
        r.query(i); tq += time.time() - t0
    if r.mismatches:
        print("first mismatch at", kind, i, r.mismatches[:3], flush=True)
        break
r.final_compare()
print("config1:", time.time() - t, "frames", tf, "queries", tq, "mismatches", r.mismatches[:5], "att", r.att_err, flush=True)
print("stats", r.kv.maint_stats(), r.ref.maint_stats())
