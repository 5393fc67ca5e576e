"""Debug: compare async decode against the synchronous run query by query."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import pyoracle as po
from paper_2604_10060_b200 import ClusterKVCache
from tests.harness import product_config

s = po.gen_stream_restated(po.StreamCfg.make(n_scenes=6, frames_per_scene=16, tokens_per_frame=16, d=32, L=4,
                                             scene_cycle=2, drift_rate=0.06, semantic_noise=0.05, n_queries=24,
                                             queries_at_end=0, seed=7))
ecfg = po.EngineCfg.make(build_batch_frames=8, offload_horizon_frames=4, prefetch_enabled=1, device_capacity_entries=1500)
def run(mode):
    kw = {} if mode.startswith("sync") else dict(parity_mode=0, check_invariants=0)
    kv = ClusterKVCache(product_config(ecfg, **kw), s.d, s.L)
    outs, keep, settled = [], [], []
    for kind, i in s.events():
        if kind == "frame":
            kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
        elif mode == "synchost":
            outs.append(torch.from_numpy(kv.query(i, s.q[i]).copy()))
        else:
            o = torch.zeros(s.L, s.d, device="cuda")
            qd = torch.from_numpy(np.ascontiguousarray(s.q[i])).cuda()
            torch.cuda.synchronize()
            kv.query(i, qd, out=o)
            keep.append(qd); outs.append(o)
            if mode == "flush":
                settled.append(int(kv.maint_stats()[4]))
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in outs], kv.maint_stats().tolist(), settled
a = run("sync"); b = run("async"); c = run("flush"); h = run("synchost")
print("stats", a[1], b[1], c[1])
print("settled per query (flush run)", c[2])
for name, r in (("async", b), ("flush", c), ("synchost", h)):
    bad = [(qi, [l for l in range(s.L) if not np.array_equal(x[l], y[l])]) for qi, (x, y) in enumerate(zip(r[0], a[0])) if not np.array_equal(x, y)]
    print(name, "differing queries:", bad[:10])
