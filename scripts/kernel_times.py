"""Per-kernel device times (CUPTI via torch.profiler) of a few decode steps of one workload.
Instrumentation for development; a number printed here is never a bench value.

    python scripts/kernel_times.py token|cluster [steps]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "token"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
D, T, NF, C = 112, 196, 334, 128
N = NF * T
st = workload.clustered_state(D, N, C, 128, T, seed=500)
if mode == "token":
    cfg = Config.make(kv_dtype=DTYPE_BF16, token_mode=1, token_budget=16 * 512, window_frames=4,
                      pool_bytes=D * N * 128 * 2 * 2, max_tokens=T)
    kv = ClusterKVCache(cfg, 128, D)
    for f in range(NF):
        kv.process_frame(f, st.visual, st.keys[:, f * T:(f + 1) * T].contiguous(),
                         st.values[:, f * T:(f + 1) * T].contiguous(), want_assigned=False)
else:
    kvb = D * (N + 64 * C + 4 * T) * 128 * 4
    cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=16, window_frames=4, build_batch_frames=1,
                      offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40, pool_bytes=int(1.3 * kvb),
                      max_slots=4 * D * C, max_cluster_pages=512, max_tokens=T, host_pool_bytes=0)
    kv = ClusterKVCache(cfg, 128, D)
    kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
q = workload.queries_near(st, steps + 2, seed=9)
out = torch.zeros(D, 128, device="cuda")
for i in range(2):
    kv.query(i, q[i], out=out)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(2, steps + 2):
        kv.query(i, q[i], out=out)
    torch.cuda.synchronize()
agg = {}
for e in prof.events():
    if e.device_type.name != "CUDA":
        continue
    import re

    m = re.search(r"\b(k_\w+)", e.name)
    name = m.group(1) if m else e.name[:40]
    agg.setdefault(name, []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{k:42s} n={len(v):3d} mean={np.mean(v):9.1f} us total={sum(v):10.1f} us")
if mode == "token":
    nbs = [kv.layer_meta(l).n_predicted for l in range(D)]
    print("boundary rows per domain: mean", np.mean(nbs), "max", max(nbs), "argmax", int(np.argmax(nbs)))
if mode == "token":
    print("select phase cycles (radix, classify, boundary, stats, list):", kv.resolve_profile()[:5].round(0))
