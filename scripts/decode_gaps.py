"""Device timeline of end-to-end decode steps (pinned host query / output through the public API):
per-step device busy time and the idle gap between consecutive steps (CUPTI via torch.profiler).
Development instrumentation only.

    python scripts/decode_gaps.py [steps]
"""
import os
import re
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
D, T, C, N = 112, 196, 256, 196 * 669
cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=16, window_frames=4, build_batch_frames=1,
                  offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                  pool_bytes=int(1.25 * D * (N + 64 * C + 400 * T) * 128 * 4), max_slots=4 * D * C,
                  max_cluster_pages=512, max_tokens=T)
kv = ClusterKVCache(cfg, 128, D)
st = workload.clustered_state(D, N, C, 128, T, seed=42)
kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
q = workload.queries_near(st, steps + 5, seed=11).cpu().pin_memory().numpy()
out = torch.zeros(D, 128).pin_memory().numpy()
for i in range(5):
    kv.query(i, q[i], out=out)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    h0 = time.perf_counter()
    for i in range(5, steps + 5):
        kv.query(i, q[i], out=out)
    wall = (time.perf_counter() - h0) * 1e6 / steps
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
k4 = [e for e in ev if re.search(r"k_select3|k_score_select", e.name)]
k6 = [e for e in ev if "k_attend" in e.name]
gaps = [k4[i + 1].time_range.start - k6[i].time_range.end for i in range(min(len(k4) - 1, len(k6)))]
k4k6 = [k6[i].time_range.start - k4[i].time_range.end for i in range(min(len(k4), len(k6)))]
print(f"wall per step {wall:.1f} us; K4 {np.mean([e.time_range.end - e.time_range.start for e in k4]):.1f} us, "
      f"K6 {np.mean([e.time_range.end - e.time_range.start for e in k6]):.1f} us, K4->K6 gap {np.mean(k4k6):.1f} us, "
      f"K6 end -> next K4 start {np.mean(gaps):.1f} us (min {np.min(gaps):.1f})")
others = {}
for e in ev:
    if e in k4 or e in k6:
        continue
    others.setdefault(e.name[:40], []).append(e.time_range.end - e.time_range.start)
for k, v in others.items():
    print(f"  other device op {k:40s} n={len(v)} mean {np.mean(v):.1f} us")
