"""Device timeline of pipelined frame ingest (CUPTI via torch.profiler): per-kernel durations and
the idle gaps between consecutive device operations. Development instrumentation only.

    python scripts/ingest_gaps.py [frames]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload  # noqa: E402

nf = int(sys.argv[1]) if len(sys.argv) > 1 else 12
D, T, C, N = 112, 196, 256, 196 * 669
cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=16, window_frames=4, build_batch_frames=1,
                  offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                  pool_bytes=int(1.25 * D * (N + 64 * C + 400 * T) * 128 * 4), max_slots=4 * D * C,
                  max_cluster_pages=512, max_tokens=T)
kv = ClusterKVCache(cfg, 128, D)
st = workload.clustered_state(D, N, C, 128, T, seed=42)
kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
fk, fv, fvis, fids = workload.frames_near(st, nf + 4, N // T + 1)
for i in range(4):
    kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for i in range(4, nf + 4):
        kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
    torch.cuda.synchronize()
ev = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
import re  # noqa: E402

gaps = {}
prev_end, prev_name = None, None
rows = []
for e in ev:
    m = re.search(r"\b(k_\w+)", e.name)
    name = m.group(1) if m else e.name[:28]
    s, t = e.time_range.start, e.time_range.end
    if prev_end is not None:
        g = s - prev_end
        gaps.setdefault(f"{prev_name} -> {name}", []).append(g)
    rows.append((name, t - s))
    prev_end, prev_name = max(t, prev_end or t), name
span = (ev[-1].time_range.end - ev[0].time_range.start) / nf
busy = sum(d for _, d in rows) / nf
print(f"per frame: span {span:.1f} us, busy {busy:.1f} us")
for k, v in sorted(gaps.items(), key=lambda x: -sum(x[1]))[:12]:
    print(f"{k:60s} n={len(v):4d} mean gap={np.mean(v):7.2f} us")
