"""Frame ingest on a drifting stream (frames far enough from their clusters that variance crosses
tau and the maintenance split slow path runs), with the split's 2-way k-means on the GPU
(split.cu, groups >= KVC_SPLIT_DEV_MIN rows) or on the host (KVC_SPLIT_DEV_MIN=0). Development
measurement for DESIGN.md §5c; the bench's ingest line is the near-cluster (no-split) stream.

    python scripts/drift_ingest.py [noise] [frames] [domains]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload  # noqa: E402

noise = float(sys.argv[1]) if len(sys.argv) > 1 else 0.05
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 20
D = int(sys.argv[3]) if len(sys.argv) > 3 else 16
N, C, T, HD = 65536, 128, 196, 128
MAINT = ["inserts", "absorbed", "immediate_splits", "deferred_marks", "settled_splits", "split_ops", "host_over",
         "maint_fetches", "partitions_opened"]


def run(dev_min):
    os.environ["KVC_SPLIT_DEV_MIN"] = str(dev_min)
    cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=16, window_frames=4, build_batch_frames=1,
                      offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                      pool_bytes=int(1.5 * D * (N + 64 * C + 400 * T) * HD * 4), max_slots=max(4096, 64 * D * C),
                      max_cluster_pages=512, max_tokens=T, max_candidates=4096)
    kv = ClusterKVCache(cfg, HD, D)
    st = workload.clustered_state(D, N, C, HD, T, seed=42)
    kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
    fk, fv, fvis, fids = workload.frames_near(st, frames + 2, N // T + 1, noise=noise, seed=5)
    for i in range(2):
        kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
    torch.cuda.synchronize()
    m0 = kv.maint_stats()
    t0 = time.perf_counter()
    for i in range(2, frames + 2):
        kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    m = dict(zip(MAINT, (kv.maint_stats() - m0).tolist()))
    q = workload.queries_near(st, 1, seed=3)[0]
    kv.query(0, q, out=torch.zeros(D, HD, device="cuda"))
    torch.cuda.synchronize()
    dig = [kv.digest(), len(kv.cluster_ids())]
    del kv
    torch.cuda.empty_cache()
    return dict(frames_per_s=round(frames / dt, 1), ms_per_frame=round(dt / frames * 1e3, 2), maint=m, digest=dig)


host = run(0)
dev = run(128)
dev_all = run(2)
print(json.dumps(dict(noise=noise, frames=frames, domains=D, host_split=host, gpu_split_ge128=dev, gpu_split_all=dev_all,
                      same_state=host["digest"] == dev["digest"] == dev_all["digest"])))

if os.environ.get("DRIFT_PROFILE"):  # per-kernel device time of the GPU-split run (CUPTI)
    import re

    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        t = run(128)
    agg = {}
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        m = re.search(r"\b(k_\w+)", e.name)
        agg.setdefault(m.group(1) if m else e.name[:40], []).append(e.device_time_total)
    print("wall ms/frame", t["ms_per_frame"])
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:12]:
        print(f"{k:42s} n={len(v):6d} mean={np.mean(v):9.1f} us total={sum(v) / 1e3:9.1f} ms")
