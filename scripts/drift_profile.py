"""Drift-regime ingest at config-2 shape (gen_stream dynamics, noise 0.02, drift
0.01/frame) on D domains: per-frame wall time, host events, and the host-event slow-path profile
(kvc_debug_event_profile). Development measurement.

    python scripts/drift_profile.py [domains] [frames]
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

D = int(sys.argv[1]) if len(sys.argv) > 1 else 112
F = int(sys.argv[2]) if len(sys.argv) > 2 else 12
N, C, T, HD = 669 * 196, 256, 196, 128
cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=16, window_frames=4, build_batch_frames=1,
                  offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                  pool_bytes=int(1.3 * D * (N + 64 * C + 400 * T) * HD * 4), max_slots=max(4096, 4 * D * C),
                  max_cluster_pages=512, max_tokens=T)
kv = ClusterKVCache(cfg, HD, D)
st = workload.clustered_state(D, N, C, HD, T, seed=42)
kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
PRE = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # absorb-regime frames first (as the bench does)
if PRE:
    ak, av, avis, aids = workload.frames_near(st, PRE, N // T + 1, seed=7)
    for i in range(PRE):
        kv.process_frame(int(aids[i]), avis[i], ak[i], av[i], want_assigned=False)
    kv.maint_stats()
fk, fv, fvis, fids = workload.frames_drift(st, F, N // T + 1 + 100000, seed=7)
rows = []
kv.event_profile(reset=True)
kv.wave_profile(reset=True)
TIMED = os.environ.get("DRIFT_TIMING") == "1"
kv.set_timing(TIMED)
kts = []
torch.cuda.synchronize()
T0 = time.perf_counter()
for i in range(F):
    m0 = kv.maint_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=False)
    kv.flush() if hasattr(kv, "flush") else None
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    m = kv.maint_stats() - m0
    rows.append({"frame": i, "ms": round(dt, 2), "splits": int(m[2]), "split_ops": int(m[5])})
    if TIMED:
        kts.append(np.round(kv.ingest_timing(), 1).tolist() + ["seq_last_launch_cycles"] + np.round(kv.resolve_profile()[:12], 0).tolist())
kv.maint_stats()  # completes the last frame's deferred replay
torch.cuda.synchronize()
wall = (time.perf_counter() - T0) * 1e3
# per-kernel device time of the rounds of a few more frames (CUDA events, summed over rounds)
kv.set_timing(True)
xk, xv, xvis, xids = workload.frames_drift(st, 3, N // T + 1 + 200000, seed=8)
kt = []
for i in range(3):
    kv.process_frame(int(xids[i]), xvis[i], xk[i], xv[i], want_assigned=True)
    kt.append(dict(zip(["cands", "assign", "topm", "resolve", "store_rows", "host_wait", "host_insert_loop",
                        "host_replay", "host_relaunch_issue", "host_events"], np.round(kv.ingest_timing(), 1).tolist())))
kv.set_timing(False)
prof = kv.event_profile()
wprof = kv.wave_profile()
tot = wall
print(json.dumps({"domains": D, "frames": F, "ms_per_frame": round(tot / F, 2), "rows": rows, "event_profile": prof, "wave_profile": wprof,
                  "per_event_us": {k: round(v / max(prof["events"], 1), 1) for k, v in prof.items() if k.endswith("_us")},
                  "timed_frames": kt, "all_frames_timing": kts}))
