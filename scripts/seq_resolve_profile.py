"""Per-token phase cycles of the sequential resolve kernel (k_resolve, kernels.cu) on full frames
of the config-2 shape: KVC_RESOLVE=seq forces it for every round. Development measurement.

    KVC_RESOLVE=seq [KVC_RESOLVE_PROF=1] python scripts/seq_resolve_profile.py [domains] [frames] [drift]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload  # noqa: E402

D = int(sys.argv[1]) if len(sys.argv) > 1 else 112
F = int(sys.argv[2]) if len(sys.argv) > 2 else 4
DRIFT = len(sys.argv) > 3 and sys.argv[3] == "drift"
N, C, T, HD = 669 * 196, 256, 196, 128
cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=16, window_frames=4, build_batch_frames=1,
                  offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                  pool_bytes=int(1.3 * D * (N + 64 * C + 400 * T) * HD * 4), max_slots=max(4096, 4 * D * C),
                  max_cluster_pages=512, max_tokens=T)
kv = ClusterKVCache(cfg, HD, D)
st = workload.clustered_state(D, N, C, HD, T, seed=42)
kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
if DRIFT:
    fk, fv, fvis, fids = workload.frames_drift(st, F, N // T + 1 + 100000, seed=7)
else:
    fk, fv, fvis, fids = workload.frames_near(st, F, N // T + 1, seed=7)
names = ["argmax", "hot", "eq34", "entries", "chain", "pending", "commit", "keys"]
out = []
kv.set_timing(True)
for i in range(F):
    kv.process_frame(int(fids[i]), fvis[i], fk[i], fv[i], want_assigned=True)
    tm = kv.ingest_timing()
    p = kv.resolve_profile()
    tok = max(p[10], 1)
    out.append({"kernels_us": dict(zip(["cands", "assign", "topm", "resolve", "store_rows"], np.round(tm[:5], 1).tolist())),
                "resolve_us": round(float(tm[3]), 1), "tokens_per_domain": round(float(p[10]), 1),
                "cycles_per_token": {n: round(float(p[k]) / tok, 1) for k, n in enumerate(names)},
                "slow_per_token": round(float(p[8]) / tok, 2), "entries_per_token": round(float(p[11]) / tok, 2)})
kv.set_timing(False)
print(json.dumps({"domains": D, "frames": out}, indent=1))
