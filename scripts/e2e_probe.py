"""Decode-step wall time per step on the config-2 state: device buffers (synchronised per step)
vs pinned host buffers through the public API (the bench's e2e). Development measurement."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload  # noqa: E402

D, N, C, T, HD = 112, 669 * 196, 256, 196, 128
cfg = Config.make(kv_dtype=DTYPE_BF16, k_v=1, k_s=16, window_frames=4, build_batch_frames=1,
                  offload_horizon_frames=1 << 30, device_capacity_entries=1 << 40,
                  pool_bytes=int(1.2 * D * (N + 64 * C + 400 * T) * HD * 4), max_slots=4 * D * C,
                  max_cluster_pages=512, max_tokens=T)
kv = ClusterKVCache(cfg, HD, D)
st = workload.clustered_state(D, N, C, HD, T, seed=42)
kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
nq = 60
q = workload.queries_near(st, nq, seed=11)
out_d = torch.zeros(D, HD, device="cuda")
qh = q.cpu().pin_memory().numpy()
oh = torch.zeros(D, HD).pin_memory().numpy()
stream = torch.cuda.ExternalStream(kv.stream)
for i in range(5):
    kv.query(i, q[i], out=out_d)
torch.cuda.synchronize()
def run(fn):
    t0 = time.perf_counter()
    for i in range(10, nq):
        fn(i)
    return (time.perf_counter() - t0) * 1e6 / (nq - 10)
r = {}
r["device_async"] = run(lambda i: kv.query(i, q[i], out=out_d)); torch.cuda.synchronize()
r["device_sync_each"] = run(lambda i: (kv.query(i, q[i], out=out_d), stream.synchronize()))
r["host_pinned"] = run(lambda i: kv.query(i, qh[i], out=oh))
r["host_q_dev_out"] = run(lambda i: (kv.query(i, qh[i], out=out_d), stream.synchronize()))
r["dev_q_host_out"] = run(lambda i: kv.query(i, q[i], out=oh))
print({k: round(v, 1) for k, v in r.items()})
