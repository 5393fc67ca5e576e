"""Index build time (index.cpp:364-450) at a config-2-like shape: build_batch_frames frames of
T tokens for L domains, then build_now() with the semantic k-means on the GPU (kmeans_dev.cu) or on
the host (KVC_BUILD_HOST=1). Development measurement; identical clusters are checked.

    python scripts/build_time.py [L] [frames]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 112
F = int(sys.argv[2]) if len(sys.argv) > 2 else 32
T, D = 196, 128
g = torch.Generator().manual_seed(1)
cent = torch.nn.functional.normalize(torch.randn(L, 64, D, generator=g), dim=-1)
frames = []
for f in range(F):
    idx = torch.randint(0, 64, (L, T), generator=g)
    k = torch.nn.functional.normalize(cent[torch.arange(L)[:, None], idx] + 0.1 * torch.randn(L, T, D, generator=g), dim=-1)
    v = torch.randn(L, T, D, generator=g)
    vis = torch.nn.functional.normalize(torch.randn(D, generator=g) + (f // 8) * 3.0, dim=0)
    frames.append((vis.numpy().astype(np.float32), k.bfloat16().contiguous(), v.bfloat16().contiguous()))


def run(host):
    if host:
        os.environ["KVC_BUILD_HOST"] = "1"
    else:
        os.environ.pop("KVC_BUILD_HOST", None)
    cfg = Config.make(kv_dtype=DTYPE_BF16, build_batch_frames=F + 1, max_tokens=T, window_frames=4,
                      pool_bytes=int(3 * L * F * T * D * 2 * 2), max_slots=max(65536, 4 * L * F * T // 16))
    kv = ClusterKVCache(cfg, D, L)
    for f, (vis, k, v) in enumerate(frames):
        kv.process_frame(f, vis, k, v, want_assigned=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    kv.build_now()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ids = kv.cluster_ids()
    sig = (len(ids), [kv.cluster(int(c))[1] for c in ids[:: max(1, len(ids) // 50)]])
    del kv
    return dt, sig


dev_t, dev_sig = run(False)
print(f"L={L} frames={F} rows/pool~{F * T // 4}: GPU build {dev_t * 1e3:.1f} ms, clusters {dev_sig[0]}", flush=True)
if os.environ.get("BUILD_HOST_TOO"):
    host_t, host_sig = run(True)
    print(f"host build {host_t * 1e3:.1f} ms; identical: {dev_sig == host_sig}; speed-up {host_t / dev_t:.1f}x")

if os.environ.get("BUILD_PROFILE"):
    import re

    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        run(False)
    agg = {}
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        m = re.search(r"\b(k_\w+)", e.name)
        agg.setdefault(m.group(1) if m else e.name[:40], []).append(e.device_time_total)
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1]))[:10]:
        print(f"{k:42s} n={len(v):6d} mean={np.mean(v):9.1f} us total={sum(v) / 1e3:9.1f} ms")
