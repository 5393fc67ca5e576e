"""GPU split_two (split.cu) vs the host restatement, d = 128 (development measurement).

    python scripts/split_time.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np
from oracle import pyoracle as po
from paper_2604_10060_b200 import api, ClusterKVCache
from tests.harness import product_config
for n, d in ((64, 128), (256, 128), (1024, 128), (4096, 128)):
    kv = ClusterKVCache(product_config(po.config1_engine()), d, 2)
    pts = np.random.default_rng(n).standard_normal((n, d)).astype(np.float32)
    kv.debug_split_two(pts, 1)
    t = time.perf_counter(); r = [kv.debug_split_two(pts, s) for s in range(5)]; tg = (time.perf_counter() - t) / 5
    t = time.perf_counter(); [api.host_split_two(pts, s) for s in range(5)]; th = (time.perf_counter() - t) / 5
    print(n, d, "iters", [x[2] for x in r], f"gpu {tg*1e3:.2f} ms host {th*1e3:.2f} ms")
