import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload
for tile in ("tc", "simt"):
    if tile == "simt": os.environ["KVC_ASSIGN"] = "simt"
    else: os.environ.pop("KVC_ASSIGN", None)
    L, N, C, d, T = 4, 50_000, 256, 128, 196
    cfg = Config.make(kv_dtype=DTYPE_BF16, build_batch_frames=1, max_tokens=T, max_cluster_pages=512, pool_bytes=1 << 30, max_slots=8192)
    kv = ClusterKVCache(cfg, d, L)
    st = workload.clustered_state(L, N, C, d, T, seed=3)
    kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
    keys = workload.frames_near(st, 1, 10_000)[0][0]
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    k = torch.randn(L, T, d, generator=g, device="cuda"); rk = (k / k.norm(dim=-1, keepdim=True)).to(torch.bfloat16)
    print(tile, "near", kv.assign_check(keys.contiguous(), 0), "random", kv.assign_check(rk.contiguous(), 0))
