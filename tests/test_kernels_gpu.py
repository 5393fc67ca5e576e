"""Device self-checks of arithmetic building blocks the bit-exact kernels rely on."""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("max_den,seed", [(64, 1), (4096, 2), (1 << 20, 3), ((1 << 31) - 1, 4), (0, 5), (0, 6)])
def test_reciprocal_division_is_correctly_rounded(max_den, seed):
    """resolve_spec.cu div_rcp (RN(1/b) + two FMA remainder corrections) == __ddiv_rn, bit for
    bit, on 2^26 random operands per denominator range (Eq. 3/4 and the buffer mean divide by
    integer counts; max_den 0: real divisors with float numerators, the split k-means' unit rows
    x / |x|)."""
    from paper_2604_10060_b200.api import debug_div_check

    assert debug_div_check(1 << 26, seed, max_den) == 0


@pytest.mark.parametrize("tile", ["tc", "simt"])
@pytest.mark.parametrize("keys_kind", ["near", "random"])
def test_distance_tile_error_within_margin(tile, keys_kind, monkeypatch):
    """The approximate cosine tile (tcgen05 bf16 hi/lo or fp32 SIMT) stays well inside the margin
    the resolve kernels certify with, the top-M lists are consistent with the tile, and their
    exact values equal a fresh fp64 cosine (kvc_debug_assign_check)."""
    import torch

    from paper_2604_10060_b200 import ClusterKVCache, Config, DTYPE_BF16, workload

    if tile == "simt":
        monkeypatch.setenv("KVC_ASSIGN", "simt")
    else:
        monkeypatch.delenv("KVC_ASSIGN", raising=False)
    L, N, C, d, T = 4, 50_000, 256, 128, 196
    cfg = Config.make(kv_dtype=DTYPE_BF16, build_batch_frames=1, max_tokens=T, max_cluster_pages=512,
                      pool_bytes=1 << 30, max_slots=8192)
    kv = ClusterKVCache(cfg, d, L)
    st = workload.clustered_state(L, N, C, d, T, seed=3)
    kv.bulk_load(st.visual, st.keys, st.values, st.assign, st.frame_ids, st.token_ids, C)
    if keys_kind == "near":
        keys = workload.frames_near(st, 1, 10_000)[0][0]
    else:
        g = torch.Generator(device="cuda")
        g.manual_seed(5)
        k = torch.randn(L, T, d, generator=g, device="cuda")
        keys = (k / k.norm(dim=-1, keepdim=True)).to(torch.bfloat16)
    err, viol, mism, margin = kv.assign_check(keys.contiguous(), 0)
    assert viol == 0 and mism == 0
    assert err < margin / 4, (err, margin)
