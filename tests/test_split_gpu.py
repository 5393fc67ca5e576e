"""GPU split_two (split.cu) -- the maintenance split's 2-way spherical k-means on the device --
bit-identical to the host restatement (kmeans.cpp) and, where it is built, the reference
(clustering.cpp:180-208): assignments, live count, iterations and the fp64 objective."""
import zlib

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2604_10060_b200 import api
from tests.harness import Replay, product_config

pytestmark = pytest.mark.gpu


def _kv(d):
    from paper_2604_10060_b200 import ClusterKVCache

    return ClusterKVCache(product_config(po.config1_engine()), d, 2)


def _points(kind, n, d, rng):
    if kind == "normal":
        return rng.standard_normal((n, d)).astype(np.float32)
    if kind == "blobs":  # two tight groups: converges in a few iterations
        c = rng.standard_normal((2, d)).astype(np.float32)
        lab = rng.integers(0, 2, n)
        return (c[lab] + 0.05 * rng.standard_normal((n, d))).astype(np.float32)
    if kind == "dups":  # three distinct directions repeated: exact ties everywhere
        base = rng.standard_normal((3, d)).astype(np.float32)
        return base[rng.integers(0, 3, n)].copy()
    if kind == "same":  # all equal up to scale: the degenerate (n-1, 1) partition
        v = rng.standard_normal(d).astype(np.float32)
        return (v[None, :] * rng.uniform(0.5, 2.0, (n, 1))).astype(np.float32)
    if kind == "tiny":  # small magnitudes (norms ~1e-6, above the 1e-12 cut)
        return (1e-7 * rng.standard_normal((n, d))).astype(np.float32)
    if kind == "one_off":  # all identical but one point
        p = np.repeat(rng.standard_normal((1, d)).astype(np.float32), n, 0)
        p[n // 2] = rng.standard_normal(d)
        return p
    raise ValueError(kind)


CASES = [("normal", 2, 8), ("normal", 3, 16), ("normal", 64, 64), ("normal", 257, 112), ("normal", 1000, 128),
         ("normal", 2048, 256), ("blobs", 700, 128), ("dups", 300, 64), ("dups", 2, 32), ("same", 50, 128),
         ("same", 2, 16), ("tiny", 200, 96), ("one_off", 129, 128), ("normal", 4096, 112)]


@pytest.mark.parametrize("kind,n,d", CASES)
def test_device_split_matches_host(kind, n, d):
    rng = np.random.default_rng(zlib.crc32(f"{kind}{n}{d}".encode()))
    pts = _points(kind, n, d, rng)
    kv = _kv(d)
    for seed in (1, 0x9E3779B97F4A7C15, 12345):
        a, live, iters, deg, obj = kv.debug_split_two(pts, seed)
        ha, hdeg = api.host_split_two(pts, seed)
        assert np.array_equal(a, ha), (kind, n, d, seed)
        assert deg == hdeg
        assert live == len(np.unique(ha))
        if not hdeg:  # the same spherical k-means: objective and iteration count bit-exact
            ka, klive, kobj, kit = api.host_kmeans(pts, 2, 50, 1e-9, seed)
            assert np.array_equal(ka, ha)
            assert (live, iters) == (klive, kit)
            assert obj == kobj, (obj, kobj)
        else:
            assert (live, iters, obj) == (2, 0, 1.0)


def test_device_split_matches_reference(ref_lib):
    rng = np.random.default_rng(5)
    kv = _kv(128)
    for n in (2, 33, 500, 1500):
        pts = rng.standard_normal((n, 128)).astype(np.float32)
        a = kv.debug_split_two(pts, n * 7919)[0]
        ra = np.zeros(n, np.int32)
        ref_lib.ref_prim_split_two(po._p(pts, po.f32p), n, 128, n * 7919, po._p(ra, po.i32p))
        assert np.array_equal(a, ra)


def test_device_split_zero_vector_raises():
    pts = np.random.default_rng(0).standard_normal((40, 64)).astype(np.float32)
    pts[17] = 0
    kv = _kv(64)
    with pytest.raises(api.KvcError):
        kv.debug_split_two(pts, 3)
    # the context stays usable
    pts[17] = 1
    kv.debug_split_two(pts, 3)


def test_config1_all_splits_on_device(monkeypatch):
    """The config-1 stream (~360 online splits) with every split of >= 2 rows on the GPU: routing,
    selections and digests stay bit-exact with the reference / restatement."""
    monkeypatch.setenv("KVC_SPLIT_DEV_MIN", "2")
    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine()
    ref = po.RefDriver(ecfg, s.d, s.L, checks=False) if po.reference() is not None else None
    r = Replay(s, ecfg, ref, None).run(check_attention=True)
    r.final_compare()
    assert r.mismatches == [], r.mismatches[:5]
    assert r.att_err < 1e-3
