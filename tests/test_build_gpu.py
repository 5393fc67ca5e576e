"""Batch index build on the GPU (kmeans_dev.cu): spherical k-means of many point sets in one launch,
bit-identical to the host restatement (kmeans.cpp) and, where it is built, the reference
(clustering.cpp:80-178) -- assignments, live count, iteration count and the fp64 objective."""
import zlib

import numpy as np
import pytest

from oracle import pyoracle as po
from paper_2604_10060_b200 import api
from tests.harness import product_config

pytestmark = pytest.mark.gpu


def _kv(d):
    from paper_2604_10060_b200 import ClusterKVCache

    return ClusterKVCache(product_config(po.config1_engine()), d, 2)


def _set(kind, n, d, rng):
    if kind == "normal":
        return rng.standard_normal((n, d)).astype(np.float32)
    if kind == "blobs":
        c = rng.standard_normal((6, d)).astype(np.float32)
        return (c[rng.integers(0, 6, n)] + 0.05 * rng.standard_normal((n, d))).astype(np.float32)
    if kind == "dups":  # 3 directions, many clusters: empty clusters and reseeds
        base = rng.standard_normal((3, d)).astype(np.float32)
        return base[rng.integers(0, 3, n)].copy()
    if kind == "same":
        v = rng.standard_normal(d).astype(np.float32)
        return np.repeat(v[None], n, 0)
    raise ValueError(kind)


SETS = [("normal", 1, 1), ("normal", 5, 8), ("normal", 64, 4), ("normal", 300, 16), ("blobs", 1568, 49),
        ("dups", 200, 12), ("same", 40, 5), ("normal", 2, 2), ("blobs", 700, 22), ("normal", 1000, 1)]


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("iters,tol", [(50, 1e-6), (3, 1e-6), (50, 0.0), (0, 1e-6)])
def test_batch_kmeans_matches_host(d, iters, tol):
    rng = np.random.default_rng(zlib.crc32(f"{d}{iters}{tol}".encode()))
    sets = [_set(kind, n, d, rng) for kind, n, _ in SETS]
    ks = [k for _, _, k in SETS]
    seeds = [int(rng.integers(0, 2**63)) for _ in SETS]
    kv = _kv(d)
    got = kv.debug_kmeans(sets, ks, seeds, iters, tol)
    for (kind, n, k), pts, seed, (a, live, it, obj) in zip(SETS, sets, seeds, got):
        ha, hlive, hobj, hit = api.host_kmeans(pts, k, iters, tol, seed)
        assert np.array_equal(a, ha), (kind, n, k)
        assert (live, it) == (hlive, hit), (kind, n, k)
        assert obj == hobj, (kind, n, k, obj, hobj)


def test_batch_kmeans_matches_reference(ref_lib):
    rng = np.random.default_rng(3)
    sets = [rng.standard_normal((n, 128)).astype(np.float32) for n in (50, 400, 1568)]
    ks, seeds = [4, 13, 49], [11, 22, 33]
    got = _kv(128).debug_kmeans(sets, ks, seeds, 50, 1e-6)
    import ctypes as C

    for pts, k, seed, (a, live, it, obj) in zip(sets, ks, seeds, got):
        ra = np.zeros(len(pts), np.int32)
        robj, rit = C.c_double(), C.c_int()
        rlive = ref_lib.ref_prim_kmeans(po._p(pts, po.f32p), len(pts), 128, k, 50, 1e-6, seed, po._p(ra, po.i32p),
                                        C.byref(robj), C.byref(rit))
        assert np.array_equal(a, ra)
        assert (live, it, obj) == (rlive, rit.value, robj.value)


def test_batch_kmeans_zero_vector_raises():
    pts = np.random.default_rng(0).standard_normal((30, 64)).astype(np.float32)
    pts[7] = 0
    with pytest.raises(api.KvcError):
        _kv(64).debug_kmeans([pts], [4], [1])


def test_build_device_equals_host_build(monkeypatch):
    """The whole index build (visual partitions + per-(partition, layer) k-means) with the device
    k-means and with the host one: identical clusters, members and statistics."""
    from paper_2604_10060_b200 import ClusterKVCache

    s = po.gen_stream_restated(po.config1_stream())
    ecfg = po.config1_engine()

    def build(host):
        if host:
            monkeypatch.setenv("KVC_BUILD_HOST", "1")
        else:
            monkeypatch.delenv("KVC_BUILD_HOST", raising=False)
        kv = ClusterKVCache(product_config(ecfg), s.d, s.L)
        for kind, i in s.events():
            if kind == "frame":
                kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
        kv.build_now()
        ids = kv.cluster_ids()
        return [(c, kv.cluster(c)) for c in ids]

    dev, host = build(False), build(True)
    assert len(dev) == len(host)
    for (ca, a), (cb, b) in zip(dev, host):
        assert ca == cb
        assert np.array_equal(a[0], b[0]) and a[1] == b[1]
        assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
