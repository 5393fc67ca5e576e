"""CPU tests of the product library without a GPU: the C-ABI loads and exports every entry point
include/kvc.h declares, refuses to run without a device (no CPU fallback), and its host slow
path (split / batch-build k-means, tau table, split seeds) is bit-exact with the reference."""
import os
import re

import numpy as np
import pytest

from paper_2604_10060_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "kvc.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"KVC_API\s+[\w\s\*]+?\b(kvc_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = api.lib()
    syms = declared_symbols()
    assert len(syms) >= 40
    missing = [s for s in syms if not hasattr(lib, s)]
    assert missing == []
    assert sorted(api.EXPORTED) == syms


def test_no_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(api.NoDevice):
        api.ClusterKVCache(api.Config.make(), 32, 2)


def test_config_defaults_match_reference_engine_config():
    """kvc_cfg_default == EngineConfig{} field for field (engine.hpp:21-33)."""
    from oracle import pyoracle as po

    ref = po.EngineCfg.make()
    mine = api.Config.make()
    for name, _ in po.EngineCfg._fields_:
        assert getattr(mine, name) == getattr(ref, name), name


def test_unknown_config_key_rejected():
    with pytest.raises(api.ConfigError):
        api.Config.make(not_a_key=1)


def test_host_tau_and_mix_seed_match_reference(ref_lib):
    lib = api.lib()
    for n in (0, 1, 7, 32, 100, 5000, 30000):
        assert lib.kvc_host_tau(n, 0.05, 0.3, 32.0) == ref_lib.ref_prim_tau(n, 0.05, 0.3, 32.0)
    for a, b in ((0, 2), (123, 0), (2**63 + 5, 77)):
        assert lib.kvc_host_mix_seed(a, b) == ref_lib.ref_prim_mix_seed(a, b)


def test_mt64_first_two_draws_shortcut():
    """The wave engine's k-means++ draws (kmeans.cpp mt64_first2) equal std::mt19937_64's first two
    outputs for the seeds mix_seed produces."""
    import ctypes as C

    lib = api.lib()
    rng = np.random.default_rng(5)
    seeds = [0, 1, 5489, 2**64 - 1] + [int(x) for x in rng.integers(0, 2**63, 200, dtype=np.int64)]
    seeds += [lib.kvc_host_mix_seed(42, c) for c in range(200)]
    f, r = (C.c_uint64 * 2)(), (C.c_uint64 * 2)()
    for sd in seeds:
        lib.kvc_host_rng_first2(sd, f, r)
        assert list(f) == list(r), sd


@pytest.mark.parametrize("n,d,seed", [(2, 8, 1), (3, 16, 2), (50, 32, 3), (400, 128, 4), (1000, 64, 5)])
def test_split_two_bit_exact(ref_lib, n, d, seed):
    """The split slow path (maintainer.cpp:195-242 -> clustering.cpp:180-208)."""
    from oracle import pyoracle as po

    rng = np.random.default_rng(seed)
    pts = rng.standard_normal((n, d)).astype(np.float32)
    if seed == 2:  # all-identical points: the degenerate (n-1, 1) rule
        pts[:] = pts[0]
    a, deg = api.host_split_two(pts, seed * 7919)
    ra = np.zeros(n, np.int32)
    rdeg = ref_lib.ref_prim_split_two(po._p(pts, po.f32p), n, d, seed * 7919, po._p(ra, po.i32p))
    assert np.array_equal(a, ra)
    assert deg == bool(rdeg)


@pytest.mark.parametrize("n,k,seed", [(64, 4, 1), (300, 16, 2), (196 * 4, 4, 3), (1000, 33, 4)])
def test_spherical_kmeans_bit_exact(ref_lib, n, k, seed):
    """Batch build (index.cpp:364-450 -> clustering.cpp:80-178)."""
    import ctypes as C

    from oracle import pyoracle as po

    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((k, 48))
    pts = (centers[rng.integers(0, k, n)] + 0.3 * rng.standard_normal((n, 48))).astype(np.float32)
    a, live, obj, it = api.host_kmeans(pts, k, 50, 1e-6, seed)
    ra = np.zeros(n, np.int32)
    robj = C.c_double()
    rit = C.c_int()
    rlive = ref_lib.ref_prim_kmeans(po._p(pts, po.f32p), n, 48, k, 50, 1e-6, seed, po._p(ra, po.i32p),
                                    C.byref(robj), C.byref(rit))
    assert np.array_equal(a, ra) and live == rlive and obj == robj.value and it == rit.value


def test_host_split_rejects_too_few_points():
    with pytest.raises(api.TooFewPoints):
        api.host_split_two(np.ones((1, 8), np.float32), 0)


def test_host_split_rejects_zero_vector():
    with pytest.raises(api.DegenerateVector):
        api.host_split_two(np.zeros((3, 8), np.float32), 0)


def test_cpp_dropin_library_exports_the_reference_api():
    """libkvclust_b200.so (the C++ drop-in) defines the reference's hot-path API in namespace
    kvclust: StreamEngine / run_stream (engine.hpp), HierIndex / build_index (index.hpp),
    TieredStore (store.hpp), Maintainer / updated_stats / tau (maintainer.hpp), retrieve /
    oracle_flat_topk / retrieve_token_baseline (retrieval.hpp)."""
    import subprocess

    lib = os.path.join(ROOT, "paper_2604_10060_b200", "_lib", "libkvclust_b200.so")
    if not os.path.exists(lib):
        pytest.skip("drop-in not built (needs the reference headers at build time)")
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    for sym in ["kvclust::run_stream(", "kvclust::StreamEngine::process(", "kvclust::StreamEngine::finish()",
                "kvclust::build_index(", "kvclust::HierIndex::semantic_topk(", "kvclust::HierIndex::visual_topk(",
                "kvclust::TieredStore::fetch(", "kvclust::Maintainer::on_insert(", "kvclust::Maintainer::place_frame(",
                "kvclust::Maintainer::materialize(", "kvclust::retrieve(", "kvclust::oracle_flat_topk(",
                "kvclust::retrieve_token_baseline(", "kvclust::updated_stats(", "kvclust::tau("]:
        assert sym in out, sym
