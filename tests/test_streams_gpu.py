"""Independent streams (config 5): several contexts on one GPU, each on its own CUDA stream with its
own work counters, driven interleaved; their selections, digests and attention outputs must equal
those of each stream run alone (no cross-talk through shared device state)."""
import numpy as np
import pytest

from oracle import pyoracle as po
from tests.harness import product_config

pytestmark = pytest.mark.gpu

CFG = dict(n_scenes=3, frames_per_scene=10, tokens_per_frame=32, d=64, L=4, n_queries=8, semantic_noise=0.05,
           queries_at_end=0)


def _streams(n):
    return [po.gen_stream_restated(po.StreamCfg.make(seed=11 + i, **CFG)) for i in range(n)]


def _run_alone(s, ecfg, token):
    from paper_2604_10060_b200 import ClusterKVCache

    kv = ClusterKVCache(product_config(ecfg, token_mode=1 if token else 0, token_budget=64), s.d, s.L)
    res = []
    for kind, i in s.events():
        if kind == "frame":
            kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
        else:
            out = kv.query(i, s.q[i], gt=s.gt[i])
            res.append((kv.digest(), [kv.selected(l) for l in range(s.L)], out.copy()))
    return res


@pytest.mark.parametrize("token", [False, True])
def test_interleaved_streams_equal_isolated(token):
    import torch

    from paper_2604_10060_b200 import ClusterKVCache

    ss = _streams(3)
    ecfg = po.EngineCfg.make(build_batch_frames=6, offload_horizon_frames=4)
    alone = [_run_alone(s, ecfg, token) for s in ss]
    kvs = [ClusterKVCache(product_config(ecfg, token_mode=1 if token else 0, token_budget=64, parity_mode=0,
                                         check_invariants=0), s.d, s.L) for s in ss]
    evs = [list(s.events()) for s in ss]
    outs = [[] for _ in ss]
    for step in range(max(len(e) for e in evs)):
        for k, (s, kv) in enumerate(zip(ss, kvs)):
            if step >= len(evs[k]):
                continue
            kind, i = evs[k][step]
            if kind == "frame":
                kv.process_frame(i, s.visual[i], s.keys[i], s.values[i])
            else:  # asynchronous: device query / output, contexts overlap on the GPU
                qd = torch.from_numpy(np.ascontiguousarray(s.q[i])).cuda()
                o = torch.zeros(s.L, s.d, device="cuda")
                torch.cuda.synchronize()
                kv.query(i, qd, out=o)
                outs[k].append((o, qd))
    torch.cuda.synchronize()
    for k in range(len(ss)):
        assert len(outs[k]) == len(alone[k])
        for (o, _), (_, _, ref) in zip(outs[k], alone[k]):
            np.testing.assert_allclose(o.cpu().numpy(), ref, rtol=0, atol=1e-6)
