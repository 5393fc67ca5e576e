"""Fused output exchange (kvc_set_peers) with two ranks sharing one GPU: each rank owns half the
domains; the attention kernel stores every finished output row into both ranks' exchange buffers
through CUDA IPC mappings, and a signal/wait pair orders the steps. Every rank's gathered output
must equal the concatenation of the ranks' own outputs, step after step (the decode pipeline runs
asynchronously, so steps overlap the exchange)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CFG = dict(n_scenes=3, frames_per_scene=8, tokens_per_frame=24, d=64, L=4, n_queries=6, semantic_noise=0.05,
           queries_at_end=0, seed=21)


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import pyoracle as po
    from paper_2604_10060_b200 import ClusterKVCache
    from paper_2604_10060_b200.sharding import FusedExchange, shard_domains
    from tests.harness import product_config

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        s = po.gen_stream_restated(po.StreamCfg.make(**CFG))
        a, b = shard_domains(s.L, world, rank)
        ecfg = po.EngineCfg.make(build_batch_frames=6, offload_horizon_frames=4)
        kv = ClusterKVCache(product_config(ecfg, parity_mode=0, check_invariants=0), s.d, b - a)
        ex = FusedExchange(kv, s.L)
        mine, full = [], []
        for kind, i in s.events():
            if kind == "frame":
                kv.process_frame(i, s.visual[i], np.ascontiguousarray(s.keys[i][a:b]),
                                 np.ascontiguousarray(s.values[i][a:b]))
            else:
                qd = torch.from_numpy(np.ascontiguousarray(s.q[i][a:b])).cuda()
                o = torch.zeros(b - a, s.d, device="cuda")
                g = torch.zeros(s.L, s.d, device="cuda")
                torch.cuda.synchronize()
                kv.query(i, qd, out=o)
                ex.gathered(g)
                stream = torch.cuda.ExternalStream(kv.stream)
                stream.synchronize()
                mine.append(o.cpu().numpy())
                full.append(g.cpu().numpy())
        allmine = [None] * world
        dist.all_gather_object(allmine, mine)
        ok = all(np.array_equal(full[t], np.concatenate([allmine[r][t] for r in range(world)], 0))
                 for t in range(len(full)))
        q.put((rank, ok, len(full)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, repr(e), 0))


def test_two_ranks_on_one_gpu():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, n in res:
        assert ok is True, (rank, ok)
        assert n > 0
