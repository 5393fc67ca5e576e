"""Per-shard parity of the multi-GPU layout: two ranks (processes, gloo process
group, both on cuda:0 here -- the same code runs one rank per GPU) each own a contiguous block of
the config-1 stream's 8 domains with their own context, and each rank is checked against ITS OWN
reference instance over the same domain subset (the reference's split counter and LRU are per
instance, maintainer.cpp:222 / store.cpp:144-181, so a single-process reference is not
decomposable into shards). Per frame: routed ids; per step: ranked / selected / digest and the
attention outputs vs the fp64 restatement; at the end: every cluster bitwise. The fused output
exchange (K6 storing every finished row into every rank's buffer through CUDA IPC) must hand
each rank the concatenation of all ranks' outputs."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import pyoracle as po
    from paper_2604_10060_b200 import ClusterKVCache
    from paper_2604_10060_b200.sharding import FusedExchange, shard_domains
    from tests.harness import attention_oracle, compare_state, product_config, rel_err

    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        s = po.gen_stream_restated(po.config1_stream())
        a, b = shard_domains(s.L, world, rank)
        ecfg = po.config1_engine()
        kv = ClusterKVCache(product_config(ecfg), s.d, b - a)
        ref = po.RefDriver(ecfg, s.d, b - a, checks=False)
        ex = FusedExchange(kv, s.L)
        g = torch.zeros(s.L, s.d, device="cuda")
        torch.cuda.synchronize()  # the context's stream does not order after torch's stream
        mism, att_err, mine, full = [], 0.0, [], []
        for kind, i in s.events():
            if kind == "frame":
                k = np.ascontiguousarray(s.keys[i][a:b])
                v = np.ascontiguousarray(s.values[i][a:b])
                pid, asg = kv.process_frame(i, s.visual[i], k, v)
                rpid, rasg = ref.frame(i, s.visual[i], k, v)
                if pid != rpid or not np.array_equal(asg, rasg):
                    mism.append(("frame", i))
            else:
                qq = np.ascontiguousarray(s.q[i][a:b])
                out = kv.query(i, qq, gt=s.gt[i])
                ref.query(i, qq, s.gt[i])
                for l in range(b - a):
                    if kv.ranked(l) != ref.ranked(l) or kv.selected(l) != ref.selected(l):
                        mism.append(("query", i, l))
                    fr, tk = ref.attended(l)
                    att_err = max(att_err, rel_err(out[l], attention_oracle(s, fr, tk, a + l, qq[l])))
                if kv.digest() != ref.digest():
                    mism.append(("digest", i))
                ex.gathered(g)
                torch.cuda.ExternalStream(kv.stream).synchronize()
                mine.append(out.copy())
                full.append(g.cpu().numpy())
        kv_ms, ref_ms = kv.maint_stats(), ref.maint_stats()
        if not np.array_equal(kv_ms, ref_ms):
            mism.append(("maint_stats", kv_ms.tolist(), ref_ms.tolist()))
        mism.extend(compare_state(kv, ref))
        allmine = [None] * world
        dist.all_gather_object(allmine, mine)
        exch_ok = all(np.array_equal(full[t], np.concatenate([allmine[r][t] for r in range(world)], 0))
                      for t in range(len(full)))
        q.put((rank, mism[:5], att_err, exch_ok, len(full), int(kv_ms[2] + kv_ms[3])))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        q.put((rank, [repr(e)], 1.0, False, 0, 0))


def test_each_rank_matches_its_own_reference_instance(ref_lib):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, mism, att_err, exch_ok, n, splits in res:
        assert mism == [], (rank, mism)
        assert att_err < 1e-3, (rank, att_err)
        assert exch_ok, rank
        assert n == 32 and splits > 0
