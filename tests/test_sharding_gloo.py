"""Multi-rank host logic on CPU (gloo, world_size 2): domain sharding + the output all-gather give
exactly the single-process decode outputs (fp64 attention oracle over each domain)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_10060_b200.sharding import gather_domain_outputs, shard_domains, shard_streams


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_out(rng_seed, D, n, d):
    from oracle import pyoracle as po

    lib = po.restatement()
    rng = np.random.default_rng(rng_seed)
    q = rng.standard_normal((D, d)).astype(np.float32)
    K = rng.standard_normal((D, n, d)).astype(np.float32)
    V = rng.standard_normal((D, n, d)).astype(np.float32)
    out = np.zeros((D, d))
    for l in range(D):
        o = np.zeros(d)
        lib.kvo_attend_f32(po._p(q[l], po.f32p), po._p(np.ascontiguousarray(K[l]), po.f32p),
                           po._p(np.ascontiguousarray(V[l]), po.f32p), n, d, d ** -0.5, po._p(o, po.f64p))
        out[l] = o
    return out


def _worker(rank, world, port, D, n, d, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = _oracle_out(5, D, n, d)  # every rank can regenerate the same synthetic inputs
    a, b = shard_domains(D, world, rank)
    local = torch.from_numpy(full[a:b].copy())
    gathered = gather_domain_outputs(local, D)
    q.put((rank, np.array_equal(gathered.numpy(), full)))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_domains_partition():
    for D in (8, 14, 112, 640, 113):
        for world in (1, 2, 4, 8):
            spans = [shard_domains(D, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == D
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard_domains(4, 8, 0)
    assert shard_streams(32, 8, 3) == [3, 11, 19, 27]


@pytest.mark.parametrize("D", [8, 7])
def test_gloo_world2_gather_equals_single_process(D):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, D, 33, 16, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]
