"""World-size-2 (and 3) gloo runs of the one-process-per-GPU path on CPU:
rank ranges tile the walk, partials travel through torch.distributed, rank
0's fixed-order reduction matches a single-process reduction of the same
ranges bit for bit. The per-rank walk is the C oracle here (test
infrastructure); on the GPU box the same function walks on the rank's GPU."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
import paper_2502_16577_b200 as pk
from paper_2502_16577_b200.distributed import combine_real, rank_span
from paper_2502_16577_b200.precision import AccumulatorPolicy


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_walker(m, policy, lo, hi):
    a = np.array(m.data, dtype=np.float64).reshape(m.n, m.n)
    return oracle.dense_f64_range(a, lo, hi, policy.value)


def _worker(rank, world, port, n, policy, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_16577_b200.distributed import permanent_distributed
        m = pk.random_real(n, 31, 0.0, 1.0)
        v = permanent_distributed(m, policy, walker=_oracle_walker)
        q.put((rank, v.hex()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_ranks_reduce_like_one_process(world):
    n, policy = 16, "kahan"
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, policy, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = dict(q.get() for _ in range(world))
    assert len(set(got.values())) == 1  # every rank holds the same bits
    m = pk.random_real(n, 31, 0.0, 1.0)
    pol = AccumulatorPolicy.KAHAN
    parts = [_oracle_walker(m, pol, *rank_span(n, r, world)) for r in range(world)]
    assert got[0] == combine_real(m, pol, parts).hex()
    a = np.array(m.data).reshape(n, n)
    whole = oracle.dense_f64_permanent(a, "kahan", tau=1)
    assert abs(float.fromhex(got[0]) - whole) <= 1e-12 * abs(whole)


def test_rank_spans_tile_the_walk():
    for n in (2, 3, 5, 12, 20, 40, 63):
        for world in (1, 2, 3, 4, 8, 16):
            T = pk.total_iterates(n)
            pos = 1
            for r in range(world):
                lo, hi = rank_span(n, r, world)
                if lo > hi:
                    continue
                assert lo == pos
                pos = hi + 1
            assert pos == T + 1
            if world & (world - 1) == 0 and (1 << (n - 1)) >= 64 * world:
                lo, _ = rank_span(n, 1 % world, world)
                assert (lo - 1) % ((1 << (n - 1)) // world) == 0
