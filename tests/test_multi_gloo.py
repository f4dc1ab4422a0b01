"""Multi-process (world_size 2, gloo, CPU) coverage of the table-wise sharded
path: plan -> per-rank tables, the pooled-row all-to-all layout, and the
inverse gradient exchange. Each rank's local pooled block is produced by the
CPU oracle here (the device kernel is covered by the GPU parity tests); the
exchanged rows must equal the single-process oracle forward of all tables."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist

    import paper_2208_06399_b200 as P
    from oracle import Oracle
    from paper_2208_06399_b200.sharded import PooledExchange, a2a_layout, local_tables
    from helpers import to_oracle_tables

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        o = Oracle()
        pool = P.generate_pool(0, 7, P.GeneratorConfig(dim_choices=(16, 32, 64), hash_size_max=2e4,
                                                      pooling_mean_target=10.0))
        B = 67  # uneven sample split (B % world != 0)
        task = P.ShardingTask(pool, world, [10 ** 12] * world)
        plan = P.greedy_shard(task, P.HeuristicKind.kLookupGreedy)
        mine = local_tables(task, plan, rank)
        wl = P.generate_workload(0, mine, B)  # subset-stable streams
        st = [(wl.find(t.id).offsets, wl.find(t.id).indices) for t in mine]
        local = o.forward_f64(to_oracle_tables(mine), B, st, wseed=3).astype(np.float32)
        lay = a2a_layout(task, plan, B)
        ex = PooledExchange(lay, rank)
        recv = ex.forward(torch.from_numpy(local))
        # reference: all tables on one process, rows of this rank's samples
        wl_all = P.generate_workload(0, pool, B)
        st_all = [(wl_all.find(t.id).offsets, wl_all.find(t.id).indices) for t in pool]
        full = o.forward_f64(to_oracle_tables(pool), B, st_all, wseed=3).astype(np.float32)
        cols = np.cumsum([0] + [t.dim for t in pool])
        rows = slice(lay.row_start[rank], lay.row_start[rank + 1])
        ok = True
        for i, t in enumerate(pool):
            got = ex.table_rows(recv, i).numpy()
            ok &= np.array_equal(got, full[rows, cols[i]:cols[i] + t.dim])
        # inverse exchange: grad of recv = recv (loss 1/2|.|^2) -> own block back
        back = ex.backward(recv.clone())
        ok &= np.array_equal(back.numpy(), local)
        result_q.put((rank, bool(ok), [len(m) for m in lay.shard_tables]))
    finally:
        dist.destroy_process_group()


def test_two_rank_pooled_exchange_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res), res
    assert sum(res[0][2]) == 7


def test_layout_splits_and_locate(P):
    from paper_2208_06399_b200.sharded import a2a_layout

    pool = P.generate_pool(0, 10)
    task = P.ShardingTask(pool, 4, [10 ** 12] * 4)
    plan = P.random_shard(task, 3)
    lay = a2a_layout(task, plan, 4096)
    assert sum(lay.shard_dims) == sum(t.dim for t in pool)
    for r in range(4):
        assert sum(lay.send_splits(r)) == 4096 * lay.shard_dims[r]
    assert sum(lay.recv_splits(0)) == 1024 * sum(t.dim for t in pool)
    for i in range(10):
        k, col = lay.locate(i)
        assert plan.assignment[i] == k
    odd = a2a_layout(task, plan, 4095)  # uneven: 1024, 1024, 1024, 1023 rows
    assert odd.row_start == [0, 1024, 2048, 3072, 4095]
    assert sum(sum(odd.send_splits(r)) for r in range(4)) == 4095 * sum(odd.shard_dims)
    assert sum(sum(odd.recv_splits(r)) for r in range(4)) == 4095 * sum(odd.shard_dims)
    with pytest.raises(ValueError):
        a2a_layout(task, plan, 3)


def test_peer_bases_match_receive_layout():
    """as_set_peer_outputs addresses (fused exchange) = receive buffer + the owner's block offset."""
    import paper_2208_06399_b200 as P
    from paper_2208_06399_b200.sharded import a2a_layout, peer_bases

    pool = P.generate_pool(0, 9, P.GeneratorConfig(dim_choices=(16, 32, 64)))
    task = P.ShardingTask(pool, 3, [1 << 40] * 3)
    plan = P.random_shard(task, 2)
    lay = a2a_layout(task, plan, 97)  # rows 33, 32, 32
    bases = [1 << 20, 2 << 20, 3 << 20]
    for k in range(3):
        got = peer_bases(lay, k, bases)
        assert got == [b + 4 * lay.rows(q) * sum(lay.shard_dims[:k]) for q, b in enumerate(bases)]
