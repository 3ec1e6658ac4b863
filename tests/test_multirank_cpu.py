"""CPU, world_size 2 over gloo: the multi-GPU partition logic.

Each rank computes its shard of the decode step (here with the CPU oracle,
standing in for its GPU) from the shared SeededRng streams, the outputs are
gathered with the same helper the multi-GPU verification uses, and rank 0
checks them against the unsharded computation. Also checks that
partition_units / partition_batch cover every unit exactly once.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2404_18057_b200.sharding import partition_batch, partition_units, units_by_row


def test_partitions_cover_units_once():
    for batch, n_kv, world in [(8, 32, 8), (32, 8, 8), (3, 5, 2), (1, 8, 4), (7, 1, 3)]:
        seen = []
        for r in range(world):
            seen += partition_units(batch, n_kv, world, r)
        assert sorted(seen) == [(b, k) for b in range(batch) for k in range(n_kv)]
        sizes = [len(partition_units(batch, n_kv, world, r)) for r in range(world)]
        assert max(sizes) - min(sizes) <= 1
        rows = [partition_batch(batch, world, r) for r in range(world)]
        assert sum(c for _, c in rows) == batch
        assert all(rows[i][0] + rows[i][1] == rows[i + 1][0] for i in range(world - 1))
    assert units_by_row([(0, 1), (0, 2), (1, 0)]) == {0: [1, 2], 1: [0]}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result):
    import torch
    import torch.distributed as dist

    from oracle.oracle import Restatement, synth_matrix
    from paper_2404_18057_b200.sharding import gather_rows, partition_batch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora = Restatement()
    B, n, h, s, N = 5, 4, 16, 40, 7
    d = n * h
    q = synth_matrix(1, B, d)
    k = synth_matrix(2, s * B, d)
    v = synth_matrix(3, s * B, d)
    start, cnt = partition_batch(B, world, rank)
    rows = list(range(start, start + cnt))
    # the rank's shard: its request rows (position-major rows of those batches)
    ksh = k.reshape(s, B, d)[:, rows].reshape(s * cnt, d)
    vsh = v.reshape(s, B, d)[:, rows].reshape(s * cnt, d)
    out, idx, w, dr = ora.decode_topn(q[rows], ksh, vsh, cnt, n, n, h, s, N, False)
    full = gather_rows(torch.from_numpy(out), B)
    if rank == 0:
        ref_out = ora.decode_topn(q, k, v, B, n, n, h, s, N, False)[0]
        result.put(bool(np.array_equal(full.numpy(), ref_out)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_sharded_step_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert all(p.exitcode == 0 for p in procs)


def _units_worker(rank, world, port, result):
    """sharding.UnitShard over the CPU oracle: each rank serves a contiguous run
    of (batch, kv head) units as one flattened batch-1 cache (GQA group 2)."""
    import torch
    import torch.distributed as dist

    from oracle.oracle import Restatement, synth_matrix
    from paper_2404_18057_b200.sharding import UnitShard, gather_units

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ora = Restatement()
    B, n, n_kv, h, s, N = 3, 6, 3, 16, 40, 7
    G = n // n_kv
    q = synth_matrix(1, B, n * h)
    k = synth_matrix(2, s * B, n_kv * h)
    v = synth_matrix(3, s * B, n_kv * h)
    sh = UnitShard(B, n_kv, G, h, world, rank)
    out = ora.decode_topn(sh.q_rows(q), sh.kv_rows(k), sh.kv_rows(v), 1, sh.n_units * G, sh.n_units, h, s, N,
                          False)[0]
    full = gather_units(torch.from_numpy(out), sh)
    if rank == 0:
        ref_out = ora.decode_topn(q, k, v, B, n, n_kv, h, s, N, False)[0]
        result.put(bool(np.array_equal(full.numpy(), ref_out)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gloo_world2_unit_shards_match_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_units_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert all(p.exitcode == 0 for p in procs)


def _max_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2404_18057_b200.sharding import max_over_ranks
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        got = max_over_ranks([10.0 + rank, 5.0 - rank, 1.5])
        out.put((rank, got))
    finally:
        dist.destroy_process_group()


def test_bench_timing_is_the_slowest_rank():
    """bench.py's step time is the element-wise max over ranks (gloo, world 2)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_max_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res[0] == res[1] == [11.0, 5.0, 1.5]
