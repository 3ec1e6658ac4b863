"""GPU, world_size 2 over gloo: the (batch, kv head) unit partition of
SURVEY.md 8(e) running the CUDA product.

Both ranks drive their own TieredKVCache on cuda:0 (one GPU in this run)
holding only their units (sharding.UnitShard: batch 1, the rank's units as kv
heads), with the unsharded cache's split length (kc_score_chunk_plan). The
per-rank outputs, selections and dropped mass are all-gathered over gloo
(sharding.gather_units) and rank 0 checks them BIT FOR BIT against the
unsharded GPU call; the per-rank H2D ledgers add up to the unsharded one.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


CASES = {
    "mha": dict(B=3, n=8, n_kv=8, h=128, s=1500, N=64, L=2, renorm=False),
    "gqa4": dict(B=5, n=8, n_kv=2, h=128, s=2100, N=48, L=2, renorm=True),
}


def _worker(rank, world, port, case, result):
    import torch
    import torch.distributed as dist

    from oracle.oracle import synth_matrix
    from paper_2404_18057_b200 import kcache as kc
    from paper_2404_18057_b200.sharding import UnitShard, gather_units

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = CASES[case]
        B, n, n_kv, h, s, N, L = (c[x] for x in ("B", "n", "n_kv", "h", "s", "N", "L"))
        G = n // n_kv
        chunk = kc.score_chunk_plan(s, B * n_kv, G)
        shard = UnitShard(B, n_kv, G, h, world, rank)
        cache = kc.TieredKVCache(shard.model_config(kc, L, s), 1, kc.TierPlacement.kcache(0, L, 2, "f16"))
        cache.set_tuning("score_chunk", chunk)
        ks = [synth_matrix(2 + 100 * l, s * B, n_kv * h) for l in range(L)]
        vs = [synth_matrix(3 + 100 * l, s * B, n_kv * h) for l in range(L)]
        qs = [synth_matrix(1 + 100 * l, B, n * h) for l in range(L)]
        for l in range(L):
            cache.append_kv(l, shard.kv_rows(ks[l]), shard.kv_rows(vs[l]))
            cache.offload_prefill_v(l)
        cache.begin_decode()
        outs, sels, drops, h2d = [], [], [], 0
        for l in range(L):
            r = kc.decode_attention_topn(shard.q_rows(qs[l]), cache, l, N, c["renorm"])
            outs.append(gather_units(torch.from_numpy(r.out), shard).numpy())
            nc = r.selection.indices.shape[1]
            gi = gather_units(torch.from_numpy(r.selection.indices.astype(np.int64)).reshape(shard.n_units, G * nc),
                              _ShardView(shard, G * nc))
            gd = gather_units(torch.from_numpy(r.selection.dropped_mass).reshape(shard.n_units, G),
                              _ShardView(shard, G))
            sels.append(gi.numpy().reshape(B * n, nc))
            drops.append(gd.numpy().reshape(B * n))
            h2d += r.h2d_bytes
        cache.close()
        h2d_all = [0] * world
        dist.all_gather_object(h2d_all, h2d)
        if rank == 0:
            full = kc.TieredKVCache(kc.small_config(L, n * h, n, s, kv_heads=n_kv), B,
                                    kc.TierPlacement.kcache(0, L, 2, "f16"))
            ok = True
            ref_h2d = 0
            for l in range(L):
                full.append_kv(l, ks[l], vs[l])
                full.offload_prefill_v(l)
            full.begin_decode()
            for l in range(L):
                r = kc.decode_attention_topn(qs[l], full, l, N, c["renorm"])
                ok &= np.array_equal(outs[l], r.out)
                ok &= np.array_equal(sels[l], r.selection.indices.astype(np.int64))
                ok &= np.array_equal(drops[l], r.selection.dropped_mass)
                ref_h2d += r.h2d_bytes
            full.close()
            result.put((bool(ok), sum(h2d_all), ref_h2d))
        dist.barrier()
    finally:
        dist.destroy_process_group()


class _ShardView:
    """gather_units over per-unit rows of another width (selections, dropped)."""

    def __init__(self, shard, width):
        self.batch, self.n_kv, self.units, self.n_units = shard.batch, shard.n_kv, shard.units, shard.n_units
        self.G, self.h = 1, width


@pytest.mark.timeout(600)
@pytest.mark.parametrize("case", sorted(CASES))
def test_unit_shards_on_gpu_equal_unsharded_bitwise(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, h2d_sum, h2d_ref = q.get(timeout=500)
    for p in procs:
        p.join(timeout=60)
    assert ok
    assert h2d_sum == h2d_ref
    assert all(p.exitcode == 0 for p in procs)
