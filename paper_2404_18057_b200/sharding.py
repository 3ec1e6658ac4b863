"""Multi-GPU partitioning of the decode-attention work.

The units of the path are independent (batch row, KV head) pairs: scoring,
selection, recall and P.V never cross units (proj/core/src/attention.cpp:
134-154,160-188). Each GPU therefore owns a shard of units -- its K slice in
HBM and its V slice in its own pinned host arena -- and the hot path needs no
collective. NCCL (or gloo on CPU) is used only to gather the [batch, d] outputs
to one rank for verification.

Two partitions:
* ``partition_batch``: whole request rows per rank (bench.py ``--shard
  batch``: each rank serves its own batch, weak scaling);
* ``partition_units``: contiguous runs of (batch, kv head) units, balanced to
  within one unit, for a fixed global batch split across ranks (bench.py
  ``--shard units``, strong scaling, e.g. config 3's 32 x 8 units).

A rank's unit shard is served by ONE TieredKVCache whose "sequence" is the
rank's units laid side by side: batch 1, n_kv_heads = units, n_heads =
units x G (``UnitShard``). The store's arena is [row][pos][h] per layer with
row = (batch, kv head), so a unit is a row either way and every kernel does
per unit exactly what it does in the unsharded cache; with the same split
length (``kc_score_chunk_plan`` of the unsharded shape) the shard's outputs
are bit-identical to the unsharded call's (tests/test_gpu_multirank.py).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def partition_batch(global_batch: int, world: int, rank: int) -> Tuple[int, int]:
    """(first row, row count) of ``rank``'s share of the request batch."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def partition_units(batch: int, n_kv: int, world: int, rank: int) -> List[Tuple[int, int]]:
    """(batch row, kv head) units of ``rank``: a contiguous run of the
    batch-major unit order, sizes differing by at most one."""
    total = batch * n_kv
    start, count = partition_batch(total, world, rank)
    return [divmod(u, n_kv) for u in range(start, start + count)]


def units_by_row(units: List[Tuple[int, int]]) -> dict:
    """{batch row: [kv heads]} for building one cache per rank."""
    out: dict = {}
    for b, k in units:
        out.setdefault(b, []).append(k)
    return out


class UnitShard:
    """The (batch row, kv head) units of one rank as one flattened cache.

    Unit u = (b, k) becomes kv head u of a batch-1 cache: its K/V columns are
    K[pos*B + b, k*h:(k+1)*h], its G q heads are q[b, k*G*h:(k+1)*G*h]."""

    def __init__(self, batch: int, n_kv: int, group: int, head_dim: int, world: int, rank: int):
        self.batch, self.n_kv, self.G, self.h = batch, n_kv, group, head_dim
        self.units = partition_units(batch, n_kv, world, rank)
        self.world, self.rank = world, rank

    @property
    def n_units(self) -> int:
        return len(self.units)

    def model_config(self, kc, n_layers: int, max_seq: int):
        """ModelConfig of the rank's cache (kc = the kcache module)."""
        n = self.n_units * self.G
        d = n * self.h
        return kc.ModelConfig(n_layers, d, n, self.h, kc.ModelConfig.default_ffn_hidden(d), 32000, max_seq,
                              self.n_units)

    def _index(self, x):
        """(batch rows, kv heads) of the units as index arrays of x's kind."""
        b = [u[0] for u in self.units]
        k = [u[1] for u in self.units]
        if isinstance(x, np.ndarray):
            return np.array(b), np.array(k)
        import torch
        return torch.tensor(b, device=x.device), torch.tensor(k, device=x.device)

    def kv_rows(self, kv_full):
        """[s*B, n_kv*h] position-major K or V rows -> the shard's [s, units*h]."""
        s = kv_full.shape[0] // self.batch
        b, k = self._index(kv_full)
        x = kv_full.reshape(s, self.batch, self.n_kv, self.h)[:, b, k, :]
        return x.reshape(s, self.n_units * self.h)

    def q_rows(self, q_full):
        """[B, n_kv*G*h] q -> the shard's [1, units*G*h]."""
        b, k = self._index(q_full)
        x = q_full.reshape(self.batch, self.n_kv, self.G * self.h)[b, k, :]
        return x.reshape(1, self.n_units * self.G * self.h)

    def slots(self):
        """Global (batch, q head) slot of each of the shard's q heads, in order."""
        return [b * self.n_kv * self.G + k * self.G + g for b, k in self.units for g in range(self.G)]


def gather_units(local_out, shard: "UnitShard", group=None):
    """All-gather of every rank's shard output ([1, units*G*h] or [units*G, h])
    into the full [B, n_kv*G*h] output on every rank (torch tensors; gloo or
    NCCL). Verification only: the decode path itself never calls it."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    gh = shard.G * shard.h
    counts = [len(partition_units(shard.batch, shard.n_kv, world, r)) for r in range(world)]
    pad = max(counts)
    buf = torch.zeros(pad, gh, dtype=local_out.dtype, device=local_out.device)
    buf[: shard.n_units] = local_out.reshape(shard.n_units, gh)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    # units are contiguous in batch-major order: rank r's units follow rank r-1's
    full = torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
    return full.reshape(shard.batch, shard.n_kv * gh)


def gather_rows(local, global_batch: int, group=None):
    """All-gather of per-rank output rows ([rows_r, d] tensors, rank-ordered
    shares of ``partition_batch``) into the full [global_batch, d] tensor on
    every rank. Verification only: the decode path itself never calls it."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [partition_batch(global_batch, world, r)[1] for r in range(world)]
    width = local.shape[1]
    pad = max(counts)
    buf = torch.zeros(pad, width, dtype=local.dtype, device=local.device)
    buf[: local.shape[0]] = local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def gpu_numa_node(device: int) -> int:
    """NUMA node of CUDA device ``device`` from sysfs (-1 when unknown): the
    node its pinned V arena is bound to, so each GPU's recall reads host
    memory local to its own PCIe root."""
    try:
        import torch
        p = torch.cuda.get_device_properties(device)
        bdf = "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
        with open(f"/sys/bus/pci/devices/{bdf}/numa_node") as f:
            node = int(f.read().strip())
        return node if node >= 0 else -1
    except Exception:
        return -1


def host_mem_available() -> int:
    """MemAvailable of this host in bytes (0 when unknown)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def max_over_ranks(values, device=None):
    """Element-wise max of per-rank timings over the default process group
    (bench.py: the job's step time is the slowest rank's). A list of floats
    in, the reduced list out; identity without an initialised group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]
