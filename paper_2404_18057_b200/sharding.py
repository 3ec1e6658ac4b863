"""Multi-GPU partitioning of the decode-attention work.

The units of the path are independent (batch row, KV head) pairs: scoring,
selection, recall and P.V never cross units (proj/core/src/attention.cpp:
134-154,160-188). Each GPU therefore owns a shard of units -- its K slice in
HBM and its V slice in its own pinned host arena -- and the hot path needs no
collective. NCCL (or gloo on CPU) is used only to gather the [batch, d] outputs
to one rank for verification.

Two partitions:
* ``partition_batch``: whole request rows per rank (what bench.py uses: each
  rank serves its own batch, weak scaling);
* ``partition_units``: contiguous runs of (batch, kv head) units, balanced to
  within one unit, for a fixed global batch split across ranks (strong
  scaling, e.g. config 3's 32 x 8 units).
"""
from __future__ import annotations

from typing import List, Tuple


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
