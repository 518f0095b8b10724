"""Multi-GPU sieve: block-cyclic p-row partitioning + cross-rank reduction.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch). Rows p are
grouped in the reference's p/100 blocks (the ScanStats::block_r_max key,
engine.hpp:229-236); rank g of G owns the blocks b with b % G == g, which
balances the linearly growing row lengths and keeps every block on one rank.
Each rank sieves its blocks into device buffers (cgpu_sieve_launch_dev) and
the ranks then combine exactly as ScanStats::merge does (engine.hpp:121-134):

    sum  : pairs_tested, survivors, first-killer histogram
    max  : block r_max (0 marks blocks a rank does not own)
    cat  : survivor lists, then sorted to canonical (p, q)

reduce_packed does all three in one all_reduce(SUM) (one owner per block, one
slice per rank); reduce_results + gather_survivors is the plain form.

The same reduction code runs on CPU tensors over gloo (tests) and on CUDA
tensors over NCCL (the product path and bench.py).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def owned_blocks(p_lo: int, p_hi: int, G: int, g: int) -> list[int]:
    """Blocks b = p // 100 in [p_lo // 100, p_hi // 100] with b % G == g."""
    if p_hi < p_lo:
        return []
    b0, b1 = p_lo // 100, p_hi // 100
    first = b0 + ((g - b0) % G)
    return list(range(first, b1 + 1, G))


def owned_rows(p_lo: int, p_hi: int, G: int, g: int):
    """(lo, hi) row intervals of rank g's shard, clipped to [p_lo, p_hi]."""
    return [(max(p_lo, 100 * b), min(p_hi, 100 * b + 99)) for b in owned_blocks(p_lo, p_hi, G, g)]


def reduce_results(acc, brm, group=None):
    """In place: acc = [pairs, survivors, hist...] (int64) summed over ranks,
    brm (int32 block r_max, 0 = not owned) max-reduced."""
    import torch.distributed as dist
    dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(brm, op=dist.ReduceOp.MAX, group=group)
    return acc, brm


def reduce_packed(acc, brm, keys, count: int, cap: int, group=None, stored=None):
    """The whole cross-rank merge in ONE all-reduce(SUM) of a packed int64
    buffer [acc | block r_max | per-rank count | per-rank survivor slices]:
    block r_max needs no MAX because every p/100 block has exactly one owner
    (the others hold 0), and each rank's survivors land in its own zeroed
    slice, so the sum is the gather. Falls back to gather_survivors when some
    rank has more than `cap` survivors. `stored` (default `count`) is how many
    of this rank's `count` survivors its buffer holds: a rank whose device
    buffer overflowed still joins every collective, and the per-rank counts
    returned let every rank see it. Returns (acc, brm, sorted (p, q), counts)."""
    import torch
    import torch.distributed as dist
    stored = count if stored is None else min(stored, count)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    na, nb = acc.numel(), brm.numel()
    # [acc | brm | count per rank | stored per rank | survivor slices]
    buf = torch.zeros(na + nb + 2 * world + world * cap, dtype=torch.int64, device=acc.device)
    buf[:na] = acc
    buf[na:na + nb] = brm.to(torch.int64)
    buf[na + nb + rank] = count
    buf[na + nb + world + rank] = stored
    k = min(stored, cap)
    base = na + nb + 2 * world + rank * cap
    buf[base:base + k] = keys[:k]
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    acc.copy_(buf[:na])
    brm.copy_(buf[na:na + nb].to(brm.dtype))
    counts = buf[na + nb:na + nb + world].cpu().numpy()
    held = buf[na + nb + world:na + nb + 2 * world].cpu().numpy()
    if held.max() > cap:
        return acc, brm, gather_survivors(keys, stored, group), counts
    surv = buf[na + nb + 2 * world:].view(world, cap).cpu().numpy()
    allk = np.concatenate([surv[r][:held[r]] for r in range(world)]).astype(np.uint64)
    allk.sort()
    return acc, brm, np.stack([allk >> np.uint64(32), allk & np.uint64(0xFFFFFFFF)], 1), counts


def check_survivor_capacity(counts, surv_cap: int):
    """After the collectives: raise on EVERY rank if any rank's survivors
    exceeded its device buffer (raising before them would leave the other
    ranks blocked in the all-reduce)."""
    over = [r for r, c in enumerate(np.asarray(counts).tolist()) if c > surv_cap]
    if over:
        raise N.CudaSieveError(N.ERR_CAPACITY, f"ranks {over} have more survivors than their "
                               f"{surv_cap}-entry buffers (counts {np.asarray(counts).tolist()})")


def gather_survivors(keys, count: int, group=None):
    """All-gather variable-length survivor lists. keys: int64 tensor holding
    this rank's `count` survivors as (p << 32) | q (any order). Returns a
    sorted numpy uint64 array of (p, q) rows -- the canonical order of the
    reference's sink (engine.hpp:272-277)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = torch.tensor([count], dtype=torch.int64, device=keys.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts)
    if m == 0:
        return np.zeros((0, 2), np.uint64)
    pad = torch.zeros(m, dtype=torch.int64, device=keys.device)
    pad[:count] = keys[:count]
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    allk = np.concatenate([p[:c].cpu().numpy() for p, c in zip(parts, counts)]).astype(np.uint64)
    allk.sort()
    return np.stack([allk >> np.uint64(32), allk & np.uint64(0xFFFFFFFF)], 1)


def primes_by_cube(primes, G: int, g: int) -> list[int]:
    """Rank g's share of an exhaustive table build (BASELINE C2) over G ranks:
    primes dealt largest r^3 first onto the least-loaded rank (ties to the
    lowest rank), returned ascending. Every prime lands on exactly one rank
    and the largest load exceeds the mean by at most one table's r^3."""
    loads = [0] * G
    mine = []
    for r in sorted(primes, reverse=True):
        k = loads.index(min(loads))
        loads[k] += r ** 3
        if k == g:
            mine.append(r)
    return sorted(mine)


def table_slice(total: int, G: int, g: int) -> tuple[int, int, int]:
    """Rank g's share of a G-way table upload: (lo, hi, chunk) with equal
    chunks of ceil(total / G) bytes (the last rank's slice may be short or
    empty); the concatenation of all slices is the whole set."""
    chunk = -(-total // G) if total else 0
    lo = min(total, g * chunk)
    return lo, min(total, lo + chunk), chunk


def allgather_tables(host, device=None, group=None):
    """Every rank's copy of the host table set `host` (uint8 tensor, pinned
    for the NCCL path) with each rank moving only 1/G of it to its GPU: rank g
    copies its slice (table_slice) and one all-gather assembles the whole set
    -- over NVLink under NCCL, into a tensor on `device`, ordered on torch's
    current stream. On gloo the slices and the result stay in host memory."""
    import torch
    import torch.distributed as dist
    G = dist.get_world_size(group)
    g = dist.get_rank(group)
    total = host.numel()
    lo, hi, chunk = table_slice(total, G, g)
    nccl = dist.get_backend(group) == "nccl"
    where = device if nccl else torch.device("cpu")
    mine = torch.zeros(max(chunk, 1), dtype=torch.uint8, device=where)
    mine[:hi - lo].copy_(host[lo:hi], non_blocking=nccl)
    if nccl:
        full = torch.empty(mine.numel() * G, dtype=torch.uint8, device=where)
        dist.all_gather_into_tensor(full, mine, group=group)
    else:
        parts = [torch.empty_like(mine) for _ in range(G)]
        dist.all_gather(parts, mine, group=group)
        full = torch.cat(parts)
    return full[:total]


def load_tables_sharded(dev, primes, host, group=None, async_=False):
    """Make the host table set resident on every rank's GPU through
    allgather_tables (1/G of the bytes over each rank's PCIe link), then load
    it from device memory (cgpu_tables_load_dev: padding check, device
    layouts) on torch's current stream, which must be the context's stream.
    async_: the asynchronous load (no host wait; check dev.load_status_copy).
    Returns the gathered tensor (keep it alive until the stream has run)."""
    import torch
    import torch.distributed as dist
    pr = np.ascontiguousarray(primes, dtype=np.uint32)
    full = allgather_tables(host, torch.device("cuda", dev.device), group)
    if full.is_cuda:
        dev.load_dev(pr, full.data_ptr(), full.numel(), async_=async_)
    else:
        dev.load(pr, full.numpy().tobytes())
    return full


class ShardedSieve:
    """The product multi-GPU path: this rank's shard on its own GPU, results
    reduced over the default process group (NCCL)."""

    def __init__(self, dev, primes, surv_cap: int = 1 << 20):
        import torch
        self.dev = dev
        self.primes = list(primes)
        self.surv_cap = surv_cap
        self.cuda = torch.device("cuda", dev.device)
        self.acc = torch.zeros(2 + len(self.primes), dtype=torch.int64, device=self.cuda)
        self.surv = torch.zeros(max(surv_cap, 1), dtype=torch.int64, device=self.cuda)
        self.brm = None

    def launch(self, p_lo, p_hi, mode=N.TRIANGLE, q_start=0):
        import torch
        import torch.distributed as dist
        G = dist.get_world_size() if dist.is_initialized() else 1
        g = dist.get_rank() if dist.is_initialized() else 0
        nb = p_hi // 100 - p_lo // 100 + 1 if p_hi >= p_lo else 0
        if self.brm is None or self.brm.numel() < max(nb, 1):
            self.brm = torch.zeros(max(nb, 1), dtype=torch.int32, device=self.cuda)
        self.nb = nb
        N.check(N.lib().cgpu_sieve_launch_dev(
            self.dev._ctx, int(p_lo), int(q_start), int(p_hi), int(mode), G, g,
            C.c_void_p(self.acc.data_ptr()), C.c_void_p(self.acc.data_ptr() + 16),
            C.c_void_p(self.brm.data_ptr()), max(nb, 1), C.c_void_p(self.surv.data_ptr()),
            self.surv_cap))

    def reduce(self):
        """Reduce over ranks; returns (pairs, survivors, hist, block_rmax, survivor_pairs)."""
        import torch.distributed as dist
        self.dev.synchronize()  # the context stream may differ from torch's current stream
        local_surv = int(self.acc[1].item())
        keys = self.surv
        if dist.is_initialized() and dist.get_world_size() > 1:
            _, _, pairs, counts = reduce_packed(self.acc, self.brm[:max(self.nb, 1)], keys, local_surv,
                                                cap=4096, stored=min(local_surv, self.surv_cap))
            check_survivor_capacity(counts, self.surv_cap)
        else:
            check_survivor_capacity([local_surv], self.surv_cap)
            k = np.sort(keys[:local_surv].cpu().numpy().astype(np.uint64))
            pairs = np.stack([k >> np.uint64(32), k & np.uint64(0xFFFFFFFF)], 1)
        a = self.acc.cpu().numpy()
        return int(a[0]), int(a[1]), a[2:].copy(), self.brm[:self.nb].cpu().numpy(), pairs
