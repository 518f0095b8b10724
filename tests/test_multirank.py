"""Host-side multi-rank logic on the CPU (gloo, world_size 2 and 3): the
block-cyclic partitioner covers every row exactly once, and the cross-rank
reduction + survivor gather of paper_1601_00636_b200.parallel turns per-rank
shard results into exactly the single-process result (ScanStats::merge,
engine.hpp:121-134; split/merge tests test_engine.cpp:134-175). Per-rank shard
results come from the C oracle here, laid out exactly as the device writes
them (cgpu_sieve_launch_dev)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import port
from paper_1601_00636_b200 import parallel
from paper_1601_00636_b200.primes import default_primes, odd_primes


def test_partition_covers_rows_once():
    for (lo, hi) in [(2, 10000), (152, 5000), (100001, 300000), (1, 99), (250, 251), (7, 6)]:
        for G in (1, 2, 3, 4, 8):
            seen = []
            for g in range(G):
                for b in parallel.owned_blocks(lo, hi, G, g):
                    assert b % G == g
                for (a, z) in parallel.owned_rows(lo, hi, G, g):
                    seen.extend(range(a, z + 1))
            assert sorted(seen) == list(range(lo, hi + 1))


def test_partition_balances_triangle_work():
    """Block-cyclic over 8 ranks keeps C5's per-rank pair counts within 1%."""
    work = []
    for g in range(8):
        work.append(sum((a + z) * (z - a + 1) // 2 for a, z in parallel.owned_rows(100001, 300000, 8, g)))
    assert max(work) / min(work) < 1.01


def test_exhaustive_build_split_by_cube():
    """The C2 build's prime split: a partition, balanced in r^3 to within the
    largest single table."""
    P = odd_primes(256)
    for G in (1, 2, 3, 8):
        parts = [parallel.primes_by_cube(P, G, g) for g in range(G)]
        assert sorted(r for part in parts for r in part) == sorted(P)
        loads = [sum(r ** 3 for r in part) for part in parts]
        assert max(loads) - sum(loads) / G <= max(P) ** 3


def test_table_slices_cover_the_set_once():
    for total in (0, 1, 7, 21873, 25869968):
        for G in (1, 2, 3, 8):
            got = []
            for g in range(G):
                lo, hi, chunk = parallel.table_slice(total, G, g)
                assert 0 <= hi - lo <= chunk and (hi - lo == chunk or hi == total)
                got.append((lo, hi))
            assert got[0][0] == 0 and got[-1][1] == total
            assert all(got[i][1] == got[i + 1][0] for i in range(G - 1))


def _gather_worker(rank, world, port_, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    for k in (32, 64):
        tb, _ = port.build_set(odd_primes(k))
        host = torch.frombuffer(bytearray(tb), dtype=torch.uint8)
        full = parallel.allgather_tables(host)
        out[(rank, k)] = full.numpy().tobytes() == tb
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_table_upload_reassembles_the_set(world):
    """Each rank contributes only its 1/G slice of the host tables; every rank
    ends up with the byte-identical set (the e2e multi-GPU upload path)."""
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_gather_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert len(out) == 2 * world and all(out.values())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_result(tb, P, offs, lo, hi, mode, G, g, q_start):
    """Oracle shard result in the device output layout."""
    n = len(P)
    acc = np.zeros(2 + n, np.int64)
    nb = hi // 100 - lo // 100 + 1
    brm = np.zeros(nb, np.int32)
    keys = []
    for (a, z) in parallel.owned_rows(lo, hi, G, g):
        o = port.sieve(tb, P, offs, a, z, mode, q_start=q_start if a == lo else 0)
        acc[0] += o["pairs_tested"]
        acc[1] += o["survivors"]
        acc[2:] += o["hist"].astype(np.int64)
        for i, v in enumerate(o["row_rmax"]):
            b = (a + i) // 100 - lo // 100
            brm[b] = max(brm[b], int(v))
        keys.extend((int(p) << 32) | int(q) for p, q in o["survivor_pairs"])
    rng = np.random.default_rng(g)
    keys = np.array(keys, np.int64)
    rng.shuffle(keys)  # device survivors come out unordered
    return acc, brm, keys


def _worker(rank, world, port_, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P, lo, hi, mode, q_start = case
    tb, offs = port.build_set(P)
    acc, brm, keys = _shard_result(tb, P, offs, lo, hi, mode, world, rank, q_start)
    acc_t, brm_t = torch.from_numpy(acc), torch.from_numpy(brm)
    keys_t = torch.zeros(max(len(keys), 1), dtype=torch.int64)
    keys_t[:len(keys)] = torch.from_numpy(keys)
    acc2, brm2 = acc_t.clone(), brm_t.clone()
    parallel.reduce_results(acc_t, brm_t)
    surv = parallel.gather_survivors(keys_t, len(keys))
    # the single-collective form, with a cap small enough to hit the fallback too
    _, _, surv2, counts = parallel.reduce_packed(acc2, brm2, keys_t, len(keys), cap=64)
    assert int(sum(counts)) == int(acc_t[1])
    assert acc2.tolist() == acc_t.tolist() and brm2.tolist() == brm_t.tolist()
    assert surv2.tolist() == surv.tolist()
    out[rank] = (acc_t.numpy().tolist(), brm_t.numpy().tolist(), surv.tolist())
    dist.destroy_process_group()


CASES = [
    (odd_primes(32), 2, 2000, port.TRIANGLE, 0),        # C1
    ([11], 2, 700, port.TRIANGLE, 0),                   # weak sieve: heavy survivor gather
    (default_primes(), 152, 1400, port.REGION, 3),      # reference region
    ([11, 13], 160, 555, port.REGION, 777),             # mid-row start, survivors
]


@pytest.mark.parametrize("world,case", [(2, 0), (2, 1), (2, 2), (3, 3)])
def test_gloo_reduction_equals_single_process(world, case):
    P, lo, hi, mode, q_start = CASES[case]
    tb, offs = port.build_set(P)
    full = port.sieve(tb, P, offs, lo, hi, mode, q_start=q_start)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), CASES[case], out), nprocs=world, join=True)
    want_brm = {}
    for i, v in enumerate(full["row_rmax"]):
        b = (lo + i) // 100
        want_brm[b] = max(want_brm.get(b, 0), int(v))
    for r in range(world):
        acc, brm, surv = out[r]
        assert acc[0] == full["pairs_tested"] and acc[1] == full["survivors"]
        assert acc[2:] == full["hist"].astype(np.int64).tolist()
        assert {lo // 100 + i: v for i, v in enumerate(brm)} == want_brm
        assert surv == full["survivor_pairs"].tolist()


def _overflow_worker(rank, world, port_, out):
    """Rank 1's device buffer held only 3 of its 10 survivors: both ranks
    finish the collectives and both raise (raising before the
    all-reduce left the other ranks blocked in it)."""
    from paper_1601_00636_b200 import _native as N
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    acc = torch.zeros(4, dtype=torch.int64)
    brm = torch.zeros(2, dtype=torch.int32)
    count = 10 if rank == 1 else 2
    acc[1] = count
    keys = torch.arange(1, 4, dtype=torch.int64) + (1000 << 32) * (rank + 1)
    _, _, pairs, counts = parallel.reduce_packed(acc, brm, keys, count, cap=64, stored=min(count, 3))
    try:
        parallel.check_survivor_capacity(counts, 3)
        out[rank] = "no error"
    except N.CudaSieveError as e:
        out[rank] = ("raised", e.code, counts.tolist(), len(pairs))
    dist.destroy_process_group()


def test_survivor_overflow_raises_on_every_rank():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_overflow_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    from paper_1601_00636_b200 import _native as N
    for r in range(2):
        assert out[r] == ("raised", N.ERR_CAPACITY, [2, 10], 5)  # the 2 + 3 survivors held
