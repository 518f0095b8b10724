#!/usr/bin/env python
"""Benchmark of the modulo-primes cuboid sieve on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5|C4|C3]
    python bench.py --impl reference ...      # the reference CPU path (oracle/_ref)

One "step" = one pass of the hot path over the workload: the (p,q) pair sieve
of BASELINE.json's config against resident residue tables, with the
cross-rank reduction of its results (ONE NCCL all-reduce(SUM) of a packed
buffer: pair/survivor counts, the first-killer histogram, block r_max -- each
block has one owner, the others hold 0 -- and per-rank survivor slices). Rows are split block-cyclically over ranks (p/100 blocks), so the
total work is fixed as N grows ("strong" scaling).

`value` = pairs sieved per second over the timed steps, inputs resident in HBM,
device time from CUDA events on the launching stream, max over ranks; L2 is
flushed between steps. `e2e` = the same metric through the C ABI with HOST
buffers: each step uploads the reference-format tables (pinned host memory),
sieves, reduces and reads the reduced results back. `table_build` = BASELINE
config 2 (exhaustive Q evaluation over Z_r^3 for the first 256 odd primes) in
Q evals/s. `roofline` uses the INT32 throughput measured on this GPU in the
same run (cgpu_int32_peak). `cpu_baseline` = the reference itself
(oracle/_ref, the unmodified headers) on a bounded seed-chosen sample of the
same workload, on all host cores.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "(p,q) pairs sieved/s"
SEED = 20160401
WORKLOADS = {
    # BASELINE.json configs; C5 is the largest and the headline
    "C5": dict(k=256, p_lo=100001, p_hi=300000, pairs=24317097730,
               desc="C5: TRIANGLE sieve 1e5<p<=3e5, 1<=q<p coprime, 256 odd primes 3..1621"),
    "C4": dict(k=128, p_lo=2, p_hi=100000, pairs=3039650753,
               desc="C4: TRIANGLE sieve p<=1e5, 1<=q<p coprime, 128 odd primes 3..727"),
    "C1": dict(k=32, p_lo=2, p_hi=2000, pairs=1216587,
               desc="C1: TRIANGLE sieve p<=2000, 1<=q<p coprime, 32 odd primes 3..137"),
    "C3": dict(k=64, p_lo=2, p_hi=10000, pairs=30397485,
               desc="C3: TRIANGLE sieve p<=1e4, 1<=q<p coprime, 64 odd primes 3..313"),
}
GATHER_CAP = 128  # survivors per rank gathered inside the step (C1..C5 have 0; overflow fails parity)


# ---- host-side workload constants ------------------------------------------------------

def phi_and_omega(n):
    """Euler phi and the number of distinct prime factors for 0..n."""
    phi = np.arange(n + 1, dtype=np.int64)
    omega = np.zeros(n + 1, dtype=np.int64)
    for p in range(2, n + 1):
        if phi[p] == p:
            phi[p::p] -= phi[p::p] // p
            omega[p::p] += 1
    return phi, omega


def ops_per_pair(primes, killable, hist, survivors, pairs, p_lo, p_hi):
    """7 * D_eff + 4 * omega_bar INT32 ops per candidate pair
    for the reference algorithm (Barrett q mod r + bit probe per probe into a
    table that can kill, one Barrett divisibility test per distinct prime
    factor of p for coprimality). D_eff is exact from this run's histogram."""
    kill_idx = np.cumsum(np.asarray(killable, dtype=np.int64))  # probes made when rank k kills
    np_ = int(kill_idx[-1]) if len(kill_idx) else 0
    probes = float(np.dot(np.asarray(hist, dtype=np.float64), kill_idx)) + survivors * np_
    d_eff = probes / max(pairs, 1)
    phi, omega = phi_and_omega(p_hi)
    w = phi[max(p_lo, 2):p_hi + 1].astype(np.float64)
    omega_bar = float(np.dot(w, omega[max(p_lo, 2):p_hi + 1]) / w.sum())
    return 7.0 * d_eff + 4.0 * omega_bar, d_eff, omega_bar


def golden_parity(workload, primes, pairs, survivors, hist, brm, wl):
    """The step's result against the reference's own full-range statistics
    (tests/golden/golden.json, generated from oracle/_ref by
    tests/golden/make_golden.py): pair and survivor counts, the first-killer
    histogram by prime and every p/100 block's r_max (engine.hpp:229-291)."""
    path = os.path.join(ROOT, "tests", "golden", "golden.json")
    g = json.load(open(path))["sieve"].get(workload) if os.path.exists(path) else None
    if g is None:
        return {"ok": False, "against": f"no reference golden for {workload}"}
    got_hist = {str(primes[k]): int(c) for k, c in enumerate(hist) if c}
    blk0 = wl["p_lo"] // 100
    got_brm = {str(blk0 + i): int(v) for i, v in enumerate(brm) if v}
    checks = {"pairs": pairs == g["pairs_tested"], "survivors": survivors == g["survivors"],
              "kill_histogram": got_hist == g["kill_histogram"],
              "block_r_max": got_brm == g["block_r_max"]}
    return {"ok": all(checks.values()), "checks": checks,
            "against": f"tests/golden/golden.json sieve.{workload} (oracle/_ref, full range)"}


# ---- clocks -------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---- CPU legs (the checker / reference; the product never runs these) ------------------

class CpuReference:
    """The reference (oracle/_ref: the unmodified headers) TRIANGLE loop --
    SieveSet::is_unsolvable in rank order, verify_small_region's pattern over
    q < p -- on a seed-chosen contiguous block of rows of the workload, sized to
    ~budget_s, on `threads` host threads. Falls back to the C restatement
    (oracle/cuboid_oracle.c, one thread) if oracle/_ref is absent."""

    def __init__(self, wl, primes, threads):
        from oracle import ref as refmod
        self.wl, self.primes = wl, primes
        span = wl["p_hi"] - wl["p_lo"] + 1
        self.span = span
        self.p0 = wl["p_lo"] + (SEED % max(span - 40000, 1))
        if refmod.available():
            rs = refmod.RefSet.build(primes)
            self._run = lambda lo, hi: refmod.triangle(rs, lo, hi, threads, with_sink=False).pairs_tested
            self.kind, self.cores = "reference", threads
        else:
            from oracle import port
            tb, offs = port.build_set(primes)
            self._run = lambda lo, hi: port.sieve(tb, primes, offs, lo, hi, port.TRIANGLE)["pairs_tested"]
            self.kind, self.cores = "port", 1
        t = time.perf_counter()
        self._run(self.p0, self.p0 + 199)
        self.sec_per_row = max(time.perf_counter() - t, 1e-4) / 200

    def sample(self, budget_s):
        rows = int(min(max(budget_s / self.sec_per_row, 20), self.wl["p_hi"] - self.p0 + 1, 40000))
        t = time.perf_counter()
        pairs = self._run(self.p0, self.p0 + rows - 1)
        return dict(pairs=pairs, seconds=time.perf_counter() - t, rows=(self.p0, self.p0 + rows - 1),
                    kind=self.kind, cores=self.cores)


def reference_api_leg(args, wl, primes):
    """C5 through the reference's own C++ API with the drop-in
    (cpp/bench_dropin: cuboid::gpu::scan_triangle on a reference SieveSet,
    results in the reference's ScanStats maps), tables resident and tables
    re-uploaded from the host every call; the histogram is checked against
    the reference golden. None when the binary was not built (it needs the
    reference headers at build time)."""
    exe = os.path.join(ROOT, "cpp", "_build", "bench_dropin")
    if args.workload != "C5" or not os.path.exists(exe):
        return None
    r = subprocess.run([exe, str(args.steps), str(args.warmup)], capture_output=True, text=True, timeout=300)
    if r.returncode != 0:
        return {"error": r.stderr[-300:]}
    d = json.loads(r.stdout.strip().splitlines()[-1])
    path = os.path.join(ROOT, "tests", "golden", "golden.json")
    g = json.load(open(path))["sieve"]["C5"]
    ok = (d["pairs"] == g["pairs_tested"] and d["survivors"] == g["survivors"] and
          d["kill_histogram"] == g["kill_histogram"] and d["blocks"] == len(g["block_r_max"]) and
          d["same_both_legs"])
    return {"path": "cuboid::gpu::scan_triangle(reference SieveSet, 100001, 300000) -> reference ScanStats",
            "resident": {"value": d["pairs"] / d["resident_s"], "unit": "pairs/s", "ms_per_call": 1e3 * d["resident_s"]},
            "upload_every_call": {"value": d["pairs"] / d["upload_s"], "unit": "pairs/s",
                                  "ms_per_call": 1e3 * d["upload_s"],
                                  "h2d_bytes_per_call": 25869968},
            "parity": "ok" if ok else "MISMATCH", "steps": d["steps"]}


def cpu_table_baseline(P256, tables_c2=None):
    """the reference's production build_table for all
    256 primes (1 thread and all cores) and its definition build_table_oracle
    on the first 64 primes (all cores), oracle/_ref on the host cores."""
    from oracle import ref as refmod
    if not refmod.available():
        return None
    threads = os.cpu_count() or 1
    out = {"kind": "reference", "cores": threads}
    _, t1 = refmod.build_tables(P256, oracle=False, nthreads=1)
    _, tn = refmod.build_tables(P256, oracle=False, nthreads=threads)
    out["build_table_256"] = {"seconds_1thread": t1, f"seconds_{threads}threads": tn,
                              "what": "production build_table (sievetable.hpp:123-141), 256 primes"}
    P64 = P256[:64]
    _, to = refmod.build_tables(P64, oracle=True, nthreads=threads)
    cube64 = sum(r ** 3 for r in P64)
    out["build_table_oracle_64"] = {
        "seconds": to, "threads": threads, "cube_evals": cube64, "value": cube64 / to,
        "unit": "cube-equivalent evals/s",
        "what": "build_table_oracle (sievetable.hpp:102-115, early exit per (p,q)) on the first 64 "
                "odd primes; the full 256-prime definition is ~5 h on 1 thread"}
    out["value"], out["unit"] = cube64 / to, "cube-equivalent evals/s"
    return out


def run_reference_arm(args, wl, primes):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    per_step = max(1.0, min(6.0, 150.0 / max(args.steps + args.warmup, 1)))
    samples = []
    ref = CpuReference(wl, primes, threads)
    for i in range(args.warmup + args.steps):
        s = ref.sample(per_step)
        if i >= args.warmup:
            samples.append(s)
    pairs = sum(s["pairs"] for s in samples)
    secs = sum(s["seconds"] for s in samples)
    v = pairs / secs
    s0 = samples[0]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "pairs/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / len(samples), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (deterministic enumeration)",
        "config": {"workload": wl["desc"], "primes": len(primes),
                   "p_range": [wl["p_lo"], wl["p_hi"]], "mode": "TRIANGLE"},
        "cpu_baseline": {"value": v, "unit": "pairs/s", "cores": s0["cores"], "kind": s0["kind"],
                         "sample": f"rows p={s0['rows'][0]}..{s0['rows'][1]} of {wl['desc'].split(':')[0]} "
                                   f"({s0['pairs']} pairs per step), SieveSet::is_unsolvable rank-ordered "
                                   f"loop of verify_small_region over q<p, {s0['cores']} threads"},
        "e2e": {"value": v, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---- the B200 arm -----------------------------------------------------------------------

def run_ours(args, wl, primes):
    import torch
    import torch.distributed as dist

    from paper_1601_00636_b200 import _native as N
    from paper_1601_00636_b200.device import Device
    from paper_1601_00636_b200 import parallel

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:  # plumbing test only: every rank on GPU 0, gloo collectives on the CPU
        local = 0
    torch.cuda.set_device(local)
    gloo = args.backend == "gloo"
    if not args.same_device and local >= torch.cuda.device_count():
        raise SystemExit(f"bench: rank {rank} needs GPU {local}, only {torch.cuda.device_count()} visible")
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        print(f"bench: rank {rank}/{dist.get_world_size()} on cuda:{local}, "
              f"{'gloo' if gloo else 'NCCL %s' % '.'.join(map(str, torch.cuda.nccl.version()))} "
              f"communicator of {dist.get_world_size()} ranks", file=sys.stderr, flush=True)
    cuda = torch.device("cuda", local)
    cdev = torch.device("cpu") if gloo else cuda  # where collectives run
    stream = torch.cuda.Stream(device=cuda)  # the context and all torch work share it
    torch.cuda.set_stream(stream)
    L = N.lib()

    def allreduce_max(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            if gloo:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    dev = Device(local, stream=stream.cuda_stream)

    # INT32 peaks of this GPU (roofline denominators)
    clk = ClockSampler(local).__enter__()  # sampled over the whole GPU run
    peaks = (C.c_double * 4)()
    N.check(L.cgpu_int32_peak(local, peaks))
    int_peak = {"alu_lop3": peaks[0], "fma_imad": peaks[1], "imad_lop3_3reg": peaks[2],
                "imad_lop3_imm": peaks[3], "best": max(peaks)}
    fpk = (C.c_double * 2)()
    N.check(L.cgpu_fp32_peak(local, fpk))
    fp_peak = {"ffma2_lane_fmas": fpk[0], "cube_mix_evals": fpk[1]}

    # ---- table build (BASELINE config 2): exhaustive Z_r^3, 256 primes --------------
    from paper_1601_00636_b200.primes import odd_primes
    P256 = odd_primes(256)
    # At N > 1 the primes are split over the ranks, balanced by r^3 (largest
    # first onto the least-loaded rank); each rank builds its share and the
    # job's rate is all evaluations over the slowest rank's build time.
    mine = parallel.primes_by_cube(P256, world, rank)
    tb_ms = []
    my_bytes = b""
    for i in range(3):
        if mine:
            my_bytes, evals = dev.build(mine, N.BUILD_EXHAUSTIVE, download=(i == 2))
        if i:
            tb_ms.append(dev.timings_ms()["plan"] if mine else 0.0)  # ms[0] = build kernels
    cube_ms = allreduce_max(float(np.mean(tb_ms)))
    tb_evals = sum(r ** 3 for r in P256)
    tb_parity = None
    if world > 1:  # assemble the shares on every rank and compare with a whole production build
        objs = [None] * world
        dist.all_gather_object(objs, (mine, my_bytes))
        full_prod, _ = dev.build(P256, N.BUILD_PRODUCTION)
        offs, _ = Device.layout(P256)
        pos = {r: int(o) for r, o in zip(P256, offs)}
        ok = True
        for primes_k, bytes_k in objs:
            if not primes_k:
                continue
            offs_k, _ = Device.layout(primes_k)
            for j, r in enumerate(primes_k):
                nb = (r * r + 7) // 8
                ok &= bytes_k[int(offs_k[j]):int(offs_k[j]) + nb] == full_prod[pos[r]:pos[r] + nb]
        tb_parity = "ok" if ok else "MISMATCH"
    prod_t = []
    for i in range(3):
        dev.build(P256, N.BUILD_PRODUCTION, download=False)
        if i:
            prod_t.append(dev.timings_ms()["plan"])
    table_build = {
        "metric": "table-build Q evals/s", "value": tb_evals / (cube_ms * 1e-3), "unit": "evals/s",
        "config": "C2: first 256 odd primes (3..1621), every (a,b,t) in Z_r^3, sum r^3 = "
                  f"{tb_evals} evals, 25,869,968 B of tables",
        "ms": cube_ms, "production_build_ms": float(np.mean(prod_t)),
        "ranks": world, "sharded_parity": tb_parity,
        # k_cube_f2 evaluates A = c0 + c1 s + ... + c4 s^4 exactly in FP32 (balanced
        # residues, |A| < 2^22, on top of 1.5 * 2^23) with two (a,b) pairs per
        # FFMA2, then tests (A + s^5) for divisibility by r with one IMAD by
        # r^-1 mod 2^32 and an unsigned min: 2 FFMA2 + 1 IMAD + 1 min per eval.
        # The bound is that mix's measured throughput (cgpu_fp32_peak).
        # frac: against the FMA-pipe model of that mix (2 FFMA2 + 1 IMAD per eval at
        # the pipes' separately measured rates); the self-chain microbenchmark of
        # the same instruction mix is kept beside it.
        "roofline": {"bound": "fp32_fma_pipes", "instr_per_eval": "2 FFMA2 + 1 IMAD + 1 VIMNMX",
                     "achieved": tb_evals / (cube_ms * 1e-3),
                     "peak": world / (2.0 / (fp_peak["ffma2_lane_fmas"] / 2) + 1.0 / int_peak["fma_imad"]),
                     "unit": "evals/s",
                     "frac": tb_evals / (cube_ms * 1e-3) / world / (
                         1.0 / (2.0 / (fp_peak["ffma2_lane_fmas"] / 2) + 1.0 / int_peak["fma_imad"])),
                     "self_chain_peak": fp_peak["cube_mix_evals"] * world,
                     "frac_vs_self_chain": tb_evals / (cube_ms * 1e-3) / (fp_peak["cube_mix_evals"] * world),
                     "fp32_peaks": fp_peak,
                     # the same bound from the pipes alone: 2 FFMA2 + 1 IMAD per eval
                     # issued at their separately measured chain rates
                     "fma_pipe_model_evals": 1.0 / (2.0 / (fp_peak["ffma2_lane_fmas"] / 2)
                                                    + 1.0 / int_peak["fma_imad"]),
                     "frac_vs_fma_pipe_model": tb_evals / (cube_ms * 1e-3) / world / (
                         1.0 / (2.0 / (fp_peak["ffma2_lane_fmas"] / 2) + 1.0 / int_peak["fma_imad"])),
                     "imad_path_peak_evals": int_peak["fma_imad"] / 5,
                     "horner_ops_per_eval_survey": 27,
                     "note": "SURVEY 8(d) counts 27 INT32 ops/eval for Horner; the kernel issues 4 "
                             "(+ shared loads and loop control amortised over 16 pairs per thread). "
                             "imad_path_peak_evals = the ceiling of the previous all-IMAD kernel "
                             "(5 IMAD/eval), still used for r = 2 and r > 2039"},
    }

    # ---- the paper's historical scan, for the published figure ------
    historical = None
    if world == 1:
        from paper_1601_00636_b200.primes import default_primes
        DP = default_primes()
        dev.build(DP, N.BUILD_PRODUCTION, download=False)
        hms = []
        for i in range(3):
            r = dev.sieve(1, 154000, N.REGION, surv_cap=1 << 16)
            hms.append(dev.timings_ms()["sieve"])
        hk = max((DP[k] for k, c in enumerate(r.hist) if c), default=0)
        t_h = min(hms) * 1e-3
        prefilter = sum(59 * p for p in range(1, 154001))  # the paper's N = 699,626,543,000
        historical = {
            "config": "REGION scan p=1..154000, q_low(p)<=q<=59p, 96 primes 11..541 (PAPER.md:852-870)",
            "pairs_tested": r.pairs_tested, "survivors": r.survivors, "max_killer": hk,
            "kernel_ms": 1e3 * t_h, "pairs_per_s": r.pairs_tested / t_h,
            "sec_per_prefilter_pair": t_h / prefilter, "paper_sec_per_pair": 3.54e-7,
            "paper_wall": "4130 min on a Pentium 4 (1 thread)",
            "pin_ok": r.survivors == 0 and hk == 137,
        }

    # ---- the other BASELINE sieve configs, one GPU, device time ----------------------
    other = {}
    if world == 1:
        for name in ("C1", "C3", "C4"):
            o = WORKLOADS[name]
            dev.build(odd_primes(o["k"]), N.BUILD_PRODUCTION, download=False)
            ms = []
            for _ in range(4):
                r = dev.sieve(o["p_lo"], o["p_hi"], N.TRIANGLE, surv_cap=1 << 16)
                ms.append(dev.timings_ms()["total"])
            other[name] = {"workload": o["desc"], "pairs": r.pairs_tested,
                           "parity": r.pairs_tested == o["pairs"] and r.survivors == 0,
                           "ms": min(ms[1:]), "pairs_per_s": r.pairs_tested / (min(ms[1:]) * 1e-3)}

    # ---- resident set for the workload ------------------------------------------------
    tables, _ = dev.build(primes, N.BUILD_PRODUCTION)
    killable = dev.killable()
    n = len(primes)

    # ---- per-rank compute of the N-GPU strong-scaling shapes, on this one GPU ------------
    # (plan + sieve of every block-cyclic shard g of G; the slowest one against
    # the whole launch / G -- what an N-rank run's compute can reach before its
    # all-reduce; the collective itself needs N GPUs)
    shard_scaling = None
    if world == 1:
        def best_total(shard, k=3):
            t = []
            for _ in range(k):
                dev.sieve(wl["p_lo"], wl["p_hi"], N.TRIANGLE, shard=shard, surv_cap=1 << 16)
                t.append(dev.timings_ms()["total"])
            return min(t)
        full_ms = best_total((1, 0))
        shard_scaling = {"full_ms": full_ms,
                         "note": "per-rank plan+sieve device time of block-cyclic shards on one GPU; "
                                 "no collective, no L2 flush"}
        for G in (2, 4, 8):
            worst = max(best_total((G, g)) for g in range(G))
            shard_scaling[str(G)] = {"slowest_shard_ms": worst, "ideal_ms": full_ms / G,
                                     "efficiency": full_ms / G / worst}
    G, g = world, rank
    nblocks = wl["p_hi"] // 100 - wl["p_lo"] // 100 + 1
    # One int64 exchange buffer, reduced by ONE all-reduce(SUM) per step:
    #   [pairs, survivors, hist(n) | block r_max (nblocks) | survivors (world x cap)]
    # Block r_max needs no MAX: every p/100 block is owned by exactly one rank
    # and the others hold 0 (k_init_blocks). Each rank writes its survivors
    # into its own slice of a zeroed region, so the SUM is the gather.
    n_acc, n_surv = 2 + n, world * GATHER_CAP
    # + 1 slot: the asynchronous table load's status word (e2e steps; 0 = verified)
    buf = torch.zeros(n_acc + nblocks + n_surv + 1, dtype=torch.int64, device=cuda)
    acc = buf[:n_acc]
    brm_sum = buf[n_acc:n_acc + nblocks]
    surv_all = buf[n_acc + nblocks:n_acc + nblocks + n_surv]
    brm = torch.zeros(nblocks, dtype=torch.int32, device=cuda)  # the kernel writes u32 r_max
    surv_mine = surv_all[g * GATHER_CAP:(g + 1) * GATHER_CAP]
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=cuda)  # > 126 MB L2

    def launch():
        if world > 1:
            surv_all.zero_()
        N.check(L.cgpu_sieve_launch_dev(
            dev._ctx, wl["p_lo"], 0, wl["p_hi"], N.TRIANGLE, G, g,
            C.c_void_p(acc.data_ptr()), C.c_void_p(acc.data_ptr() + 16), C.c_void_p(brm.data_ptr()),
            nblocks, C.c_void_p(surv_mine.data_ptr()), GATHER_CAP))

    def exchange():
        if world == 1:
            return
        brm_sum.copy_(brm)
        if gloo:  # stage through host memory
            h = buf.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.SUM)
            buf.copy_(h)
        else:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM)

    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for _ in range(args.warmup):
        launch()
        exchange()
    barrier()
    step_ms, kern_ms, launches = [], [], 0
    for _ in range(args.steps):
        flush.zero_()
        e0.record(stream)
        launch()
        exchange()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        kern_ms.append(dev.timings_ms()["sieve"])
        launches += dev.launch_count()
    barrier()
    local_ms = float(np.sum(step_ms))
    total_ms = allreduce_max(local_ms)

    # results of the last step (already reduced across ranks)
    res = acc.cpu().numpy()
    pairs, survivors, hist = int(res[0]), int(res[1]), res[2:]
    brm_final = (brm_sum if world > 1 else brm).cpu().numpy().astype(np.int64)
    parity = golden_parity(args.workload, primes, pairs, survivors, hist, brm_final, wl)
    parity_ok = parity["ok"]
    local_pairs = pairs if world == 1 else None

    # ---- e2e: host tables in, host results out, through the C ABI -------------------------
    # Every step uploads the host tables (cgpu_tables_load from pinned memory),
    # sieves, reduces and reads the result vector back to the host. Two
    # contexts, each on its own stream with its own buffers, form a 2-deep
    # pipeline: step i+1's upload runs on the copy engine while step i sieves.
    pinned = torch.empty(len(tables), dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = np.frombuffer(tables, np.uint8)
    pr = np.ascontiguousarray(primes, dtype=np.uint32)

    class Lane:
        def __init__(self, d, s):
            self.dev, self.stream = d, s
            self.buf = torch.zeros_like(buf)
            self.brm = torch.zeros_like(brm)
            self.h = torch.empty(buf.numel(), dtype=torch.int64, pin_memory=True)
            self.done = torch.cuda.Event()

        def issue(self):
            b = self.buf
            with torch.cuda.stream(self.stream):
                # asynchronous loads: no host wait inside the step; the load is
                # verified on the device and its status word rides in the result
                # vector (checked below)
                if world > 1:  # 1/G of the bytes per rank over PCIe, all-gathered over NVLink
                    self.full = parallel.load_tables_sharded(self.dev, pr, pinned, async_=True)
                else:
                    self.dev.load_host_async(pr, pinned.data_ptr(), len(tables))
                if world > 1:  # survivor slices and the status slot are summed over ranks
                    b[n_acc + nblocks:].zero_()
                self.dev.load_status_copy(b[-1:].data_ptr())
                N.check(L.cgpu_sieve_launch_dev(
                    self.dev._ctx, wl["p_lo"], 0, wl["p_hi"], N.TRIANGLE, G, g,
                    C.c_void_p(b.data_ptr()), C.c_void_p(b.data_ptr() + 16), C.c_void_p(self.brm.data_ptr()),
                    nblocks, C.c_void_p(b[n_acc + nblocks + g * GATHER_CAP:].data_ptr()), GATHER_CAP))
                b[n_acc:n_acc + nblocks].copy_(self.brm)
                if world > 1:
                    if gloo:
                        hb = b.cpu()
                        dist.all_reduce(hb, op=dist.ReduceOp.SUM)
                        b.copy_(hb)
                    else:
                        dist.all_reduce(b, op=dist.ReduceOp.SUM)
                self.h.copy_(b, non_blocking=True)
                self.done.record(self.stream)

    s2 = torch.cuda.Stream(device=cuda)
    lanes = [Lane(dev, stream), Lane(Device(local, stream=s2.cuda_stream), s2)]

    def e2e_run(k):
        lanes[0].issue()
        for i in range(1, k):
            lanes[i % 2].issue()
            lanes[(i - 1) % 2].done.synchronize()
        lanes[(k - 1) % 2].done.synchronize()
        return lanes[(k - 1) % 2].h

    e2e_run(max(2, args.warmup))
    barrier()
    t = time.perf_counter()
    h_buf = e2e_run(args.steps)
    e2e_s = [time.perf_counter() - t]
    barrier()
    e2e_total = allreduce_max(float(np.sum(e2e_s)))
    clk.__exit__()
    e2e_res = h_buf.numpy()
    load_status = int(e2e_res[-1])  # summed over ranks: 0 iff every rank's asynchronous load verified
    e2e_parity = golden_parity(args.workload, primes, int(e2e_res[0]), int(e2e_res[1]),
                               e2e_res[2:n_acc], e2e_res[n_acc:n_acc + nblocks], wl)
    parity_ok = parity_ok and e2e_parity["ok"] and load_status == 0
    e2e_parity["load_status"] = load_status

    # ---- roofline of the dominant kernel (k_sieve), rank-local ------------------------------
    if world > 1:  # this rank's own pairs for the per-launch figure
        N.check(L.cgpu_sieve_launch_dev(
            dev._ctx, wl["p_lo"], 0, wl["p_hi"], N.TRIANGLE, G, g,
            C.c_void_p(acc.data_ptr()), C.c_void_p(acc.data_ptr() + 16), C.c_void_p(brm.data_ptr()),
            nblocks, C.c_void_p(surv_mine.data_ptr()), GATHER_CAP))
        local_pairs = int(acc[0].item())
        overflow = allreduce_max(float(int(acc[1].item()) > GATHER_CAP)) > 0
    else:
        overflow = survivors > GATHER_CAP
    parity_ok = parity_ok and not overflow  # every survivor must have been gathered
    opp, d_eff, omega_bar = ops_per_pair(primes, killable, hist, survivors, pairs,
                                         wl["p_lo"], wl["p_hi"])
    kavg = float(np.mean(kern_ms))
    kname = dev.sieve_kernel() or "k_sieve"  # the wheel sieve k_wsieve for C5, the window sieve otherwise
    achieved = local_pairs * opp / (kavg * 1e-3)
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(kname, {}).get(wl["desc"][:2], {}).get("dram_bytes")
        except (ValueError, AttributeError):
            traffic = None
    ncu = None
    if os.path.exists(prof):
        try:
            x = json.load(open(prof)).get(kname, {}).get(wl["desc"][:2], {})
            ncu = {k: x.get(k) for k in ("round", "duration_ms", "issue_active_pct", "alu_pipe_pct",
                                          "xu_pipe_pct", "lsu_pipe_pct", "l1tex_throughput_pct",
                                          "smem_wavefront_pct", "fma_pipe_pct", "warps_active_pct",
                                          "registers")}
            if x.get("duration_ms"):
                ncu["dram_gbs"] = x.get("dram_bytes", 0) / (x["duration_ms"] * 1e-3) / 1e9
        except (ValueError, AttributeError):
            ncu = None
    # The hardware fraction: k_sieve's warp instructions per launch (ncu,
    # profiles/ncu_summary.json, same kernel build and workload) x 32 lanes
    # over this run's CUDA-event kernel time, against the measured INT32 issue
    # peak -- i.e. the issue utilisation the live kernel sustains. Shared-memory
    # wavefronts (1 per clock per SM) beside it. At N > 1 a rank's launch
    # holds its share of the instructions (scaled by its pairs).
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    clocks = clk.summary()
    nk = (json.load(open(prof)).get(kname, {}).get(wl["desc"][:2], {})
          if os.path.exists(prof) else {})
    share = local_pairs / max(pairs, 1)
    hw = {}
    if nk.get("warp_inst"):
        lanes_s = nk["warp_inst"] * share * 32 / (kavg * 1e-3)
        hw = {"achieved": lanes_s, "frac": lanes_s / int_peak["best"]}
    if nk.get("smem_wavefronts") and clocks.get("sm_mhz"):
        hw["smem_wavefront_frac"] = nk["smem_wavefronts"] * share / (
            kavg * 1e-3 * sms * clocks["sm_mhz"] * 1e6)
    roof = {"bound": "int32_issue", "achieved": hw.get("achieved"), "peak": int_peak["best"],
            "unit": "thread-instructions/s", "frac": hw.get("frac"), "traffic": traffic,
            "smem_wavefront_frac": hw.get("smem_wavefront_frac"),
            "kernel": kname, "kernel_ms": kavg, "pairs_per_launch": local_pairs,
            "warp_inst_per_launch": nk.get("warp_inst", 0) * share or None,
            "smem_wavefronts_per_launch": nk.get("smem_wavefronts", 0) * share or None,
            "ncu_round": nk.get("round"), "sms": sms,
            "how": "frac = warp_inst x 32 / live kernel_ms / peak (issue utilisation); "
                   "smem_wavefront_frac = wavefronts / (kernel_ms x SMs x median SM clock); "
                   "warp_inst and wavefronts from profiles/ncu_summary.json (ncu --set full of "
                   "the same kernel on the same workload), kernel_ms from CUDA events in this run",
            "peak_source": "measured in this run: best of cgpu_int32_peak's INT32 chains "
                           "(nominal issue limit 148 SM x 128 lanes x clock = 3.72e13 at 1965 MHz)",
            "int32_peaks": int_peak,
            "ncu_pipes": ncu,
            "reference_algorithm": {
                "ops_per_pair": opp, "d_eff": d_eff, "omega_bar": omega_bar,
                "achieved": achieved, "unit": "INT32 ops/s", "frac": achieved / int_peak["best"],
                "note": "SURVEY 8(d)'s count for the reference algorithm (7 D_eff + 4 omega_bar "
                        "per pair); the kernel is bit-sliced (one probe answers 32 q), so this "
                        "ratio exceeds 1 -- it is the work-efficiency figure, not a pipe fraction"}}

    if rank == 0:
        value = pairs * args.steps / (total_ms * 1e-3)
        line = {
            "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (deterministic enumeration of the BASELINE config)",
            "config": {"workload": wl["desc"], "primes": n, "p_range": [wl["p_lo"], wl["p_hi"]],
                       "mode": "TRIANGLE", "pairs_per_step": pairs,
                       "l2": "flushed between steps (512 MiB write)",
                       "parallelism": f"dp{world}: p/100 blocks block-cyclic over ranks, one NCCL "
                                      "all-reduce(SUM) of counts/histogram/block r_max/survivor slices"},
            "parity": "ok" if parity_ok else "MISMATCH",
            "parity_detail": parity,
            "parity_detail_e2e": e2e_parity,
            "e2e": {"value": pairs * args.steps / e2e_total, "unit": "pairs/s",
                    "h2d_bytes_per_step": (parallel.table_slice(len(tables), world, 0)[2] if world > 1
                                           else len(tables)) + 4 * n,
                    "d2h_bytes_per_step": 8 * buf.numel(),
                    "ms_per_step": 1e3 * e2e_total / args.steps,
                    "path": "per step: cgpu_tables_load_async(pinned host tables; no host wait, "
                            "verified on the device, status word in the result vector) + "
                            "cgpu_sieve_launch_dev + reduce + D2H of the result vector; two "
                            "contexts/streams pipelined 2 deep "
                            "(step i+1's upload overlaps step i's sieve); at N>1 each rank uploads "
                            "1/N of the tables (h2d bytes are per rank) and one all-gather assembles "
                            "the set (parallel.load_tables_sharded, cgpu_tables_load_dev)"},
            "gpu_launches": launches,
            "roofline": roof,
            "table_build": table_build,
            "historical_region_scan": historical,
            "other_configs": other or None,
            "strong_scaling_per_rank": shard_scaling,
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            s = CpuReference(wl, primes, os.cpu_count() or 1).sample(args.cpu_budget)
            line["cpu_baseline"] = {
                "value": s["pairs"] / s["seconds"], "unit": "pairs/s", "cores": s["cores"],
                "kind": s["kind"],
                "sample": f"rows p={s['rows'][0]}..{s['rows'][1]} of {wl['desc'].split(':')[0]} "
                          f"({s['pairs']} pairs, {s['seconds']:.1f} s)"}
            line["e2e_reference_api"] = reference_api_leg(args, wl, primes)
            s1 = CpuReference(wl, primes, 1).sample(args.cpu_budget / 2)
            line["cpu_baseline_1thread"] = {
                "value": s1["pairs"] / s1["seconds"], "unit": "pairs/s", "cores": 1, "kind": s1["kind"],
                "sample": f"rows p={s1['rows'][0]}..{s1['rows'][1]} of {wl['desc'].split(':')[0]} "
                          f"({s1['pairs']} pairs, {s1['seconds']:.1f} s), the reference's own "
                          "single-thread execution model (engine.hpp:494)"}
            line["table_build"]["cpu_baseline"] = cpu_table_baseline(P256, tables_c2=None)
        print(json.dumps(line), flush=True)
    dev.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: start N ranks on this node (one
    process per GPU, LOCAL_RANK = device) through torch.distributed.run on
    127.0.0.1 with the same arguments; rank 0's JSON line is the output."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench: launching {args.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def launch_check(args):
    """Every rank joins the process group and all-reduces 1; rank 0 prints the
    world it saw (the CPU test of the launcher uses gloo)."""
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group(args.backend)
    t = torch.ones(1, dtype=torch.int64)
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": world, "ranks_seen": int(t.item()),
                          "backend": args.backend if world > 1 else None}), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="C5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU sample")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl")
    ap.add_argument("--same-device", action="store_true",
                    help="plumbing test: all ranks on GPU 0 (use with --backend gloo)")
    ap.add_argument("--launch-check", action="store_true",
                    help="launcher test: init the process group, count the ranks, print, exit")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    if args.launch_check:
        return launch_check(args)
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    from paper_1601_00636_b200.primes import odd_primes
    wl = WORKLOADS[args.workload]
    primes = odd_primes(wl["k"])
    if args.impl == "reference":
        return run_reference_arm(args, wl, primes)
    return run_ours(args, wl, primes)


if __name__ == "__main__":
    sys.exit(main())
