"""The reference's `bench` subcommand (cli.hpp:213-248, cmd_bench) on the GPU:
load the table files, scan() the REGION rows [p_start, p_end] from q_low
`repeat` times and print the same lines -- pairs and seconds per run, the
seconds per pair against the paper's 3.54e-07 s/pair, and the run-to-run
variation. scan() here is cuboid.scan (the device sieve); elapsed is its wall
time including the host handoff, like ScanStats::elapsed.

    python -m paper_1601_00636_b200.bench_cmd --tables T.bin --index P.bin 152 5000 [--repeat 3]
"""
from __future__ import annotations

import argparse
import sys

from . import cuboid


def cmd_bench(tables_path: str, index_path: str, p_start: int, p_end: int, repeat: int,
              p_limit: int = cuboid.P_LIMIT_32BIT, batch_pairs: int = 1 << 16, out=sys.stdout) -> int:
    s = cuboid.SieveSet.load_files(tables_path, index_path)
    opt = cuboid.ScanOptions(p_limit=p_limit, batch_pairs=batch_pairs)
    q0 = cuboid.q_bounds(p_start)[0]
    rates = []
    for run in range(repeat):
        st = cuboid.scan(s, (p_start, q0), p_end, opt=opt)
        secs = st.elapsed
        out.write(f"run {run + 1}: {st.pairs_tested} pairs in {secs:g} s")
        if st.pairs_tested == 0:
            out.write(" (empty range)\n")
            continue
        dt = secs / st.pairs_tested
        rates.append(dt)
        out.write(f", dt={dt:g} s/pair\n")
    if rates:
        out.write("reference dt: 3.54e-07 s/pair\n")
        if len(rates) > 1:
            lo, hi = min(rates), max(rates)
            out.write(f"run-to-run variation: {(hi - lo) / hi * 100.0:g}%\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="bench", description=__doc__.split("\n")[0])
    ap.add_argument("--tables", default="Cuboid_pq_bit_tables.bin")
    ap.add_argument("--index", default="Cuboid_primes.bin")
    ap.add_argument("--p-limit", type=int, default=cuboid.P_LIMIT_32BIT)
    ap.add_argument("--batch-pairs", type=int, default=1 << 16)
    ap.add_argument("--repeat", type=int, default=3)
    ap.add_argument("p_start", type=int)
    ap.add_argument("p_end", type=int)
    a = ap.parse_args(argv)
    return cmd_bench(a.tables, a.index, a.p_start, a.p_end, a.repeat, a.p_limit, a.batch_pairs)


if __name__ == "__main__":
    sys.exit(main())
