"""Generates tests/golden/golden.json from the REFERENCE ITSELF (oracle/_ref:
the unmodified /root/reference/proj/include headers compiled by oracle/Makefile).

Run in the build container (needs oracle/_ref/libcuboid_ref.so):
    python tests/golden/make_golden.py
The fixture is committed; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_1601_00636_b200.primes import default_primes, odd_primes  # noqa: E402

THREADS = os.cpu_count() or 1


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def stats_json(st, primes, with_surv=False):
    d = {
        "pairs_tested": st.pairs_tested,
        "survivors": st.survivors,
        "kill_histogram": {str(primes[k]): c for k, c in enumerate(st.hist_by_rank) if c},
        "block_r_max": {str(b): r for b, r in sorted(st.block_r_max.items())},
    }
    if with_surv:
        flat = ",".join(f"{p}:{q}" for p, q, _ in st.survivor_pairs)
        d["survivor_sha256"] = sha(flat.encode())
        d["survivor_kinds"] = sorted({k for _, _, k in st.survivor_pairs})
        d["first_survivors"] = [[p, q, k] for p, q, k in st.survivor_pairs[:20]]
    return d


def main():
    g = {"generator": "oracle/_ref (reference headers, unmodified)", "tables": {}, "sieve": {}}
    sets = {"odd32": odd_primes(32), "odd64": odd_primes(64), "odd128": odd_primes(128),
            "odd256": odd_primes(256), "default96": default_primes()}
    rsets = {}
    for name, P in sets.items():
        t0 = time.time()
        s = ref.RefSet.build(P)
        rsets[name] = s
        tb = s.tables()
        g["tables"][name] = {"primes": [P[0], P[-1], len(P)], "bytes": len(tb), "sha256": sha(tb),
                             "index_bytes": len(s.index_bytes()),
                             "index_sha256": sha(s.index_bytes()),
                             "per_table_sha256": [sha(tb[s.offsets[k]:(s.offsets[k + 1] if k + 1 < len(P) else len(tb))])
                                                  for k in range(len(P))]}
        print(name, len(tb), f"{time.time() - t0:.1f}s", flush=True)
    g["tables"]["r11_bytes"] = ref.build_table(11).hex()

    def tri(name, setname, p_lo, p_hi, with_surv=False):
        t0 = time.time()
        st = ref.triangle(rsets[setname], p_lo, p_hi, THREADS, with_sink=with_surv)
        g["sieve"][name] = dict(mode="TRIANGLE", set=setname, p_lo=p_lo, p_hi=p_hi,
                                **stats_json(st, sets[setname], with_surv))
        print(name, st.pairs_tested, f"{time.time() - t0:.1f}s", flush=True)

    def reg(name, setname, p_lo, q_start, p_hi, small_p=False, with_surv=False):
        t0 = time.time()
        st = ref.scan(rsets[setname], p_lo, q_start, p_hi, small_p=small_p, with_sink=with_surv)
        g["sieve"][name] = dict(mode="REGION", set=setname, p_lo=p_lo, q_start=q_start, p_hi=p_hi,
                                resume=[st.resume_p, st.resume_q],
                                **stats_json(st, sets.get(setname, [11]), with_surv))
        print(name, st.pairs_tested, f"{time.time() - t0:.1f}s", flush=True)

    tri("C1", "odd32", 2, 2000, with_surv=True)
    tri("C3", "odd64", 2, 10000)
    tri("C5_sub", "odd256", 200001, 201000)
    tri("C4", "odd128", 2, 100000)
    reg("R152", "default96", 152, 3, 152)
    reg("R152_300", "default96", 152, 3, 300)
    reg("R152_2000", "default96", 152, 3, 2000)
    reg("R153_5000tail", "default96", 153, 5000, 153)
    t0 = time.time()
    st = ref.scan_mt(rsets["default96"], 152, 5000, THREADS)
    g["sieve"]["R152_5000"] = dict(mode="REGION", set="default96", p_lo=152, q_start=3, p_hi=5000,
                                   **stats_json(st, sets["default96"]))
    print("R152_5000", st.pairs_tested, f"{time.time() - t0:.1f}s", flush=True)
    # weak sieve: heavy survivor output
    sets["weak11"] = [11]
    rsets["weak11"] = ref.RefSet.build([11])
    reg("W_row1", "weak11", 1, 1, 1, small_p=True, with_surv=True)
    reg("W_1_40", "weak11", 1, 1, 40, small_p=True, with_surv=True)
    tri("W_T300", "weak11", 2, 300, with_surv=True)
    # small-p region (p < 152 needs small_p), default set
    reg("R1_151", "default96", 1, 1, 151, small_p=True, with_surv=True)
    g["verify_small_region"] = ref.verify_small_region(rsets["default96"])
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(out, "w") as f:
        json.dump(g, f, indent=1, sort_keys=True)
    print("wrote", out)


if __name__ == "__main__":
    main()
