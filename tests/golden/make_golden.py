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


def c4_subsample(g, rset, primes):
    """C4's phi-weighted coprime 10^6-pair subsample (tests/subsample.py):
    first-killer rank of every pair from the reference's is_unsolvable in rank
    order (sievetable.hpp:199-205), stored as hashes plus the rank histogram."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import subsample
    t0 = time.time()
    pq = subsample.sample()
    ranks = ref.classify(rset, pq, THREADS)
    hist = np.bincount(ranks + 1, minlength=len(primes) + 1)
    g["sieve"]["C4_subsample"] = {
        "set": "odd128", "seed": subsample.SEED, "n": int(len(pq)), "p_max": subsample.P_MAX,
        "pairs_sha256": sha(pq.tobytes()), "ranks_sha256": sha(ranks.astype("<i4").tobytes()),
        "survivors": int(hist[0]),
        "rank_histogram": {str(primes[k]): int(c) for k, c in enumerate(hist[1:]) if c},
    }
    print("C4_subsample", len(pq), f"{time.time() - t0:.1f}s", flush=True)


def main(only=()):
    """Regenerate everything, or (with names) only those sieve entries, merged
    into the committed golden.json (e.g. `make_golden.py C5` -- the headline
    config, ~10 min on 8 host threads)."""
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    if only:
        with open(out) as f:
            g = json.load(f)
    else:
        g = {"generator": "oracle/_ref (reference headers, unmodified)", "tables": {}, "sieve": {}}
    sets = {"odd32": odd_primes(32), "odd64": odd_primes(64), "odd128": odd_primes(128),
            "odd256": odd_primes(256), "default96": default_primes()}
    rsets = {}
    for name, P in sets.items():
        if only:
            rsets[name] = ref.RefSet.build(P)
            continue
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

    if only:
        if "C5" in only:
            # BASELINE config 5, the headline: 10^5 < p <= 3*10^5 against the
            # 256-prime set, whole range (engine.hpp:259-277, sievetable.hpp:199-205)
            tri("C5", "odd256", 100001, 300000, with_surv=True)
        if "C4S" in only:
            c4_subsample(g, rsets["odd128"], sets["odd128"])
        with open(out, "w") as f:
            json.dump(g, f, indent=1, sort_keys=True)
        print("updated", out, only)
        return
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
    main(tuple(sys.argv[1:]))
