"""Experiment: per-warp busy time of k_sieve (needs a library built with
-DCGPU_WARP_CLOCKS, passed as CUBOID_GPU_LIB). Prints the spread of warp end
times and per-SM busy times -- the load-balance evidence."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1601_00636_b200 import device as D, _native as N, odd_primes  # noqa: E402

cfg = {"C3": (64, 2, 10000), "C4": (128, 2, 100000), "C5": (256, 100001, 300000)}
dev = D.Device(0)
L = N.lib()
for spec in sys.argv[1].split(","):  # NAME or NAME/G/g (block-cyclic shard g of G)
    name, *sh = spec.split("/")
    shard = (int(sh[0]), int(sh[1])) if sh else (1, 0)
    k, lo, hi = cfg[name]
    dev.build(odd_primes(k), N.BUILD_PRODUCTION, download=False)
    for _ in range(3):
        dev.sieve(lo, hi, N.TRIANGLE, shard=shard)
    ms = dev.timings_ms()["sieve"]
    buf = (C.c_ulonglong * (3 * 8192))()
    assert L.cgpu_debug_warp_clocks(buf, 8192) == 0
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 3)
    a = a[a[:, 1] > 0]
    t0 = a[:, 0].min()
    st, en, sm = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, a[:, 2]
    busy = en - st
    print(f"{spec}: kernel {ms * 1e3:.0f} us, warps {len(a)}; start max {st.max():.1f} us; "
          f"end min/p10/p50/p90/max {np.percentile(en, [0, 10, 50, 90, 100]).round(1).tolist()}; "
          f"busy mean {busy.mean():.1f} std {busy.std():.1f}")
    sm_end = np.array([en[sm == s].max() for s in np.unique(sm)])
    if os.environ.get("WCLK_DUMP"):  # per-SM last-warp end and busy sum, for offline analysis
        np.save(os.path.join(os.environ["WCLK_DUMP"], spec.replace("/", "_") + ".npy"),
                np.stack([np.arange(len(a)), st, en, sm], 1))  # warp index (blockIdx * warps + w), start, end, smid
    print(f"   per-SM last warp end: min {sm_end.min():.1f} mean {sm_end.mean():.1f} max {sm_end.max():.1f}")
    order = np.argsort(-en)[:8]
    print("   latest warps (idx, end us, sm):", [(int(i), round(float(en[i]), 1), int(sm[i])) for i in order])
    wpc = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cta = np.arange(len(a)) // wpc
    spread = [en[cta == c].max() - en[cta == c].min() for c in np.unique(cta)]
    print(f"   within-CTA end spread: mean {np.mean(spread):.1f} max {np.max(spread):.1f} us")
    # correlation of end time with the warp's position in the unit order
    idx = np.arange(len(a))
    print("   end time by warp-index decile:",
          [round(float(en[(idx * 10 // len(a)) == d].mean()), 1) for d in range(10)])
