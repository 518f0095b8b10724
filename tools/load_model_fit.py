"""Offline analysis of k_sieve's static load balance: replays k_plan's work
units for a TRIANGLE launch on the host (same factorisation, drain weights and
row charge as sieve.cu), cuts the unit space into the per-warp slices the
kernel uses, and regresses the measured per-SM finish times (warp-clock dumps
of tools/warp_clocks.py, WCLK_DUMP) against per-slice features -- row setups,
windows by factor-count variant, expected drained windows. Tells which terms
the planner's unit model under- or over-charges.

    python tools/load_model_fit.py <dump.npy> <k primes> <p_lo> <p_hi> [G g]
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import port  # noqa: E402  (analysis tool: table popcounts)
from paper_1601_00636_b200.primes import odd_primes  # noqa: E402

ROW_COST, ALPHA, WARPS_PER_CTA, REG = 800, 12.0, 24, [11, 13, 17, 19, 23, 29, 31, 37]


def kill_fractions(k):
    P = odd_primes(k)
    tb, offs = port.build_set(P)
    out = {}
    for r in REG:
        j = P.index(r)
        bits = [(tb[offs[j] + ((r + b) >> 3)] >> ((r + b) & 7)) & 1 for b in range(r)]  # row 1
        out[r] = sum(bits) / r
    return out


def factor(p):
    f, n, d = [], p, 2
    while d * d <= n:
        if n % d == 0:
            f.append(d)
            while n % d == 0:
                n //= d
        d += 1
    if n > 1:
        f.append(n)
    return f


def rows(p_lo, p_hi, G, g, kill):
    out = []
    for blk in range(p_lo // 100, p_hi // 100 + 1):
        if blk % G != g:
            continue
        for p in range(blk * 100, blk * 100 + 100):
            if p < p_lo or p > p_hi or p < 2:
                out.append((p, 0, 0, 0, 0.0, 0))
                continue
            fs = factor(p)
            odd = [f for f in fs if f != 2]
            even = 2 in fs
            windows = (p - 1 + 31) // 32
            surv = 1.0
            for r in REG:
                if p % r:
                    surv *= 1 - kill[r]
            cop = 0.5 if even else 1.0
            for f in odd:
                cop *= 1 - 1 / f
            wt = 1 + ALPHA * (1 - math.exp(-32 * cop * surv))
            shift = 3 if wt >= 6 else 2 if wt >= 3 else 1 if wt >= 1.5 else 0
            qprob = 1 - math.exp(-32 * cop * surv)  # P(window queued for the drain)
            out.append((p, windows, shift, len(odd), qprob, ROW_COST + (windows << shift)))
    return out


def main():
    dump, k, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    G, g = (int(sys.argv[5]), int(sys.argv[6])) if len(sys.argv) > 6 else (1, 0)
    a = np.load(dump)
    idx, st, en, sm = a[:, 0].astype(int), a[:, 1], a[:, 2], a[:, 3].astype(int)
    nw = len(idx)
    R = rows(lo, hi, G, g, kill_fractions(k))
    units = np.array([r[5] for r in R], dtype=np.float64)
    pre = np.concatenate([[0], np.cumsum(units)])
    W = pre[-1]
    feats = np.zeros((nw, 6))  # segs, windows nf<=2, nf3, nf4-5, nf>5, queued windows
    for w in range(nw):
        ws, we = W * w // nw, W * (w + 1) // nw
        s = np.searchsorted(pre, ws, side="right") - 1
        while s < len(R) and pre[s] < we:
            rs, re = pre[s], pre[s + 1]
            u0, u1 = max(ws, rs) - rs, min(we, re) - rs
            p, win, sh, nf, qp, _ = R[s]
            if win and u1 > ROW_COST:
                w0 = 0 if u0 <= ROW_COST else min(win, -(-(u0 - ROW_COST) // (1 << sh)))
                w1 = min(win, -(-(u1 - ROW_COST) // (1 << sh)))
                if w1 > w0:
                    n = w1 - w0
                    feats[w, 0] += 1
                    feats[w, 1 + (0 if nf <= 2 else 1 if nf == 3 else 2 if nf <= 5 else 3)] += n
                    feats[w, 5] += n * qp
            s += 1
    cta = idx // WARPS_PER_CTA
    X = np.array([feats[cta == c].sum(0) for c in range(cta.max() + 1)])
    y = np.array([en[cta == c].max() for c in range(cta.max() + 1)])  # SM finish time (us)
    A = np.column_stack([X, np.ones(len(X))])
    coef, *_ = np.linalg.lstsq(A, y, rcond=None)
    pred = A @ coef
    names = ["segments", "win_nf<=2", "win_nf3", "win_nf4-5", "win_nf>5", "queued_win", "const"]
    print(f"{dump}: SMs {len(y)}, finish mean {y.mean():.1f} max {y.max():.1f} us, "
          f"R^2 {1 - ((y - pred) ** 2).sum() / ((y - y.mean()) ** 2).sum():.3f}")
    base = coef[1] if coef[1] else 1
    for n_, c_ in zip(names, coef):
        print(f"   {n_:12s} {c_: .4e} us   ({c_ / base: .2f} x a plain window)")
    print("   per-SM feature spread (min/max):", [f"{n_}:{X[:, i].min():.0f}/{X[:, i].max():.0f}"
                                               for i, n_ in enumerate(names[:-1])])


if __name__ == "__main__":
    main()
