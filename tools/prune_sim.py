#!/usr/bin/env python
"""Candidate-pruning simulator (design tool, CPU, numpy only).

Emulates the R12 loss of every candidate of a window for a sample of blocks
(FP32 products, FMA emulated in FP64 then rounded: close enough for counting)
and counts how many full candidate evaluations a WARP executes under several
pruning strategies, 32 blocks per warp:

  scan      : the shipped order (0, +1..+P, -1..-N), one-element bound on
              f <= -3, warp-uniform skip (all 32 lanes prune)
  lane-B1   : evaluate f = 0 and a prior list for every lane, then each lane
              evaluates only its own survivors (bound <= incumbent); the warp
              runs max-over-lanes iterations.  Bound: the max element.
  lane-Bk   : the same with the subset bound over the k largest elements

    python tools/prune_sim.py --kind weight_outlier --rows 4096 --cols 4096 --window -8:8
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

E2M1 = np.array([0, 0.5, 1, 1.5, 2, 3, 4, 6], np.float32)


def e4m3_val(c):
    c = np.asarray(c)
    e, m = c >> 3, c & 7
    return np.where(e == 0, m * 2.0 ** -9, (1 + m / 8.0) * 2.0 ** (e - 7.0)).astype(np.float32)


def e4m3_code(v):
    # nearest code 0..126, ties to even code (v >= 0)
    vals = e4m3_val(np.arange(127))
    idx = np.searchsorted(vals, v)
    idx = np.clip(idx, 1, 126)
    lo, hi = vals[idx - 1], vals[idx]
    dlo, dhi = v - lo, hi - v
    pick_hi = (dhi < dlo) | ((dhi == dlo) & (idx % 2 == 0))
    code = np.where(pick_hi, idx, idx - 1)
    return np.where(v >= 448, 126, code)


def e2m1_round(t):
    a = np.abs(t)
    mids = np.array([0.25, 0.75, 1.25, 1.75, 2.5, 3.5, 5.0], np.float32)
    idx = np.searchsorted(mids, a, side="left")  # a == mid -> lower index
    # ties: at a mid the lower code is idx; go to even code
    is_mid = np.isin(a, mids)
    up_tie = is_mid & (idx % 2 == 1)  # lower code odd -> round up to even
    idx = idx + up_tie
    q = E2M1[np.minimum(idx, 7)]
    return np.copysign(q, t).astype(np.float32)


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32)


def losses(y, codes):
    """y: [nb,16] f32 block values, codes: [nb,C] candidate codes (0 = zero scale)."""
    s = e4m3_val(codes)  # [nb,C]
    rho = np.where(codes == 0, np.float32(0), f32(1.0 / np.where(codes == 0, 1, s)))
    t = f32(y[:, None, :] * rho[:, :, None])
    q = e2m1_round(t)
    d = f32(y[:, None, :].astype(np.float64) - q.astype(np.float64) * s[:, :, None])
    dd = d.astype(np.float64) ** 2
    a = f32(dd[..., 0])
    b = f32(dd[..., 1])
    for i in range(2, 16, 2):
        a = f32(dd[..., i] + a)
        b = f32(dd[..., i + 1] + b)
    return f32(a.astype(np.float64) + b), d


def subset_bound(y, codes, k):
    """R12 loss restricted to the k largest |y| of each block (chain order kept)."""
    order = np.argsort(-np.abs(y), axis=1)[:, :k]
    mask = np.zeros_like(y, bool)
    np.put_along_axis(mask, order, True, axis=1)
    s = e4m3_val(codes)
    rho = np.where(codes == 0, np.float32(0), f32(1.0 / np.where(codes == 0, 1, s)))
    t = f32(y[:, None, :] * rho[:, :, None])
    q = e2m1_round(t)
    d = f32(y[:, None, :].astype(np.float64) - q.astype(np.float64) * s[:, :, None])
    dd = np.where(mask[:, None, :], d.astype(np.float64) ** 2, 0.0)
    a = f32(dd[..., 0])
    b = f32(dd[..., 1])
    for i in range(2, 16, 2):
        a = f32(dd[..., i] + a)
        b = f32(dd[..., i + 1] + b)
    return f32(a.astype(np.float64) + b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="weight_outlier")
    ap.add_argument("--rows", type=int, default=2048)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--window", default="-8:8")
    ap.add_argument("--prior", default="5,4,-1")
    ap.add_argument("--max-blocks", type=int, default=1 << 17)
    a = ap.parse_args()
    import ssgen
    fmin, fmax = (int(v) for v in a.window.split(":"))
    x = ssgen.generate(a.kind, a.rows, a.cols, seed=ssgen.workloads.BASE_SEED, tid=1000)
    x = x.float().numpy().reshape(-1, 16)[: a.max_blocks]
    A = np.abs(x).max()
    G = np.float32(2688.0) / np.float32(A)
    y = f32(x * G)
    m = np.abs(y).max(1)
    c0 = e4m3_code(f32(m * np.float32(1 / 6)))
    offs = np.arange(fmin, fmax + 1)
    cc = c0[:, None] + offs[None, :]
    valid = (cc >= 1) & (cc <= 126)
    cc = np.clip(cc, 1, 126)
    cc[:, offs == 0] = c0[:, None]
    L, _ = losses(y, cc)
    L = np.where(valid | (offs == 0)[None, :], L, np.inf)
    # winner: lexicographic (loss, code)
    key = L.astype(np.float64) * 1e6 + 0  # loss first
    best = L.min(1)
    win = np.where(L == best[:, None], cc, 10 ** 6).min(1)
    f_star = win - c0
    hist = {int(f): int((f_star == f).sum()) for f in offs}
    print("blocks", len(y), "hist", hist)
    nb = len(y) // 32 * 32
    W = nb // 32

    def warp_max(cnt):
        return cnt[:nb].reshape(W, 32).max(1).mean()

    i0 = int(np.where(offs == 0)[0][0])
    prior = [int(v) for v in a.prior.split(",") if v] if a.prior else []
    pi = [int(np.where(offs == f)[0][0]) for f in prior if fmin <= f <= fmax]
    inc = L[:, [i0] + pi].min(1)
    rest = [i for i in range(len(offs)) if i != i0 and i not in pi]
    for k in (1, 2, 3, 4, 6, 8):
        Bk = subset_bound(y, cc, k)
        surv = ((Bk[:, rest] <= inc[:, None]) & np.isfinite(L[:, rest])).sum(1)
        print("k=%d per-block survivors %.2f  warp iterations %.2f  -> evals/warp %.2f"
              % (k, surv.mean(), warp_max(surv), 1 + len(pi) + warp_max(surv)))
    # all-candidates evaluation
    print("full window evals", len(offs), "valid mean", (valid | (offs == 0)).sum(1).mean())



def chain_prefix(y, codes):
    """RN(a_k + b_k) after k = 1..8 pairs (k = 8: the loss) -> [nb, C, 8]."""
    s = e4m3_val(codes)
    rho = np.where(codes == 0, np.float32(0), f32(1.0 / np.where(codes == 0, 1, s)))
    t = f32(y[:, None, :] * rho[:, :, None])
    q = e2m1_round(t)
    d = f32(y[:, None, :].astype(np.float64) - q.astype(np.float64) * s[:, :, None])
    dd = d.astype(np.float64) ** 2
    a = f32(dd[..., 0])
    b = f32(dd[..., 1])
    out = [f32(a.astype(np.float64) + b)]
    for i in range(2, 16, 2):
        a = f32(dd[..., i] + a)
        b = f32(dd[..., i + 1] + b)
        out.append(f32(a.astype(np.float64) + b))
    return np.stack(out, -1)


def lb_max(y, codes):
    """cand_lb: RN(d^2) of the max element; and its saturation flag."""
    m = np.abs(y).max(1)
    s = e4m3_val(codes)
    rho = np.where(codes == 0, np.float32(0), f32(1.0 / np.where(codes == 0, 1, s)))
    t = f32(m[:, None] * rho)
    q = e2m1_round(t)
    d = f32(m[:, None].astype(np.float64) - q.astype(np.float64) * s)
    return f32(d.astype(np.float64) ** 2), t >= 6


def simulate_order(P, offs, order, checks, lbneg_from=None, warp=32, cost_pair=6, cost_chk=4,
                   cost_cand=5, cost_lex=2, lb=None, sat=None):
    """Warp cost (instructions per lane) of one strategy.  P: [nb, C, 8] prefixes.
    order: offsets in evaluation order (first must be 0).  checks: pair counts after
    which a warp-uniform early exit is tested.  lbneg_from: apply the max-element
    bound (warp vote) to f <= -lbneg_from before evaluating."""
    nb = P.shape[0] // warp * warp
    W = nb // warp
    Pw = P[:nb].reshape(W, warp, P.shape[1], 8)
    idx = {int(f): i for i, f in enumerate(offs)}
    best = np.full((W, warp), np.inf, np.float32)
    cost = np.zeros(W)
    evals = np.zeros(W)
    alive = np.ones(W, bool)  # negative-side break (sat) per warp
    for f in order:
        ci = idx[f]
        pref = Pw[:, :, ci, :]
        run = np.ones(W, bool)
        if lbneg_from is not None and f <= -lbneg_from:
            lbw = lb[:nb, ci].reshape(W, warp)
            sw = sat[:nb, ci].reshape(W, warp)
            pr = lbw > best
            brk = (pr & sw).all(1)
            alive &= ~brk
            cost += np.where(alive | brk, 8, 0)  # bound evaluation + votes
            run = alive & ~pr.all(1)
        cost += run * cost_cand + run * cost_lex
        done_pairs = np.zeros(W)
        cont = run.copy()
        last = 0
        for k in list(checks) + [8]:
            cost += cont * (k - last) * cost_pair
            evals += cont * (k - last) / 8.0
            last = k
            if k == 8:
                break
            cost += cont * cost_chk
            pk = pref[:, :, k - 1]
            cont &= ~(pk > best).all(1)
        full = cont
        lw = pref[:, :, 7]
        upd = full[:, None] & (lw < best)
        best = np.where(upd, lw, best)
    return cost.mean(), evals.mean()


def main_order():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="weight_outlier")
    ap.add_argument("--rows", type=int, default=512)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--window", default="-8:8")
    a = ap.parse_args(sys.argv[2:])
    import ssgen
    fmin, fmax = (int(v) for v in a.window.split(":"))
    x = ssgen.generate(a.kind, a.rows, a.cols, seed=ssgen.workloads.BASE_SEED, tid=1000)
    x = x.float().numpy().reshape(-1, 16)
    G = np.float32(2688.0) / np.float32(np.abs(x).max())
    y = f32(x * G)
    m = np.abs(y).max(1)
    c0 = e4m3_code(f32(m * np.float32(1 / 6)))
    offs = np.arange(fmin, fmax + 1)
    cc = np.clip(c0[:, None] + offs[None, :], 1, 126)
    cc[:, offs == 0] = c0[:, None]
    P = chain_prefix(y, cc)
    lb, sat = lb_max(y, cc)
    shipped = [0] + list(range(1, fmax + 1)) + list(range(-1, fmin - 1, -1))
    prio = [0, 5, 4, -1, 1, 6, 3, -2, 2, 7, 8] + list(range(-3, fmin - 1, -1))
    prio = [f for f in prio if fmin <= f <= fmax] + [f for f in range(fmin, fmax + 1) if f not in prio]
    print("shipped (lb on f<=-3):", simulate_order(P, offs, shipped, [], 3, lb=lb, sat=sat, cost_lex=0))
    for chk in ([], [4], [2, 4], [2, 4, 6], [3, 6], [4, 6]):
        print("prio checks", chk, simulate_order(P, offs, prio, chk))
        print("prio checks", chk, "+lb", simulate_order(P, offs, prio, chk, 3, lb=lb, sat=sat))


if __name__ == "__main__" and len(sys.argv) > 1 and sys.argv[1] == "order":
    main_order()
    sys.exit(0)


if __name__ == "__main__":
    main()
