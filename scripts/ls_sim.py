"""Critical-path model of the level-synchronous Gauss-Seidel programs (gs_ls.cu, one
compute warp per group; written for the first record format, still the model behind DESIGN §5.1):
K contiguous groups, rows in (DAG level, width, index) order inside a group,
<= 32 rows per step; a step starts after the group's previous step and after
every step (of the previous group) it imports from, plus a hop.  Calibrated on
B200 on c5 level 2: step cost ~115 ns + 5 ns/row, effective hop
~3 us (it overestimates c4 level 2 by ~35 %: a model, not a predictor).

    python scripts/ls_sim.py LEVEL.npz K[,K...] [h0_us h1_us hop_us]

LEVEL.npz from scripts/dump_levels.py.
"""
import sys

import numpy as np


def build(rp, ci, lev, K, fwd=True):
    n = len(rp)-1
    gstart = (np.arange(K+1, dtype=np.int64)*n//K)
    t_of_row = np.arange(n) if fwd else n-1-np.arange(n)
    gid = np.empty(n, np.int64)
    for g in range(K):
        ts = np.arange(gstart[g], gstart[g+1]); rows = ts if fwd else n-1-ts
        gid[rows] = g
    # deps
    rows_of = np.repeat(np.arange(n), np.diff(rp))
    dep = (ci < rows_of) if fwd else (ci > rows_of)
    di, dj = rows_of[dep], ci[dep]
    if np.any((gid[dj] != gid[di]) & (gid[dj] != gid[di]-1)): return None
    nd = np.bincount(di, minlength=n)
    # per group order: (lev, nd, t)
    step_of = np.empty(n, np.int64); steps=[]  # steps: list of (g, rows)
    sidx = 0; gsteps=[]
    for g in range(K):
        ts = np.arange(gstart[g], gstart[g+1]); rows = ts if fwd else n-1-ts
        order = rows[np.lexsort((np.arange(len(rows)), nd[rows], lev[rows]))]
        L = lev[order]
        first = sidx
        u = 0; m = len(order)
        # split into runs of equal level, chunks of 32
        bounds = np.flatnonzero(np.diff(L)) + 1
        starts = np.concatenate(([0], bounds)); ends = np.concatenate((bounds, [m]))
        for s0, e0 in zip(starts, ends):
            for s in range(s0, e0, 32):
                step_of[order[s:min(s+32,e0)]] = sidx; sidx += 1
        gsteps.append((first, sidx))
    return gid, step_of, gsteps, di, dj, nd

def simulate(b, h=0.09, c=1.0, hw=None):
    gid, step_of, gsteps, di, dj, nd = b
    S = gsteps[-1][1]
    # cross deps per step: max producer step
    cross = gid[dj] != gid[di]
    need = np.full(S, -1, np.int64)
    np.maximum.at(need, step_of[di[cross]], step_of[dj[cross]])
    T = np.zeros(S)
    for g,(s0,s1) in enumerate(gsteps):
        t = 0.0
        for s in range(s0, s1):
            p = need[s]
            if p >= 0: t = max(t, T[p] + c)
            t += h
            T[s] = t
    return T, [T[s1-1] for (s0,s1) in gsteps], S

def step_rows(b):
    gid, step_of, gsteps, di, dj, nd = b
    S = gsteps[-1][1]
    rows = np.bincount(step_of, minlength=S)
    wid = np.zeros(S, np.int64)
    np.maximum.at(wid, step_of, nd)
    return rows, wid

def simulate2(b, hfun, c=1.8):
    gid, step_of, gsteps, di, dj, nd = b
    S = gsteps[-1][1]
    rows, wid = step_rows(b)
    hs = hfun(rows, wid)
    cross = gid[dj] != gid[di]
    need = np.full(S, -1, np.int64)
    np.maximum.at(need, step_of[di[cross]], step_of[dj[cross]])
    T = np.zeros(S)
    ends = []
    for g,(s0,s1) in enumerate(gsteps):
        t = 0.0
        for s in range(s0, s1):
            p = need[s]
            if p >= 0 and T[p] + c > t: t = T[p] + c
            t += hs[s]
            T[s] = t
        ends.append(t)
    return np.array(ends)

def simulate3(b, hfun, Wc, c_l2=3.0, c_sm=0.1):
    """groups g -> CTA g // Wc; cross-group hop c_sm inside a CTA, c_l2 across"""
    gid, step_of, gsteps, di, dj, nd = b
    S = gsteps[-1][1]
    rows, wid = step_rows(b)
    hs = hfun(rows, wid)
    cross = gid[dj] != gid[di]
    need = np.full(S, -1, np.int64)
    np.maximum.at(need, step_of[di[cross]], step_of[dj[cross]])
    g_of_step = np.empty(S, np.int64)
    for g,(s0,s1) in enumerate(gsteps): g_of_step[s0:s1] = g
    T = np.zeros(S); ends=[]
    for g,(s0,s1) in enumerate(gsteps):
        t = 0.0
        for s in range(s0, s1):
            p = need[s]
            if p >= 0:
                c = c_sm if g_of_step[p] // Wc == g // Wc else c_l2
                if T[p] + c > t: t = T[p] + c
            t += hs[s]
            T[s] = t
        ends.append(t)
    return np.array(ends)

def build_b(rp, ci, lev, gstart, fwd=True):
    n = len(rp)-1; K = len(gstart)-1
    gid = np.empty(n, np.int64)
    for g in range(K): gid[gstart[g]:gstart[g+1]] = g
    rows_of = np.repeat(np.arange(n), np.diff(rp))
    dep = (ci < rows_of)
    di, dj = rows_of[dep], ci[dep]
    if np.any((gid[dj] != gid[di]) & (gid[dj] != gid[di]-1)): return None
    nd = np.bincount(di, minlength=n)
    step_of = np.empty(n, np.int64); sidx = 0; gsteps=[]
    for g in range(K):
        rows = np.arange(gstart[g], gstart[g+1])
        order = rows[np.lexsort((rows, nd[rows], lev[rows]))]
        L = lev[order]; first = sidx; m=len(order)
        bounds = np.flatnonzero(np.diff(L)) + 1
        starts = np.concatenate(([0], bounds)); ends = np.concatenate((bounds, [m]))
        for s0, e0 in zip(starts, ends):
            for s in range(s0, e0, 32):
                step_of[order[s:min(s+32,e0)]] = sidx; sidx += 1
        gsteps.append((first, sidx))
    return gid, step_of, gsteps, di, dj, nd

def equal_steps_partition(lev, K, n):
    # weight of a prefix: sum over rows of 1/rows-in-its-level-window approximated by
    # per-row cost w_i = max(1/32, 1/cnt(level of i within a local window))
    # simple: cumulative cost = number of distinct (level) runs ~ use per-level row counts in sliding window
    W = 2048
    cost = np.empty(n)
    for s in range(0, n, W):
        L = lev[s:s+W]
        cnt = np.bincount(L - L.min())
        c = cnt[L - L.min()]
        cost[s:s+W] = np.maximum(1.0/32, 1.0/c)
    cum = np.concatenate(([0], np.cumsum(cost)))
    tgt = np.linspace(0, cum[-1], K+1)
    gs = np.searchsorted(cum, tgt).astype(np.int64); gs[0]=0; gs[-1]=n
    return gs


if __name__ == "__main__":
    z = np.load(sys.argv[1])
    rp, ci, lf = z["rp"], z["ci"], z["lf"]
    h0, h1, hop = (float(x) for x in sys.argv[3:6]) if len(sys.argv) > 5 else (0.115, 0.005, 3.0)
    print(f"n {len(rp) - 1} DAG depth {lf.max() + 1}")
    for K in (int(k) for k in sys.argv[2].split(",")):
        b = build(rp, ci, lf, K)
        if b is None:
            print(f"K={K}: not eligible (a dependency beyond the previous group)")
            continue
        e = simulate2(b, lambda r, w: h0 + h1 * r, hop)
        print(f"K={K}: steps {b[2][-1][1]}  modelled sweep {e.max():.0f} us")
