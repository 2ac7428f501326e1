#!/usr/bin/env python3
"""CPU simulation of the Gauss-Seidel systolic pipeline kernel's schedule.

Development aid (not product, not a test oracle): mirrors gs2d.cu's
pipe::gs2d_pipe_kernel — warps as coroutines with the same progress waits,
ring indexing, staging ranges and edge/wrap buffers — so deadlocks and index
errors show up in seconds instead of as a spinning GPU.  Compares against the
in-place lexicographic Gauss-Seidel.

    python tools/sim_gs_pipe.py N T
"""
import sys

import numpy as np

import os

NW, RS = int(os.environ.get("SIM_NW", 12)), int(os.environ.get("SIM_RS", 64))
S, IRS, SG = 8, 64, 64
BIG = 1 << 20


def reference(F, N, T):
    a = F.copy()
    a[0, :] = a[-1, :] = a[:, 0] = a[:, -1] = 0.0
    for _ in range(T):
        for i in range(1, N - 1):
            for j in range(1, N - 1):
                s = a[i - 1, j - 1] + a[i - 1, j]
                s = s + a[i - 1, j + 1]
                s = s + a[i, j - 1]
                s = s + a[i, j]
                s = s + a[i, j + 1]
                s = s + a[i + 1, j - 1]
                s = s + a[i + 1, j]
                s = s + a[i + 1, j + 1]
                a[i, j] = s / 9.0
    return a


class Sim:
    def __init__(self, N, T, F, seed=0):
        self.N, self.T, self.seed = N, T, seed
        self.nb = (N - 2 + 31) // 32
        self.a = F.copy()
        self.a[0, :] = self.a[-1, :] = self.a[:, 0] = self.a[:, -1] = 0.0
        self.wb = [np.full((N, N), np.nan), np.full((N, N), np.nan)]
        self.eb = np.full(((T + 1) * self.nb * 2, N + 2), np.nan)
        self.gp = np.zeros((T + 1) * self.nb, dtype=np.int64)
        self.nclk = N + 63
        self.fin = ((self.nclk + S - 1) // S) * S - 1
        self.rb = [np.full((NW, 32, RS), np.nan) for _ in range(self.nb)]
        self.ir = [np.full((32, IRS), np.nan) for _ in range(self.nb)]
        self.ab = [np.full((NW, SG), np.nan) for _ in range(self.nb)]
        self.be = [np.full((NW, SG), np.nan) for _ in range(self.nb)]
        self.prog = [np.zeros(NW, dtype=np.int64) for _ in range(self.nb)]

    def need(self, v):
        return min(v, self.fin)

    def warp(self, b, w):
        N, T, nb = self.N, self.T, self.nb
        i0 = 1 + 32 * b
        has_above, has_below = b > 0, i0 + 32 <= N - 2
        prog, rb, ir, ab, be = self.prog[b], self.rb[b], self.ir[b], self.ab[b], self.be[b]
        for t in range(w + 1, T + 1, NW):
            lvl, plvl, clvl = t * BIG, (t - 1) * BIG, (t + 1) * BIG
            nchunk = (self.nclk + S - 1) // S

            def eb_row(level, cta, side):
                return self.eb[(level * nb + cta) * 2 + side]

            def prefetch(k):
                c_lo, c_hi = k * S - 1, (k + 1) * S - 2
                if has_above:
                    while self.gp[t * nb + b - 1] < self.need(c_hi + 64):
                        yield "above"
                if has_below and t > 1:
                    while self.gp[(t - 1) * nb + b + 1] < self.need(c_hi - 60):
                        yield "below"
                if w == 0 and t > 1:
                    while prog[NW - 1] < plvl + self.need(c_hi + 5):
                        yield "wrap"
                for col in range(c_lo + 1, c_hi + 2):
                    if 0 <= col < N:
                        ab[w, col & (SG - 1)] = eb_row(t, b - 1, 1)[col] if has_above else 0.0
                for col in range(c_lo - 61, c_hi - 60):
                    if 0 <= col < N:
                        if has_below:
                            src = self.a[i0 + 32] if t - 1 == 0 else eb_row(t - 1, b + 1, 0)
                            be[w, col & (SG - 1)] = src[col]
                        else:
                            be[w, col & (SG - 1)] = 0.0
                if w == 0:
                    src = self.a if t - 1 == 0 else self.wb[((t - 1) // NW) & 1]
                    for r in range(32):
                        for p in range(c_lo - 2 * r + 1, c_hi - 2 * r + 4):
                            if 0 <= p < N:
                                row = i0 + r
                                ir[r, p & (IRS - 1)] = src[row, p] if row <= N - 1 else 0.0

            st = {"a1": np.zeros(32), "a2": np.zeros(32), "a3": np.zeros(32), "c1": np.zeros(32),
                  "c2": np.zeros(32), "d1": np.zeros(32), "d2": np.zeros(32), "d3": np.zeros(32),
                  "out": np.zeros(32)}
            for k in range(nchunk):
                c_lo = k * S - 1
                c_hi = c_lo + S - 1
                yield from prefetch(k)
                if w > 0:
                    while prog[w - 1] < plvl + self.need(c_hi + 5):
                        yield "prod"
                if w < NW - 1:
                    rel = c_hi + 1 - (RS - 4)
                    if rel > 0:
                        while t + 1 <= T and prog[w + 1] < clvl + self.need(rel):
                            yield "cons"
                    elif t + 1 - NW >= 1:
                        while prog[w + 1] < (t + 1 - NW) * BIG + self.fin:
                            yield "cons_prev"
                for c in range(c_lo, c_hi + 1):
                    out = st["out"].copy()
                    sh = np.concatenate([[0.0], out[:31]])
                    newout = np.zeros(32)
                    for lane in range(32):
                        i = i0 + lane
                        j = c - 2 * lane
                        q = j + 1
                        st["a1"][lane] = st["a2"][lane]
                        st["a2"][lane] = st["a3"][lane]
                        st["a3"][lane] = sh[lane] if lane else ab[w, q & (SG - 1)]
                        st["c1"][lane] = st["c2"][lane]
                        prow = rb[w - 1, lane] if w else ir[lane]
                        pmask = (RS if w else IRS) - 1
                        st["c2"][lane] = prow[q & pmask]
                        st["d1"][lane] = st["d2"][lane]
                        st["d2"][lane] = st["d3"][lane]
                        if lane < 31:
                            prow1 = rb[w - 1, lane + 1] if w else ir[lane + 1]
                            st["d3"][lane] = prow1[q & pmask]
                        else:
                            st["d3"][lane] = be[w, q & (SG - 1)]
                        v = 0.0
                        if i <= N - 2 and 1 <= j <= N - 2:
                            s = st["a1"][lane] + st["a2"][lane]
                            for term in (st["a3"][lane], out[lane], st["c1"][lane], st["c2"][lane],
                                         st["d1"][lane], st["d2"][lane], st["d3"][lane]):
                                s = s + term
                            v = s / 9.0
                            if t == T:
                                self.a[i, j] = v
                        newout[lane] = v
                        rb[w, lane, j & (RS - 1)] = v  # every slot, as the kernel
                        if 0 <= j < N:
                            if lane == 0:
                                self.eb[(t * nb + b) * 2 + 0, j] = v
                            if lane == 31:
                                self.eb[(t * nb + b) * 2 + 1, j] = v
                            if w == NW - 1 and t < T and i <= N - 1:
                                self.wb[(t // NW) & 1][i, j] = v
                    st["out"] = newout
                prog[w] = lvl + c_hi + 1
                self.gp[t * nb + b] = c_hi + 1

    def run(self):
        gens = [self.warp(b, w) for b in range(self.nb) for w in range(NW)]
        alive = list(range(len(gens)))
        rng = np.random.default_rng(self.seed)
        skip = rng.random(len(gens)) ** 3 * 0.97  # a few warps run much slower
        while alive:
            progressed = False
            nxt = []
            order = list(alive)
            if self.seed:
                rng.shuffle(order)
            for g in order:
                if self.seed and rng.random() < skip[g]:  # adversarial: skip a turn
                    nxt.append(g)
                    continue
                try:
                    r = next(gens[g])
                    nxt.append(g)
                    # a yield means waiting; try others
                except StopIteration:
                    progressed = True
            # detect deadlock: run each alive gen until it yields twice in a row
            if not progressed:
                states = [self.prog[b].copy() for b in range(self.nb)] + [self.gp.copy()]
                # one more sweep to see if anything moved
                moved = False
                for g in nxt:
                    try:
                        next(gens[g])
                    except StopIteration:
                        moved = True
                after = [self.prog[b].copy() for b in range(self.nb)] + [self.gp.copy()]
                if not moved and all((x == y).all() for x, y in zip(states, after)):
                    raise RuntimeError("deadlock: prog=%s gp=%s" % (self.prog, self.gp))
            alive = nxt
        return self.a


def main():
    N, T = int(sys.argv[1]), int(sys.argv[2])
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    rng = np.random.default_rng(1)
    F = rng.random((N, N))
    got = Sim(N, T, F, seed).run()
    want = reference(F, N, T)
    bad = np.argwhere(got != want)
    print("N=%d T=%d exact=%s nbad=%d first=%s" % (N, T, len(bad) == 0, len(bad), bad[:5].tolist()))


if __name__ == "__main__":
    main()
