"""Python restatement of the segmented-ring exchange protocol (TEST
INFRASTRUCTURE): the same data flow as csrc/shard_kernels.cuh +
csrc/tb_kernel.cuh + csrc/sharded.cu, written with plain integers so it can
run under torch.distributed (gloo) on CPU and be checked against the oracle.

Per launch of K steps on every rank g (segment [lo_g, lo_{g+1}) of ids):
  pack    -- record = first 16 cars + the origin-cone slots this rank owns
  gather  -- all-gather of the records
  plan    -- assemble the cone window, simulate it K steps -> W_j, c_j
  halo    -- the next rank's first 16 cars
  advance -- own cars + halo, K steps, draws indexed by global rank
"""
from __future__ import annotations

M = 2147483647
A = 48271
HEAD = 16


def seeded(seed: int) -> int:
    s = seed % M
    return 1 if s == 0 else s


def threshold(p: float) -> int:
    lo, hi = 0, M
    while lo < hi:
        mid = (lo + hi) // 2
        if float(mid) / float(M) < p:
            lo = mid + 1
        else:
            hi = mid
    return lo


def step_cars(xs, vs, ids, L, vmax, tp, s0, t, N, W):
    """One synchronous step of consecutive cars (leader = next entry; the
    last entry's leader is unknown and its result is garbage).  Returns the
    number of wraps and the new arrays."""
    n = len(xs)
    nx, nv, wraps = [0] * n, [0] * n, []
    for i in range(n):
        x, v = xs[i], vs[i]
        xl = xs[i + 1] if i + 1 < n else x
        gap = (xl - x - 1) % L
        v = min(v + 1, vmax, gap)
        rank = (ids[i] + W) % N
        s = s0 * pow(A, (t * N + 1 + rank) % (M - 1), M) % M
        if s < tp and v > 0:
            v -= 1
        nxp = x + v
        wraps.append(nxp >= L)
        nx[i], nv[i] = nxp % L, v
    return nx, nv, wraps


class Shard:
    def __init__(self, L, N, vmax, p, seed, G, g, x_id, v_id, K):
        self.L, self.N, self.vmax, self.G, self.g, self.K = L, N, vmax, G, g, K
        self.tp, self.s0 = threshold(p), seeded(seed)
        self.lo = [k * N // G for k in range(G + 1)]
        a, b = self.lo[g], self.lo[g + 1]
        self.ids = list(range(a, b))
        self.x = [int(u) for u in x_id[a:b]]
        self.v = [int(u) for u in v_id[a:b]]
        self.t, self.W = 0, 0
        self.sumv = []  # this rank's partial velocity sum per step

    def cone_ids(self):
        Mc = self.K * self.vmax
        h = (self.N - self.W) % self.N
        return [(h - Mc + i) % self.N for i in range(Mc + self.K)]

    def pack(self):
        own = {gid: (self.x[k], self.v[k]) for k, gid in enumerate(self.ids)}
        cone = [own.get(gid) for gid in self.cone_ids()]
        return {"g": self.g, "head": list(zip(self.x[:HEAD], self.v[:HEAD])), "cone": cone}

    def plan(self, records):
        recs = {r["g"]: r for r in records}
        Mc = self.K * self.vmax
        ids = self.cone_ids()
        xs, vs = [], []
        for i, gid in enumerate(ids):
            owner = max(k for k in range(self.G) if self.lo[k] <= gid)
            xv = recs[owner]["cone"][i]
            xs.append(xv[0])
            vs.append(xv[1])
        Ws, cs, W = [], [], self.W
        for j in range(self.K):
            xs, vs, wr = step_cars(xs, vs, ids, self.L, self.vmax, self.tp, self.s0, self.t + j,
                                   self.N, W)
            c = sum(1 for i in range(Mc) if wr[i])
            Ws.append(W)
            cs.append(c)
            W = (W + c) % self.N
        self.halo = recs[(self.g + 1) % self.G]["head"]
        return Ws, cs

    def advance(self, Ws, cs):
        xs = self.x + [h[0] for h in self.halo]
        vs = self.v + [h[1] for h in self.halo]
        ids = self.ids + [(self.ids[-1] + 1 + i) % self.N for i in range(HEAD)]
        n = len(self.x)
        for j in range(self.K):
            xs, vs, _ = step_cars(xs, vs, ids, self.L, self.vmax, self.tp, self.s0, self.t + j,
                                  self.N, Ws[j])
            self.sumv.append(sum(vs[:n]))
        self.x, self.v = xs[:n], vs[:n]
        self.t += self.K
        self.W = (Ws[-1] + cs[-1]) % self.N


def rank_order(x_id, v_id, W, N):
    """ID order -> increasing-position (rank) order: rank(id) = (id+W) mod N."""
    xr, vr = [0] * N, [0] * N
    for gid in range(N):
        r = (gid + W) % N
        xr[r], vr[r] = x_id[gid], v_id[gid]
    return xr, vr
