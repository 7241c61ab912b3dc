"""Synthetic workloads of BASELINE.json's configs (host-side input source).

The reference draws ids from a Zipf law whose rank maps straight to the row
id (low ids hot, src/data.cpp:85-98,128-136) with a fixed pooling fan-in.
The B200 configs extend that with per-table rows/dims and power-law bag
lengths; data are synthetic, seeded, and identical for
every implementation they are fed to.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# Criteo Kaggle (DAC) categorical cardinalities, clipped at 10M rows
# (sum 33,631,350 -- SURVEY.md 8(d) cfg2).
CRITEO_KAGGLE = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194, 27,
                 14992, 5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572]


@dataclass
class Workload:
    name: str
    rows: list
    dims: list
    batch: int                      # per GPU
    zipf: float = 1.05
    fixed_len: int | None = None    # pooling factor (reference: ids_per_sample)
    len_lo: int = 1                 # power-law bag lengths on [len_lo, len_hi]
    len_hi: int = 50
    len_alpha: float = 1.0
    mesh: tuple = (1, 1)            # (N = MP ranks per group, M = DP groups)
    dtype: str = "fp32"
    strategy: str = "table-wise"
    c: float = 1.0
    eta: float = 0.05
    scramble: bool = False          # hashed id -> row bijection (balances row-wise owners)
    describe: str = ""
    _cdf: dict = field(default_factory=dict, repr=False)

    @property
    def F(self) -> int:
        return len(self.rows)

    @property
    def sum_dims(self) -> int:
        return int(sum(self.dims))

    def mean_len(self) -> float:
        if self.fixed_len is not None:
            return float(self.fixed_len)
        L = np.arange(self.len_lo, self.len_hi + 1, dtype=np.float64)
        p = L ** (-self.len_alpha)
        return float((L * p).sum() / p.sum())

    # ---- planning cost ----
    # One distinct row costs about as much as UNIQUE_WEIGHT id contributions
    # (segment flush: moment + row read-modify-write, an L2 miss for big
    # tables): fitted on B200 from per-rank lookup + update times of a 4x1
    # config-3 run (≈0.135 ns per id, ≈0.44 ns per distinct row).  The
    # table-wise LPT of plan_greedy is fed expected ids plus weighted expected
    # distinct rows as each table's "expected lookups".
    UNIQUE_WEIGHT = 3.0

    def expected_unique(self, f: int, n: float) -> float:
        """E[#distinct rows] among n Zipf draws from table f."""
        rows, s = int(self.rows[f]), self.zipf
        if rows > 20_000_000:
            return float(min(n, rows))
        k = np.arange(1, rows + 1, dtype=np.float64)
        p = k ** (-s)
        p /= p.sum()
        return float(np.sum(-np.expm1(n * np.log1p(-p))))

    def plan_cost(self, f: int, n_req: int) -> float:
        ids = self.batch * self.mean_len() * n_req
        return ids + self.UNIQUE_WEIGHT * self.expected_unique(f, ids)

    def table_plan(self, n_mp: int) -> list:
        """Table-wise plan for an MP group of n_mp: the reference LPT
        (plan_greedy over plan_cost) refined by local search -- move a table
        off the most loaded rank, or swap two tables, while that lowers the
        maximum load.  On config 2 this takes max/mean from 1.055 to 1.001 at
        N = 4 and from 1.13 to 1.06 at N = 8."""
        from . import api

        F = self.F
        cost = [self.plan_cost(f, n_mp) for f in range(F)]
        prof = [(f, int(self.rows[f]) * int(self.dims[f]) * 4, float(cost[f]), int(self.rows[f])) for f in range(F)]
        plan = api.plan_greedy(prof, n_mp, "table-wise")
        if n_mp <= 1:
            return plan
        assign = [0] * F
        for e in plan:
            assign[e["table_id"]] = e["local_rank"]
        load = np.zeros(n_mp)
        for f, r in enumerate(assign):
            load[r] += cost[f]
        for _ in range(10 * F):
            hi = int(np.argmax(load))
            cur, best = load.max(), None
            mine = [f for f in range(F) if assign[f] == hi]
            for f in mine:
                for r2 in range(n_mp):
                    if r2 == hi:
                        continue
                    nl = load.copy()
                    nl[hi] -= cost[f]
                    nl[r2] += cost[f]
                    if nl.max() < cur - 1e-9 and (best is None or nl.max() < best[0]):
                        best = (nl.max(), f, None, r2)
                    for g in [g for g in range(F) if assign[g] == r2]:
                        nl = load.copy()
                        nl[hi] += cost[g] - cost[f]
                        nl[r2] += cost[f] - cost[g]
                        if nl.max() < cur - 1e-9 and (best is None or nl.max() < best[0]):
                            best = (nl.max(), f, g, r2)
            if best is None:
                break
            _, f, g, r2 = best
            load[hi] -= cost[f]
            load[r2] += cost[f]
            assign[f] = r2
            if g is not None:
                load[r2] -= cost[g]
                load[hi] += cost[g]
                assign[g] = hi
        return [{"table_id": f, "row_lo": 0, "row_hi": int(self.rows[f]), "local_rank": int(assign[f])}
                for f in range(F)]

    # ---- sampling ----
    def _sample_ids(self, rng, rows: int, n: int) -> np.ndarray:
        if n == 0:
            return np.zeros(0, np.uint32)
        s = self.zipf
        u = rng.random(n)
        if rows <= 20_000_000:
            key = (rows, s)
            cdf = self._cdf.get(key)
            if cdf is None:
                k = np.arange(1, rows + 1, dtype=np.float64)
                cdf = np.cumsum(k ** (-s))
                cdf /= cdf[-1]
                self._cdf[key] = cdf
            ids = np.searchsorted(cdf, u, side="right")
        else:  # continuous inverse-CDF approximation for huge tables
            if abs(s - 1.0) < 1e-9:
                x = np.exp(u * np.log(rows + 1.0))
            else:
                a = 1.0 - s
                x = (1.0 + u * ((rows + 1.0) ** a - 1.0)) ** (1.0 / a)
            ids = np.floor(x).astype(np.int64) - 1
        ids = np.minimum(ids, rows - 1).astype(np.uint64)
        if self.scramble:
            ids = _bijection(ids, rows)
        return ids.astype(np.uint32)

    def lengths(self, rng, batch: int | None = None) -> np.ndarray:
        B, F = batch or self.batch, self.F
        if self.fixed_len is not None:
            return np.full(B * F, self.fixed_len, np.uint32)
        L = np.arange(self.len_lo, self.len_hi + 1)
        p = L.astype(np.float64) ** (-self.len_alpha)
        p /= p.sum()
        return rng.choice(L, size=B * F, p=p).astype(np.uint32)

    def batch_for(self, seed: int, step: int, rank: int, batch: int | None = None):
        """(lengths[B*F], ids[nnz]) of one rank's batch: sample-major bags
        (batch overrides B, e.g. for a bounded CPU sample)."""
        batch = batch or self.batch
        rng = np.random.default_rng([seed, step, rank, 1])
        lengths = self.lengths(rng, batch)
        F = self.F
        off = np.zeros(len(lengths) + 1, np.int64)
        np.cumsum(lengths, out=off[1:])
        ids = np.empty(int(off[-1]), np.uint32)
        for f in range(F):  # table f's item positions in ascending order, O(its ids)
            bags = np.arange(f, batch * F, F)
            lf = lengths[bags].astype(np.int64)
            n = int(lf.sum())
            if n == 0:
                self._sample_ids(rng, int(self.rows[f]), 0)
                continue
            first = np.zeros(len(lf), np.int64)
            np.cumsum(lf[:-1], out=first[1:])
            pos = np.repeat(off[bags] - first, lf) + np.arange(n, dtype=np.int64)
            ids[pos] = self._sample_ids(rng, int(self.rows[f]), n)
        return lengths, ids

    def upstream_for(self, seed: int, step: int, rank: int, batch: int | None = None) -> np.ndarray:
        """Synthetic per-sample upstream gradient f32(1e-3 * N(0,1))."""
        rng = np.random.default_rng([seed, step, rank, 2])
        out = rng.standard_normal((batch or self.batch, self.sum_dims), dtype=np.float32)
        out *= np.float32(1e-3)
        return out


def _bijection(ids: np.ndarray, rows: int) -> np.ndarray:
    """Fixed permutation of [0, rows): multiplicative hash by an odd constant
    coprime with rows, then modulo (documented id -> row scramble)."""
    mult = 2654435761
    while np.gcd(mult, rows) != 1:
        mult += 2
    return (ids.astype(np.uint64) * np.uint64(mult)) % np.uint64(rows)


def get(name: str, **over) -> Workload:
    """The five BASELINE.json configs."""
    if name == "cfg1":
        w = Workload("cfg1", [100_000] * 8, [64] * 8, 512, zipf=1.0, fixed_len=20, c=1.0, eta=0.1,
                     describe="8 tables x 100K rows x D=64 fp32, B=512, pooling 20, Zipf 1.0, 1x1")
    elif name == "cfg2":
        rows = [min(r, 10_000_000) for r in CRITEO_KAGGLE]
        w = Workload("cfg2", rows, [128] * 26, 16384, zipf=1.05, c=1.0,
                     describe="26 Criteo-Kaggle tables (clipped 10M rows, 33.6M total) x D=128 fp32, "
                              "B=16384/GPU, bag length power-law [1,50] alpha=1 (mean 11.1), Zipf 1.05 ids")
    elif name == "cfg3":
        rows = [min(r, 10_000_000) for r in CRITEO_KAGGLE]
        w = Workload("cfg3", rows, [128] * 26, 16384, zipf=1.05, mesh=(8, 1),
                     describe="cfg2 tables, B=16384/GPU, 2D mesh sweep")
    elif name == "cfg4":
        w = Workload("cfg4", [200_000_000] * 4, [128] * 4, 16384, zipf=1.05, mesh=(4, 2), dtype="bf16",
                     strategy="row-wise", c=2.0,
                     describe="4 tables x 200M rows x D=128 bf16 / fp32 accumulators, row-wise, 4x2")
    elif name == "cfg5":
        rng = np.random.default_rng(500)
        dims = (rng.integers(4, 33, size=500) * 8).tolist()
        rows = np.exp(rng.uniform(np.log(1e3), np.log(2e6), size=500)).astype(int).tolist()
        w = Workload("cfg5", rows, dims, 32768, zipf=1.05, len_lo=1, len_hi=200, mesh=(2, 4), c=4.0,
                     describe="500 tables, D in [32,256], pooling power-law [1,200], B=32768/GPU, 2x4")
    else:
        raise ValueError(name)
    for k, v in over.items():
        setattr(w, k, v)
    return w
