"""Parity oracle for the 2D-sparse-parallel embedding step.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline / reference legs may import this package; the
product package (``paper_2508_03854_b200``) never does.

Two interchangeable backends with one interface:

* ``Oracle("port")`` -- ``oracle/s2d_oracle.c``, a plain-C restatement of the
  reference algorithm (each function cites the reference file:line it follows).
* ``Oracle("reference")`` -- ``oracle/_ref/libs2dref.so``: the UNMODIFIED
  reference sources (``/root/reference/proj/src``) compiled by
  ``oracle/Makefile`` and driven through their public API by
  ``oracle/ref_harness.cpp``.

Parity status: pinned.  ``tests/test_oracle.py`` checks the port against the
reference's own known-answer tests and against ``tests/golden/`` vectors that
``tests/golden/make_golden.py`` produced with the compiled reference.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libs2dref.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build(force: bool = False) -> None:
    """Compile the checkers (make -C oracle).  The reference part is built only
    where /root/reference exists; elsewhere the prebuilt _ref/ is used."""
    if force or not os.path.exists(PORT_SO) or (
        os.path.isdir("/root/reference/proj") and not os.path.exists(REF_SO)
    ):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def reference_available() -> bool:
    return os.path.exists(REF_SO)


class _OrCfg(C.Structure):
    _fields_ = [
        ("F", C.c_uint32), ("N", C.c_uint32), ("B", C.c_uint32),
        ("rows", C.c_void_p), ("dims", C.c_void_p),
        ("n_entries", C.c_uint32), ("plan", C.c_void_p),
        ("eta", C.c_double), ("eps", C.c_double), ("c", C.c_double),
        ("sgd", C.c_int),
        ("mean", C.c_void_p),
    ]


class _OrDump(C.Structure):
    _fields_ = [
        ("dem_len", C.c_void_p), ("dem_ids", C.c_void_p), ("dem_nnz", C.c_void_p),
        ("mask", C.c_void_p), ("part", C.c_void_p), ("part_cnt", C.c_void_p),
        ("grad", C.c_void_p), ("grad_cnt", C.c_void_p),
        ("cap_ids", C.c_uint64), ("cap_floats", C.c_uint64),
    ]


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _ptr_array(arrs):
    return (C.c_void_p * len(arrs))(*[_ptr(a) for a in arrs])


@dataclass
class MeshSpec:
    """Tables, plan, mesh and optimizer of one run (the reference's
    TrainerOptions restricted to the embedding path, trainer.hpp:47-70)."""

    rows: np.ndarray                # [F] uint32
    dims: np.ndarray                # [F] uint32
    plan: np.ndarray                # [E,4] uint32 (table_id,row_lo,row_hi,local_rank)
    T: int = 1
    M: int = 1
    B: int = 1
    eta: float = 0.1
    eps: float = 1e-8
    c: float = 1.0
    sgd: bool = False
    mean: np.ndarray | None = None  # [F] uint8 per-table mean pooling (None: all sum)

    @property
    def N(self) -> int:
        return self.T // self.M

    @property
    def F(self) -> int:
        return len(self.rows)

    @property
    def sum_dims(self) -> int:
        return int(self.dims.sum())

    def replica_floats(self) -> int:
        return int((self.rows.astype(np.uint64) * self.dims).sum())

    def replica_rows(self) -> int:
        return int(self.rows.astype(np.uint64).sum())

    def woff(self) -> np.ndarray:
        o = np.zeros(self.F + 1, np.uint64)
        o[1:] = np.cumsum(self.rows.astype(np.uint64) * self.dims)
        return o

    def voff(self) -> np.ndarray:
        o = np.zeros(self.F + 1, np.uint64)
        o[1:] = np.cumsum(self.rows.astype(np.uint64))
        return o


@dataclass
class Dump:
    dem_len: np.ndarray
    dem_ids: list
    mask: np.ndarray
    part: list  # part[o][n] float32 arrays
    grad: list  # grad[n][o]


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        if kind == "port":
            build()
            self.lib = C.CDLL(PORT_SO)
        elif kind == "reference":
            build()
            if not os.path.exists(REF_SO):
                raise FileNotFoundError(REF_SO)
            self.lib = C.CDLL(REF_SO)
        else:
            raise ValueError(kind)
        L = self.lib
        p = "or_" if kind == "port" else "ref_"
        self._p = p
        if kind == "port":
            L.or_init_rows.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _f32p]
            L.or_group_step.argtypes = [C.c_void_p] * 9
            L.or_group_step.restype = C.c_int
            L.or_synthetic_upstream.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _f32p]
            L.or_mix64.restype = C.c_uint64
            L.or_mix64.argtypes = [C.c_uint64]
        else:
            L.ref_init_rows.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, _f32p]
            L.ref_init_rows.restype = C.c_int
            L.ref_group_step.argtypes = [
                C.c_uint32, C.c_uint32, C.c_uint32, _u32p, _u32p, C.c_uint32, _u32p,
                C.c_double, C.c_double, C.c_double, C.c_int,
                C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, _f32p, _f32p, C.c_void_p, C.c_uint32,
                C.POINTER(C.c_double)]
            L.ref_group_step.restype = C.c_int
            L.ref_last_error.restype = C.c_char_p
            L.ref_gen_batch_ids.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                            C.c_double, C.c_uint32, C.c_uint32, _u32p]
            L.ref_gen_batch_ids.restype = C.c_int
        getattr(L, p + "pool_ids").restype = C.c_int
        getattr(L, p + "adagrad_row_step").restype = C.c_double
        getattr(L, p + "effective_lr").restype = C.c_double
        getattr(L, p + "effective_lr").argtypes = [C.c_double] * 4
        getattr(L, p + "plan_greedy").restype = C.c_int
        getattr(L, p + "plan_greedy").argtypes = [C.c_uint32, _u32p, _f64p, _u64p, C.c_uint32, C.c_int, _u32p]
        getattr(L, p + "sync").restype = C.c_int
        getattr(L, p + "sync").argtypes = [C.c_uint32, C.c_uint32, _u32p, _u32p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]

    # ---- function-level API -------------------------------------------------
    def init_rows(self, table_id, rows, lo, hi, dim, seed) -> np.ndarray:
        out = np.empty((hi - lo) * dim, np.float32)
        if self.kind == "port":
            self.lib.or_init_rows(table_id, lo, hi, dim, seed, out)
        else:
            rc = self.lib.ref_init_rows(table_id, rows, lo, hi, dim, seed, out)
            if rc:
                raise ValueError(self.lib.ref_last_error().decode())
        return out.reshape(hi - lo, dim)

    def init_rows_list(self, table_id, rows, dim, seed) -> np.ndarray:
        """init_table rows for a list of row ids (port), n x dim."""
        rows = np.ascontiguousarray(rows, np.uint32)
        out = np.empty((rows.size, dim), np.float32)
        fn = self.lib.or_init_rows_list
        fn.argtypes = [C.c_uint32, _u32p, C.c_uint64, C.c_uint32, C.c_uint64, _f32p]
        fn(table_id, rows, rows.size, dim, seed, out)
        return out

    def row_gradients(self, rows, dims, B, lengths, ids, upstream):
        """(keys, g): every touched (table, row) of one N = 1 step in
        ascending (table, row) order (key = table << 32 | row) and its f64
        gradient (item-order sum x 1/B, optimizer.cpp:25-59), zero-padded to
        max(dims) columns (port)."""
        rows = np.ascontiguousarray(rows, np.uint32)
        dims = np.ascontiguousarray(dims, np.uint32)
        lengths = np.ascontiguousarray(lengths, np.uint32)
        ids = np.ascontiguousarray(ids, np.uint32)
        upstream = np.ascontiguousarray(upstream, np.float32)
        cap = int(min(ids.size, int(rows.astype(np.uint64).sum()))) + 1
        keys = np.zeros(cap, np.uint64)
        g = np.zeros((cap, int(dims.max())), np.float64)
        fn = self.lib.or_row_gradients
        fn.argtypes = [C.c_uint32, _u32p, _u32p, C.c_uint32, _u32p, _u32p, _f32p, C.c_uint64, _u64p, _f64p]
        fn.restype = C.c_int64
        u = fn(len(rows), rows, dims, B, lengths, ids, upstream, cap, keys, g)
        if u < 0:
            raise RuntimeError("row_gradients capacity")
        return keys[:u], g[:u]

    def init_replica(self, spec: MeshSpec, seed: int):
        w = np.empty(spec.replica_floats(), np.float32)
        woff = spec.woff()
        for f in range(spec.F):
            w[woff[f]:woff[f + 1]] = self.init_rows(f, int(spec.rows[f]), 0, int(spec.rows[f]),
                                                    int(spec.dims[f]), seed).ravel()
        v = np.zeros(spec.replica_rows(), np.float32)
        return w, v

    def pool_ids(self, w: np.ndarray, dim: int, shards, ids) -> np.ndarray:
        w = np.ascontiguousarray(w, np.float32)
        lohi = np.ascontiguousarray(np.array(shards, np.uint32).ravel())
        ids = np.ascontiguousarray(np.array(ids, np.uint32))
        out = np.empty(dim, np.float32)
        if self.kind == "port":
            rc = self.lib.or_pool_ids(C.c_void_p(_ptr(w)), C.c_uint32(dim), C.c_uint32(len(shards)),
                                      C.c_void_p(_ptr(lohi)), C.c_void_p(_ptr(ids)), C.c_uint32(len(ids)),
                                      C.c_void_p(_ptr(out)))
        else:
            rows = w.size // dim
            rc = self.lib.ref_pool_ids(C.c_void_p(_ptr(w)), C.c_uint32(rows), C.c_uint32(dim),
                                       C.c_uint32(len(shards)), C.c_void_p(_ptr(lohi)),
                                       C.c_void_p(_ptr(ids)), C.c_uint32(len(ids)), C.c_void_p(_ptr(out)))
        if rc == -2:
            raise IndexError("lookup id outside shard ranges")
        if rc:
            raise ValueError("pool_ids failed")
        return out

    def apply_row_update(self, w: np.ndarray, v: np.ndarray, dim: int, shard, row: int, delta, new_moment):
        """apply_row_update (embedding.cpp:108-129) in place on a whole table
        (w rows x dim f32, v rows f32) through shard = (row_lo, row_hi)."""
        assert w.dtype == np.float32 and v.dtype == np.float32 and w.flags.c_contiguous
        d = np.ascontiguousarray(delta, np.float64)
        if d.size != dim:
            raise ValueError("delta length mismatch")
        lo, hi = shard
        if self.kind == "port":
            rc = self.lib.or_apply_row_update(C.c_void_p(_ptr(w)), C.c_void_p(_ptr(v)), C.c_uint32(lo),
                                              C.c_uint32(hi), C.c_uint32(dim), C.c_uint32(row),
                                              C.c_void_p(_ptr(d)), C.c_double(new_moment))
        else:
            rc = self.lib.ref_apply_row_update(C.c_void_p(_ptr(w)), C.c_void_p(_ptr(v)), C.c_uint32(v.size),
                                               C.c_uint32(lo), C.c_uint32(hi), C.c_uint32(dim), C.c_uint32(row),
                                               C.c_void_p(_ptr(d)), C.c_double(new_moment))
        if rc == -2:
            raise IndexError(f"row {row} outside shard range [{lo},{hi})")
        if rc:
            raise ValueError("new_moment must be finite and >= 0")

    def adagrad_row_step(self, w, v, g, eta=0.1, eps=1e-8, c=1.0):
        w = np.array(w, np.float32)
        vv = np.array([v], np.float32)
        g = np.ascontiguousarray(np.array(g, np.float64))
        err = C.c_int(0)
        lr = getattr(self.lib, self._p + "adagrad_row_step")(
            C.c_void_p(_ptr(w)), C.c_void_p(_ptr(vv)), C.c_void_p(_ptr(g)), C.c_uint32(len(g)),
            C.c_double(eta), C.c_double(eps), C.c_double(c), C.byref(err))
        if err.value:
            raise ValueError("nonfinite row gradient")
        return {"w": w, "v": vv[0], "effective_lr": lr}

    def effective_lr(self, v, eta=0.1, eps=1e-8, c=1.0) -> float:
        return getattr(self.lib, self._p + "effective_lr")(v, eta, eps, c)

    def plan_greedy(self, profiles, n, strategy="table-wise") -> np.ndarray:
        """profiles: list of (table_id, size_bytes, lookups, num_rows)."""
        ids = np.array([p[0] for p in profiles], np.uint32)
        lk = np.array([p[2] for p in profiles], np.float64)
        nr = np.array([p[3] for p in profiles], np.uint64)
        out = np.zeros(4 * len(profiles) * max(n, 1), np.uint32)
        cnt = getattr(self.lib, self._p + "plan_greedy")(len(profiles), ids, lk, nr, n,
                                                         1 if strategy == "row-wise" else 0, out)
        if cnt < 0:
            raise ValueError("plan_greedy failed")
        return out[: 4 * cnt].reshape(cnt, 4)

    def metrics_row(self, v: np.ndarray, eta=0.05, eps=1e-8, c=1.0) -> dict:
        """MetricsRow moment columns (trainer.cpp:745-771) over a replica's
        moments (port restatement)."""
        v = np.ascontiguousarray(v, np.float32)
        out = np.zeros(3, np.float64)
        fn = self.lib.or_metrics_row
        fn.argtypes = [_f32p, C.c_uint64, C.c_double, C.c_double, C.c_double, _f64p]
        fn.restype = C.c_int
        if fn(v, v.size, eta, eps, c, out):
            raise ValueError("metrics_row failed")
        return {"eff_lr_p50": out[0], "eff_lr_p99": out[1], "v_mean": out[2]}

    def synthetic_upstream(self, seed, step, rank, B, dims) -> np.ndarray:
        dims = np.ascontiguousarray(dims, np.uint32)
        out = np.empty(B * int(dims.sum()), np.float32)
        self.lib.or_synthetic_upstream(seed, step, rank, B, len(dims), dims, out)
        return out.reshape(B, int(dims.sum()))

    def gen_batch_ids(self, seed, step, rank, F, rows, zipf, L, B) -> np.ndarray:
        """DataGenerator ids (data.cpp:70-136); rows / zipf / L scalars or per-table."""
        rows = np.ascontiguousarray(np.broadcast_to(np.asarray(rows, np.uint32), (F,)))
        zipf = np.ascontiguousarray(np.broadcast_to(np.asarray(zipf, np.float64), (F,)))
        L = np.ascontiguousarray(np.broadcast_to(np.asarray(L, np.uint32), (F,)))
        out = np.empty(int(B) * int(L.astype(np.uint64).sum()), np.uint32)
        fn = getattr(self.lib, "or_gen_batch_ids" if self.kind == "port" else "ref_gen_batch_ids_tables")
        fn.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, _u32p, _f64p, _u32p, C.c_uint32, _u32p]
        fn.restype = C.c_int
        rc = fn(seed, step, rank, F, rows, zipf, L, B, out)
        if rc:
            raise ValueError("gen_batch_ids failed" if self.kind == "port" else self.lib.ref_last_error().decode())
        return out

    # ---- one MP group / the full mesh ---------------------------------------
    def group_step(self, spec: MeshSpec, lengths, ids, upstream, w, v, dirty=None,
                   want_dump=False, threads=1):
        self.last_compute_seconds = None
        """lengths/ids/upstream: per local rank of the group.  Returns
        (pooled per rank, Dump|None).  w, v, dirty are updated in place."""
        N, B, F = spec.N, spec.B, spec.F
        lengths = [np.ascontiguousarray(x, np.uint32) for x in lengths]
        ids = [np.ascontiguousarray(x, np.uint32) for x in ids]
        upstream = [np.ascontiguousarray(x, np.float32) for x in upstream]
        pooled = [np.zeros((B, spec.sum_dims), np.float32) for _ in range(N)]
        rows = np.ascontiguousarray(spec.rows, np.uint32)
        dims = np.ascontiguousarray(spec.dims, np.uint32)
        plan = np.ascontiguousarray(spec.plan, np.uint32)
        mean = None if spec.mean is None else np.ascontiguousarray(spec.mean, np.uint8)
        keep = [lengths, ids, upstream, pooled, rows, dims, plan, mean]
        dump = None
        if mean is not None and mean.any() and self.kind != "port":
            raise ValueError("mean pooling has no reference path (embedding.cpp:39-92 is sum-only); use the port")
        if self.kind == "port":
            cfg = _OrCfg(F, N, B, _ptr(rows), _ptr(dims), len(plan), _ptr(plan),
                         spec.eta, spec.eps, spec.c, int(spec.sgd), _ptr(mean) if mean is not None else None)
            dmp = None
            if want_dump:
                cap_ids = int(sum(int(x.sum()) for x in lengths)) + 1
                cap_floats = int(sum(int(x.sum()) for x in lengths)) * int(dims.max()) + 1
                dd = dict(
                    dem_len=np.zeros(N * N * B * F, np.uint32),
                    dem_ids=np.zeros(N * cap_ids, np.uint32),
                    dem_nnz=np.zeros(N, np.uint64),
                    mask=np.zeros(N * B * F, np.uint32),
                    part=np.zeros(N * cap_floats, np.float32),
                    part_cnt=np.zeros(N * N, np.uint64),
                    grad=np.zeros(N * cap_floats, np.float32),
                    grad_cnt=np.zeros(N * N, np.uint64),
                )
                keep.append(dd)
                dmp = _OrDump(*[_ptr(dd[k]) for k in ["dem_len", "dem_ids", "dem_nnz", "mask", "part",
                                                       "part_cnt", "grad", "grad_cnt"]],
                              cap_ids, cap_floats)
            rc = self.lib.or_group_step(
                C.byref(cfg), _ptr_array(lengths), _ptr_array(ids), _ptr_array(upstream),
                _ptr_array(pooled), C.c_void_p(_ptr(w)), C.c_void_p(_ptr(v)),
                C.c_void_p(_ptr(dirty) if dirty is not None else None),
                C.byref(dmp) if dmp is not None else None)
            if want_dump and rc == 0:
                part, grad = [], []
                for o in range(N):
                    row, at = [], 0
                    for n in range(N):
                        cnt = int(dd["part_cnt"][o * N + n])
                        row.append(dd["part"][o * cap_floats + at: o * cap_floats + at + cnt].copy())
                        at += cnt
                    part.append(row)
                for n in range(N):
                    row, at = [], 0
                    for o in range(N):
                        cnt = int(dd["grad_cnt"][n * N + o])
                        row.append(dd["grad"][n * cap_floats + at: n * cap_floats + at + cnt].copy())
                        at += cnt
                    grad.append(row)
                dump = Dump(
                    dem_len=dd["dem_len"].reshape(N, N, B * F),
                    dem_ids=[dd["dem_ids"][o * cap_ids: o * cap_ids + int(dd["dem_nnz"][o])].copy()
                             for o in range(N)],
                    mask=dd["mask"].reshape(N, B * F),
                    part=part, grad=grad)
        else:
            secs = C.c_double(0.0)
            rc = self.lib.ref_group_step(
                F, N, B, rows, dims, len(plan), plan, spec.eta, spec.eps, spec.c, int(spec.sgd),
                _ptr_array(lengths), _ptr_array(ids), _ptr_array(upstream), _ptr_array(pooled),
                w, v, C.c_void_p(_ptr(dirty) if dirty is not None else None), threads, C.byref(secs))
            self.last_compute_seconds = secs.value
        if rc == -2:
            raise IndexError("lookup id outside shard ranges")
        if rc == -3:
            raise ValueError("nonfinite row gradient / invalid argument")
        if rc:
            raise RuntimeError(f"group_step failed rc={rc}")
        del keep
        return pooled, dump

    def save_checkpoint(self, path: str, rows, dims, w: np.ndarray, v: np.ndarray) -> None:
        """S2DCKPT1 of the flat replica (embedding.cpp:133-185); table_id = f."""
        rows = np.ascontiguousarray(rows, np.uint32)
        dims = np.ascontiguousarray(dims, np.uint32)
        w = np.ascontiguousarray(w, np.float32)
        v = np.ascontiguousarray(v, np.float32)
        fn = getattr(self.lib, self._p + "save_checkpoint")
        fn.argtypes = [C.c_char_p, C.c_uint32, _u32p, _u32p, _f32p, _f32p]
        fn.restype = C.c_int
        if fn(path.encode(), len(rows), rows, dims, w, v) != 0:
            raise RuntimeError("checkpoint write failed")

    def load_checkpoint(self, path: str, rows, dims):
        """(w, v) flat replica from an S2DCKPT1 file (reference loader only)."""
        if self.kind != "reference":
            return read_checkpoint(path)[1:]
        rows = np.ascontiguousarray(rows, np.uint32)
        dims = np.ascontiguousarray(dims, np.uint32)
        w = np.empty(int((rows.astype(np.uint64) * dims).sum()), np.float32)
        v = np.empty(int(rows.astype(np.uint64).sum()), np.float32)
        fn = self.lib.ref_load_checkpoint
        fn.argtypes = [C.c_char_p, C.c_uint32, _u32p, _u32p, _f32p, _f32p]
        fn.restype = C.c_int
        if fn(path.encode(), len(rows), rows, dims, w, v) != 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return w, v

    def sync(self, spec: MeshSpec, ws, vs, dirties):
        M = len(ws)
        rows = np.ascontiguousarray(spec.rows, np.uint32)
        dims = np.ascontiguousarray(spec.dims, np.uint32)
        getattr(self.lib, self._p + "sync")(M, spec.F, rows, dims, int(spec.sgd), _ptr_array(ws),
                                            _ptr_array(vs), _ptr_array(dirties))


class RefTrainerOpts(C.Structure):
    """TrainerOptions subset (trainer.hpp:47-70) of ref_harness.cpp."""

    _fields_ = [("T", C.c_uint32), ("M", C.c_uint32), ("F", C.c_uint32), ("rows", C.c_uint32), ("dim", C.c_uint32),
                ("dense_hidden", C.c_uint32), ("over_hidden", C.c_uint32), ("dense_dim", C.c_uint32),
                ("ids_per_sample", C.c_uint32), ("B", C.c_uint32), ("strategy", C.c_int32), ("zipf", C.c_double),
                ("eta", C.c_double), ("eps", C.c_double), ("c", C.c_double), ("sgd", C.c_int32),
                ("sync_interval", C.c_uint32), ("data_seed", C.c_uint64), ("init_seed", C.c_uint64),
                ("eval_seed", C.c_uint64), ("steps", C.c_uint32)]


def trainer_options(T, M, F=3, rows=64, dim=8, B=4, L=3, steps=4, strategy="row-wise", zipf=1.0, eta=0.1, c=None,
                    sgd=False, sync_interval=1, dense_hidden=6, over_hidden=10, dense_dim=4, seeds=(1, 2, 3)):
    return RefTrainerOpts(T, M, F, rows, dim, dense_hidden, over_hidden, dense_dim, L, B,
                          1 if strategy == "row-wise" else 0, zipf, eta, 1e-8, float(M if c is None else c),
                          1 if sgd else 0, sync_interval, seeds[0], seeds[1], seeds[2], steps)


def reference_trainer(o: RefTrainerOpts):
    """The REAL reference Trainer (trainer.cpp, compiled into oracle/_ref):
    Trainer(opts).step_n(steps).  Returns (ws[g], vs[g], plan [E,4])."""
    lib = C.CDLL(REF_SO)
    fn = lib.ref_trainer_run
    fn.argtypes = [C.POINTER(RefTrainerOpts), C.c_void_p, C.c_void_p, _u32p, C.POINTER(C.c_uint32)]
    fn.restype = C.c_int
    ws = [np.zeros(o.F * o.rows * o.dim, np.float32) for _ in range(o.M)]
    vs = [np.zeros(o.F * o.rows, np.float32) for _ in range(o.M)]
    plan = np.zeros(4 * o.F * (o.T // o.M), np.uint32)
    n = C.c_uint32(0)
    if fn(C.byref(o), _ptr_array(ws), _ptr_array(vs), plan, C.byref(n)):
        lib.ref_last_error.restype = C.c_char_p
        raise RuntimeError(lib.ref_last_error().decode())
    return ws, vs, plan[: 4 * n.value].reshape(-1, 4)


def reference_trainer_model(o: RefTrainerOpts):
    """The REAL reference Trainer with its dense model's outputs:
    (ws[g], vs[g], rank_model(0) as {"dense_arch": (w1, b1, w2, b2),
    "over_arch": (...)}, per-step MetricsRow [steps, 6]: step, loss, ne,
    eff_lr_p50, eff_lr_p99, v_mean)."""
    lib = C.CDLL(REF_SO)
    fn = lib.ref_trainer_run_model
    fn.argtypes = [C.POINTER(RefTrainerOpts), C.c_void_p, C.c_void_p, _f32p,
                   np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")]
    fn.restype = C.c_int
    F, D = o.F, o.dim
    shapes = [("dense_arch", o.dense_dim, o.dense_hidden, D), ("over_arch", F * D + D, o.over_hidden, 1)]
    total = sum(h * i + h + n * h + n for _, i, h, n in shapes)
    flat = np.zeros(total, np.float32)
    loss = np.zeros((o.steps, 6), np.float64)
    ws = [np.zeros(o.F * o.rows * o.dim, np.float32) for _ in range(o.M)]
    vs = [np.zeros(o.F * o.rows, np.float32) for _ in range(o.M)]
    if fn(C.byref(o), _ptr_array(ws), _ptr_array(vs), flat, loss):
        lib.ref_last_error.restype = C.c_char_p
        raise RuntimeError(lib.ref_last_error().decode())
    model, at = {}, 0
    for name, i, h, n in shapes:
        parts = []
        for shape in [(h, i), (h,), (n, h), (n,)]:
            k = int(np.prod(shape))
            parts.append(flat[at:at + k].reshape(shape))
            at += k
        model[name] = tuple(parts)
    return ws, vs, model, loss


def restated_trainer(o: RefTrainerOpts):
    """The same loop composed from the reference's public API
    (ref_harness.cpp ref_restated_run), recording every step's per-rank
    embedding-path inputs: (ws, vs, lengths[step][rank], ids[step][rank],
    upstream[step][rank], pooled[step][rank])."""
    lib = C.CDLL(REF_SO)
    fn = lib.ref_restated_run
    fn.argtypes = [C.POINTER(RefTrainerOpts), _u32p, _u32p, _f32p, _f32p, C.c_void_p, C.c_void_p]
    fn.restype = C.c_int
    S, T, BF = o.steps, o.T, o.B * o.F
    ln = np.zeros((S, T, BF), np.uint32)
    ids = np.zeros((S, T, BF * o.ids_per_sample), np.uint32)
    up = np.zeros((S, T, o.B, o.F * o.dim), np.float32)
    pooled = np.zeros((S, T, o.B, o.F * o.dim), np.float32)
    ws = [np.zeros(o.F * o.rows * o.dim, np.float32) for _ in range(o.M)]
    vs = [np.zeros(o.F * o.rows, np.float32) for _ in range(o.M)]
    if fn(C.byref(o), ln, ids, up, pooled, _ptr_array(ws), _ptr_array(vs)):
        lib.ref_last_error.restype = C.c_char_p
        raise RuntimeError(lib.ref_last_error().decode())
    return ws, vs, ln, ids, up, pooled


@dataclass
class MeshState:
    """Full-replica state of every DP group, as the reference keeps it
    (trainer.cpp:216-224): ws[g], vs[g], dirty[g]."""

    spec: MeshSpec
    ws: list = field(default_factory=list)
    vs: list = field(default_factory=list)
    dirty: list = field(default_factory=list)

    @classmethod
    def init(cls, oracle: Oracle, spec: MeshSpec, seed: int) -> "MeshState":
        w, v = oracle.init_replica(spec, seed)
        st = cls(spec)
        for _ in range(spec.M):
            st.ws.append(w.copy())
            st.vs.append(v.copy())
            st.dirty.append(np.zeros(spec.replica_rows(), np.uint8))
        return st

    def step(self, oracle: Oracle, lengths, ids, upstream, do_sync: bool, threads=1):
        """lengths/ids/upstream per GLOBAL rank (T of them).  One run_step
        (trainer.cpp:615-663) minus input generation and the dense MLP."""
        spec = self.spec
        N = spec.N
        pooled = []
        for g in range(spec.M):
            sl = slice(g * N, (g + 1) * N)
            p, _ = oracle.group_step(spec, lengths[sl], ids[sl], upstream[sl], self.ws[g], self.vs[g],
                                     self.dirty[g], threads=threads)
            pooled.extend(p)
        if spec.M > 1 and do_sync:
            oracle.sync(spec, self.ws, self.vs, self.dirty)
        return pooled


def row_wise_plan(rows, n) -> np.ndarray:
    """plan_greedy row-wise ranges (planner.cpp:46-56), numpy form for tests."""
    out = []
    for t, r in enumerate(rows):
        for j in range(n):
            lo, hi = int(r) * j // n, int(r) * (j + 1) // n
            if hi > lo:
                out.append((t, lo, hi, j))
    return np.array(out, np.uint32).reshape(-1, 4)


def read_checkpoint(path: str):
    """Parse an S2DCKPT1 file (embedding.cpp:187-219): (tables, w, v) with
    tables = [(version, table_id, rows, dim)] and the flat replica arrays."""
    b = open(path, "rb").read()
    if b[:8] != b"S2DCKPT1":
        raise RuntimeError("not a checkpoint file: " + path)
    (count,) = np.frombuffer(b, np.uint32, 1, 8)
    off, tables, ws, vs = 12, [], [], []
    for _ in range(int(count)):
        ver, tid = np.frombuffer(b, np.uint32, 2, off)
        rows, dim = np.frombuffer(b, np.uint64, 2, off + 8)
        off += 24
        n = int(rows) * int(dim)
        ws.append(np.frombuffer(b, np.float32, n, off))
        off += 4 * n
        vs.append(np.frombuffer(b, np.float32, int(rows), off))
        off += 4 * int(rows)
        tables.append((int(ver), int(tid), int(rows), int(dim)))
    if off != len(b):
        raise RuntimeError("trailing bytes in checkpoint: " + path)
    cat = lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.float32)
    return tables, cat(ws), cat(vs)


def reference_train_toy(overrides: dict) -> dict:
    """The REAL reference run_train (src/experiment.cpp:23-34, config.cpp and
    trainer.cpp in oracle/_ref) for train_toy's {dotted_key: value} config."""
    lib = C.CDLL(REF_SO)
    fn = lib.ref_train_toy
    fn.argtypes = [C.c_uint32, C.POINTER(C.c_char_p), C.POINTER(C.c_char_p), C.POINTER(C.c_double),
                   C.POINTER(C.c_double), C.c_char_p]
    fn.restype = C.c_int
    ks = (C.c_char_p * max(1, len(overrides)))(*[k.encode() for k in overrides])
    vs = (C.c_char_p * max(1, len(overrides)))(*[str(v).encode() for v in overrides.values()])
    ne, ctr = C.c_double(0), C.c_double(0)
    h = C.create_string_buffer(17)
    if fn(len(overrides), ks, vs, C.byref(ne), C.byref(ctr), h):
        lib.ref_last_error.restype = C.c_char_p
        raise RuntimeError(lib.ref_last_error().decode())
    return {"final_ne": ne.value, "baseline_ctr": ctr.value, "config_hash": h.value.decode()}


def reference_aggregate(rows, grads, group_batch: int):
    """The REAL reference aggregate_group_gradient (optimizer.cpp:25-59):
    (rows [U], g [U, dim] f64, sample_count [U])."""
    lib = C.CDLL(REF_SO)
    fn = lib.ref_aggregate
    fn.restype = C.c_int
    r = np.ascontiguousarray(rows, np.uint32)
    g = np.ascontiguousarray(grads, np.float64)
    n, dim = g.shape
    out_r = np.zeros(max(n, 1), np.uint32)
    out_g = np.zeros((max(n, 1), dim), np.float64)
    out_c = np.zeros(max(n, 1), np.uint32)
    m = C.c_uint32(0)
    if fn(C.c_void_p(_ptr(r)), C.c_void_p(_ptr(g)), C.c_uint32(n), C.c_uint32(group_batch), C.c_uint32(dim),
          C.c_void_p(_ptr(out_r)), C.c_void_p(_ptr(out_g)), C.c_void_p(_ptr(out_c)), C.byref(m)):
        lib.ref_last_error.restype = C.c_char_p
        raise ValueError(lib.ref_last_error().decode())
    U = m.value
    return out_r[:U], out_g[:U], out_c[:U]
