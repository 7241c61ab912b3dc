"""Python surface of the B200 2D-sparse-parallel embedding step.

Reference-named functions keep the signatures of the reference's pybind11
module (proj/bindings/module.cpp:35-164, proj/python/sparse2d/__init__.py):
``Topology``, ``plan_greedy``, ``imbalance_ratio``, ``effective_lr``,
``adagrad_row_step``.  The step itself is ``Sparse2DEmbedding``: one object
per GPU rank, the drop-in for the embedding phases of
``Trainer::Impl::run_step`` (proj/src/trainer.cpp:615-663).

All compute runs in libsparse2d_b200.so (hand-written sm_100a kernels + NCCL);
this module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _lib as L


def _lib():
    return L.load()


# ---- Topology (include/sparse2d/topology.hpp:13-26) -------------------------

class Topology:
    """T ranks split into M groups of N = T/M; rank r -> (r // N, r % N)."""

    def __init__(self, total_ranks: int, groups: int):
        t = L.TopologyC()
        L.check(_lib().s2d_topology_init(total_ranks, groups, C.byref(t)))
        self.total_ranks = t.total_ranks
        self.groups = t.groups
        self.ranks_per_group = t.ranks_per_group

    def group_of(self, rank: int) -> int:
        return rank // self.ranks_per_group

    def local_of(self, rank: int) -> int:
        return rank % self.ranks_per_group

    def rank_of(self, group: int, local: int) -> int:
        return group * self.ranks_per_group + local

    def __repr__(self):
        return f"Topology(total_ranks={self.total_ranks}, groups={self.groups})"


# ---- planner (src/planner.cpp) ----------------------------------------------

def _profiles(profiles) -> tuple:
    arr = (L.TableLoadProfile * len(profiles))()
    for i, (tid, size, lookups, rows) in enumerate(profiles):
        arr[i] = L.TableLoadProfile(int(tid), int(size), float(lookups), int(rows))
    return arr


def plan_greedy(profiles: Sequence[tuple], ranks: int, strategy: str = "table-wise") -> list[dict]:
    """profiles: (table_id, size_bytes, expected_lookups, num_rows) tuples
    (bindings/module.cpp:109-131).  Returns [{table_id,row_lo,row_hi,local_rank}]."""
    if strategy not in ("table-wise", "row-wise"):
        raise ValueError("unknown sharding strategy: " + str(strategy))
    prof = _profiles(profiles)
    cap = max(1, len(profiles) * max(1, ranks))
    out = (L.PlanEntry * cap)()
    n = C.c_uint32(0)
    L.check(_lib().s2d_plan_greedy(prof, len(profiles), ranks,
                                   L.S2D_ROW_WISE if strategy == "row-wise" else L.S2D_TABLE_WISE,
                                   out, cap, C.byref(n)))
    return [dict(table_id=out[i].table_id, row_lo=out[i].row_lo, row_hi=out[i].row_hi,
                 local_rank=out[i].local_rank) for i in range(n.value)]


def _plan_array(plan: Iterable[dict]):
    plan = list(plan)
    arr = (L.PlanEntry * max(1, len(plan)))()
    for i, e in enumerate(plan):
        arr[i] = L.PlanEntry(e["table_id"], e["row_lo"], e["row_hi"], e["local_rank"])
    return arr, len(plan)


def validate_plan(plan: Iterable[dict], ranks_per_group: int, profiles: Sequence[tuple]) -> None:
    arr, n = _plan_array(plan)
    prof = _profiles(profiles)
    L.check(_lib().s2d_validate_plan(arr, n, ranks_per_group, prof, len(profiles)))


def owner_of(plan: Iterable[dict], table_id: int, row: int) -> int:
    arr, n = _plan_array(plan)
    o = C.c_uint32(0)
    L.check(_lib().s2d_plan_owner_of(arr, n, table_id, row, C.byref(o)))
    return o.value


def imbalance_ratio(loads: Sequence[float]) -> float:
    a = (C.c_double * max(1, len(loads)))(*loads)
    out = C.c_double(0)
    L.check(_lib().s2d_imbalance_ratio(a, len(loads), C.byref(out)))
    return out.value


# ---- optimizer (src/optimizer.cpp) ------------------------------------------

@dataclass
class OptimizerConfig:
    """OptimizerConfig (include/sparse2d/optimizer.hpp:15-22)."""

    eta: float = 0.05
    eps: float = 1e-8
    c: float = 1.0
    variant: str = "rowwise-adagrad"  # | "sgd"

    def to_c(self) -> L.OptimizerConfigC:
        if self.variant not in ("rowwise-adagrad", "sgd"):
            raise ValueError("unknown optimizer variant: " + str(self.variant))
        return L.OptimizerConfigC(self.eta, self.eps, self.c,
                                  L.S2D_SGD if self.variant == "sgd" else L.S2D_ROWWISE_ADAGRAD)


def effective_lr(v: float, eta: float = 0.1, eps: float = 1e-8, c: float = 1.0) -> float:
    """eta / (sqrt(v / c) + eps) (optimizer.cpp:61-63), validated like the binding."""
    cfg = OptimizerConfig(eta, eps, c).to_c()
    out = C.c_double(0)
    L.check(_lib().s2d_effective_lr(v, C.byref(cfg), C.byref(out)))
    return out.value


def adagrad_row_step(w, v, g, eta: float = 0.1, eps: float = 1e-8, c: float = 1.0) -> dict:
    """Fused moment-scaled row-wise AdaGrad step on one row, executed by the
    same sm_100a row-update code as the training step
    (bindings/module.cpp:93-107).  Returns {w, v, effective_lr}."""
    return adagrad_rows([w], [v], [g], eta=eta, eps=eps, c=c)[0]


def adagrad_rows(ws, vs, gs, eta=0.1, eps=1e-8, c=1.0, variant="rowwise-adagrad") -> list[dict]:
    w = np.ascontiguousarray(np.array(ws, np.float32))
    if w.ndim != 2:
        raise ValueError("rows must share one dim")
    g = np.ascontiguousarray(np.array(gs, np.float64))
    if g.shape != w.shape:
        raise ValueError("gradient dim mismatch")
    v = np.ascontiguousarray(np.array(vs, np.float32).reshape(-1))
    lr = np.zeros(len(v), np.float64)
    cfg = OptimizerConfig(eta, eps, c, variant).to_c()
    L.check(_lib().s2d_adagrad_rows(C.byref(cfg), w.shape[0], w.shape[1], w.ctypes.data, v.ctypes.data,
                                    g.ctypes.data, lr.ctypes.data))
    return [dict(w=w[i].tolist(), v=float(v[i]), effective_lr=float(lr[i])) for i in range(len(v))]


# ---- analytic helpers of the reference module (bindings/module.cpp:43-89, 133-145)

def _dbl(fn, *args) -> float:
    out = C.c_double(0)
    L.check(fn(*args, C.byref(out)))
    return out.value


def memory_overhead(table_size_gb: float, groups: int, total_gpus: int) -> float:
    """S (M-1) / T (src/cost_model.cpp:24-28)."""
    return _dbl(_lib().s2d_memory_overhead, table_size_gb, groups, total_gpus)


def sync_latency(table_size_gb: float, groups: int, total_gpus: int, sync_bw_gbps: float) -> float:
    """2 memory_overhead / bandwidth (src/cost_model.cpp:30-34)."""
    return _dbl(_lib().s2d_sync_latency, table_size_gb, groups, total_gpus, sync_bw_gbps)


def qps_scaling_factor(qps_base: float, gpus_base: float, qps_new: float, gpus_new: float) -> float:
    """(qps_new / qps_base) / (gpus_new / gpus_base) (src/cost_model.cpp:46-55)."""
    return _dbl(_lib().s2d_qps_scaling_factor, qps_base, gpus_base, qps_new, gpus_new)


def evaluate_ne(probs, labels) -> dict:
    """Normalized entropy (src/trainer.cpp:14-43): {ne, baseline_ctr, eval_samples}."""
    p = np.ascontiguousarray(probs, np.float64)
    y = np.ascontiguousarray(labels, np.float32)
    if p.size != y.size:
        raise ValueError("evaluate_ne: empty or mismatched inputs")
    ne, ctr = C.c_double(0), C.c_double(0)
    L.check(_lib().s2d_evaluate_ne(p.ctypes.data, y.ctypes.data, p.size, C.byref(ne), C.byref(ctr)))
    return {"ne": ne.value, "baseline_ctr": ctr.value, "eval_samples": int(p.size)}


def closed_form_ratio(mu_norm: float, sigma: float, dim: int, batch: int, groups: int) -> float:
    """Proposition 1 closed form (src/moment_analysis.cpp:128-141)."""
    return _dbl(_lib().s2d_closed_form_ratio, mu_norm, sigma, dim, batch, groups)


def recommend_c(mu_norm: float, sigma: float, dim: int, batch: int, groups: int) -> float:
    """The AdaGrad moment scaling factor c recommended for M groups
    (src/moment_analysis.cpp:143-146)."""
    return _dbl(_lib().s2d_recommend_c, mu_norm, sigma, dim, batch, groups)


def estimate_increment_ratio(mu_norm: float, sigma: float, dim: int, batch: int, groups: int, trials: int,
                             seed: int = 1) -> dict:
    """Monte Carlo E|g_group|^2 / E|g_full|^2 (src/moment_analysis.cpp:69-124)."""
    r, se = C.c_double(0), C.c_double(0)
    L.check(_lib().s2d_estimate_increment_ratio(mu_norm, sigma, dim, batch, groups, trials, seed, C.byref(r),
                                                C.byref(se)))
    return {"ratio_estimate": r.value, "std_error": se.value, "trials": int(trials), "groups": int(groups)}


# ---- the step engine -----------------------------------------------------------

@dataclass
class TableConfig:
    """One embedding table: FeatureSpec / EmbeddingTable shape
    (data.hpp:11-18, embedding.hpp:12-23) with per-table rows and dim."""

    rows: int
    dim: int
    expected_lookups: float = 1.0  # expected lookups per batch (planner load)
    pooling: str = "sum"  # "sum" (the reference's pool_ids) | "mean"

    def pooling_code(self) -> int:
        if self.pooling not in ("sum", "mean"):
            raise ValueError("pooling must be 'sum' or 'mean'")
        return L.S2D_POOL_MEAN if self.pooling == "mean" else L.S2D_POOL_SUM


def launch_count() -> int:
    """Kernels launched by libsparse2d_b200 in this process."""
    return int(_lib().s2d_launch_count())


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    L.check(_lib().s2d_nccl_unique_id(buf))
    return buf.raw


def _numel(x) -> int:
    return int(x.numel()) if hasattr(x, "numel") else int(x.size)


def _ptr_kind(x, dtype, writable=False):
    """(pointer, mem kind, keepalive) for a numpy array or torch tensor of a
    4-byte `dtype` (np.uint32 or np.float32)."""
    try:
        import torch  # plumbing only: device memory / pinned host buffers
        if isinstance(x, torch.Tensor):
            ok = (torch.float32,) if dtype == np.float32 else (torch.int32, getattr(torch, "uint32", torch.int32))
            if x.dtype not in ok:
                raise TypeError(f"tensor dtype {x.dtype} does not match {np.dtype(dtype).name}")
            if not x.is_contiguous():
                raise ValueError("tensor must be contiguous")
            return x.data_ptr(), (L.S2D_DEVICE if x.is_cuda else L.S2D_HOST), x
    except ImportError:
        pass
    if writable:
        if not (isinstance(x, np.ndarray) and x.dtype == dtype and x.flags.c_contiguous):
            raise TypeError(f"output must be a C-contiguous {np.dtype(dtype).name} array")
        return x.ctypes.data, L.S2D_HOST, x
    a = np.ascontiguousarray(x, dtype)
    return a.ctypes.data, L.S2D_HOST, a


def traces_to_csv(rows: Iterable[dict], config_hash: str = "") -> str:
    """Trace CSV in the reference schema (experiment.cpp:47-62):
    ``# config_hash=…`` comments, header ``step,kernel,rank,bytes,latency_s``,
    latency printed ``%.9g`` (csv.cpp:11-15).  Rows are measured
    (Sparse2DEmbedding.trace_rows, gathered over ranks by the caller), not
    modelled by the alpha-beta bandwidth model."""
    out = [f"# config_hash={config_hash}",
           "# bytes = bytes sent by the rank to other ranks (self-delivery stays in HBM)",
           "# latency_s = measured device time of the kernels carrying the exchange",
           "step,kernel,rank,bytes,latency_s"]
    def order(r):
        # lookup / grad a2a: one trace per MP group, participants in local
        # order -> global rank order; table_allreduce: one trace per local
        # rank o over its replicas g = 0..M-1 (trainer.cpp:598-610,
        # topology.cpp:128-131) -> (local, group)
        if r["kernel"] == "table_allreduce":
            sub = (r.get("local", r["rank"]), r.get("group", 0))
        else:
            sub = (r["rank"], 0)
        return (r["step"], _TRACE_ORDER.get(r["kernel"], 9)) + sub

    for r in sorted(rows, key=order):
        out.append(f"{r['step']},{r['kernel']},{r['rank']},{r['bytes']},{r['latency_s']:.9g}")
    return "\n".join(out) + "\n"


_TRACE_ORDER = {"lookup_a2a": 0, "grad_a2a": 1, "table_allreduce": 2}


class LocalHub:
    """In-process rendezvous of a single-process mesh (s2d_hub_create): the
    T virtual ranks of one process, each driven by its own thread, as the
    reference Trainer runs its ranks (trainer.cpp:80-97).  Pass it as
    ``hub=`` to every rank's Sparse2DEmbedding; ranks may share one GPU."""

    def __init__(self, total_ranks: int):
        self.lib = _lib()
        self.total_ranks = int(total_ranks)
        self._h = C.c_void_p()
        L.check(self.lib.s2d_hub_create(self.total_ranks, C.byref(self._h)))

    def close(self):
        if self._h:
            self.lib.s2d_hub_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_ranks(fn, n: int, timeout: float | None = 600.0) -> list:
    """Run fn(rank) for rank in [0, n) on n threads (one host thread per
    virtual rank; the C calls release the GIL) and return the results in rank
    order.  The first exception raised by any rank is re-raised."""
    import threading

    out, errs = [None] * n, [None] * n

    def body(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001  (re-raised below)
            errs[r] = e

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(n)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
        if t.is_alive():
            raise TimeoutError("a virtual rank did not finish")
    for e in errs:
        if e is not None:
            raise e
    return out


def local_mesh(tables, topology: Topology, devices=None, **kw) -> list:
    """All T ranks of a mesh in this process (virtual ranks on one LocalHub).
    devices: per-rank CUDA device (default: all on device 0).  Creation is
    collective, so the engines are built on T threads.  Returns the engines in
    rank order; each keeps the hub alive."""
    T = topology.total_ranks
    hub = LocalHub(T)
    devs = list(devices) if devices is not None else [0] * T
    engines = run_ranks(lambda r: Sparse2DEmbedding(tables, topology, rank=r, device=devs[r], hub=hub, **kw), T)
    hub.close()  # the contexts hold their own references
    return engines


class Sparse2DEmbedding:
    """Per-rank engine of the 2D-sparse-parallel embedding step.

    One instance per GPU; rank r of T with M DP groups (N = T/M ranks per MP
    group).  Every rank registers the same tables and plan (the plan is
    identical in every group) and owns the shards its local rank
    is assigned.  ``nccl_id`` (128 bytes from rank 0, e.g. broadcast over
    torch.distributed) is required when T > 1 across processes; ``hub`` (a
    LocalHub) instead makes this rank a virtual rank of a single-process mesh
    (see local_mesh / run_ranks).
    """

    def __init__(self, tables: Sequence[TableConfig], topology: Topology, rank: int = 0, device: int = 0,
                 strategy: str = "table-wise", plan: Sequence[dict] | None = None,
                 optimizer: OptimizerConfig | None = None, weight_dtype: str = "fp32",
                 nccl_id: bytes | None = None, strict: bool = True, hub: LocalHub | None = None):
        self.lib = _lib()
        self.topology = topology
        self.rank = rank
        self._device = device
        self.tables = list(tables)
        self.F = len(self.tables)
        self.dims = np.array([t.dim for t in self.tables], np.uint32)
        self.rows = np.array([t.rows for t in self.tables], np.uint64)
        self.sum_dims = int(self.dims.sum())
        N = topology.ranks_per_group
        if plan is None:
            prof = [(i, t.rows * t.dim * 4, t.expected_lookups, t.rows) for i, t in enumerate(self.tables)]
            plan = plan_greedy(prof, N, strategy)
        self.plan = [dict(e) for e in plan]
        self._ctx = C.c_void_p()
        if hub is not None:
            L.check(self.lib.s2d_ctx_create_local(device, topology.total_ranks, topology.groups, rank, hub._h,
                                                  C.byref(self._ctx)))
        else:
            L.check(self.lib.s2d_ctx_create(device, topology.total_ranks, topology.groups, rank,
                                            nccl_id if nccl_id is not None else None, C.byref(self._ctx)))
        self.set_strict(strict)
        td = (L.TableDesc * self.F)(*[L.TableDesc(i, t.rows, t.dim, t.pooling_code()) for i, t in enumerate(self.tables)])
        parr, n = _plan_array(self.plan)
        if weight_dtype not in ("fp32", "bf16"):
            raise ValueError("weight_dtype must be fp32 or bf16")
        self.weight_dtype = weight_dtype
        L.check(self.lib.s2d_register_tables(self._ctx, td, self.F, parr, n,
                                             L.S2D_BF16 if weight_dtype == "bf16" else L.S2D_F32))
        self.optimizer = optimizer or OptimizerConfig()
        self.set_optimizer(self.optimizer)
        self._batch = None

    # -- lifecycle --
    def close(self):
        if self._ctx:
            self.lib.s2d_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_strict(self, strict: bool):
        L.check(self.lib.s2d_ctx_set_strict(self._ctx, 1 if strict else 0))

    def save_tables(self, path: str):
        """S2DCKPT1 checkpoint of DP group 0's replica (Trainer::save_tables,
        trainer.cpp:875-878); collective over every rank of the mesh."""
        L.check(self.lib.s2d_save_tables(self._ctx, os.fsencode(path)))

    def load_tables(self, path: str):
        """Load an S2DCKPT1 checkpoint into every replica (Trainer::load_tables,
        trainer.cpp:880-896)."""
        L.check(self.lib.s2d_load_tables(self._ctx, os.fsencode(path)))

    def gen_batch(self, seed: int, step: int, rank: int, batch: int, zipf, ids_per_sample, device: bool = True):
        """The reference DataGenerator's ids for one rank's batch, generated on
        the GPU (s2d_gen_batch; data.cpp:85-136).  zipf / ids_per_sample are
        per-table (or scalars).  Returns (lengths[B*F], ids) as CUDA tensors
        (device=True) or numpy arrays."""
        z = np.ascontiguousarray(np.broadcast_to(np.asarray(zipf, np.float64), (self.F,)))
        L_ = np.ascontiguousarray(np.broadcast_to(np.asarray(ids_per_sample, np.uint32), (self.F,)))
        n_ids = int(batch) * int(L_.astype(np.uint64).sum())
        if device:
            import torch

            dev = torch.device("cuda", self._device)
            lengths = torch.empty(batch * self.F, dtype=torch.int32, device=dev)
            ids = torch.empty(max(n_ids, 1), dtype=torch.int32, device=dev)[:n_ids]
            lp, ip, mem = lengths.data_ptr(), ids.data_ptr(), L.S2D_DEVICE
        else:
            lengths = np.empty(batch * self.F, np.uint32)
            ids = np.empty(n_ids, np.uint32)
            lp, ip, mem = lengths.ctypes.data, ids.ctypes.data, L.S2D_HOST
        L.check(self.lib.s2d_gen_batch(self._ctx, seed, step, rank, batch, z.ctypes.data, L_.ctypes.data, lp, ip,
                                       mem))
        return lengths, ids

    def set_async_host(self, on: bool):
        """Host-memory pooled output completes asynchronously (s2d_ctx_set_async_host)."""
        L.check(self.lib.s2d_ctx_set_async_host(self._ctx, 1 if on else 0))

    def set_stream(self, stream_ptr: int | None):
        L.check(self.lib.s2d_ctx_set_stream(self._ctx, stream_ptr))

    def set_optimizer(self, cfg: OptimizerConfig):
        c = cfg.to_c()
        L.check(self.lib.s2d_set_optimizer(self._ctx, C.byref(c)))
        self.optimizer = cfg

    # -- state --
    def init_tables(self, seed: int):
        """init_table (embedding.cpp:17-37) for every owned shard, on device."""
        L.check(self.lib.s2d_init_tables(self._ctx, seed))

    def owned_range(self, table: int) -> tuple[int, int]:
        lo, hi = C.c_uint32(0), C.c_uint32(0)
        L.check(self.lib.s2d_shard_range(self._ctx, table, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def read_rows(self, table: int, lo: int, hi: int):
        d = int(self.dims[table])
        w = np.zeros((hi - lo, d), np.float32)
        v = np.zeros(hi - lo, np.float32)
        L.check(self.lib.s2d_shard_read(self._ctx, table, lo, hi, w.ctypes.data, v.ctypes.data))
        return w, v

    def gather_rows(self, table: int, rows):
        """Weights (n x dim fp32) and moments of owned rows by global id."""
        r = np.ascontiguousarray(rows, np.uint32).ravel()
        d = int(self.dims[table]) if 0 <= table < self.F else 0
        w = np.zeros((r.size, d), np.float32)
        v = np.zeros(r.size, np.float32)
        L.check(self.lib.s2d_shard_gather(self._ctx, table, r.size, r.ctypes.data, w.ctypes.data, v.ctypes.data))
        return w, v

    def set_debug_grad(self, on: bool):
        """Record each backward's f64 row gradients (debug(7))."""
        L.check(self.lib.s2d_ctx_set_debug_grad(self._ctx, 1 if on else 0))

    def write_rows(self, table: int, lo: int, w=None, v=None):
        n = len(w) if w is not None else len(v)
        wa = None if w is None else np.ascontiguousarray(w, np.float32)
        va = None if v is None else np.ascontiguousarray(v, np.float32)
        L.check(self.lib.s2d_shard_write(self._ctx, table, lo, lo + n,
                                          wa.ctypes.data if wa is not None else None,
                                          va.ctypes.data if va is not None else None))

    # -- the step --
    def apply_row_updates(self, table: int, rows, delta, new_moment):
        """apply_row_update (embedding.cpp:108-129) on owned rows of `table`:
        w += delta (f64 add, rounded to storage), v = new_moment.  rows are
        global row ids; delta is len(rows) x dim; a repeated row is updated in
        call order.  IndexError outside the owned range, ValueError for a
        negative or nonfinite moment (nothing written then)."""
        r = np.ascontiguousarray(rows, np.uint32).ravel()
        n = r.size
        D = int(self.dims[table]) if 0 <= table < self.F else 0
        d = np.ascontiguousarray(delta, np.float64).reshape(-1)
        m = np.ascontiguousarray(new_moment, np.float64).ravel()
        if d.size != n * D or m.size != n:
            raise ValueError("delta length mismatch")
        L.check(self.lib.s2d_apply_row_updates(self._ctx, table, n, r.ctypes.data, d.ctypes.data, m.ctypes.data))

    def forward(self, lengths, ids, pooled=None, batch: int | None = None):
        """Pooled embeddings of this rank's batch.  lengths: [B*F] sample-major
        bag lengths, ids: concatenated global row ids.  numpy / CPU tensors are
        host buffers (copied inside); CUDA tensors stay on device."""
        lp, lk, lka = _ptr_kind(lengths, np.uint32)
        ip, ik, ika = _ptr_kind(ids, np.uint32)
        nnz, nb = _numel(ika), _numel(lka)
        if batch is None:
            if nb % self.F:
                raise ValueError("len(lengths) must be a multiple of the table count")
            batch = nb // self.F
        if lk != ik:
            raise ValueError("lengths and ids must both be host or both be device buffers")
        if isinstance(pooled, str) and pooled == "engine":
            # zero-copy: results land in the engine-owned, peer-mapped buffer
            # (pooled_buffer_ptr()); owners store single-owner tables' rows there
            if lk != L.S2D_DEVICE:
                raise ValueError("engine output needs device inputs")
            L.check(self.lib.s2d_lookup_forward(self._ctx, batch, lp, ip, nnz, None, lk))
            self._batch = batch
            return None
        if pooled is None:
            if lk == L.S2D_DEVICE:
                import torch
                pooled = torch.empty((batch, self.sum_dims), dtype=torch.float32, device=lka.device)
            else:
                pooled = np.zeros((batch, self.sum_dims), np.float32)
        pp, pk, pka = _ptr_kind(pooled, np.float32, writable=True)
        if pk != lk:
            raise ValueError("pooled must live where the inputs live")
        L.check(self.lib.s2d_lookup_forward(self._ctx, batch, lp, ip, nnz, pp, lk))
        self._batch = batch
        return pooled

    def backward_update(self, upstream):
        """Gradient all-to-all + dedup + fused moment-scaled row-wise AdaGrad for
        the batch of the last forward.  upstream: [B][sum dims] fp32."""
        up, uk, _ua = _ptr_kind(upstream, np.float32)
        L.check(self.lib.s2d_backward_update(self._ctx, up, uk))

    def pooled_buffer_ptr(self) -> int:
        """Device address of the engine-owned pooled output (see forward(...,
        pooled="engine")); [batch][sum dims] fp32."""
        p = C.c_void_p()
        L.check(self.lib.s2d_pooled_buffer(self._ctx, C.byref(p)))
        return p.value or 0

    def sync_replicas(self):
        """Weight + moment mean of dirty rows across the DP group
        (trainer.cpp:547-596).  No-op for M = 1."""
        L.check(self.lib.s2d_replica_sync(self._ctx))

    def synchronize(self):
        L.check(self.lib.s2d_synchronize(self._ctx))

    def stats(self) -> dict:
        s = L.StepStats()
        L.check(self.lib.s2d_get_step_stats(self._ctx, C.byref(s)))
        return {k: getattr(s, k) for k, _ in L.StepStats._fields_}

    PHASES = ("input", "bucket", "a2a_ids", "lookup", "a2a_lookup", "combine", "grad_gather", "a2a_grad",
              "sort", "count_sync", "update", "sync", "sync_push", "sync_mean", "sync_scatter")

    def set_profiling(self, on, hot_only: bool = False):
        """Phase events on the engine stream; hot_only brackets only the fused
        update (s2d_ctx_set_profiling levels 1 / 2)."""
        L.check(self.lib.s2d_ctx_set_profiling(self._ctx, (2 if hot_only else 1) if on else 0))

    def phase_times(self) -> dict:
        """{phase: (ms, launches)} summed since the last call (CUDA events on
        the engine's stream)."""
        n = len(self.PHASES)
        ms = (C.c_double * n)()
        cnt = (C.c_uint32 * n)()
        L.check(self.lib.s2d_get_phase_times(self._ctx, ms, cnt, n))
        return {p: (ms[i], cnt[i]) for i, p in enumerate(self.PHASES)}

    # Phases whose device time carries each reference collective.  The
    # exchanges are fused into their producing kernels (owner lookup stores
    # pooled rows into the requester's buffer over NVLink; the grad gather
    # pulls upstream rows from peers), so a collective's latency is the time
    # of the kernels that move its bytes.
    TRACE_PHASES = {
        "lookup_a2a": ("a2a_ids", "lookup", "a2a_lookup", "combine"),
        "grad_a2a": ("grad_gather", "a2a_grad"),
        "table_allreduce": ("sync", "sync_push", "sync_mean", "sync_scatter"),
    }

    def trace_rows(self, step: int) -> list[dict]:
        """Measured CollectiveTrace rows of this rank since the last
        phase_times() call (topology.hpp:53-61, one row per participant as
        traces_to_csv writes them, experiment.cpp:47-62).  Needs
        set_profiling(True) around the step.  bytes = bytes this rank sent to
        other ranks (ids + pooled rows for lookup_a2a); self-delivery stays in
        HBM and is not counted, unlike the simulated trace.  table_allreduce
        appears only when a replica sync ran."""
        times = self.phase_times()
        if times["lookup"][1] > 1:
            # the byte counters describe the last step only
            raise ValueError(f"trace_rows covers {times['lookup'][1]} forwards; call phase_times() right before "
                             "the step to be traced")
        st = self.stats()
        sent = {
            "lookup_a2a": st["ids_bytes_sent"] + st["lookup_bytes_sent"],
            "grad_a2a": st["grad_bytes_sent"],
            "table_allreduce": st["sync_bytes"],
        }
        rows = []
        for kernel, phases in self.TRACE_PHASES.items():
            if kernel == "table_allreduce" and (times["sync"][1] == 0 or not self._owns_rows()):
                continue  # the reference traces only local ranks with a non-empty shard
            ms = sum(times[p][0] for p in phases)
            rows.append({"step": int(step), "kernel": kernel, "rank": self.rank,
                         "group": self.topology.group_of(self.rank), "local": self.topology.local_of(self.rank),
                         "bytes": int(sent[kernel]), "latency_s": ms * 1e-3})
        return rows

    def metrics_row(self) -> dict:
        """MetricsRow moment columns (trainer.hpp:72-79, trainer.cpp:745-771)
        of this rank's MP-group replica: eff_lr_p50, eff_lr_p99, v_mean over
        every row of every table.  Collective over the MP group."""
        m = L.MetricsRowC()
        L.check(self.lib.s2d_metrics(self._ctx, C.byref(m)))
        return {"eff_lr_p50": m.eff_lr_p50, "eff_lr_p99": m.eff_lr_p99, "v_mean": m.v_mean, "rows": int(m.rows)}

    def _owns_rows(self) -> bool:
        return any(hi > lo for lo, hi in (self.owned_range(f) for f in range(self.F)))

    def gen_upstream(self, seed: int, step: int, rank: int, batch: int) -> np.ndarray:
        """The synthetic upstream gradient (s2d_gen_upstream) as a host array."""
        out = np.zeros((batch, self.sum_dims), np.float32)
        L.check(self.lib.s2d_gen_upstream(self._ctx, seed, step, rank, batch, out.ctypes.data, L.S2D_HOST))
        return out

    def debug(self, which: int) -> np.ndarray:
        """Wire buffers of the last step (see s2d_debug_read)."""
        n = C.c_uint64(0)
        L.check(self.lib.s2d_debug_read(self._ctx, which, None, 0, C.byref(n)))
        dt = np.float32 if which in (2, 3, 6) else (np.float64 if which == 7 else np.uint32)
        out = np.zeros(n.value, dt)
        L.check(self.lib.s2d_debug_read(self._ctx, which, out.ctypes.data, n.value, C.byref(n)))
        return out


# ---- Trainer facade (include/sparse2d/trainer.hpp:106-132) -----------------------

@dataclass
class TrainerOptions:
    """TrainerOptions (trainer.hpp:47-70): topology, tables (num_tables x
    rows_per_table x dim), the DataGenerator's Zipf exponent and pooling
    fan-in, per-rank batch, steps, sync cadence, seeds, optimizer, and the
    dense model (DlrmConfig dense_hidden / over_hidden, DataParams dense_dim
    and ground truth; model.hpp:68-77, data.hpp:51-56).  dense_model=False
    trains on the synthetic upstream instead of the device MLPs."""

    total_ranks: int = 1
    groups: int = 1
    num_tables: int = 8
    rows_per_table: int = 10000
    dim: int = 16
    strategy: str = "row-wise"
    zipf_exponent: float = 1.0
    ids_per_sample: int = 2
    per_rank_batch: int = 4
    steps: int = 1000
    sync_interval: int = 1
    data_seed: int = 1
    init_seed: int = 2
    optimizer: OptimizerConfig | None = None
    weight_dtype: str = "fp32"
    devices: Sequence[int] | None = None
    dense_model: bool = True
    dense_dim: int = 8
    dense_hidden: int = 32
    over_hidden: int = 64
    gt_id_scale: float = 0.25
    gt_dense_scale: float = 0.35
    gt_bias: float = -0.8
    eval_cadence: int = 0
    eval_samples: int = 100000
    eval_seed: int = 3


class _DevArray:
    """A raw CUDA pointer as __cuda_array_interface__ (for torch.as_tensor)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3}


class Trainer:
    """The reference's one-object training loop over the 2D mesh
    (Trainer, trainer.hpp:106-132): every rank a virtual rank of this
    process (s2d_trainer_*).  The upstream gradient of each step comes from
    ``set_upstream(fn)`` -- fn(rank, step, lengths, pooled, upstream) with
    torch CUDA tensor views, fn filling ``upstream`` (the dense model's
    backward) -- or, by default, from the dense model on the device (the
    reference's toy DLRM MLPs, dense.h), or with ``dense_model=False`` the
    synthetic f32(1e-3 N(0,1)) gradient."""

    def __init__(self, opts: TrainerOptions):
        self.lib = _lib()
        self.opts = opts
        opt = (opts.optimizer or OptimizerConfig()).to_c()
        devs = list(opts.devices) if opts.devices else []
        self._devs = (C.c_int32 * max(1, len(devs)))(*devs) if devs else None
        if opts.strategy not in ("table-wise", "row-wise"):
            raise ValueError("unknown sharding strategy: " + str(opts.strategy))
        c = L.TrainerOptionsC(opts.total_ranks, opts.groups, opts.num_tables, opts.rows_per_table, opts.dim,
                              L.S2D_ROW_WISE if opts.strategy == "row-wise" else L.S2D_TABLE_WISE,
                              opts.zipf_exponent, opts.ids_per_sample, opts.per_rank_batch, opts.steps,
                              opts.sync_interval, opts.data_seed, opts.init_seed, opt,
                              L.S2D_BF16 if opts.weight_dtype == "bf16" else L.S2D_F32, len(devs),
                              C.cast(self._devs, C.POINTER(C.c_int32)) if devs else None,
                              1 if opts.dense_model else 0, opts.dense_dim, opts.dense_hidden, opts.over_hidden,
                              opts.gt_id_scale, opts.gt_dense_scale, opts.gt_bias, opts.eval_cadence,
                              opts.eval_samples, opts.eval_seed)
        self._t = C.c_void_p()
        L.check(self.lib.s2d_trainer_create(C.byref(c), C.byref(self._t)))
        self._cb = None

    def close(self):
        if self._t:
            self.lib.s2d_trainer_destroy(self._t)
            self._t = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_upstream(self, fn):
        """fn(rank, step, lengths, pooled, upstream) -> None, called on the
        rank's thread after each forward; tensors are CUDA views (lengths
        [B*F] int32, pooled and upstream [B, F*D] fp32)."""
        if fn is None:
            L.check(self.lib.s2d_trainer_set_upstream(self._t, L.UPSTREAM_FN(), None))
            self._cb = None
            return
        import torch

        o = self.opts
        F, D = o.num_tables, o.dim

        def cb(_user, rank, step, batch, lengths, pooled, upstream, _stream):
            try:
                dev = torch.device("cuda", (list(o.devices) if o.devices else [0])[rank % max(1, len(o.devices or [0]))])
                with torch.cuda.device(dev):
                    ln = torch.as_tensor(_DevArray(lengths, (batch * F,), "<i4"), device=dev)
                    pl = torch.as_tensor(_DevArray(pooled, (batch, F * D), "<f4"), device=dev)
                    up = torch.as_tensor(_DevArray(upstream, (batch, F * D), "<f4"), device=dev)
                    fn(int(rank), int(step), ln, pl, up)
                    torch.cuda.synchronize(dev)
                return 0
            except Exception:  # noqa: BLE001  (reported as a failed step)
                import traceback

                traceback.print_exc()
                return 1

        self._cb = L.UPSTREAM_FN(cb)
        L.check(self.lib.s2d_trainer_set_upstream(self._t, self._cb, None))

    def step_n(self, count: int):
        """Trainer::step_n (trainer.hpp:117)."""
        L.check(self.lib.s2d_trainer_step_n(self._t, count))

    def run(self):
        """Trainer::run: the remaining of opts.steps."""
        L.check(self.lib.s2d_trainer_run(self._t))

    @property
    def steps_done(self) -> int:
        n = C.c_uint64(0)
        L.check(self.lib.s2d_trainer_steps_done(self._t, C.byref(n)))
        return n.value

    def plan(self) -> list[dict]:
        n = C.c_uint32(0)
        L.check(self.lib.s2d_trainer_plan(self._t, None, 0, C.byref(n)))
        out = (L.PlanEntry * max(1, n.value))()
        L.check(self.lib.s2d_trainer_plan(self._t, out, n.value, C.byref(n)))
        return [dict(table_id=out[i].table_id, row_lo=out[i].row_lo, row_hi=out[i].row_hi,
                     local_rank=out[i].local_rank) for i in range(n.value)]

    def rank_model(self, rank: int) -> dict:
        """Trainer::rank_model(rank) (trainer.hpp:125): {"dense_arch": (w1, b1,
        w2, b2), "over_arch": (...)} fp32, w1 [hidden, in], w2 [out, hidden]."""
        o = self.opts
        F, D = o.num_tables, o.dim
        out = {}
        for arch, (name, i, h, n) in enumerate([("dense_arch", o.dense_dim, o.dense_hidden, D),
                                                  ("over_arch", F * D + D, o.over_hidden, 1)]):
            w1 = np.zeros((h, i), np.float32)
            b1 = np.zeros(h, np.float32)
            w2 = np.zeros((n, h), np.float32)
            b2 = np.zeros(n, np.float32)
            L.check(self.lib.s2d_trainer_rank_model(self._t, rank, arch, w1.ctypes.data, b1.ctypes.data,
                                                    w2.ctypes.data, b2.ctypes.data))
            out[name] = (w1, b1, w2, b2)
        return out

    @property
    def last_loss(self) -> float:
        """MetricsRow::loss of the last step: the global-batch mean log-loss."""
        x = C.c_double(0)
        L.check(self.lib.s2d_trainer_last_loss(self._t, C.byref(x)))
        return x.value

    def metrics(self) -> list[dict]:
        """TrainResult::metrics so far: one MetricsRow dict (step, loss, ne,
        eff_lr_p50, eff_lr_p99, v_mean) per eval_cadence-th step and after
        the last step (dense model only)."""
        n = C.c_uint32(0)
        L.check(self.lib.s2d_trainer_metrics_rows(self._t, None, 0, C.byref(n)))
        out = (L.TrainMetricsRowC * max(1, n.value))()
        L.check(self.lib.s2d_trainer_metrics_rows(self._t, C.cast(out, C.c_void_p), n.value, C.byref(n)))
        return [{k: getattr(out[i], k) for k, _ in L.TrainMetricsRowC._fields_} for i in range(n.value)]

    def finalize(self) -> dict:
        """Trainer::finalize (trainer.hpp:118): {"final_ne": {ne, baseline_ctr,
        eval_samples}, "metrics": [...]}; evaluates unless the last step did."""
        rep = L.NEReportC()
        L.check(self.lib.s2d_trainer_final_ne(self._t, C.byref(rep)))
        return {"final_ne": {"ne": rep.ne, "baseline_ctr": rep.baseline_ctr, "eval_samples": rep.eval_samples},
                "metrics": self.metrics()}

    def replica_tables(self, group: int) -> list[tuple]:
        """[(weights [rows, dim] fp32, moments [rows] fp32)] per table of DP
        group `group` (Trainer::replica_tables, trainer.hpp:123)."""
        o = self.opts
        out = []
        for f in range(o.num_tables):
            w = np.zeros((o.rows_per_table, o.dim), np.float32)
            v = np.zeros(o.rows_per_table, np.float32)
            L.check(self.lib.s2d_trainer_replica_table(self._t, group, f, w.ctypes.data, v.ctypes.data))
            out.append((w, v))
        return out

    def tables(self) -> list[tuple]:
        """Consensus view: group 0's replica (Trainer::tables, trainer.hpp:122)."""
        return self.replica_tables(0)

    def save_tables(self, path: str):
        L.check(self.lib.s2d_trainer_save_tables(self._t, os.fsencode(path)))

    def load_tables(self, path: str):
        L.check(self.lib.s2d_trainer_load_tables(self._t, os.fsencode(path)))

    def metrics_row(self) -> dict:
        m = L.MetricsRowC()
        L.check(self.lib.s2d_trainer_metrics(self._t, C.byref(m)))
        return {"eff_lr_p50": m.eff_lr_p50, "eff_lr_p99": m.eff_lr_p99, "v_mean": m.v_mean, "rows": int(m.rows)}


# ---- train_toy (bindings/module.cpp:148-163, src/experiment.cpp:23-34) ------

# ExperimentConfig's keys and defaults (src/config.cpp:24-60)
_CONFIG_DEFAULTS = {
    "topology.total_ranks": "8", "topology.groups": "1",
    "data.tables": "8", "data.rows_per_table": "10000", "data.ids_per_sample": "2", "data.zipf_exponent": "1.0",
    "data.dense_dim": "8", "data.gt_id_scale": "0.25", "data.gt_dense_scale": "0.35", "data.gt_bias": "-0.8",
    "model.dim": "16", "model.dense_hidden": "32", "model.over_hidden": "64",
    "optimizer.variant": "rowwise-adagrad", "optimizer.eta": "0.1", "optimizer.eps": "1e-8", "optimizer.c": "1.0",
    "run.steps": "1000", "run.per_rank_batch": "4", "run.sync_interval": "1", "run.eval_cadence": "0",
    "run.eval_samples": "100000", "run.seed": "1", "run.threads": "1", "run.trace": "false",
    "sharding.strategy": "row-wise",
    "bandwidth.alpha_s": "2e-6", "bandwidth.inter_bytes_per_s": "2.5e10", "bandwidth.intra_bytes_per_s": "",
    "bandwidth.ranks_per_host": "8", "compute.flops_per_s": "2e12",
    "seeds.data": "", "seeds.init": "", "seeds.eval": "",
}

_M64 = (1 << 64) - 1


def _mix64(x: int) -> int:
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & _M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def _make_key(*fields: int) -> int:
    """rng.hpp make_key: fold fields through mix64."""
    h = 0x8A5CD789635D2DFF
    for f in fields:
        h = _mix64((h + 0x9E3779B97F4A7C15 + f) & _M64)
    return h


def _resolve_config(values: dict) -> tuple:
    """ExperimentConfig::resolve (src/config.cpp:200-289): every issue is
    collected and raised together as ValueError; seeds derive from run.seed
    as make_key({master, lane}) unless given."""
    issues = []

    def u64(key, lo, hi):
        raw = values[key]
        try:
            v = int(raw, 10)
        except ValueError:
            issues.append(f"{key} = '{raw}' is not a valid integer")
            return lo
        if v < lo or v > hi:
            issues.append(f"{key} = {raw} out of range [{lo}, {hi}]")
            return lo
        return v

    def dbl(key, lo, hi):
        raw = values[key]
        try:
            v = float(raw)
        except ValueError:
            issues.append(f"{key} = '{raw}' is not a valid number")
            return lo
        if not math.isfinite(v) or v < lo or v > hi:
            issues.append(f"{key} = {raw} out of range")
            return lo
        return v

    total = u64("topology.total_ranks", 1, 1 << 20)
    groups = u64("topology.groups", 1, 1 << 20)
    if total % groups:
        issues.append("topology.groups must divide topology.total_ranks")
    o = dict(
        total_ranks=total, groups=groups, num_tables=u64("data.tables", 1, 4096),
        rows_per_table=u64("data.rows_per_table", 1, 100000000), ids_per_sample=u64("data.ids_per_sample", 0, 1024),
        zipf_exponent=dbl("data.zipf_exponent", 0.0, 100.0), dense_dim=u64("data.dense_dim", 1, 4096),
        gt_id_scale=dbl("data.gt_id_scale", 0.0, 1e6), gt_dense_scale=dbl("data.gt_dense_scale", 0.0, 1e6),
        gt_bias=dbl("data.gt_bias", -1e6, 1e6), dim=u64("model.dim", 1, 512),
        dense_hidden=u64("model.dense_hidden", 1, 65536), over_hidden=u64("model.over_hidden", 1, 65536),
        steps=u64("run.steps", 1, 1 << 40), per_rank_batch=u64("run.per_rank_batch", 1, 1 << 20),
        sync_interval=u64("run.sync_interval", 1, 1 << 20), eval_cadence=u64("run.eval_cadence", 0, 1 << 40),
        eval_samples=u64("run.eval_samples", 1, 100000000))
    variant = values["optimizer.variant"]
    if variant not in ("rowwise-adagrad", "sgd"):
        issues.append(f"unknown optimizer variant: {variant}")
    opt = OptimizerConfig(eta=dbl("optimizer.eta", 1e-12, 1e6), eps=dbl("optimizer.eps", 1e-30, 1e6),
                          c=dbl("optimizer.c", 1e-12, 1e9), variant=variant)
    master = u64("run.seed", 0, _M64)
    u64("run.threads", 1, 1024)
    if values["run.trace"] not in ("true", "1", "false", "0"):
        issues.append(f"run.trace = '{values['run.trace']}' is not a boolean (true/false)")
    strategy = values["sharding.strategy"]
    if strategy not in ("row-wise", "table-wise"):
        issues.append(f"unknown sharding strategy: {strategy}")
    dbl("bandwidth.alpha_s", 0.0, 1.0)
    dbl("bandwidth.inter_bytes_per_s", 1.0, 1e18)
    if values["bandwidth.intra_bytes_per_s"]:
        dbl("bandwidth.intra_bytes_per_s", 1.0, 1e18)
    u64("bandwidth.ranks_per_host", 1, 1 << 20)
    dbl("compute.flops_per_s", 1.0, 1e24)

    def seed(key, lane):
        return _make_key(master, lane) if not values[key] else u64(key, 0, _M64)

    o.update(data_seed=seed("seeds.data", 1), init_seed=seed("seeds.init", 2), eval_seed=seed("seeds.eval", 3))
    if issues:
        raise ValueError(f"configuration invalid ({len(issues)} issue(s)):" + "".join("\n  - " + i for i in issues))
    return o, opt, strategy


def _config_hash(values: dict) -> str:
    """ExperimentConfig::hash_hex (src/config.cpp:291-316): FNV-1a 64 over the
    sorted 'key=value\\n' entries."""
    h = 0xCBF29CE484222325
    for k in sorted(values):
        for c in (k + "=" + values[k] + "\n").encode():
            h = ((h ^ c) * 0x100000001B3) & _M64
    return f"{h:016x}"


def train_toy(overrides: dict | None = None) -> dict:
    """run_train for a config given as {dotted_key: value} (the reference
    module's train_toy): the Trainer facade with the device dense model on
    this process's GPUs.  Returns final_ne, baseline_ctr, config_hash, the
    metrics rows, and qps_sim -- here MEASURED samples/s of the whole run
    (global batch x steps / wall seconds; the reference's alpha-beta
    simulation is out of scope) -- and peak_mem_bytes, the reference's
    footprint formula without its simulated all-to-all term (owned shard
    state + MLP + one resident batch, trainer.cpp:796-829)."""
    import time

    values = dict(_CONFIG_DEFAULTS)
    for k, v in (overrides or {}).items():
        if k not in values:
            raise ValueError(f"unknown config key '{k}'")
        values[k] = str(v)
    o, opt, strategy = _resolve_config(values)
    tr = Trainer(TrainerOptions(optimizer=opt, strategy=strategy, dense_model=True, **o))
    try:
        t0 = time.perf_counter()
        tr.run()
        fin = tr.finalize()
        wall = time.perf_counter() - t0
        N = o["total_ranks"] // o["groups"]
        shard = max(sum(e["row_hi"] - e["row_lo"] for e in tr.plan() if e["local_rank"] == n) for n in range(N))
        D, F = o["dim"], o["num_tables"]
        mlp = (o["dense_hidden"] * o["dense_dim"] + o["dense_hidden"] + D * o["dense_hidden"] + D
               + o["over_hidden"] * (F * D + D) + 2 * o["over_hidden"] + 1)
        batch = (F * o["ids_per_sample"] * 4 + o["dense_dim"] * 4 + 4) * o["per_rank_batch"]
        return {"final_ne": fin["final_ne"]["ne"], "baseline_ctr": fin["final_ne"]["baseline_ctr"],
                "qps_sim": o["total_ranks"] * o["per_rank_batch"] * o["steps"] / wall,
                "peak_mem_bytes": shard * (D + 1) * 4 + mlp * 4 + batch, "config_hash": _config_hash(values),
                "metrics": fin["metrics"]}
    finally:
        tr.close()


# ---- function-level forms of the path's reductions (embedding.hpp, optimizer.hpp) ----

def lookup_and_pool(weights, shards, per_sample_ids, table_id: int = 0) -> np.ndarray:
    """lookup_and_pool / pool_ids (embedding.hpp:41-58) on the device:
    weights [rows, dim] fp32 (the whole table, global row index), shards
    [(row_lo, row_hi)] in presentation order, per_sample_ids a list of id
    lists -> pooled [len(per_sample_ids), dim] fp32.  IndexError (the
    reference's out_of_range) for an id no shard covers."""
    w = np.ascontiguousarray(weights, np.float32)
    if w.ndim != 2:
        raise ValueError("weights must be [rows, dim]")
    lo = np.ascontiguousarray([int(s[0]) for s in shards], np.uint32)
    hi = np.ascontiguousarray([int(s[1]) for s in shards], np.uint32)
    lens = np.array([len(x) for x in per_sample_ids], np.uint64)
    off = np.zeros(len(lens) + 1, np.uint64)
    np.cumsum(lens, out=off[1:])
    ids = (np.concatenate([np.asarray(x, np.uint32) for x in per_sample_ids]) if len(lens) and off[-1]
           else np.zeros(1, np.uint32))
    out = np.zeros((len(lens), w.shape[1]), np.float32)
    L.check(_lib().s2d_pool_ids(w.ctypes.data, w.shape[0], w.shape[1], int(table_id), len(lo), lo.ctypes.data,
                                hi.ctypes.data, len(lens), off.ctypes.data, ids.ctypes.data, out.ctypes.data))
    return out


def pool_ids(weights, shards, ids, table_id: int = 0) -> np.ndarray:
    """pool_ids (embedding.hpp:52-53): one bag -> [dim] fp32."""
    return lookup_and_pool(weights, shards, [list(ids)], table_id)[0]


def aggregate_group_gradient(rows, grads, group_batch: int) -> list[dict]:
    """aggregate_group_gradient (optimizer.hpp:36-44) on the device:
    contributions (rows[i], grads[i] f64 [dim]) in arrival order ->
    [{"row", "g" (f64 [dim]), "sample_count"}] by ascending row."""
    r = np.ascontiguousarray(rows, np.uint32)
    g = np.ascontiguousarray(grads, np.float64)
    if g.ndim != 2 or g.shape[0] != len(r):
        raise ValueError("grads must be [n, dim] with one row per contribution")
    lib = _lib()
    n = C.c_uint64(0)
    L.check(lib.s2d_aggregate_group_gradient(r.ctypes.data, g.ctypes.data, len(r), int(group_batch), g.shape[1],
                                             None, None, None, 0, C.byref(n)))
    U = n.value
    out_r = np.zeros(max(U, 1), np.uint32)
    out_g = np.zeros((max(U, 1), g.shape[1]), np.float64)
    out_c = np.zeros(max(U, 1), np.uint32)
    if U:
        L.check(lib.s2d_aggregate_group_gradient(r.ctypes.data, g.ctypes.data, len(r), int(group_batch), g.shape[1],
                                                 out_r.ctypes.data, out_g.ctypes.data, out_c.ctypes.data, U,
                                                 C.byref(n)))
    return [{"row": int(out_r[k]), "g": out_g[k], "sample_count": int(out_c[k])} for k in range(U)]
