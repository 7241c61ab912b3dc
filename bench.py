#!/usr/bin/env python3
"""Benchmark of the 2D-sparse-parallel embedding step (fwd + bwd + fused
moment-scaled row-wise AdaGrad [+ replica sync]) -- BASELINE.json metric
"embedding fwd+bwd+update samples/s; HBM GB/s vs peak".

    python bench.py                               # N=1, cfg2, defaults
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W
    python bench.py --impl reference ...          # reference CPU path (oracle/_ref)

One JSON line on rank 0.  `value` = whole-job samples/s with inputs resident
in HBM (CUDA events on the engine's stream, max over ranks); `e2e` = the same
through the public API with pinned HOST buffers (H2D of lengths+ids+upstream
and D2H of the pooled output inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default=None, help="cfg1..cfg5 (default: cfg2 at N=1, cfg3 at N>1)")
    p.add_argument("--mesh", default=None, help="NxM (MP ranks per group x DP groups); default N x 1")
    p.add_argument("--batch", type=int, default=None, help="per-GPU batch override")
    p.add_argument("--strategy", default=None)
    p.add_argument("--scramble", action="store_true", help="hashed id -> row bijection (balances row-wise owners)")
    p.add_argument("--c", type=float, default=None, help="AdaGrad moment scaling factor (default: the config's, c = M)")
    p.add_argument("--nbatches", type=int, default=3, help="distinct input batches cycled")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e legs (very large configs)")
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="CPU baseline sample budget")
    p.add_argument("--seed", type=int, default=1234)
    p.add_argument("--trace-csv", default=None, help="write one measured step's collective trace (reference schema)")
    p.add_argument("--plan-rotate", type=int, default=0, help="experiment: rotate the plan's local ranks by k")
    p.add_argument("--no-phases", action="store_true", help="experiment: no phase events in the timed region")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, world):
    from paper_2508_03854_b200 import workloads

    name = args.config or ("cfg2" if world == 1 else "cfg3")
    w = workloads.get(name)
    if args.mesh:
        n, m = (int(x) for x in args.mesh.lower().split("x"))
    else:
        n, m = (world, 1) if world > 1 else (1, 1)
    if n * m != world:
        raise SystemExit(f"mesh {n}x{m} needs {n * m} ranks, have {world}")
    w.mesh = (n, m)
    if m > 1:
        w.c = float(m)  # paper default c = M
    if args.batch:
        w.batch = args.batch
    if args.strategy:
        w.strategy = args.strategy
    if args.scramble:
        w.scramble = True
    if args.c is not None:
        w.c = args.c
    return w


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled through NVML every
    ~10 ms DURING the timed region (in-process thread; the device calls of the
    timed loop release the GIL).  Falls back to `nvidia-smi -lms 20`."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, dev):
        self.dev = dev
        self.sm, self.reasons, self.mx = [], set(), None
        self._stop = threading.Event()
        self.t = None
        self.proc = None
        self.lines = []

    def _handle(self, nv):
        import torch
        try:
            pr = torch.cuda.get_device_properties(self.dev)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.dev)

    def _poll(self, nv, h):
        masks = [(n, getattr(nv, a, 0)) for n, a in self.REASONS]
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for n, m in masks:
                    if m and (r & m):
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.010)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._handle(nv)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, args=(nv, h), daemon=True)
            self.t.start()
        except Exception:
            try:
                q = "clocks.sm,clocks.max.sm," + ",".join("clocks_event_reasons." + n for n, _ in self.REASONS[:4])
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                     "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.t = threading.Thread(target=self._read, daemon=True)
                self.t.start()
            except Exception:
                self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            try:
                self.sm.append(float(parts[0]))
                self.mx = float(parts[1])
            except (ValueError, IndexError):
                continue
            for (nm, _), val in zip(self.REASONS, parts[2:6]):
                if val.lower() in ("active", "1"):
                    self.reasons.add(nm)

    def __exit__(self, *a):
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.mx, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


def algorithmic_bytes(w, nnz_own, unique, entries, n_mp, dirty=0):
    """Algorithmic HBM bytes per step of each phase, SURVEY.md 8(d):
    4 nnz (ids) + s_w D nnz (row gathers) + 4 D E_owned (partials out)
    + 4 D E_local (partials in) + 4 D B F (pooled out) + 4 D B F (upstream in)
    + 4 D E_owned (grads in at the owner) + 2 U (s_w D + 4) (row + moment RMW)
    + 2 U_dirty (s_w D + 4) (sync); the partial terms vanish at N = 1 and the
    sort passes are implementation overhead (excluded).  `lookup_unique`
    replaces the per-id row gathers by one HBM read per distinct row (the
    Zipf-hot repeats are L2 hits): the HBM-side view of the same kernel."""
    sw = 2 if w.dtype == "bf16" else 4
    D = float(np.mean(w.dims))
    BF = w.batch * w.F
    pooled = 4.0 * D * BF
    if n_mp > 1:
        part = 4.0 * D * entries  # partials out (owner) + the same count in at the requesters
        lookup = 4 * nnz_own + sw * D * nnz_own + part + part + pooled
        lookup_unique = 4 * nnz_own + sw * D * unique + part + part + pooled
        update = pooled + 4.0 * D * entries + 2 * unique * (sw * D + 4)  # upstream in, grads in, RMW
    else:
        lookup = 4 * nnz_own + sw * D * nnz_own + pooled
        lookup_unique = 4 * nnz_own + sw * D * unique + pooled
        update = pooled + 2 * unique * (sw * D + 4)
    return {"lookup": lookup, "lookup_unique": lookup_unique, "update": update,
            "sync": 2 * dirty * (sw * D + 4), "conversions": {"lookup": nnz_own * D, "update": nnz_own * D}}


# B200 XU (F2F) rate used for the conversion ceiling: 16 lanes / clk / SM
XU_PER_CLK_SM = 16


PHASE_KERNELS = {"lookup": ("k_lookup_ring",), "update": ("k_update_ring", "k_range_partials", "k_group_partials")}


def traffic_from_profiles(phase):
    """DRAM bytes (read + write) per step of a phase's kernels from the
    committed `ncu --set full` captures (profiles/traffic.json, written by
    tools/ncu_summarize.py); None if a kernel of the phase has no capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tj = json.load(f)
        tot, src = 0.0, []
        for k in PHASE_KERNELS[phase]:
            t = tj.get(k)
            if t is None:
                if k == "k_group_partials":  # tiny; missing capture adds nothing material
                    continue
                return None, f"no capture of {k}"
            tot += t["dram_bytes_per_launch"] * t.get("launches_per_step", 1)
            src.append(f"profiles/{t['round']}/{t['source']}")
        return tot, " + ".join(src)
    except Exception:
        return None, None


# ----------------------------------------------------------------------------
# reference CPU arm: the unmodified reference library (oracle/_ref) on a
# bounded sample of the same workload
# ----------------------------------------------------------------------------

def reference_step_sample(w, seed, n_samples, threads, step):
    """One bounded-sample step of the reference CPU path for one MP group of
    the arm's mesh (N = w.mesh[0] virtual ranks, each with n_samples of its
    own batch, the reference's group step incl. its all-to-all copies).
    Tables are compacted to the rows the sample touches (each row's
    arithmetic is independent); the plan is the reference
    plan_greedy over the compacted tables with the arm's strategy.  Returns
    (seconds of ref_group_step, samples processed)."""
    from oracle import MeshSpec, Oracle

    ref = Oracle("reference")
    n_mp = w.mesh[0]
    F = w.F
    B = min(n_samples, w.batch)
    L, I, U, feats = [], [], [], []
    for r in range(n_mp):  # a B-sample batch per rank, same distributions as the arm's
        lengths, ids = w.batch_for(seed, step, r, batch=B)
        L.append(lengths)
        I.append(ids)
        feats.append(np.repeat(np.tile(np.arange(F), B), lengths))
        U.append(w.upstream_for(seed, step, r, batch=B))
    rows = np.zeros(F, np.uint32)
    cI = [np.empty_like(x) for x in I]
    for f in range(F):
        sel = [ft == f for ft in feats]
        u, inv = np.unique(np.concatenate([x[m] for x, m in zip(I, sel)]), return_inverse=True)
        rows[f] = max(1, len(u))
        o = 0
        for r in range(n_mp):
            k = int(sel[r].sum())
            cI[r][sel[r]] = inv[o:o + k].astype(np.uint32)
            o += k
    dims = np.array(w.dims, np.uint32)
    if n_mp == 1:
        plan = np.array([[f, 0, int(rows[f]), 0] for f in range(F)], np.uint32)
    else:
        prof = [(f, int(rows[f]) * int(dims[f]) * 4, w.plan_cost(f, n_mp), int(rows[f])) for f in range(F)]
        plan = ref.plan_greedy(prof, n_mp, w.strategy)
    spec = MeshSpec(rows=rows, dims=dims, plan=plan, T=n_mp, M=1, B=B, eta=w.eta, c=w.c)
    rng = np.random.default_rng(seed)
    wt = (rng.standard_normal(spec.replica_floats()) * 0.05).astype(np.float32)
    vt = np.zeros(spec.replica_rows(), np.float32)
    ref.group_step(spec, L, cI, U, wt, vt, None, threads=threads)
    return ref.last_compute_seconds, B * n_mp


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = workload(args, world)
    from oracle import reference_available

    threads = os.cpu_count() or 1
    kind = "reference" if reference_available() else "port"
    if kind != "reference":
        _emit({"impl": "reference", "unavailable": "oracle/_ref/libs2dref.so not built"})
        return
    # calibrate the sample to ~target seconds per step
    target = max(0.5, min(6.0, 150.0 / max(1, args.steps + args.warmup)))
    t, b = reference_step_sample(w, args.seed, 256, threads, 0)
    n = int(max(64, min(w.batch, 256 * target / max(t, 1e-3))))
    for k in range(args.warmup):
        reference_step_sample(w, args.seed, n, threads, k)
    tot_t, tot_s = 0.0, 0
    for k in range(args.steps):
        t, b = reference_step_sample(w, args.seed, n, threads, args.warmup + k)
        tot_t += t
        tot_s += b
    sps = tot_s / tot_t
    line = {
        "impl": "reference", "metric": "embedding fwd+bwd+update samples/s", "value": sps,
        "unit": "samples/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "storage_dtype": "f32", "data": "synthetic",
        "config": {"workload": w.name + ": " + w.describe, "mesh": f"{w.mesh[0]}x{w.mesh[1]}",
                   "simulated": f"one MP group of {w.mesh[0]} virtual ranks (reference group step, all host threads)",
                   "global_batch": n * w.mesh[0],
                   "sample": f"{n} of {w.batch} samples per rank per step, tables compacted to touched rows"},
        "cpu_baseline": {"value": sps, "unit": "samples/s", "cores": threads, "kind": kind, "cpu_model": cpu_model(),
                         "sample": f"{n} of {w.batch} samples per rank x {w.mesh[0]} ranks per step, touched-row tables"},
        "e2e": {"value": sps, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    _emit(line)


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2508_03854_b200 as s2d

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workload(args, world)
    n_mp, m = w.mesh
    topo = s2d.Topology(world, m)
    nid = None
    if world > 1:
        obj = [s2d.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    # expected lookups = ids + weighted distinct rows per table (Workload.plan_cost)
    tables = [s2d.TableConfig(int(r), int(d), w.plan_cost(f, n_mp)) for f, (r, d) in enumerate(zip(w.rows, w.dims))]
    plan = w.table_plan(n_mp) if (w.strategy == "table-wise" and n_mp > 1) else None
    if args.plan_rotate:
        prof = [(i, t.rows * t.dim * 4, t.expected_lookups, t.rows) for i, t in enumerate(tables)]
        plan = s2d.plan_greedy(prof, n_mp, w.strategy)
        for e in plan:
            e["local_rank"] = (e["local_rank"] + args.plan_rotate) % n_mp
    eng = s2d.Sparse2DEmbedding(tables, topo, rank=rank, device=local, strategy=w.strategy, plan=plan,
                                optimizer=s2d.OptimizerConfig(eta=w.eta, eps=1e-8, c=w.c),
                                weight_dtype=w.dtype, nccl_id=nid, strict=False)
    # a real (non-NULL) stream shared by the engine and the timing events
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    eng.init_tables(args.seed)
    # inputs: NB distinct batches, resident in HBM for `value`
    NB = max(1, args.nbatches)
    host = []
    for k in range(NB):
        lengths, ids = w.batch_for(args.seed, k, rank)
        up = w.upstream_for(args.seed, k, rank)
        host.append((lengths, ids, up))
    dev = [(torch.from_numpy(l.view(np.int32)).cuda(), torch.from_numpy(i.view(np.int32)).cuda(),
            torch.from_numpy(u).cuda()) for l, i, u in host]
    nnz_mean = float(np.mean([len(h[1]) for h in host]))

    host_s = {"forward": 0.0, "backward": 0.0}

    def step(k):
        l, i, u = dev[k % NB]
        t0 = time.perf_counter()
        eng.forward(l, i, "engine", batch=w.batch)  # zero-copy output (engine buffer)
        t1 = time.perf_counter()
        eng.backward_update(u)
        host_s["forward"] += t1 - t0
        host_s["backward"] += time.perf_counter() - t1
        if m > 1:
            eng.sync_replicas()

    def barrier():
        if world > 1:
            dist.barrier()

    for k in range(args.warmup):
        step(k)
    eng.synchronize()
    torch.cuda.synchronize()
    eng.phase_times()  # reset
    # kernel events inside the timed region, on the engine stream: only around
    # the three hot kernels (each event pair drains the stream between two
    # kernels); the full phase split comes from a separate profiled pass
    eng.set_profiling(not args.no_phases, hot_only=True)
    barrier()
    torch.cuda.synchronize()
    launches0 = s2d.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    host_s["forward"] = host_s["backward"] = 0.0
    wait0 = eng.stats()["host_wait_ns"]
    with ClockSampler(local) as clk:
        # a step-boundary event per step (recording does not drain the stream)
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ev0.record(stream)
        for k in range(args.steps):
            step(args.warmup + k)
            evs[k].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = s2d.launch_count() - launches0
    eng.synchronize()
    eng.set_profiling(False)
    phases = eng.phase_times()
    ms = ev0.elapsed_time(ev1)
    host_timed = dict(host_s)  # host time of the timed steps only
    host_timed["blocked_on_counts"] = (eng.stats()["host_wait_ns"] - wait0) * 1e-9
    # full phase split (every phase bracketed) from a separate pass of the same steps
    eng.set_profiling(True)
    n_split = min(args.steps, 20)
    for k in range(n_split):
        step(args.warmup + k)
    eng.synchronize()
    eng.set_profiling(False)
    split = {p: v for p, v in eng.phase_times().items() if v[1]}
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * w.batch * args.steps / (ms_max / 1e3)
    st = eng.stats()
    step_ms = [round(ev0.elapsed_time(evs[0]), 4)] + [round(evs[k - 1].elapsed_time(evs[k]), 4)
                                                       for k in range(1, args.steps)]
    mine = {"nnz_owned": st["nnz_owned"], "unique_rows": st["unique_rows"], "ms": ms, "step_ms": step_ms,
            "phase_ms": {p: round(v[0] / max(1, n_split), 4) for p, v in split.items()},
            "host_ms_per_step": {k: round(1e3 * v / max(1, args.steps), 4) for k, v in host_timed.items()}}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    if args.trace_csv:
        # one more profiled step -> measured trace rows in the reference's
        # trace.csv schema (experiment.cpp:47-62), written by rank 0
        eng.set_profiling(True)
        eng.phase_times()
        step(0)
        eng.synchronize()
        eng.set_profiling(False)
        rows = eng.trace_rows(0)
        allrows = [rows]
        if world > 1:
            allrows = [None] * world
            dist.all_gather_object(allrows, rows)
        if rank == 0:
            with open(args.trace_csv, "w") as f:
                f.write(s2d.traces_to_csv([r for rr in allrows for r in rr], f"{w.name}-{n_mp}x{m}-seed{args.seed}"))

    # ---- e2e through the public API with pinned host buffers ----
    K2 = args.e2e_steps or max(3, min(args.steps, 10))
    pin = [(torch.from_numpy(l.view(np.int32)).pin_memory(), torch.from_numpy(i.view(np.int32)).pin_memory(),
            torch.from_numpy(u).pin_memory()) for l, i, u in host]
    pooled_hs = [torch.empty((w.batch, w.sum_dims), dtype=torch.float32).pin_memory() for _ in range(2)]
    pooled_h = pooled_hs[0]

    def step_host(k, sync_each):
        l, i, u = pin[k % NB]
        eng.forward(l, i, pooled_hs[k % 2], batch=w.batch)
        eng.backward_update(u)
        if m > 1:
            eng.sync_replicas()
        if sync_each:
            eng.synchronize()  # the step's pooled rows are in host memory

    def pcie_probe(nbytes):
        """Pinned host <-> device copy bandwidth of this GPU with both
        directions in flight (two streams), best of 3."""
        nb = max(1 << 20, int(nbytes)) // 4 * 4
        hs = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
        hd = torch.empty(nb // 4, dtype=torch.float32).pin_memory()
        ds = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
        dd = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        best = (0.0, 0.0)
        for _ in range(3):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            torch.cuda.synchronize()
            with torch.cuda.stream(s1):
                e[0].record()
                ds.copy_(hs, non_blocking=True)
                e[1].record()
            with torch.cuda.stream(s2):
                e[2].record()
                hd.copy_(dd, non_blocking=True)
                e[3].record()
            torch.cuda.synchronize()
            up, down = nb / (e[0].elapsed_time(e[1]) / 1e3) / 1e9, nb / (e[2].elapsed_time(e[3]) / 1e3) / 1e9
            best = (max(best[0], up), max(best[1], down))
        del hs, hd, ds, dd
        return {"h2d_gbs": best[0], "d2h_gbs": best[1], "bytes": nb,
                "how": "pinned tensors, H2D and D2H copies in flight together on two streams, best of 3"}

    def time_e2e(async_host, sync_each):
        eng.set_async_host(async_host)
        step_host(0, True)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k in range(K2):
            step_host(k, sync_each)
        eng.synchronize()  # every step's pooled rows are in host memory
        torch.cuda.synchronize()
        te = torch.tensor([(time.perf_counter() - t0) * 1e3], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        return world * w.batch * K2 / (float(te.item()) / 1e3)

    # serial: the read-back completes inside forward; per-step: copies on the
    # context's copy streams, host waits at the end of every step; pipelined
    # (the headline): no host wait between steps -- step k's read-back
    # overlaps step k+1's upload, lookup and update; one synchronize at the end
    # the device-resident inputs are no longer needed: their HBM goes to the
    # host-mode staging buffers
    del dev
    torch.cuda.empty_cache()
    if args.no_e2e:
        e2e_serial = e2e_step = e2e = None
    else:
        e2e_serial = time_e2e(False, True)
        e2e_step = time_e2e(True, True)
        e2e = time_e2e(True, False)
    eng.set_async_host(False)
    h2d = int(sum(x.numel() * 4 for x in pin[0]) / 1)
    d2h = int(pooled_h.numel() * 4)
    # the e2e ceiling: this GPU's pinned-host copy bandwidth, both directions
    # at once (as the e2e loop drives them), measured now
    pcie = None if args.no_e2e else pcie_probe(min(h2d, d2h))
    if pcie and e2e:
        floor_ms = 1e3 * max(h2d / (pcie["h2d_gbs"] * 1e9), d2h / (pcie["d2h_gbs"] * 1e9))
        pcie["e2e_floor_samples_per_s"] = world * w.batch / (floor_ms / 1e3)
        pcie["e2e_frac"] = e2e / pcie["e2e_floor_samples_per_s"]

    # ---- roofline of the dominant phase (SURVEY.md 8(d) bytes) ----
    peak, peak_src = load_peaks()
    ab = algorithmic_bytes(w, st["nnz_owned"] or nnz_mean, st["unique_rows"] or 0, st["entries_owned"], n_mp,
                           st.get("dirty_rows", 0))
    clk_now = clk.summary()
    sm_hz = (clk_now["sm_mhz"] or 1965.0) * 1e6
    # per-launch times: the update from the timed region (its events are the
    # only ones there), lookup / sort from the split pass
    per_phase = {}
    ms_step_local = ms / max(1, args.steps)
    for p in ("lookup", "sort", "update"):
        src, where = (phases, "timed region") if phases.get(p, (0, 0))[1] else (split, "split pass")
        if p in src and src[p][1]:
            pl = src[p][0] / src[p][1]
            ent = {"ms_per_launch": pl, "share": pl / max(ms_step_local, 1e-9), "measured_in": where}
            if p in ("lookup", "update"):
                ent["algo_bytes"] = ab[p]
                ent["algo_gbs"] = ab[p] / (pl / 1e3) / 1e9
                ent["frac"] = ent["algo_gbs"] / peak
                # f32 -> f64 widening of every gathered column on the XU pipe
                xu_ms = 1e3 * ab["conversions"][p] / (148 * XU_PER_CLK_SM * sm_hz)
                ent["xu_floor_ms"] = xu_ms
                ent["xu_frac"] = xu_ms / pl
            if p == "lookup":
                ent["unique_row_bytes"] = ab["lookup_unique"]
                ent["unique_row_frac"] = ab["lookup_unique"] / (pl / 1e3) / 1e9 / peak
            per_phase[p] = ent
    dom = max(per_phase, key=lambda p: per_phase[p]["ms_per_launch"]) if per_phase else "update"
    if dom == "sort":  # the sort is implementation overhead (no 8(d) bytes): report the heavier of the others
        dom = max((p for p in per_phase if p != "sort"), key=lambda p: per_phase[p]["ms_per_launch"], default="update")
    kname = {"lookup": "k_lookup_ring", "update": "k_update_ring+k_range_partials"}[dom]
    achieved = per_phase.get(dom, {}).get("algo_gbs", 0.0)
    traffic = traffic_from_profiles(dom)
    if (w.name, n_mp, m, w.batch) != ("cfg2", 1, 1, 16384):  # captured on cfg2 1x1 only
        traffic = (None, "no ncu capture for this workload/mesh (profiles/ hold cfg2 1x1)")
    wbytes = 2 if w.dtype == "bf16" else 4
    table_gb = sum(int(r) * (int(d) * wbytes + 4) for r, d in zip(w.rows, w.dims)) / 1e9
    line = {
        "metric": "embedding fwd+bwd+update samples/s", "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64",  # arithmetic type of the path (f64 accumulation, as the reference)
        "storage_dtype": "bf16" if w.dtype == "bf16" else "f32",
        "data": "synthetic (seeded Zipf ids, power-law bag lengths, N(0,1e-3) upstream)",
        "config": {"workload": w.name + ": " + w.describe + (" (ids scrambled)" if w.scramble else ""),
                   "global_batch": world * w.batch,
                   "per_gpu_batch": w.batch, "tables": w.F, "dim": int(np.max(w.dims)),
                   "mesh": f"{n_mp}x{m}", "strategy": w.strategy, "optimizer": f"rowwise-adagrad c={w.c}",
                   "parallelism": f"mp{n_mp}xdp{m}", "nnz_per_gpu": nnz_mean,
                   "l2": f"inputs larger than L2 (tables {table_gb:.1f} GB, upstream "
                         f"{w.batch * w.sum_dims * 4 / 1e6:.0f} MB/step), {NB} distinct batches cycled"},
        "roofline": {"bound": "hbm", "kernel": kname, "phase": dom, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
                     "traffic": traffic[0], "traffic_source": traffic[1],
                     "dram_frac": (traffic[0] / (per_phase[dom]["ms_per_launch"] / 1e3) / 1e9 / peak
                                   if traffic[0] and dom in per_phase else None),
                     "algorithmic_bytes_per_launch": ab[dom],
                     "bytes_model": "SURVEY.md 8(d): update = upstream (or owner gradient rows) read once + "
                                    "2 U (s_w D + 4) row/moment read-modify-write; lookup = ids + s_w D per id "
                                    "+ pooled rows out; sort passes excluded",
                     "xu_ceiling": {p: {"floor_ms": per_phase[p]["xu_floor_ms"], "frac": per_phase[p]["xu_frac"]}
                                    for p in ("lookup", "update") if p in per_phase},
                     "xu_note": "f32->f64 widening of nnz x D gathered columns (F2F on the XU pipe, "
                                "16/clk/SM) at the sampled SM clock: the conversion-throughput floor"},
        "phases": per_phase,
        "phase_split_ms": {p: v[0] / max(1, n_split) for p, v in split.items()},
        "phase_split_note": f"every phase bracketed, separate pass of {n_split} steps (rank 0)",
        "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "forward(pinned host ids -> pinned host pooled) -> backward_update(pinned host upstream) "
                       "every step, synchronize after the last; wall clock around the loop (max over ranks)",
                "copy_overlap": "inputs on the H2D copy stream, pooled read-back on the D2H stream; at N = 1 two "
                                "staging buffers per direction let step k's read-back overlap step k+1",
                "per_step_sync_value": e2e_step, "serial_value": e2e_serial, "pcie_ceiling": pcie},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "step_stats": {k: st[k] for k in ("nnz_owned", "unique_rows", "long_segments", "a2a_bytes_sent",
                                          "sync_bytes", "dirty_rows", "sync_mode")},
        "per_rank": per_rank,
    }
    if world > 1:
        # NVLink roofline of the exchanges (rank 0): bytes this rank stores into
        # peers / the time of the kernels that carry them (the profiled split
        # pass), against the measured peer-store ceiling (tools/nvlink_probe.cu,
        # profiles/r01/nvlink_probe.json: 690 GB/s one way, 652 per direction both
        # ways; 900 nominal)
        def ph_ms(*names):
            return sum(split[p][0] / max(1, n_split) for p in names if p in split)

        nv = {}
        for name, nbytes, phs in (("C1_ids", st["ids_bytes_sent"], ("bucket", "a2a_ids")),
                                  ("C1_pooled", st["lookup_bytes_sent"], ("lookup",)),
                                  ("C2_grad", st["grad_bytes_sent"], ("grad_gather",)),
                                  ("C3_sync", st["sync_bytes"], ("sync_push", "sync_mean"))):
            pm = ph_ms(*phs)
            if pm and nbytes:
                gbs = nbytes / (pm / 1e3) / 1e9
                nv[name] = {"bytes": nbytes, "ms": pm, "achieved_gbs": gbs, "frac": gbs / 652.4,
                            "phases": list(phs)}
        line["nvlink"] = {"peak_gbs": 652.4, "peak_source": "measured peer stores per direction, both directions "
                                                            "active (profiles/r01/nvlink_probe.json)",
                          "exchanges": nv}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(w, args)
    if rank == 0:
        _emit(line)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_baseline(w, args):
    from oracle import reference_available

    threads = os.cpu_count() or 1
    if not reference_available():
        return None
    t, b = reference_step_sample(w, args.seed, 256, threads, 0)
    n = int(max(64, min(w.batch, 256 * 4.0 / max(t, 1e-3))))
    tot_t, tot_s, k = 0.0, 0, 0
    while tot_t < args.cpu_seconds and k < 20:
        t, b = reference_step_sample(w, args.seed, n, threads, k)
        tot_t += t
        tot_s += b
        k += 1
    return {"value": tot_s / tot_t, "unit": "samples/s", "cores": threads, "kind": "reference",
            "cpu_model": cpu_model(),
            "sample": f"{k} steps x {n} of {w.batch} samples, tables compacted to touched rows"}


def _emit(line):
    """The ONE JSON line, on the real stdout (C-level prints were moved off it)."""
    os.write(_JSON_FD, (json.dumps(line) + "\n").encode())


_JSON_FD = 1


def main():
    global _JSON_FD
    # Libraries print to fd 1 from C (e.g. NCCL's version banner under
    # NCCL_DEBUG=VERSION); keep stdout for the JSON line alone.
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
