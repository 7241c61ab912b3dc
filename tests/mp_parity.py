"""Multi-GPU parity of the 2D step, run under torchrun (one process per GPU):

    python -m torch.distributed.run --nproc-per-node T --master-addr 127.0.0.1 \
        --master-port 29531 tests/mp_parity.py --groups M [--strategy row-wise]

Every rank runs the sm_100a step through the C ABI with NCCL between ranks.
Rank 0 replays the whole T-rank mesh with the CPU oracle on identical inputs
and checks, bit for bit: every rank's pooled output of every step, the wire
layouts of the last step on every rank (demand lengths and ids received,
pooled partials sent, gradient payload sent, unique rows updated), and every
rank's shard of its group's replica (weights + moments) at the end.
torch.distributed (gloo) only carries the NCCL bootstrap id and the results.
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


class _ThreadDist:
    """torch.distributed's object collectives for virtual ranks on threads
    (--local): every call is a rendezvous of all `world` threads."""

    def __init__(self, world):
        import threading

        self.world = world
        self.bar = threading.Barrier(world, timeout=900)
        self.box = [None] * world

    def view(self, rank):
        return _RankDist(self, rank)


class _RankDist:
    def __init__(self, hub, rank):
        self.h, self.rank = hub, rank

    def _exchange(self, obj):
        self.h.box[self.rank] = obj
        self.h.bar.wait()
        out = list(self.h.box)
        self.h.bar.wait()
        return out

    def broadcast_object_list(self, lst, src=0):
        lst[0] = self._exchange(lst[0])[src]

    def gather_object(self, obj, out, dst=0):
        got = self._exchange(obj)
        if self.rank == dst:
            out[:] = got

    def all_gather_object(self, out, obj):
        out[:] = self._exchange(obj)

    def barrier(self):
        self._exchange(None)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=1)
    ap.add_argument("--strategy", default="row-wise")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--sync-interval", type=int, default=1)
    ap.add_argument("--sgd", action="store_true")
    ap.add_argument("--batch", type=int, default=48)
    ap.add_argument("--engine-out", action="store_true", help="zero-copy pooled output (owners write it)")
    ap.add_argument("--mean", action="store_true", help="tables 0, 2, 4 use mean pooling")
    ap.add_argument("--mixed-out", action="store_true",
                    help="even ranks take the engine-owned output, odd ranks their own device buffer")
    ap.add_argument("--ckpt", action="store_true", help="S2DCKPT1 save from the mesh + load into every replica")
    ap.add_argument("--bad-id", action="store_true",
                    help="rank 1 sends an id past its table's rows: some rank must raise IndexError")
    ap.add_argument("--bf16", action="store_true",
                    help="bf16 shards: the oracle is re-seeded every step from the mesh's (widened) weights")
    ap.add_argument("--local", type=int, default=0,
                    help="run T virtual ranks as threads of this process on one GPU (LocalHub), no torchrun")
    args = ap.parse_args()

    if args.local:
        import paper_2508_03854_b200 as s2d

        hub = s2d.LocalHub(args.local)
        td = _ThreadDist(args.local)
        rc = s2d.run_ranks(lambda r: rank_main(args, r, args.local, 0, td.view(r), hub), args.local, timeout=1200)
        sys.exit(max(int(x or 0) for x in rc))
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    sys.exit(rank_main(args, rank, world, local, dist, None))


def rank_main(args, rank, world, local, dist, hub):
    import torch

    import paper_2508_03854_b200 as s2d
    from cases import make_batch, upstream

    torch.cuda.set_device(local)
    M = args.groups
    N = world // M
    rows = np.array([300, 41, 7, 1000, 128], np.uint32)
    dims = np.array([64, 64, 64, 64, 64], np.uint32)
    F, B = len(rows), args.batch
    eta, c = 0.1, float(M)
    profiles = [(f, int(rows[f]) * int(dims[f]) * 4, float(10 - f), int(rows[f])) for f in range(F)]
    plan = s2d.plan_greedy(profiles, N, args.strategy)
    nid = [s2d.nccl_unique_id() if rank == 0 and hub is None else None]
    dist.broadcast_object_list(nid, src=0)
    mean = np.array([1 if (args.mean and f % 2 == 0) else 0 for f in range(F)], np.uint8)
    tables = [s2d.TableConfig(int(rows[f]), int(dims[f]), pooling="mean" if mean[f] else "sum") for f in range(F)]
    opt = s2d.OptimizerConfig(eta=eta, eps=1e-8, c=c, variant="sgd" if args.sgd else "rowwise-adagrad")
    eng = s2d.Sparse2DEmbedding(tables, s2d.Topology(world, M), rank=rank, device=local, plan=plan, optimizer=opt,
                                weight_dtype="bf16" if args.bf16 else "fp32", nccl_id=nid[0], hub=hub)
    eng.init_tables(31)
    if args.bf16:
        return run_bf16(args, eng, dist, rank, world, M, N, rows, dims, B, eta, c, plan)
    if args.bad_id:
        return run_bad_id(eng, dist, rank, world, rows, dims, B)

    def inputs(step, r):
        rng = np.random.default_rng([step, r, 77])
        lengths, ids = make_batch(rng, rows, B, max_len=9, zipf=1.1)
        return lengths, ids, upstream(rng, B, int(dims.sum()))

    pooled_mine, layouts = [], None
    trace = None
    sync_modes = []
    for step in range(args.steps):
        if step == args.steps - 1:  # measured trace covers the last step only
            eng.set_profiling(True)
            eng.phase_times()
        lengths, ids, up = inputs(step, rank)
        if args.engine_out or (args.mixed_out and rank % 2 == 0):
            import torch

            dl = torch.from_numpy(lengths.view(np.int32)).cuda()
            di = torch.from_numpy(ids.view(np.int32)).cuda()
            eng.forward(dl, di, "engine", batch=B)
            eng.synchronize()
            pooled_mine.append(eng.debug(6).reshape(B, -1).copy())
        else:  # caller-owned device output: every partial travels through the receive buffer
            dl = torch.from_numpy(lengths.view(np.int32)).cuda()
            di = torch.from_numpy(ids.view(np.int32)).cuda()
            out = torch.empty((B, int(dims.sum())), dtype=torch.float32, device="cuda")
            eng.forward(dl, di, out, batch=B)
            eng.synchronize()
            pooled_mine.append(out.cpu().numpy())
        eng.backward_update(up)
        if M > 1 and (step + 1) % args.sync_interval == 0:
            eng.sync_replicas()
            sync_modes.append(eng.stats()["sync_mode"])
        if step == args.steps - 1:
            layouts = {k: eng.debug(k) for k in (0, 1, 2, 3, 4, 5)}
            eng.synchronize()
            trace = eng.trace_rows(step)
            eng.set_profiling(False)
    shard = {}
    for f in range(F):
        lo, hi = eng.owned_range(f)
        if hi > lo:
            shard[f] = (lo, hi) + eng.read_rows(f, lo, hi)
    ckpt_path, loaded = None, {}
    if args.ckpt:
        import tempfile

        box = [tempfile.mkdtemp(prefix="s2d_ckpt_") + "/mesh.ckpt" if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        ckpt_path = box[0]
        eng.save_tables(ckpt_path)
        eng.init_tables(12345)  # clobber, then restore from the file
        eng.load_tables(ckpt_path)
        for f in range(F):
            lo, hi = eng.owned_range(f)
            if hi > lo:
                loaded[f] = (lo, hi) + eng.read_rows(f, lo, hi)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object((pooled_mine, layouts, shard, loaded, trace, sync_modes), gathered, dst=0)
    eng.close()
    if rank != 0:
        dist.barrier()
        return 0

    from oracle import MeshSpec, MeshState, Oracle

    port = Oracle("port")
    plan_arr = np.array([[e["table_id"], e["row_lo"], e["row_hi"], e["local_rank"]] for e in plan], np.uint32)
    spec = MeshSpec(rows=rows, dims=dims, plan=plan_arr, T=world, M=M, B=B, eta=eta, c=c, sgd=args.sgd, mean=mean)
    st = MeshState.init(port, spec, 31)
    st_prev = ([w.copy() for w in st.ws], [v.copy() for v in st.vs])
    fails = []
    for step in range(args.steps):
        ins = [inputs(step, r) for r in range(world)]
        L = [x[0] for x in ins]
        I = [x[1] for x in ins]
        U = [x[2] for x in ins]
        want = st.step(port, L, I, U, do_sync=(M > 1 and (step + 1) % args.sync_interval == 0))
        for r in range(world):
            got = gathered[r][0][step]
            if not np.array_equal(got.view(np.uint32), want[r].view(np.uint32)):
                fails.append(f"pooled step {step} rank {r}: max|d|={np.max(np.abs(got - want[r]))}")
        if step == args.steps - 1:
            # wire layouts of the last step, per MP group (oracle dump on a copy)
            for g in range(M):
                sl = slice(g * N, (g + 1) * N)
                w0, v0 = st_prev[0][g].copy(), st_prev[1][g].copy()
                _, dump = port.group_step(spec, L[sl], I[sl], U[sl], w0, v0, None, want_dump=True)
                for l in range(N):
                    r = g * N + l
                    lay = gathered[r][1]
                    if N > 1:
                        if not np.array_equal(lay[0], dump.dem_len[l].ravel()):
                            fails.append(f"demand lengths rank {r}")
                        if not np.array_equal(lay[1], dump.dem_ids[l]):
                            fails.append(f"demand ids rank {r}")
                        # partials received by requester l, by owner; gradient
                        # rows received by owner l, by requester
                        want_p = np.concatenate([dump.part[o][l] for o in range(N)])
                        want_g = np.concatenate([dump.grad[n][l] for n in range(N)])
                        # (engine output: single-owner tables' rows bypass the partial buffer)
                        engine_r = args.engine_out or (args.mixed_out and r % 2 == 0)
                        if not engine_r and not np.array_equal(lay[2].view(np.uint32), want_p.view(np.uint32)):
                            fails.append(f"partial payload rank {r}")
                        if not np.array_equal(lay[3].view(np.uint32), want_g.view(np.uint32)):
                            fails.append(f"grad payload rank {r}")
                        if not np.array_equal(lay[4], dump.mask[l]):
                            fails.append(f"owner mask rank {r}")
        st_prev = ([w.copy() for w in st.ws], [v.copy() for v in st.vs])
    woff, voff = spec.woff(), spec.voff()
    for r in range(world):
        g = r // N
        for f, (lo, hi, w, v) in gathered[r][2].items():
            D = int(dims[f])
            ww = st.ws[g][woff[f] + lo * D: woff[f] + hi * D].reshape(hi - lo, D)
            vv = st.vs[g][voff[f] + lo: voff[f] + hi]
            if not np.array_equal(w.view(np.uint32), ww.view(np.uint32)):
                fails.append(f"weights rank {r} table {f}: max|d|={np.max(np.abs(w - ww))}")
            if not np.array_equal(v.view(np.uint32), vv.view(np.uint32)):
                fails.append(f"moments rank {r} table {f}")
    if args.ckpt:
        # bytes of the mesh's checkpoint == the oracle's group-0 replica
        # written by the S2DCKPT1 restatement; every replica reloads it
        want_path = ckpt_path + ".oracle"
        port.save_checkpoint(want_path, rows, dims, st.ws[0], st.vs[0])
        if open(ckpt_path, "rb").read() != open(want_path, "rb").read():
            fails.append("checkpoint bytes")
        for r in range(world):
            for f, (lo, hi, w, v) in gathered[r][3].items():
                D = int(dims[f])
                ww = st.ws[0][woff[f] + lo * D: woff[f] + hi * D].reshape(hi - lo, D)
                vv = st.vs[0][voff[f] + lo: voff[f] + hi]
                if not (np.array_equal(w.view(np.uint32), ww.view(np.uint32))
                        and np.array_equal(v.view(np.uint32), vv.view(np.uint32))):
                    fails.append(f"checkpoint reload rank {r} table {f}")
    # which replica-sync path ran: the pair snapshot exchange (1) at M = 2,
    # the slice push / mean / scatter (2) otherwise or when the environment
    # forces it, NCCL (3) when forced
    want_mode = (3 if os.environ.get("S2D_SYNC_NCCL") == "1"
                 else 2 if os.environ.get("S2D_SYNC_SNAPSHOT") == "0" or M != 2 else 1)
    for r in range(world):
        if any(md not in (0, want_mode) for md in gathered[r][5]) or (M > 1 and want_mode not in gathered[r][5]):
            fails.append(f"rank {r} sync modes {gathered[r][5]} (want {want_mode})")
    # measured trace of the last step (reference trace.csv schema)
    last_sync = M > 1 and args.steps % args.sync_interval == 0
    for r in range(world):
        kinds = [t["kernel"] for t in gathered[r][4]]
        if kinds != ["lookup_a2a", "grad_a2a"] + (["table_allreduce"] if last_sync else []):
            fails.append(f"trace kernels rank {r}: {kinds}")
    if N > 1 and sum(t["bytes"] for r in range(world) for t in gathered[r][4] if t["kernel"] != "table_allreduce") == 0:
        fails.append("trace: no MP exchange bytes")
    if fails:
        print("MP PARITY FAIL", world, M, args.strategy, *fails[:20], sep="\n  ")
        dist.barrier()
        return 1
    print(f"MP PARITY OK T={world} M={M} N={N} {args.strategy} steps={args.steps} sgd={args.sgd} ckpt={args.ckpt}"
          + (" local" if hub is not None else ""))
    dist.barrier()
    return 0


def run_bad_id(eng, dist, rank, world, rows, dims, B):
    """An id >= rows (no bounds check in the reference's build_demand,
    trainer.cpp:293-299; std::out_of_range in pool_ids, embedding.cpp:61-63)
    must surface as IndexError (S2D_ERANGE) on the rank that detects it: the
    requester's bucketing for multi-owner tables, the owner's lookup for
    single-owner tables."""
    from cases import make_batch, upstream

    eng.set_strict(False)
    rng = np.random.default_rng([5, rank])
    lengths, ids = make_batch(rng, rows, B, max_len=9, zipf=1.1)
    if rank == 1:
        ids = ids.copy()
        ids[0] = rows[0] + 7  # bag (0, 0) belongs to table 0
    raised = 0
    try:
        eng.forward(lengths, ids)
        eng.backward_update(upstream(rng, B, int(dims.sum())))
        eng.synchronize()
    except IndexError:
        raised = 1
    flags = [None] * world
    dist.all_gather_object(flags, raised)
    if rank == 0:
        ok = sum(flags) >= 1
        print(("MP PARITY OK" if ok else "MP PARITY FAIL") + f" bad-id raised on ranks {flags}")
    dist.barrier()
    return 0 if sum(flags) >= 1 else 1


def _shards(eng, F):
    out = {}
    for f in range(F):
        lo, hi = eng.owned_range(f)
        if hi > lo:
            out[f] = (lo, hi) + eng.read_rows(f, lo, hi)
    return out


def run_bf16(args, eng, dist, rank, world, M, N, rows, dims, B, eta, c, plan):
    """bf16 storage has no reference path (embedding.hpp:16): every step the
    oracle is seeded from the mesh's bf16 weights (widened exactly) and must
    give bit-equal pooled outputs (f64 pooling of bf16 rows is exact), moments
    within 1e-5 and weights within 1e-2 relative after the step (one bf16
    rounding).  Sync every step (sync_interval = 1)."""
    from cases import make_batch, upstream
    from oracle import MeshSpec, MeshState, Oracle

    F = len(rows)
    port = Oracle("port") if rank == 0 else None
    plan_arr = np.array([[e["table_id"], e["row_lo"], e["row_hi"], e["local_rank"]] for e in plan], np.uint32)
    spec = MeshSpec(rows=rows, dims=dims, plan=plan_arr, T=world, M=M, B=B, eta=eta, c=c, sgd=False)
    woff, voff = spec.woff(), spec.voff()
    fails = []

    def assemble(gathered):  # per-group replicas from every rank's shards
        ws = [np.zeros(spec.replica_floats(), np.float32) for _ in range(M)]
        vs = [np.zeros(spec.replica_rows(), np.float32) for _ in range(M)]
        for r in range(world):
            g = r // N
            for f, (lo, hi, w, v) in gathered[r].items():
                D = int(dims[f])
                ws[g][woff[f] + lo * D: woff[f] + hi * D] = w.ravel()
                vs[g][voff[f] + lo: voff[f] + hi] = v
        return ws, vs

    def close(a, b, tol, atol=1e-30):
        a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
        return bool(np.all(np.abs(a - b) <= tol * np.maximum(np.abs(b), 1e-30) + atol))

    for step in range(args.steps):
        pre = [None] * world if rank == 0 else None
        dist.gather_object(_shards(eng, F), pre, dst=0)
        rng = np.random.default_rng([step, rank, 77])
        lengths, ids = make_batch(rng, rows, B, max_len=9, zipf=1.1)
        up = upstream(rng, B, int(dims.sum()))
        got = eng.forward(lengths, ids)
        eng.backward_update(up)
        if M > 1:
            eng.sync_replicas()
        ins = [None] * world if rank == 0 else None
        dist.gather_object((lengths, ids, up, got, _shards(eng, F)), ins, dst=0)
        if rank != 0:
            continue
        ws, vs = assemble(pre)
        st = MeshState(spec, ws, vs, [np.zeros(spec.replica_rows(), np.uint8) for _ in range(M)])
        want = st.step(port, [x[0] for x in ins], [x[1] for x in ins], [x[2] for x in ins], do_sync=M > 1)
        post_w, post_v = assemble([x[4] for x in ins])
        for r in range(world):
            if not np.array_equal(ins[r][3].view(np.uint32), want[r].view(np.uint32)):
                fails.append(f"bf16 pooled step {step} rank {r}")
        for g in range(M):
            if not close(post_v[g], st.vs[g], 1e-5):
                fails.append(f"bf16 moments step {step} group {g}")
            # the replica mean of two bf16-rounded rows can cancel (opposite
            # updates of a near-zero weight), so the relative bar gets an
            # absolute floor of one bf16 ulp at the table's RMS magnitude
            atol = 2.0 ** -8 * float(np.sqrt(np.mean(np.square(st.ws[g], dtype=np.float64))))
            if not close(post_w[g], st.ws[g], 1e-2, atol):
                d = np.abs(post_w[g].astype(np.float64) - st.ws[g])
                fails.append(f"bf16 weights step {step} group {g}: max|d|={d.max():.3g} atol={atol:.3g}")
    eng.close()
    if rank == 0:
        if fails:
            print("MP PARITY FAIL", world, M, "bf16", *fails[:20], sep="\n  ")
            dist.barrier()
            return 1
        print(f"MP PARITY OK T={world} M={M} N={N} bf16 steps={args.steps}")
    dist.barrier()
    return 0


if __name__ == "__main__":
    main()
