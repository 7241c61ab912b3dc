"""CPU, world_size 2 (gloo): the multi-rank wire protocol of the N > 1 step.

Each process plays one rank of an MP group and moves real payloads through
torch.distributed (gloo) using exactly the bookkeeping of the device path
(paper_2508_03854_b200/csrc/ctx.cu): per-owner dense bag lengths and id
blocks from K1, id offsets = exclusive scan of counts flattened [owner][bag],
entry float offsets = exclusive scan of (count > 0 ? dim : 0), blocks
concatenated by peer rank.  The received demand, the pooled-partial and
gradient payloads and the combined pooled output must equal the oracle's
(trainer.cpp:283-457 layouts) bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _a2a(dist, blocks):
    """all-to-all of per-destination numpy blocks over gloo (via all_gather)."""
    world = dist.get_world_size()
    got = [None] * world
    dist.all_gather_object(got, blocks)
    me = dist.get_rank()
    return [got[src][me] for src in range(world)]


def _worker(rank, world, port, strategy, out_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from cases import make_batch, upstream
    from oracle import MeshSpec, MeshState, Oracle, row_wise_plan

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        port_o = Oracle("port")
        N, B = world, 12
        rows = np.array([50, 9, 300, 4], np.uint32)
        dims = np.array([8, 4, 12, 8], np.uint32)
        F = len(rows)
        plan = row_wise_plan(rows, N) if strategy == "row-wise" else port_o.plan_greedy(
            [(f, 0, float(F - f), int(rows[f])) for f in range(F)], N)
        spec = MeshSpec(rows=rows, dims=dims, plan=plan, T=N, M=1, B=B, eta=0.1, c=1.0)
        batches = [make_batch(np.random.default_rng([r, 5]), rows, B, max_len=7) for r in range(N)]
        ups = [upstream(np.random.default_rng([r, 6]), B, int(dims.sum())) for r in range(N)]
        lengths, ids = batches[rank]
        BF = B * F

        def owner(f, i):
            for e in plan:
                if e[0] == f and e[1] <= i < e[2]:
                    return int(e[3])
            raise IndexError

        # ---- K1: counts, dense lengths per owner, id blocks (canonical order)
        cnt = np.zeros((N, BF), np.uint32)
        blocks = [[] for _ in range(N)]
        off = 0
        for b in range(BF):
            for i in ids[off:off + lengths[b]]:
                o = owner(b % F, int(i))
                cnt[o, b] += 1
                blocks[o].append(int(i))
            off += int(lengths[b])
        dimv = np.tile(dims, B)
        eoff_req = np.concatenate([[0], np.cumsum(np.where(cnt.ravel() > 0, np.tile(dimv, N), 0))]).astype(np.uint64)
        # ---- id + lengths all-to-all
        recv = _a2a(dist, [(cnt[o], np.array(blocks[o], np.uint32)) for o in range(N)])
        recv_len = np.stack([x[0] for x in recv])            # [N requester][BF]
        recv_ids = np.concatenate([x[1] for x in recv]).astype(np.uint32)
        # ---- oracle reference for this group
        st = MeshState.init(port_o, spec, 8)
        w0, v0 = st.ws[0].copy(), st.vs[0].copy()
        L = [x[0] for x in batches]
        I = [x[1] for x in batches]
        pooled_want, dump = port_o.group_step(spec, L, I, ups, w0, v0, None, want_dump=True)
        assert np.array_equal(recv_len.ravel(), dump.dem_len[rank].ravel()), "demand lengths"
        assert np.array_equal(recv_ids, dump.dem_ids[rank]), "demand ids"
        # ---- owner partials (f64 in occurrence order -> f32), entries in [n][bag] order
        own_idoff = np.concatenate([[0], np.cumsum(recv_len.ravel().astype(np.int64))]).astype(np.int64)
        woff = spec.woff()
        parts = []
        for n in range(N):
            blk = []
            for b in range(BF):
                k = n * BF + b
                cnt_nb = int(recv_len[n, b])
                if not cnt_nb:
                    continue
                f, D = b % F, int(dims[b % F])
                tbl = st.ws[0][woff[f]:woff[f + 1]]
                blk.append(port_o.pool_ids(tbl, D, [(0, int(rows[f]))],
                                           recv_ids[own_idoff[k]:own_idoff[k] + cnt_nb]))
            parts.append(np.concatenate(blk) if blk else np.zeros(0, np.float32))
        assert np.array_equal(np.concatenate(parts).view(np.uint32),
                              np.concatenate(dump.part[rank]).view(np.uint32)), "partial payload"
        # ---- C1 all-to-all + requester combine (ascending owner)
        precv = _a2a(dist, parts)
        recv_part = np.concatenate(precv)
        sumD = int(dims.sum())
        coff = np.concatenate([[0], np.cumsum(dims.astype(np.int64))]).astype(np.int64)
        pooled = np.zeros((B, sumD), np.float32)
        for b in range(BF):
            s, f = b // F, b % F
            acc = np.zeros(int(dims[f]), np.float64)
            for o in range(N):
                if cnt[o, b]:
                    e = int(eoff_req[o * BF + b])
                    acc += recv_part[e:e + int(dims[f])].astype(np.float64)
            pooled[s, coff[f]:coff[f + 1]] = acc.astype(np.float32)
        assert np.array_equal(pooled.view(np.uint32), pooled_want[rank].view(np.uint32)), "pooled"
        # ---- C2 send layout
        gsend = np.zeros(int(eoff_req[-1]), np.float32)
        for o in range(N):
            for b in range(BF):
                if cnt[o, b]:
                    s, f = b // F, b % F
                    e = int(eoff_req[o * BF + b])
                    gsend[e:e + int(dims[f])] = ups[rank][s, coff[f]:coff[f + 1]]
        assert np.array_equal(gsend.view(np.uint32), np.concatenate(dump.grad[rank]).view(np.uint32)), "grad payload"
        out_q.put((rank, "ok"))
    except Exception as e:  # surfaced to the parent
        out_q.put((rank, f"{type(e).__name__}: {e}"))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("strategy", ["row-wise", "table-wise"])
def test_two_rank_wire_protocol(strategy):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, strategy, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def _trace_worker(rank, world, port, out_q, N=None):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    import paper_2508_03854_b200 as s2d

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # per-rank measured rows as Sparse2DEmbedding.trace_rows returns them
        N = N or world
        mine = [{"step": 3, "kernel": k, "rank": rank, "group": rank // N, "local": rank % N,
                 "bytes": 100 * (rank + 1) + i, "latency_s": 1e-4 * (rank + 1)}
                for i, k in enumerate(("lookup_a2a", "grad_a2a", "table_allreduce"))]
        allrows = [None] * world
        dist.all_gather_object(allrows, mine)  # the gather bench.py --trace-csv does
        if rank == 0:
            out_q.put(s2d.traces_to_csv([r for rr in allrows for r in rr], "h"))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_trace_rows_gathered_over_ranks_gloo():
    """world_size 2 (gloo): rank 0 writes every rank's measured trace rows in
    the reference's per-collective, per-participant order
    (experiment.cpp:53-60)."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_trace_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    text = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    body = [l for l in text.splitlines() if not l.startswith("#")]
    assert body == ["step,kernel,rank,bytes,latency_s",
                    "3,lookup_a2a,0,100,0.0001", "3,lookup_a2a,1,200,0.0002",
                    "3,grad_a2a,0,101,0.0001", "3,grad_a2a,1,201,0.0002",
                    "3,table_allreduce,0,102,0.0001", "3,table_allreduce,1,202,0.0002"]


def test_trace_rows_2x2_mesh_table_allreduce_order_gloo():
    """world_size 4 as a 2x2 mesh (N = 2 ranks per MP group, M = 2 groups):
    the reference writes one table_allreduce trace per local rank o over its
    replicas rank_of(g, o) (trainer.cpp:598-610, topology.cpp:128-131), so
    the rows come in rank order 0, 2, 1, 3; the all-to-alls stay in rank order."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_trace_worker, args=(r, 4, port, q, 2)) for r in range(4)]
    for p in ps:
        p.start()
    text = q.get(timeout=180)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    body = [l for l in text.splitlines() if not l.startswith("#")]
    ranks = lambda k: [int(l.split(",")[2]) for l in body[1:] if l.split(",")[1] == k]
    assert ranks("lookup_a2a") == [0, 1, 2, 3]
    assert ranks("grad_a2a") == [0, 1, 2, 3]
    assert ranks("table_allreduce") == [0, 2, 1, 3]
