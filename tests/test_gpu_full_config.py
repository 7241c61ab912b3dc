"""Whole-step parity at BASELINE config shapes (not sampled): every pooled
element, the dedup (the exact set of updated rows), every row gradient and
every touched row's weights and moment after the step, against the CPU
oracle run on tables compacted to the rows the step touches (each row's
arithmetic is independent).

* cfg2: 26 Criteo tables (33.6M x 128 fp32), B = 16384, one GPU -- the
  compiled, unmodified reference (oracle/_ref) runs the compacted step.
* cfg4 shape: 2 tables x 200M rows x 128 bf16, row-wise over a 2x1 mesh of
  virtual ranks (one GPU); the oracle is seeded from the GPU's bf16 rows
  (widened exactly), 1e-2 on weights (one bf16 rounding), 1e-5 on moments.
* cfg5 shape: 500 tables, D 32..256, bag lengths 1..200, c = 4 on one GPU and
  c = 1 on a 2x1 table-wise mesh (B reduced to 512 per rank to bound the CPU
  oracle's time).

Numerics bar: pooled rows and row gradients of rows with at
most 128 contributions are bit-exact; hot rows (contributions re-associated
at fixed 128-item chunk boundaries) within 1e-5; weights / moments
bit-exact except where a tree-ordered |g|^2 or a re-associated hot-row sum
moves an f32 rounding (asserted: all within 1e-5, and the bit-exact share
reported and bounded below)."""
import os

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

K_CHUNK = 128


def _rel_ok(a, b, tol, atol=0.0):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return bool(np.all(np.abs(a - b) <= tol * np.abs(b) + atol))


def _compact(F, lengths_list, ids_list):
    """Per table: the sorted unique touched ids over all ranks, and every
    rank's ids remapped to compact indices (order preserved)."""
    keys = [(np.repeat(np.tile(np.arange(F, dtype=np.uint64), len(l) // F), l) << np.uint64(32))
            | x.astype(np.uint64) for l, x in zip(lengths_list, ids_list)]
    u, inv = np.unique(np.concatenate(keys), return_inverse=True)
    tab = (u >> np.uint64(32)).astype(np.int64)
    first = np.searchsorted(tab, np.arange(F + 1))
    uniq = [(u[first[f]:first[f + 1]] & np.uint64(0xffffffff)).astype(np.uint32) for f in range(F)]
    local = (np.arange(len(u)) - first[tab]).astype(np.uint32)
    cids, o = [], 0
    for k in keys:
        cids.append(local[inv[o:o + len(k)]])
        o += len(k)
    return uniq, cids


def _contrib_counts(F, lengths, ids):
    """(table << 32 | row) -> number of contributions, sorted by key."""
    feat = np.repeat(np.tile(np.arange(F, dtype=np.uint64), len(lengths) // F), lengths)
    k, c = np.unique((feat << np.uint64(32)) | ids.astype(np.uint64), return_counts=True)
    return k, c


def _oracle():
    from oracle import Oracle, reference_available

    return Oracle("reference") if reference_available() else Oracle("port")


def test_cfg2_full_batch_vs_reference(port):
    import paper_2508_03854_b200 as s2d
    from oracle import MeshSpec
    from paper_2508_03854_b200 import workloads

    seed = 11
    wl = workloads.get("cfg2")
    F, B, D = wl.F, wl.batch, 128
    rows = np.array(wl.rows, np.uint32)
    dims = np.array(wl.dims, np.uint32)
    eng = s2d.Sparse2DEmbedding([s2d.TableConfig(int(r), D) for r in rows], s2d.Topology(1, 1),
                                optimizer=s2d.OptimizerConfig(eta=wl.eta, eps=1e-8, c=wl.c))
    try:
        eng.init_tables(seed)
        eng.set_debug_grad(True)
        lengths, ids = wl.batch_for(seed, 0, 0)
        up = wl.upstream_for(seed, 0, 0)
        got = eng.forward(lengths, ids)
        eng.backward_update(up)
        eng.synchronize()
        urow, utab = eng.debug(5), eng.debug(8)
        g_gpu = eng.debug(7).reshape(len(urow), D)
        assert eng.stats()["unique_rows"] == len(urow)

        # dedup: exactly the touched (table, row) keys, in (table, row) order
        keys, g_ref = port.row_gradients(rows, dims, B, lengths, ids, up)
        kc, cnt = _contrib_counts(F, lengths, ids)
        assert np.array_equal(keys, kc)
        assert np.array_equal((utab.astype(np.uint64) << np.uint64(32)) | urow, keys)
        short = cnt <= K_CHUNK
        assert np.array_equal(g_gpu[short].view(np.uint64), g_ref[short].view(np.uint64)), "short-row gradients"
        assert _rel_ok(g_gpu[~short], g_ref[~short], 1e-5, 1e-300), "hot-row gradients"

        # the reference on the compacted step: pooled rows + updated rows
        uniq, cids = _compact(F, [lengths], [ids])
        crows = np.array([len(u) for u in uniq], np.uint32)
        w0 = np.concatenate([port.init_rows_list(f, uniq[f], D, seed).ravel() for f in range(F)])
        v0 = np.zeros(int(crows.sum()), np.float32)
        plan = np.array([[f, 0, int(crows[f]), 0] for f in range(F)], np.uint32)
        spec = MeshSpec(rows=crows, dims=dims, plan=plan, T=1, M=1, B=B, eta=wl.eta, c=wl.c)
        ref = _oracle()
        pooled, _ = ref.group_step(spec, [lengths], [cids[0]], [up], w0, v0, None, threads=os.cpu_count() or 1)
        assert np.array_equal(bits(got), bits(pooled[0])), "pooled rows (all %d elements)" % got.size

        woff = np.concatenate([[0], np.cumsum(crows.astype(np.int64) * D)])
        voff = np.concatenate([[0], np.cumsum(crows.astype(np.int64))])
        eq_w = eq_v = total = 0
        for f in range(F):
            w_gpu, v_gpu = eng.gather_rows(f, uniq[f])
            w_ref = w0[woff[f]:woff[f + 1]].reshape(-1, D)
            v_ref = v0[voff[f]:voff[f + 1]]
            assert _rel_ok(w_gpu, w_ref, 1e-5, 1e-30) and _rel_ok(v_gpu, v_ref, 1e-5, 1e-30), f
            eq_w += int(np.all(bits(w_gpu) == bits(w_ref), axis=1).sum())
            eq_v += int((bits(v_gpu) == bits(v_ref)).sum())
            total += len(uniq[f])
        print(f"cfg2 full step: {got.size} pooled elements bit-exact, {len(urow)} rows, "
              f"{int(short.sum())} short-row gradients bit-exact, rows bit-exact w {eq_w}/{total} v {eq_v}/{total}")
        assert eq_w >= total * (1 - 1e-3) and eq_v >= total * (1 - 1e-3)
    finally:
        eng.close()


def test_cfg4_shape_bf16_rowwise_200m_rows_2x1():
    """cfg4's table shape (200M-row bf16 tables, fp32 moments, row-wise, raw
    Zipf ids: the hot rows all land on rank 0) on a 2x1 mesh of virtual ranks;
    two tables (102 GB of bf16 weights) fit one GPU."""
    import paper_2508_03854_b200 as s2d
    from oracle import MeshSpec, Oracle
    from paper_2508_03854_b200 import workloads

    seed, T = 5, 2
    wl = workloads.get("cfg4", rows=[200_000_000] * 2, dims=[128] * 2, batch=8192)
    F, B, D = 2, wl.batch, 128
    rows = np.array(wl.rows, np.uint32)
    dims = np.array(wl.dims, np.uint32)
    tables = [s2d.TableConfig(int(r), D) for r in rows]
    engs = s2d.local_mesh(tables, s2d.Topology(T, 1), strategy="row-wise", weight_dtype="bf16",
                          optimizer=s2d.OptimizerConfig(eta=wl.eta, eps=1e-8, c=wl.c))
    try:
        s2d.run_ranks(lambda r: engs[r].init_tables(seed), T)
        ins = [wl.batch_for(seed, 0, r) for r in range(T)]
        ups = [wl.upstream_for(seed, 0, r) for r in range(T)]
        uniq, cids = _compact(F, [x[0] for x in ins], [x[1] for x in ins])
        crows = np.array([len(u) for u in uniq], np.uint32)

        def owned(r, f):
            lo, hi = engs[r].owned_range(f)
            return uniq[f][(uniq[f] >= lo) & (uniq[f] < hi)]

        # the GPU's initial bf16 rows (widened) seed the oracle's fp32 replica
        w0 = np.concatenate([np.concatenate([engs[r].gather_rows(f, owned(r, f))[0] for r in range(T)]).ravel()
                             for f in range(F)])
        v0 = np.zeros(int(crows.sum()), np.float32)
        plan = []
        for f in range(F):  # compact plan: rank r owns the compacted ids of its row range
            o = 0
            for r in range(T):
                k = len(owned(r, f))
                if k:
                    plan.append([f, o, o + k, r])
                o += k
        spec = MeshSpec(rows=crows, dims=dims, plan=np.array(plan, np.uint32), T=T, M=1, B=B, eta=wl.eta, c=wl.c)
        port = Oracle("port")
        want, _ = port.group_step(spec, [x[0] for x in ins], cids, ups, w0, v0, None)

        def go(r):
            out = engs[r].forward(ins[r][0], ins[r][1])
            engs[r].backward_update(ups[r])
            engs[r].synchronize()
            return out

        got = s2d.run_ranks(go, T)
        for r in range(T):
            assert np.array_equal(bits(got[r]), bits(want[r])), f"pooled rank {r}"
        woff = np.concatenate([[0], np.cumsum(crows.astype(np.int64) * D)])
        voff = np.concatenate([[0], np.cumsum(crows.astype(np.int64))])
        for f in range(F):
            w_gpu = np.concatenate([engs[r].gather_rows(f, owned(r, f))[0] for r in range(T)])
            v_gpu = np.concatenate([engs[r].gather_rows(f, owned(r, f))[1] for r in range(T)])
            w_ref = w0[woff[f]:woff[f + 1]].reshape(-1, D)
            atol = 2.0 ** -8 * float(np.sqrt(np.mean(np.square(w_ref, dtype=np.float64))))
            assert _rel_ok(w_gpu, w_ref, 1e-2, atol), f"bf16 weights table {f}"
            assert _rel_ok(v_gpu, v0[voff[f]:voff[f + 1]], 1e-5, 1e-30), f"moments table {f}"
        print(f"cfg4 shape: {sum(len(u) for u in uniq)} touched rows of 2 x 200M, rank-0 share of ids "
              f"{engs[0].stats()['nnz_owned'] / max(1, sum(e.stats()['nnz_owned'] for e in engs)):.3f}")
    finally:
        for e in engs:
            e.close()


@pytest.mark.parametrize("T,c", [(1, 4.0), (2, 1.0)])
def test_cfg5_shape_500_tables(T, c):
    """cfg5's tables (500 tables, rows 1e3..2e6, D 32..256, bag lengths
    power-law on [1, 200]) at B = 512 per rank: mixed dims through every
    kernel; c = 4 (moment-scaled) on one rank, c = 1 (plain row-wise AdaGrad)
    on a 2x1 table-wise mesh."""
    import paper_2508_03854_b200 as s2d
    from oracle import MeshSpec
    from paper_2508_03854_b200 import workloads

    seed = 21
    wl = workloads.get("cfg5", batch=512, c=c)
    F, B = wl.F, wl.batch
    rows = np.array(wl.rows, np.uint32)
    dims = np.array(wl.dims, np.uint32)
    tables = [s2d.TableConfig(int(r), int(d), 1.0) for r, d in zip(rows, dims)]
    opt = s2d.OptimizerConfig(eta=wl.eta, eps=1e-8, c=c)
    if T == 1:
        engs = [s2d.Sparse2DEmbedding(tables, s2d.Topology(1, 1), optimizer=opt)]
    else:
        engs = s2d.local_mesh(tables, s2d.Topology(T, 1), strategy="table-wise", optimizer=opt)
    try:
        s2d.run_ranks(lambda r: engs[r].init_tables(seed), T)
        ins = [wl.batch_for(seed, 0, r) for r in range(T)]
        ups = [wl.upstream_for(seed, 0, r) for r in range(T)]
        uniq, cids = _compact(F, [x[0] for x in ins], [x[1] for x in ins])
        crows = np.array([max(1, len(u)) for u in uniq], np.uint32)
        from oracle import Oracle

        port = Oracle("port")
        w0 = np.concatenate([port.init_rows_list(f, uniq[f], int(dims[f]), seed).ravel()
                             if len(uniq[f]) else np.zeros(int(dims[f]), np.float32) for f in range(F)])
        v0 = np.zeros(int(crows.sum()), np.float32)
        owner = {e["table_id"]: e["local_rank"] for e in engs[0].plan}
        plan = np.array([[f, 0, int(crows[f]), owner[f]] for f in range(F)], np.uint32)
        spec = MeshSpec(rows=crows, dims=dims, plan=plan, T=T, M=1, B=B, eta=wl.eta, c=c)
        want, _ = _oracle().group_step(spec, [x[0] for x in ins], cids, ups, w0, v0, None, threads=os.cpu_count() or 1)

        def go(r):
            out = engs[r].forward(ins[r][0], ins[r][1])
            engs[r].backward_update(ups[r])
            engs[r].synchronize()
            return out

        got = s2d.run_ranks(go, T)
        for r in range(T):
            assert np.array_equal(bits(got[r]), bits(want[r])), f"pooled rank {r}"
        woff = np.concatenate([[0], np.cumsum(crows.astype(np.int64) * dims)])
        voff = np.concatenate([[0], np.cumsum(crows.astype(np.int64))])
        eq = total = 0
        for f in range(F):
            if not len(uniq[f]):
                continue
            w_gpu, v_gpu = engs[owner[f]].gather_rows(f, uniq[f])
            w_ref = w0[woff[f]:woff[f + 1]].reshape(-1, int(dims[f]))
            v_ref = v0[voff[f]:voff[f] + len(uniq[f])]
            assert _rel_ok(w_gpu, w_ref, 1e-5, 1e-30) and _rel_ok(v_gpu, v_ref, 1e-5, 1e-30), f
            eq += int((np.all(bits(w_gpu) == bits(w_ref), axis=1) & (bits(v_gpu) == bits(v_ref))).sum())
            total += len(uniq[f])
        print(f"cfg5 shape T={T} c={c}: {sum(g.size for g in got)} pooled elements bit-exact, "
              f"rows bit-exact {eq}/{total}")
        assert eq >= total * (1 - 1e-3)
    finally:
        for e in engs:
            e.close()
