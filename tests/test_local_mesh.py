"""Single-process meshes (LocalHub virtual ranks on one GPU) driven directly
from pytest threads: host-side writes join the replica sync."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mesh(T, M, rows=(64, 40), dim=16):
    import paper_2508_03854_b200 as s2d

    tables = [s2d.TableConfig(r, dim) for r in rows]
    engs = s2d.local_mesh(tables, s2d.Topology(T, M), strategy="row-wise",
                          optimizer=s2d.OptimizerConfig(eta=0.1, eps=1e-8, c=float(M)))
    s2d.run_ranks(lambda r: engs[r].init_tables(5), T)
    return s2d, engs


def test_apply_row_updates_join_replica_sync():
    """apply_row_updates on one replica marks its rows dirty, so the next
    sync averages them (f32((w_0 + w_1) * 0.5), trainer.cpp:574-594) and the
    replicas agree again."""
    s2d, engs = _mesh(2, 2)
    try:
        w0, v0 = engs[0].read_rows(0, 0, 64)
        rows = np.array([3, 9, 3], np.uint32)
        delta = np.full((3, 16), 0.25, np.float64)
        engs[0].apply_row_updates(0, rows, delta, np.array([1.0, 2.0, 3.0]))
        s2d.run_ranks(lambda r: engs[r].sync_replicas(), 2)
        (wa, va), (wb, vb) = engs[0].read_rows(0, 0, 64), engs[1].read_rows(0, 0, 64)
        assert np.array_equal(wa.view(np.uint32), wb.view(np.uint32))
        assert np.array_equal(va.view(np.uint32), vb.view(np.uint32))
        w3 = np.float32(np.float32(w0[3] + 0.25) + 0.25)  # two updates of row 3 in call order (f64 adds)
        want = ((w3.astype(np.float64) + w0[3].astype(np.float64)) * 0.5).astype(np.float32)
        assert np.array_equal(wa[3].view(np.uint32), want.view(np.uint32))
        assert va[3] == np.float32((3.0 + 0.0) * 0.5) and va[9] == np.float32(1.0)
        untouched = [r for r in range(64) if r not in (3, 9)]
        assert np.array_equal(wa[untouched].view(np.uint32), w0[untouched].view(np.uint32))
    finally:
        for e in engs:
            e.close()


def test_shard_write_joins_replica_sync():
    s2d, engs = _mesh(2, 2)
    try:
        w0, v0 = engs[1].read_rows(1, 0, 40)
        engs[1].write_rows(1, 10, np.ones((2, 16), np.float32), np.full(2, 4.0, np.float32))
        s2d.run_ranks(lambda r: engs[r].sync_replicas(), 2)
        wa, va = engs[0].read_rows(1, 0, 40)
        wb, vb = engs[1].read_rows(1, 0, 40)
        assert np.array_equal(wa.view(np.uint32), wb.view(np.uint32))
        want = ((1.0 + w0[10:12].astype(np.float64)) * 0.5).astype(np.float32)
        assert np.array_equal(wa[10:12].view(np.uint32), want.view(np.uint32))
        assert np.all(va[10:12] == np.float32(2.0))
    finally:
        for e in engs:
            e.close()


def test_local_mesh_matches_oracle_2x1():
    """A 2x1 row-wise mesh driven in-process: pooled outputs and shards after
    two steps are bit-exact against the oracle."""
    from cases import make_batch, upstream
    from oracle import MeshSpec, MeshState, Oracle

    rows = np.array([64, 40], np.uint32)
    dims = np.array([16, 16], np.uint32)
    s2d, engs = _mesh(2, 1)
    try:
        port = Oracle("port")
        plan = np.array([[e["table_id"], e["row_lo"], e["row_hi"], e["local_rank"]] for e in engs[0].plan], np.uint32)
        spec = MeshSpec(rows=rows, dims=dims, plan=plan, T=2, M=1, B=8, eta=0.1, c=1.0)
        st = MeshState.init(port, spec, 5)
        for step in range(2):
            ins = []
            for r in range(2):
                rng = np.random.default_rng([step, r])
                ln, ids = make_batch(rng, rows, 8, max_len=5)
                ins.append((ln, ids, upstream(rng, 8, 32)))
            want = st.step(port, [x[0] for x in ins], [x[1] for x in ins], [x[2] for x in ins], do_sync=False)

            def go(r):
                out = engs[r].forward(ins[r][0], ins[r][1])
                engs[r].backward_update(ins[r][2])
                return out

            got = s2d.run_ranks(go, 2)
            for r in range(2):
                assert np.array_equal(got[r].view(np.uint32), want[r].view(np.uint32)), (step, r)
        off = spec.woff()
        for r in range(2):
            for f in range(2):
                lo, hi = engs[r].owned_range(f)
                w, _ = engs[r].read_rows(f, lo, hi)
                ref = st.ws[0][off[f]:off[f + 1]].reshape(int(rows[f]), 16)[lo:hi]
                assert np.array_equal(w.view(np.uint32), ref.view(np.uint32)), (r, f)
    finally:
        for e in engs:
            e.close()


def test_metrics_row_over_mp_group_shards():
    """MetricsRow is collective over the MP group: a 2x1 row-wise mesh gives
    the same statistics as the oracle on the whole replica."""
    from cases import make_batch, upstream
    from oracle import MeshSpec, MeshState, Oracle

    rows = np.array([64, 40], np.uint32)
    s2d, engs = _mesh(2, 1)
    try:
        port = Oracle("port")
        plan = np.array([[e["table_id"], e["row_lo"], e["row_hi"], e["local_rank"]] for e in engs[0].plan], np.uint32)
        spec = MeshSpec(rows=rows, dims=np.array([16, 16], np.uint32), plan=plan, T=2, M=1, B=8, eta=0.1, c=1.0)
        st = MeshState.init(port, spec, 5)
        ins = []
        for r in range(2):
            rng = np.random.default_rng([9, r])
            ln, ids = make_batch(rng, rows, 8, max_len=5)
            ins.append((ln, ids, upstream(rng, 8, 32)))
        st.step(port, [x[0] for x in ins], [x[1] for x in ins], [x[2] for x in ins], do_sync=False)

        def go(r):
            engs[r].forward(ins[r][0], ins[r][1])
            engs[r].backward_update(ins[r][2])
            return engs[r].metrics_row()

        got = s2d.run_ranks(go, 2)
        want = port.metrics_row(st.vs[0], eta=0.1, eps=1e-8, c=1.0)
        for g in got:
            assert g["eff_lr_p50"] == want["eff_lr_p50"] and g["eff_lr_p99"] == want["eff_lr_p99"]
            assert abs(g["v_mean"] - want["v_mean"]) <= 1e-12 * abs(want["v_mean"])
    finally:
        for e in engs:
            e.close()


TRAINER_MESHES = [
    dict(T=1, M=1, steps=5),
    dict(T=4, M=1),
    dict(T=4, M=2),
    dict(T=8, M=2, strategy="table-wise", sync_interval=3, steps=6),
    dict(T=4, M=2, sgd=True, sync_interval=2),
    dict(T=6, M=3, rows=50, dim=12, L=5),
]


@pytest.mark.parametrize("mesh", TRAINER_MESHES, ids=[str(m) for m in TRAINER_MESHES])
def test_gpu_mesh_matches_real_reference_trainer(mesh):
    """End to end against the REAL reference Trainer (trainer.cpp in
    oracle/_ref): its training loop, restated on the public API and pinned
    bitwise to Trainer::replica_tables (tests/test_oracle.py), records every
    step's per-rank batch and the f32 gradient its MLP sends back; the same
    T-rank mesh on the GPU (virtual ranks, one B200) consumes those inputs.
    Every pooled output of every step and every replica after the last step
    are bitwise equal to the reference's (acceptance criterion 1 shape,
    tests/acceptance/main.cpp:95-125, for M = 1 and the 2D meshes)."""
    import paper_2508_03854_b200 as s2d
    from oracle import reference_available, reference_trainer, restated_trainer, trainer_options

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    o = trainer_options(**mesh)
    ws_real, vs_real, plan = reference_trainer(o)
    _, _, ln, ids, up, pooled = restated_trainer(o)
    N = o.T // o.M
    tables = [s2d.TableConfig(o.rows, o.dim) for _ in range(o.F)]
    plan_d = [dict(table_id=int(e[0]), row_lo=int(e[1]), row_hi=int(e[2]), local_rank=int(e[3])) for e in plan]
    opt = s2d.OptimizerConfig(eta=o.eta, eps=o.eps, c=o.c, variant="sgd" if o.sgd else "rowwise-adagrad")
    engs = s2d.local_mesh(tables, s2d.Topology(o.T, o.M), plan=plan_d, optimizer=opt)
    try:
        s2d.run_ranks(lambda r: engs[r].init_tables(o.init_seed), o.T)

        def step(r, k):
            got = engs[r].forward(ln[k, r], ids[k, r])
            engs[r].backward_update(up[k, r])
            if o.M > 1 and (k + 1) % o.sync_interval == 0:
                engs[r].sync_replicas()
            return got

        for k in range(o.steps):
            got = s2d.run_ranks(lambda r: step(r, k), o.T)
            for r in range(o.T):
                assert np.array_equal(got[r].view(np.uint32), pooled[k, r].view(np.uint32)), (k, r)
        for r in range(o.T):
            g = r // N
            for f in range(o.F):
                lo, hi = engs[r].owned_range(f)
                if hi <= lo:
                    continue
                w, v = engs[r].read_rows(f, lo, hi)
                wr = ws_real[g][f * o.rows * o.dim:(f + 1) * o.rows * o.dim].reshape(o.rows, o.dim)[lo:hi]
                vr = vs_real[g][f * o.rows:(f + 1) * o.rows][lo:hi]
                assert np.array_equal(w.view(np.uint32), wr.view(np.uint32)), (r, f)
                assert np.array_equal(v.view(np.uint32), vr.view(np.uint32)), (r, f)
    finally:
        for e in engs:
            e.close()


FACADE_MESHES = [dict(T=1, M=1, steps=5), dict(T=4, M=2), dict(T=8, M=2, strategy="table-wise", sync_interval=3,
                                                                  steps=6), dict(T=4, M=2, sgd=True, sync_interval=2)]


@pytest.mark.parametrize("mesh", FACADE_MESHES, ids=[str(m) for m in FACADE_MESHES])
def test_trainer_facade_matches_real_reference_trainer(mesh):
    """The Trainer facade (s2d_trainer_*: device DataGenerator ids, plan_greedy
    over profile_from_spec, internal (step+1) % sync_interval cadence) with the
    dense model's gradient supplied through the upstream callback -- here the
    f32 gradient the reference's MLP produced, recorded by the pinned restated
    loop -- reproduces the REAL reference Trainer: same plan, the same batch
    and pooled rows at every step and rank, and every replica bitwise after
    run()."""
    import torch

    import paper_2508_03854_b200 as s2d
    from oracle import reference_available, reference_trainer, restated_trainer, trainer_options

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    o = trainer_options(**mesh)
    ws_real, vs_real, plan_real = reference_trainer(o)
    _, _, ln, _, up, pooled = restated_trainer(o)
    tr = s2d.Trainer(s2d.TrainerOptions(
        total_ranks=o.T, groups=o.M, num_tables=o.F, rows_per_table=o.rows, dim=o.dim,
        strategy="row-wise" if o.strategy else "table-wise", zipf_exponent=o.zipf, ids_per_sample=o.ids_per_sample,
        per_rank_batch=o.B, steps=o.steps, sync_interval=o.sync_interval, data_seed=o.data_seed,
        init_seed=o.init_seed, optimizer=s2d.OptimizerConfig(o.eta, o.eps, o.c, "sgd" if o.sgd else "rowwise-adagrad"),
        devices=[0]))
    try:
        seen = {}

        def fn(rank, step, lengths, pooled_t, up_t):
            seen[(rank, step)] = (np.array_equal(lengths.cpu().numpy().view(np.uint32), ln[step, rank])
                                  and np.array_equal(pooled_t.cpu().numpy().view(np.uint32),
                                                     pooled[step, rank].view(np.uint32)))
            up_t.copy_(torch.from_numpy(up[step, rank]).to(up_t.device))

        tr.set_upstream(fn)
        tr.run()
        assert tr.steps_done == o.steps
        assert len(seen) == o.T * o.steps and all(seen.values()), [k for k, v in seen.items() if not v][:5]
        got_plan = sorted((e["table_id"], e["row_lo"], e["row_hi"], e["local_rank"]) for e in tr.plan())
        assert got_plan == sorted(tuple(int(x) for x in e) for e in plan_real)
        for g in range(o.M):
            for f, (w, v) in enumerate(tr.replica_tables(g)):
                wr = ws_real[g][f * o.rows * o.dim:(f + 1) * o.rows * o.dim].reshape(o.rows, o.dim)
                assert np.array_equal(w.view(np.uint32), wr.view(np.uint32)), (g, f)
                assert np.array_equal(v.view(np.uint32), vs_real[g][f * o.rows:(f + 1) * o.rows].view(np.uint32))
    finally:
        tr.close()


def test_trainer_facade_default_upstream_checkpoint_metrics(tmp_path, port):
    """Without a callback the facade trains on the synthetic upstream
    (s2d_gen_upstream, equal to the oracle's or_synthetic_upstream); the
    replicas agree after a sync step, the S2DCKPT1 save / load round trip
    restores them, and MetricsRow comes from group 0."""
    import paper_2508_03854_b200 as s2d

    opts = s2d.TrainerOptions(total_ranks=4, groups=2, num_tables=3, rows_per_table=200, dim=16, ids_per_sample=4,
                              per_rank_batch=32, steps=3, optimizer=s2d.OptimizerConfig(eta=0.1, c=2.0),
                              devices=[0], dense_model=False)
    tr = s2d.Trainer(opts)
    try:
        tr.run()
        t0, t1 = tr.replica_tables(0), tr.replica_tables(1)
        for (w0, v0), (w1, v1) in zip(t0, t1):
            assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
            assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))
        assert any(np.any(v > 0) for _, v in t0)
        m = tr.metrics_row()
        assert m["rows"] == 600 and m["eff_lr_p50"] <= m["eff_lr_p99"]  # ascending lr percentiles
        path = str(tmp_path / "t.ckpt")
        tr.save_tables(path)
        tr.step_n(2)
        tr.load_tables(path)
        for (w0, v0), (w1, v1) in zip(t0, tr.tables()):
            assert np.array_equal(w0.view(np.uint32), w1.view(np.uint32))
    finally:
        tr.close()
    eng = s2d.Sparse2DEmbedding([s2d.TableConfig(10, 12), s2d.TableConfig(7, 4)], s2d.Topology(1, 1))
    try:
        got = eng.gen_upstream(9, 4, 3, 17)
        want = port.synthetic_upstream(9, 4, 3, 17, np.array([12, 4], np.uint32))
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    finally:
        eng.close()


DENSE_MESHES = [dict(T=1, M=1, steps=5), dict(T=4, M=2), dict(T=4, M=2, all_gpus=True),
                dict(T=4, M=1, strategy="table-wise", B=16),
                dict(T=4, M=2, sgd=True, sync_interval=2), dict(T=6, M=3, rows=50, dim=12, L=5, dense_hidden=9,
                                                                over_hidden=33, dense_dim=7)]


@pytest.mark.parametrize("mesh", DENSE_MESHES, ids=[str(m) for m in DENSE_MESHES])
def test_trainer_dense_model_matches_real_reference_trainer(mesh):
    """The Trainer facade with its own dense model (the toy DLRM MLPs on the
    device, dense.h: DataGenerator dense features + labels, forward, loss,
    backward, the dense DP step) against the REAL reference Trainer with
    ITS MLPs (trainer.cpp + model.cpp in oracle/_ref, nothing replayed):
    every rank's MLP parameters and every replica after the last step are
    bitwise equal; every step's MetricsRow (global-batch loss, NE of the
    eval set, effective-lr percentiles, mean moment) agrees."""
    import paper_2508_03854_b200 as s2d
    from oracle import reference_available, reference_trainer_model, trainer_options

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    mesh = dict(mesh)
    devices = None if mesh.pop("all_gpus", False) else [0]  # None: ranks round-robin over every GPU
    o = trainer_options(**mesh)
    ws_real, vs_real, model_real, rows_real = reference_trainer_model(o)
    tr = s2d.Trainer(s2d.TrainerOptions(
        total_ranks=o.T, groups=o.M, num_tables=o.F, rows_per_table=o.rows, dim=o.dim,
        strategy="row-wise" if o.strategy else "table-wise", zipf_exponent=o.zipf, ids_per_sample=o.ids_per_sample,
        per_rank_batch=o.B, steps=o.steps, sync_interval=o.sync_interval, data_seed=o.data_seed,
        init_seed=o.init_seed, optimizer=s2d.OptimizerConfig(o.eta, o.eps, o.c, "sgd" if o.sgd else "rowwise-adagrad"),
        devices=devices, dense_model=True, dense_dim=o.dense_dim, dense_hidden=o.dense_hidden,
        over_hidden=o.over_hidden, eval_cadence=1, eval_samples=512, eval_seed=o.eval_seed))
    try:
        losses = []
        for _ in range(o.steps):
            tr.step_n(1)
            losses.append(tr.last_loss)
        # the loss is -log(p) (trainer.cpp:412): CUDA's log may round 1 ulp
        # away from the host libm's; it feeds nothing downstream
        np.testing.assert_allclose(np.array(losses), rows_real[:, 1], rtol=1e-15, atol=0)
        # MetricsRow per step: NE of the eval set (lane kEval, pooled from
        # group 0's replica with rank 0's MLPs; CUDA exp in the sigmoid),
        # the exact effective-lr percentiles, v_mean (blocked f64 sum)
        rows = tr.metrics()
        assert [r["step"] for r in rows] == list(range(1, o.steps + 1))
        got = np.array([[r["loss"], r["ne"], r["eff_lr_p50"], r["eff_lr_p99"], r["v_mean"]] for r in rows])
        np.testing.assert_allclose(got[:, 0], rows_real[:, 1], rtol=1e-15, atol=0)
        np.testing.assert_allclose(got[:, 1], rows_real[:, 2], rtol=1e-13, atol=0)
        np.testing.assert_array_equal(got[:, 2:4], rows_real[:, 3:5])
        np.testing.assert_allclose(got[:, 4], rows_real[:, 5], rtol=1e-12, atol=0)
        fin = tr.finalize()["final_ne"]
        assert fin["ne"] == rows[-1]["ne"] and fin["eval_samples"] == 512
        for r in range(o.T):
            got = tr.rank_model(r)
            for name in ("dense_arch", "over_arch"):
                for a, b in zip(got[name], model_real[name]):
                    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (r, name)
        for g in range(o.M):
            for f, (w, v) in enumerate(tr.replica_tables(g)):
                wr = ws_real[g][f * o.rows * o.dim:(f + 1) * o.rows * o.dim].reshape(o.rows, o.dim)
                assert np.array_equal(w.view(np.uint32), wr.view(np.uint32)), (g, f)
                assert np.array_equal(v.view(np.uint32), vs_real[g][f * o.rows:(f + 1) * o.rows].view(np.uint32))
    finally:
        tr.close()


def test_train_toy_matches_reference_module():
    """train_toy (the reference module's run_train entry point,
    tests/python/test_smoke.py:62-90): the same config through the device
    Trainer + dense model and through the REAL reference run_train gives the
    same final NE, baseline CTR and config hash; reruns are deterministic."""
    import paper_2508_03854_b200 as s2d
    from oracle import reference_available, reference_train_toy

    cfg = {"topology.total_ranks": "4", "topology.groups": "2", "data.tables": "2", "data.rows_per_table": "64",
           "model.dim": "8", "model.dense_hidden": "4", "model.over_hidden": "8", "run.steps": "20",
           "run.eval_samples": "256", "run.seed": "3"}
    res = s2d.train_toy(cfg)
    assert 0.0 < res["final_ne"] < 2.0 and res["qps_sim"] > 0.0
    assert s2d.train_toy(cfg)["final_ne"] == res["final_ne"]
    assert len(res["metrics"]) == 1 and res["metrics"][0]["step"] == 20
    if not reference_available():
        pytest.skip("oracle/_ref not built")
    ref = reference_train_toy(cfg)
    assert res["config_hash"] == ref["config_hash"]
    assert res["baseline_ctr"] == ref["baseline_ctr"]
    assert abs(res["final_ne"] - ref["final_ne"]) <= 1e-12 * abs(ref["final_ne"])
