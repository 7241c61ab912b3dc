"""CPU: pins the oracle (oracle/s2d_oracle.c) to the reference.

(1) the reference's own known-answer tests, restated (test_embedding.cpp,
test_optimizer.cpp, test_planner.cpp); (2) golden vectors produced by the
compiled reference (tests/golden/make_golden.py); (3) when oracle/_ref is
built, randomized port-vs-reference agreement."""
import hashlib
import os

import numpy as np
import pytest

from conftest import bits

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name + ".npz"))


# ---- (1) reference known answers ---------------------------------------------

def test_pooling_known_answers(port):
    w = np.array([1, 0, 0, 2], np.float32)  # r0=(1,0), r1=(0,2): test_embedding.cpp:26-86
    assert list(port.pool_ids(w, 2, [(0, 2)], [1])) == [0.0, 2.0]
    assert list(port.pool_ids(w, 2, [(0, 2)], [1, 1])) == [0.0, 4.0]
    assert list(port.pool_ids(w, 2, [(0, 2)], [0, 1])) == [1.0, 2.0]
    assert list(port.pool_ids(w, 2, [(0, 2)], [])) == [0.0, 0.0]
    with pytest.raises(IndexError):
        port.pool_ids(w, 2, [(0, 2)], [7])


def test_pooling_linearity_and_sharding(port):
    t = port.init_rows(0, 40, 0, 40, 8, 5).ravel()
    ids = [1, 5, 5, 17, 39]
    a = port.pool_ids(t, 8, [(0, 40)], ids)
    b = port.pool_ids(2 * t, 8, [(0, 40)], ids)
    assert np.array_equal(b, 2 * a)  # test_embedding.cpp:88-98 (x2 exact)
    t = port.init_rows(0, 100, 0, 100, 4, 19).ravel()
    ids = [0, 29, 30, 70, 71, 99, 29]
    whole = port.pool_ids(t, 4, [(0, 100)], ids)
    split = port.pool_ids(t, 4, [(0, 30), (30, 71), (71, 100)], ids)
    assert np.allclose(whole, split, rtol=1e-6)  # 110-121


def test_adagrad_known_answers(port):
    o = port.adagrad_row_step([1, 1], 0.0, [2, 0], eta=0.1, eps=1e-8, c=4.0)  # test_optimizer.cpp:57-67
    assert abs(o["v"] - 4.0) < 1e-6 and abs(o["effective_lr"] - 0.1) < 1e-6
    assert abs(o["w"][0] - 0.8) < 1e-6 and o["w"][1] == 1.0
    o = port.adagrad_row_step([1, 1], 0.0, [2, 0], eta=0.1, eps=1e-8, c=1.0)  # 69-77
    assert abs(o["effective_lr"] - 0.05) < 1e-6 and abs(o["w"][0] - 0.9) < 1e-6
    o = port.adagrad_row_step([0.25, -0.5], 3.0, [0, 0], c=1.0)  # 79-87
    assert o["v"] == np.float32(3.0) and list(o["w"]) == [0.25, -0.5]
    with pytest.raises(ValueError):  # 89-94
        port.adagrad_row_step([0.0], 0.0, [float("nan")])
    assert port.effective_lr(4.0, eta=0.1, eps=1e-8, c=4.0) == pytest.approx(0.1, rel=1e-6)


def test_planner_known_answers(port):
    plan = port.plan_greedy([(i, 6400, float(x), 100) for i, x in enumerate([7, 5, 4, 3, 1])], 2)
    assert [int(e[3]) for e in plan] == [0, 1, 1, 0, 1]  # test_planner.cpp:60-79
    plan = port.plan_greedy([(0, 640, 5.0, 10), (1, 640, 2.0, 10)], 3, "row-wise")
    t0 = [tuple(int(x) for x in e) for e in plan if e[0] == 0]
    assert t0 == [(0, 0, 3, 0), (0, 3, 6, 1), (0, 6, 10, 2)]  # 81-91


# ---- (2) golden vectors from the compiled reference ---------------------------

def test_known_golden(port):
    g = load("known")
    w = np.array([1, 0, 0, 2], np.float32)
    for k, ids in {"single": [1], "dup": [1, 1], "two": [0, 1], "empty": []}.items():
        assert np.array_equal(bits(port.pool_ids(w, 2, [(0, 2)], ids)), bits(g[f"pool_{k}"]))
    t = port.init_rows(0, 100, 0, 100, 4, 19).ravel()
    ids = [0, 29, 30, 70, 71, 99, 29]
    assert np.array_equal(bits(port.pool_ids(t, 4, [(0, 100)], ids)), bits(g["shard_whole"]))
    assert np.array_equal(bits(port.pool_ids(t, 4, [(0, 30), (30, 71), (71, 100)], ids)), bits(g["shard_split"]))
    for c in (4, 1):
        o = port.adagrad_row_step([1.0, 1.0], 0.0, [2.0, 0.0], eta=0.1, eps=1e-8, c=float(c))
        assert np.array_equal(bits(o["w"]), bits(g[f"adagrad_c{c}_w"]))
        assert np.float32(o["v"]) == g[f"adagrad_c{c}_v"]
        assert o["effective_lr"] == g[f"adagrad_c{c}_lr"]
    for i in range(64):
        o = port.adagrad_row_step(g["rows_w"][i], g["rows_v"][i], g["rows_g"][i], eta=0.1, eps=1e-8, c=3.0)
        assert np.array_equal(bits(o["w"]), bits(g["rows_w_out"][i]))
        assert np.float32(o["v"]) == g["rows_v_out"][i]
    assert np.array_equal(port.plan_greedy([(i, 6400, float(x), 100) for i, x in enumerate([7, 5, 4, 3, 1])], 2),
                          g["lpt_plan"])
    assert np.array_equal(port.plan_greedy([(0, 640, 5.0, 10), (1, 640, 2.0, 10)], 3, "row-wise"),
                          g["rowwise_plan"])


def test_init_golden(port):
    g = load("init")
    assert np.array_equal(bits(port.init_rows(3, 100, 0, 100, 16, 11)), bits(g["t3"]))
    assert np.array_equal(bits(port.init_rows(0, 1000, 0, 1000, 64, 2)), bits(g["t0"]))
    assert np.array_equal(bits(port.init_rows(7, 5, 0, 5, 128, 123456789)), bits(g["t7"]))


@pytest.mark.parametrize("name", ["mesh_8x1_row", "mesh_4x2_row", "mesh_2x4_table", "mesh_2x2_sgd_sync3"])
def test_mesh_golden(port, name):
    from oracle import MeshSpec, MeshState

    g = load(name)
    T, M, B = int(g["T"]), int(g["M"]), int(g["B"])
    spec = MeshSpec(rows=g["rows"], dims=g["dims"], plan=g["plan"], T=T, M=M, B=B, eta=float(g["eta"]),
                    c=float(g["c"]), sgd=bool(g["sgd"]))
    st = MeshState.init(port, spec, int(g["seed"]))
    F = spec.F
    for step in range(int(g["steps"])):
        ids = [g[f"s{step}_r{r}_ids"] for r in range(T)]
        lengths = [np.full(B * F, len(ids[r]) // (B * F), np.uint32) for r in range(T)]
        up = [g[f"s{step}_r{r}_up"] for r in range(T)]
        pooled = st.step(port, lengths, ids, up, do_sync=(M > 1 and (step + 1) % int(g["sync_interval"]) == 0))
        for r in range(T):
            assert np.array_equal(bits(pooled[r]), bits(g[f"s{step}_r{r}_pooled"])), (step, r)
    for gg in range(M):
        assert np.array_equal(bits(st.ws[gg]), bits(g[f"w{gg}"]))
        assert np.array_equal(bits(st.vs[gg]), bits(g[f"v{gg}"]))
    if M > 1 and int(g["sync_interval"]) == 1:  # replica consensus (test_trainer.cpp:141-151)
        for gg in range(1, M):
            assert np.array_equal(bits(st.ws[gg]), bits(st.ws[0]))


def test_mixed_golden(port):
    from oracle import MeshSpec, MeshState, row_wise_plan

    g = load("mixed")
    spec = MeshSpec(rows=g["rows"], dims=g["dims"], plan=row_wise_plan(g["rows"], 2), T=2, M=1, B=16, eta=0.1,
                    c=2.0)
    st = MeshState.init(port, spec, 4)
    for step in range(3):
        L = [g[f"s{step}_r{r}_len"] for r in range(2)]
        I = [g[f"s{step}_r{r}_ids"] for r in range(2)]
        U = [g[f"s{step}_r{r}_up"] for r in range(2)]
        pooled = st.step(port, L, I, U, do_sync=False)
        for r in range(2):
            assert np.array_equal(bits(pooled[r]), bits(g[f"s{step}_r{r}_pooled"]))
    assert np.array_equal(bits(st.ws[0]), bits(g["w"]))
    assert np.array_equal(bits(st.vs[0]), bits(g["v"]))


@pytest.mark.parametrize("c", [1, 4])
def test_cfg1_golden(port, c):
    """BASELINE config 1 shapes: 2 steps of 8 x 100K x 64, B=512, L=20."""
    from oracle import MeshSpec, MeshState, row_wise_plan

    g = load(f"cfg1_c{c}")
    rows = np.full(8, 100_000, np.uint32)
    spec = MeshSpec(rows=rows, dims=np.full(8, 64, np.uint32), plan=row_wise_plan(rows, 1), T=1, M=1, B=512,
                    eta=0.1, c=float(c))
    st = MeshState.init(port, spec, 2)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    for step in range(2):
        up = (1e-3 * np.random.default_rng([step, 99]).standard_normal((512, 512))).astype(np.float32)
        pooled = st.step(port, [np.full(512 * 8, 20, np.uint32)], [g[f"s{step}_ids"]], [up], do_sync=False)[0]
        assert sha(pooled) == str(g[f"s{step}_pooled_sha"])
    assert sha(st.ws[0]) == str(g["w_sha"])
    assert sha(st.vs[0]) == str(g["v_sha"])


# ---- (3) port vs compiled reference on random meshes --------------------------

@pytest.mark.parametrize("T,M,strategy,sgd", [(8, 1, "row-wise", False), (8, 2, "table-wise", False),
                                              (8, 4, "row-wise", True), (6, 3, "row-wise", False)])
def test_port_matches_reference(port, ref, T, M, strategy, sgd):
    from cases import make_batch
    from oracle import MeshSpec, MeshState, row_wise_plan

    rng = np.random.default_rng(T * 10 + M)
    rows = np.array([64, 33, 7, 100, 1], np.uint32)
    dims = np.array([8, 4, 12, 8, 4], np.uint32)
    N = T // M
    plan = row_wise_plan(rows, N) if strategy == "row-wise" else port.plan_greedy(
        [(f, 0, float(9 - f), int(rows[f])) for f in range(5)], N)
    spec = MeshSpec(rows=rows, dims=dims, plan=plan, T=T, M=M, B=5, eta=0.05, c=float(M), sgd=sgd)
    a, b = MeshState.init(port, spec, 3), MeshState.init(ref, spec, 3)
    for step in range(4):
        batches = [make_batch(rng, rows, 5, max_len=6) for _ in range(T)]
        L = [x[0] for x in batches]
        I = [x[1] for x in batches]
        U = [(1e-2 * rng.standard_normal((5, int(dims.sum())))).astype(np.float32) for _ in range(T)]
        pa = a.step(port, L, I, U, True)
        pb = b.step(ref, L, I, U, True, threads=3)
        for x, y in zip(pa, pb):
            assert np.array_equal(bits(x), bits(y))
    for g in range(M):
        assert np.array_equal(bits(a.ws[g]), bits(b.ws[g]))
        assert np.array_equal(bits(a.vs[g]), bits(b.vs[g]))


def test_checkpoint_format_port_vs_reference(port, ref, tmp_path):
    """S2DCKPT1 writer restated in the port is byte-identical to the
    reference's save_checkpoint (embedding.cpp:133-185) and the reference's
    load_checkpoint reads it back (187-219)."""
    from oracle import read_checkpoint

    rng = np.random.default_rng(3)
    rows = np.array([7, 1, 300, 64], np.uint32)
    dims = np.array([4, 8, 64, 128], np.uint32)
    w = rng.standard_normal(int((rows.astype(np.uint64) * dims).sum())).astype(np.float32)
    v = rng.random(int(rows.sum())).astype(np.float32)
    a, b = str(tmp_path / "port.ckpt"), str(tmp_path / "ref.ckpt")
    port.save_checkpoint(a, rows, dims, w, v)
    ref.save_checkpoint(b, rows, dims, w, v)
    assert open(a, "rb").read() == open(b, "rb").read()
    assert not os.path.exists(a + ".tmp")
    tables, w2, v2 = read_checkpoint(a)
    assert tables == [(1, f, int(rows[f]), int(dims[f])) for f in range(len(rows))]
    assert np.array_equal(bits(w2), bits(w)) and np.array_equal(bits(v2), bits(v))
    w3, v3 = ref.load_checkpoint(a, rows, dims)
    assert np.array_equal(bits(w3), bits(w)) and np.array_equal(bits(v3), bits(v))
    with pytest.raises(RuntimeError):
        ref.load_checkpoint(a, rows[:2], dims[:2])  # table count mismatch


def test_gen_batch_ids_port_vs_reference(port, ref):
    """DataGenerator ids (data.cpp:85-136) restated in the port equal the
    reference generator's, per-table rows / exponents / pooling."""
    rows, zipf, L = [100, 3, 5000, 1, 70000], [1.0, 1.2, 0.8, 0.0, 1.05], [5, 2, 20, 1, 11]
    for seed, step, rank in ((7, 3, 1), (0, 0, 0), (12345, 9, 6)):
        a = port.gen_batch_ids(seed, step, rank, len(rows), rows, zipf, L, 48)
        b = ref.gen_batch_ids(seed, step, rank, len(rows), rows, zipf, L, 48)
        assert np.array_equal(a, b)


@pytest.mark.parametrize("kind", ["port", "reference"])
def test_apply_row_update_known_answers(kind):
    """proj/tests/test_embedding.cpp:123-165 on init_table(0, 10, 4, 3)."""
    from oracle import Oracle, reference_available

    if kind == "reference" and not reference_available():
        pytest.skip("oracle/_ref not built")
    o = Oracle(kind)
    w0 = o.init_rows(0, 10, 0, 10, 4, 3).reshape(10, 4).copy()
    v0 = np.zeros(10, np.float32)
    w, v = w0.copy(), v0.copy()
    o.apply_row_update(w, v, 4, (0, 10), 3, [0.0] * 4, float(v[3]))
    assert np.array_equal(w, w0) and np.array_equal(v, v0)
    o.apply_row_update(w, v, 4, (0, 10), 3, [0.5, -0.5, 0.25, 0.0], 2.0)
    keep = np.arange(10) != 3
    assert np.array_equal(w[keep], w0[keep]) and np.array_equal(v[keep], v0[keep])
    assert v[3] == 2.0 and w[3, 0] == np.float32(np.float64(w0[3, 0]) + 0.5)
    o.apply_row_update(w, v, 4, (0, 10), 1, [0.0] * 4, 5.0)
    o.apply_row_update(w, v, 4, (0, 10), 1, [0.0] * 4, 1.0)
    assert v[1] == 1.0
    with pytest.raises(ValueError):
        o.apply_row_update(w, v, 4, (0, 10), 1, [0.0] * 4, -0.5)
    with pytest.raises(IndexError):
        o.apply_row_update(w, v, 4, (0, 10), 42, [0.0] * 4, 0.0)


def test_apply_row_update_port_matches_reference():
    from oracle import Oracle, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    outs = []
    for kind in ("port", "reference"):
        o = Oracle(kind)
        w = o.init_rows(2, 50, 0, 50, 8, 11).reshape(50, 8).copy()
        v = np.abs(np.random.default_rng(9).standard_normal(50)).astype(np.float32)
        r2 = np.random.default_rng(4)
        for _ in range(40):
            o.apply_row_update(w, v, 8, (10, 40), int(r2.integers(10, 40)), r2.standard_normal(8) * 1e-3,
                               float(abs(r2.standard_normal())))
        outs.append((w, v))
    assert np.array_equal(outs[0][0].view(np.uint32), outs[1][0].view(np.uint32))
    assert np.array_equal(outs[0][1].view(np.uint32), outs[1][1].view(np.uint32))


def test_mean_pooling_oracle_definition(port):
    """The mean-pooling definition the oracle pins (s2d_oracle.c or_cfg.mean):
    rows r0 = (1, 0), r1 = (0, 2) (test_embedding.cpp:26-86 shapes): bag
    [0, 1] -> f32((1 + 0, 0 + 2) * (1/2)) = (0.5, 1); [1] -> (0, 2); [] -> 0.
    SGD with eta = 1, B = 1: the bag's gradient row is f32(up * (1/L)), so
    row 0 moves by -up/2 and row 1 (in both bags) by -(up/2 + up')."""
    from oracle import MeshSpec

    spec = MeshSpec(rows=np.array([2], np.uint32), dims=np.array([4], np.uint32),
                    plan=np.array([[0, 0, 2, 0]], np.uint32), T=1, M=1, B=3, eta=1.0, sgd=True,
                    mean=np.array([1], np.uint8))
    w = np.array([1, 0, 0, 0, 0, 2, 0, 0], np.float32)
    v = np.zeros(2, np.float32)
    lengths = np.array([2, 1, 0], np.uint32)
    ids = np.array([0, 1, 1], np.uint32)
    up = np.array([[3, 3, 3, 3], [1, 1, 1, 1], [9, 9, 9, 9]], np.float32)
    pooled, _ = port.group_step(spec, [lengths], [ids], [up], w, v)
    assert np.array_equal(pooled[0], np.array([[0.5, 1, 0, 0], [0, 2, 0, 0], [0, 0, 0, 0]], np.float32))
    inv_b = 1.0 / 3.0  # 1 / (N * B)
    g0 = np.float64(np.float32(3 * 0.5)) * inv_b
    g1 = (np.float64(np.float32(3 * 0.5)) + np.float64(np.float32(1.0))) * inv_b
    assert np.array_equal(w[:4], np.array([np.float32(1 - g0), np.float32(-g0), np.float32(-g0), np.float32(-g0)],
                                          np.float32))
    assert np.array_equal(w[4:], np.array([np.float32(-g1), np.float32(2 - g1), np.float32(-g1), np.float32(-g1)],
                                          np.float32))


def test_metrics_row_definition(port):
    """or_metrics_row follows make_metrics_row (trainer.cpp:745-771):
    nth_element at ceil(q n) - 1 of the per-row effective_lr, sequential
    v_sum / n."""
    rng = np.random.default_rng(3)
    v = np.concatenate([np.zeros(50, np.float32), rng.random(151).astype(np.float32) * 4])
    m = port.metrics_row(v, eta=0.1, eps=1e-8, c=2.0)
    lrs = np.sort(0.1 / (np.sqrt(v.astype(np.float64) / 2.0) + 1e-8))
    n = v.size
    assert m["eff_lr_p50"] == lrs[int(np.ceil(0.5 * n)) - 1]
    assert m["eff_lr_p99"] == lrs[int(np.ceil(0.99 * n)) - 1]
    acc = 0.0
    for x in v:
        acc += float(x)
    assert m["v_mean"] == acc / n


PIN_MESHES = [
    dict(T=1, M=1),
    dict(T=4, M=1),
    dict(T=4, M=2),
    dict(T=4, M=4, strategy="table-wise"),
    dict(T=8, M=2, strategy="table-wise", sync_interval=3, steps=6),
    dict(T=4, M=2, sgd=True, sync_interval=2),
    dict(T=6, M=3, rows=50, dim=12, L=5),
]


@pytest.mark.parametrize("mesh", PIN_MESHES, ids=[str(m) for m in PIN_MESHES])
def test_restated_loop_equals_real_trainer(mesh):
    """Oracle pin against the REAL reference Trainer (trainer.cpp compiled
    into oracle/_ref): the step composed from the public API in
    ref_harness.cpp -- DataGenerator batches, the restated build_demand /
    owner split / combine / grad payloads / owner update (ref_group_step),
    the per-rank MLPs and the replica sync -- leaves every group's replica
    bitwise equal to Trainer::replica_tables(g) (acceptance criterion 1 shape,
    tests/acceptance/main.cpp:95-125; replica consensus, test_trainer.cpp:141-151)."""
    from oracle import reference_available, reference_trainer, restated_trainer, trainer_options

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    o = trainer_options(**mesh)
    ws_real, vs_real, _ = reference_trainer(o)
    ws, vs = restated_trainer(o)[:2]
    for g in range(o.M):
        assert np.array_equal(ws[g].view(np.uint32), ws_real[g].view(np.uint32)), g
        assert np.array_equal(vs[g].view(np.uint32), vs_real[g].view(np.uint32)), g
    if o.M > 1 and o.steps % o.sync_interval == 0:  # consensus after a sync step
        for g in range(1, o.M):
            assert np.array_equal(ws_real[g].view(np.uint32), ws_real[0].view(np.uint32))
