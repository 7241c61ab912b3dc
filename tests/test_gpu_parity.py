"""GPU parity: the sm_100a step (through the C ABI) against the CPU oracle on
identical seeded inputs.  Bar (BASELINE.json north_star): bucketing, dedup
and wire layouts bit-exact; pooled outputs, accumulators and weights within
1e-5 relative for fp32 (1e-2 for bf16).  The fp32 path is bit-exact by
construction except for gradient segments longer than kChunk (hot rows),
whose f64 sums are re-associated per chunk -- those cases are checked at
the stated tolerance and additionally report their bit-equal fraction."""
import numpy as np
import pytest

from cases import make_batch, upstream
from conftest import bits

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _engine(rows, dims, strategy="table-wise", eta=0.1, c=1.0, variant="rowwise-adagrad", dtype="fp32",
            mean=None):
    import paper_2508_03854_b200 as s2d

    mean = mean if mean is not None else [0] * len(rows)
    tables = [s2d.TableConfig(int(r), int(d), pooling="mean" if m else "sum") for r, d, m in zip(rows, dims, mean)]
    return s2d.Sparse2DEmbedding(tables, s2d.Topology(1, 1), rank=0, device=0, strategy=strategy,
                                 optimizer=s2d.OptimizerConfig(eta=eta, eps=1e-8, c=c, variant=variant),
                                 weight_dtype=dtype)


def _spec(rows, dims, B, eta=0.1, c=1.0, sgd=False, mean=None):
    from oracle import MeshSpec, row_wise_plan

    rows = np.array(rows, np.uint32)
    return MeshSpec(rows=rows, dims=np.array(dims, np.uint32), plan=row_wise_plan(rows, 1), T=1, M=1, B=B,
                    eta=eta, c=c, sgd=sgd, mean=None if mean is None else np.array(mean, np.uint8))


def _download(eng, spec):
    ws, vs = [], []
    for f in range(spec.F):
        w, v = eng.read_rows(f, 0, int(spec.rows[f]))
        ws.append(w.ravel())
        vs.append(v)
    return np.concatenate(ws), np.concatenate(vs)


def _close(a, b, tol=TOL):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= tol * np.maximum(np.abs(b), 1e-30) + 1e-30)


def test_init_tables_bit_exact(port):
    from oracle import MeshState

    rows, dims = [1000, 37, 5], [64, 128, 8]
    eng = _engine(rows, dims)
    eng.init_tables(22)
    spec = _spec(rows, dims, 1)
    st = MeshState.init(port, spec, 22)
    w, v = _download(eng, spec)
    assert np.array_equal(bits(w), bits(st.ws[0]))
    assert np.all(v == 0)


def test_adagrad_row_step_known_answers():
    """test_optimizer.cpp:50-94 and tests/python/test_smoke.py:38-44 through the
    device row-update kernel."""
    import paper_2508_03854_b200 as s2d

    out = s2d.adagrad_row_step([1.0, 1.0], 0.0, [2.0, 0.0], eta=0.1, eps=1e-8, c=4.0)
    assert abs(out["v"] - 4.0) < 1e-6
    assert abs(out["effective_lr"] - 0.1) < 1e-6
    assert abs(out["w"][0] - 0.8) < 1e-6 and out["w"][1] == 1.0
    out = s2d.adagrad_row_step([1.0, 1.0], 0.0, [2.0, 0.0], eta=0.1, eps=1e-8, c=1.0)
    assert abs(out["effective_lr"] - 0.05) < 1e-6 and abs(out["w"][0] - 0.9) < 1e-6
    out = s2d.adagrad_row_step([0.25, -0.5], 3.0, [0.0, 0.0], eta=0.1, c=1.0)
    assert out["v"] == 3.0 and out["w"] == [0.25, -0.5]
    with pytest.raises(ValueError):
        s2d.adagrad_row_step([0.0], 0.0, [float("nan")])
    with pytest.raises(ValueError):
        s2d.adagrad_row_step([0.0], 0.0, [0.0], eta=0.0)


def test_adagrad_rows_bit_exact_vs_reference_formula(port):
    rng = np.random.default_rng(3)
    import paper_2508_03854_b200 as s2d

    for dim in (4, 64, 128, 256, 512, 6):
        w = rng.standard_normal((50, dim)).astype(np.float32)
        v = rng.random(50).astype(np.float32)
        g = rng.standard_normal((50, dim)) * 1e-2
        for c in (1.0, 4.0):
            got = s2d.adagrad_rows(w, v, g, eta=0.1, eps=1e-8, c=c)
            for i in range(50):
                want = port.adagrad_row_step(w[i], v[i], g[i], eta=0.1, eps=1e-8, c=c)
                assert np.array_equal(bits(got[i]["w"]), bits(want["w"])), (dim, c, i)
                assert np.float32(got[i]["v"]) == np.float32(want["v"])


@pytest.mark.parametrize("c,variant", [(1.0, "rowwise-adagrad"), (4.0, "rowwise-adagrad"), (1.0, "sgd")])
def test_single_gpu_steps_vs_oracle(port, c, variant):
    from oracle import MeshState

    rng = np.random.default_rng(11)
    rows, dims = [100, 1000, 7, 5000], [64, 64, 64, 64]
    B = 64
    spec = _spec(rows, dims, B, eta=0.1, c=c, sgd=variant == "sgd")
    eng = _engine(rows, dims, eta=0.1, c=c, variant=variant)
    eng.init_tables(5)
    st = MeshState.init(port, spec, 5)
    for step in range(4):
        lengths, ids = make_batch(rng, spec.rows, B, max_len=12)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        got = eng.forward(lengths, ids)
        assert np.array_equal(bits(got), bits(want)), f"pooled step {step}"
        eng.backward_update(up)
    w, v = _download(eng, spec)
    assert np.array_equal(bits(v), bits(st.vs[0]))
    assert np.array_equal(bits(w), bits(st.ws[0]))


def test_cfg1_shape_bit_exact(port):
    """BASELINE config 1 shape (8 x 100K x 64, B=512, L=20, Zipf 1.0, 1x1)."""
    from oracle import MeshState

    rng = np.random.default_rng(1)
    rows, dims, B = [100_000] * 8, [64] * 8, 512
    spec = _spec(rows, dims, B, eta=0.1, c=1.0)
    eng = _engine(rows, dims)
    eng.init_tables(2)
    st = MeshState.init(port, spec, 2)
    for step in range(2):
        lengths, ids = make_batch(rng, spec.rows, B, fixed_len=20, zipf=1.0)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        got = eng.forward(lengths, ids)
        assert np.array_equal(bits(got), bits(want))
        eng.backward_update(up)
    w, v = _download(eng, spec)
    assert np.array_equal(bits(v), bits(st.vs[0]))
    assert np.array_equal(bits(w), bits(st.ws[0]))


def test_async_host_copies_bit_exact(port):
    """async host mode: pooled read-back on the D2H stream, upstream upload
    on the H2D stream, pinned buffers reused every step (s2d_ctx_set_async_host)."""
    import torch

    from oracle import MeshState

    rng = np.random.default_rng(5)
    rows, dims, B = [5000, 300, 70000], [64, 64, 64], 256
    spec = _spec(rows, dims, B, eta=0.1, c=1.0)
    eng = _engine(rows, dims)
    eng.set_strict(False)
    eng.set_async_host(True)
    eng.init_tables(9)
    st = MeshState.init(port, spec, 9)
    pooled_h = torch.empty((B, spec.sum_dims), dtype=torch.float32).pin_memory()
    up_h = torch.empty((B, spec.sum_dims), dtype=torch.float32).pin_memory()
    for step in range(4):
        lengths, ids = make_batch(rng, spec.rows, B, max_len=12, zipf=1.1)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        lh = torch.from_numpy(lengths.view(np.int32)).pin_memory()
        ih = torch.from_numpy(ids.view(np.int32)).pin_memory()
        up_h.copy_(torch.from_numpy(up))
        eng.forward(lh, ih, pooled_h, batch=B)
        eng.backward_update(up_h)
        eng.synchronize()
        assert np.array_equal(bits(pooled_h.numpy()), bits(want)), step
    w, v = _download(eng, spec)
    assert np.array_equal(bits(v), bits(st.vs[0]))
    assert np.array_equal(bits(w), bits(st.ws[0]))


def test_async_host_pipelined_steps(port):
    """async host mode without a host wait between steps (the e2e loop of
    bench.py): inputs on the H2D stream into alternating staging buffers, the
    pooled read-back of step k overlapping step k+1 (N = 1); every step's
    pooled rows and the final tables bit-exact after one synchronize."""
    import torch

    from oracle import MeshState

    rng = np.random.default_rng(6)
    rows, dims, B = [5000, 300, 70000], [64, 64, 64], 256
    spec = _spec(rows, dims, B, eta=0.1, c=1.0)
    eng = _engine(rows, dims)
    eng.set_strict(False)
    eng.set_async_host(True)
    eng.init_tables(9)
    st = MeshState.init(port, spec, 9)
    outs, wants, keep = [], [], []
    for step in range(5):
        lengths, ids = make_batch(rng, spec.rows, B, max_len=12, zipf=1.1)
        up = upstream(rng, B, spec.sum_dims)
        wants.append(st.step(port, [lengths], [ids], [up], do_sync=False)[0])
        lh = torch.from_numpy(lengths.view(np.int32)).pin_memory()
        ih = torch.from_numpy(ids.view(np.int32)).pin_memory()
        uh = torch.from_numpy(up).pin_memory()
        ph = torch.empty((B, spec.sum_dims), dtype=torch.float32).pin_memory()
        keep.append((lh, ih, uh))
        outs.append(ph)
        eng.forward(lh, ih, ph, batch=B)
        eng.backward_update(uh)
    eng.synchronize()
    for step in range(5):
        assert np.array_equal(bits(outs[step].numpy()), bits(wants[step])), step
    w, v = _download(eng, spec)
    assert np.array_equal(bits(v), bits(st.vs[0]))
    assert np.array_equal(bits(w), bits(st.ws[0]))


def test_hot_rows_long_segments(port):
    """Tiny tables => segments of thousands of contributions (chunked f64
    reduction).  Within 1e-5 relative; report bit-equal share."""
    from oracle import MeshState

    rng = np.random.default_rng(7)
    rows, dims, B = [3, 10, 2000], [128, 128, 128], 1024
    spec = _spec(rows, dims, B, eta=0.1, c=2.0)
    eng = _engine(rows, dims, eta=0.1, c=2.0)
    eng.init_tables(9)
    st = MeshState.init(port, spec, 9)
    for step in range(3):
        lengths, ids = make_batch(rng, spec.rows, B, max_len=40, zipf=1.2)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        got = eng.forward(lengths, ids)
        assert np.array_equal(bits(got), bits(want))
        eng.backward_update(up)
        assert eng.stats()["long_segments"] > 0
    w, v = _download(eng, spec)
    assert _close(v, st.vs[0]) and _close(w, st.ws[0])
    print("bit-equal w share", float(np.mean(bits(w) == bits(st.ws[0]))))


def test_mixed_dims_variable_pooling_empty_bags(port):
    from oracle import MeshState

    rng = np.random.default_rng(5)
    rows, dims, B = [3, 50, 1000, 7, 200, 64], [4, 8, 12, 16, 32, 256], 40
    spec = _spec(rows, dims, B, eta=0.05, c=3.0)
    eng = _engine(rows, dims, eta=0.05, c=3.0)
    eng.init_tables(4)
    st = MeshState.init(port, spec, 4)
    for step in range(3):
        lengths, _ = make_batch(rng, spec.rows, B, max_len=30)
        lengths[::7] = 0  # empty bags pool to zero
        lengths, ids = _regen(rng, spec.rows, lengths)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        got = eng.forward(lengths, ids)
        assert np.array_equal(bits(got), bits(want))
        eng.backward_update(up)
    w, v = _download(eng, spec)
    assert np.array_equal(bits(v), bits(st.vs[0]))
    assert np.array_equal(bits(w), bits(st.ws[0]))


@pytest.mark.parametrize("variant", ["rowwise-adagrad", "sgd"])
def test_mean_pooling_bit_exact(port, variant):
    """Mean pooling (north star K2 "sum/mean"; the reference is sum-only, so
    the semantics are this build's, pinned by the oracle restatement):
    out = f32(f64(f32 sum) * (1/L)), gradient row f32(f64(up) * (1/L)).
    Mixed sum / mean tables, mixed dims, variable lengths, empty bags."""
    from oracle import MeshState

    rng = np.random.default_rng(17)
    rows, dims, B = [50, 1000, 7, 200], [8, 12, 128, 32], 48
    mean = [1, 0, 1, 1]
    spec = _spec(rows, dims, B, eta=0.05, c=2.0, sgd=variant == "sgd", mean=mean)
    eng = _engine(rows, dims, eta=0.05, c=2.0, variant=variant, mean=mean)
    eng.init_tables(9)
    st = MeshState.init(port, spec, 9)
    for step in range(3):
        lengths, _ = make_batch(rng, spec.rows, B, max_len=25)
        lengths[::5] = 0
        lengths, ids = _regen(rng, spec.rows, lengths)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        got = eng.forward(lengths, ids)
        assert np.array_equal(bits(got), bits(want)), step
        eng.backward_update(up)
    w, v = _download(eng, spec)
    assert np.array_equal(bits(v), bits(st.vs[0]))
    assert np.array_equal(bits(w), bits(st.ws[0]))


def _regen(rng, rows, lengths):
    from cases import zipf_ids

    F = len(rows)
    ids = [zipf_ids(rng, int(rows[b % F]), int(lengths[b])) for b in range(len(lengths))]
    return lengths, np.concatenate(ids).astype(np.uint32)


def test_empty_batch_and_all_empty_bags(port):
    rows, dims = [10, 20], [8, 8]
    eng = _engine(rows, dims)
    eng.init_tables(1)
    lengths = np.zeros(2 * 3, np.uint32)
    ids = np.zeros(0, np.uint32)
    got = eng.forward(lengths, ids)
    assert got.shape == (3, 16) and np.all(got == 0)
    eng.backward_update(np.ones((3, 16), np.float32))
    w0, _ = eng.read_rows(0, 0, 10)
    eng2 = _engine(rows, dims)
    eng2.init_tables(1)
    w1, _ = eng2.read_rows(0, 0, 10)
    assert np.array_equal(bits(w0), bits(w1))


def test_out_of_range_id_raises():
    eng = _engine([10, 20], [8, 8])
    eng.init_tables(1)
    lengths = np.array([1, 1], np.uint32)
    with pytest.raises(IndexError):
        eng.forward(lengths, np.array([3, 20], np.uint32))


def test_nonfinite_gradient_raises():
    eng = _engine([10, 20], [8, 8])
    eng.init_tables(1)
    eng.forward(np.array([1, 1], np.uint32), np.array([3, 4], np.uint32))
    up = np.zeros((1, 16), np.float32)
    up[0, 3] = np.nan
    with pytest.raises(ValueError):
        eng.backward_update(up)


def test_bf16_weights_within_tolerance(port):
    """bf16 storage: no reference path (embedding.hpp:16); oracle = fp32
    reference seeded each step from the GPU's bf16 weights."""
    from oracle import MeshState

    rng = np.random.default_rng(21)
    rows, dims, B = [500, 40], [128, 64], 128
    spec = _spec(rows, dims, B, eta=0.1, c=2.0)
    eng = _engine(rows, dims, eta=0.1, c=2.0, dtype="bf16")
    eng.init_tables(3)
    for step in range(3):
        w, v = _download(eng, spec)
        st = MeshState(spec, [w.copy()], [v.copy()], [np.zeros(spec.replica_rows(), np.uint8)])
        lengths, ids = make_batch(rng, spec.rows, B, max_len=10)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        got = eng.forward(lengths, ids)
        assert np.array_equal(bits(got), bits(want))  # pooling of bf16 rows is exact in f64
        eng.backward_update(up)
        w2, v2 = _download(eng, spec)
        assert _close(v2, st.vs[0], 1e-5)
        assert _close(w2, st.ws[0], 1e-2)


@pytest.mark.parametrize("dims", [[128, 128, 128], [256, 256]])
def test_bf16_uniform_dims_fast_paths(port, dims):
    """bf16 shards whose rows fill whole warp chunks (D = 128 * VPL): the
    slot-indexed lookup and the unpredicated (FULL) update paths."""
    from oracle import MeshState

    rng = np.random.default_rng(33)
    rows = [700, 3000, 9][: len(dims)]
    B = 128
    spec = _spec(rows, dims, B, eta=0.1, c=1.0)
    eng = _engine(rows, dims, eta=0.1, c=1.0, dtype="bf16")
    eng.init_tables(8)
    for step in range(3):
        w, v = _download(eng, spec)
        st = MeshState(spec, [w.copy()], [v.copy()], [np.zeros(spec.replica_rows(), np.uint8)])
        lengths, ids = make_batch(rng, spec.rows, B, max_len=14, zipf=1.2)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        got = eng.forward(lengths, ids)
        assert np.array_equal(bits(got), bits(want))
        eng.backward_update(up)
        w2, v2 = _download(eng, spec)
        assert _close(v2, st.vs[0], 1e-5)
        assert _close(w2, st.ws[0], 1e-2)


def test_fp32_full_rows_vpl2_bit_exact(port):
    """fp32 D = 256 (VPL = 2, FULL update path, slot-indexed lookup): bit-exact."""
    from oracle import MeshState

    rng = np.random.default_rng(34)
    rows, dims, B = [400, 2000], [256, 256], 96
    spec = _spec(rows, dims, B, eta=0.1, c=2.0)
    eng = _engine(rows, dims, eta=0.1, c=2.0)
    eng.init_tables(2)
    st = MeshState.init(port, spec, 2)
    for step in range(3):
        lengths, ids = make_batch(rng, spec.rows, B, max_len=12, zipf=1.1)
        up = upstream(rng, B, spec.sum_dims)
        want = st.step(port, [lengths], [ids], [up], do_sync=False)[0]
        got = eng.forward(lengths, ids)
        assert np.array_equal(bits(got), bits(want))
        eng.backward_update(up)
    w, v = _download(eng, spec)
    assert np.array_equal(bits(v), bits(st.vs[0]))
    assert np.array_equal(bits(w), bits(st.ws[0]))


def test_checkpoint_save_load_bytes(port, tmp_path):
    """s2d_save_tables writes the reference's S2DCKPT1 bytes for the trained
    tables (oracle writer on the oracle's replica); s2d_load_tables restores
    them into a fresh engine; count / shape / truncation errors raise."""
    from oracle import MeshState, read_checkpoint

    rng = np.random.default_rng(21)
    rows, dims, B = [300, 5000, 17], [64, 128, 32], 96
    spec = _spec(rows, dims, B, eta=0.1, c=1.0)
    eng = _engine(rows, dims)
    eng.init_tables(4)
    st = MeshState.init(port, spec, 4)
    for _ in range(2):
        lengths, ids = make_batch(rng, spec.rows, B, max_len=10, zipf=1.1)
        up = upstream(rng, B, spec.sum_dims)
        st.step(port, [lengths], [ids], [up], do_sync=False)
        eng.forward(lengths, ids)
        eng.backward_update(up)
    got, want = str(tmp_path / "gpu.ckpt"), str(tmp_path / "oracle.ckpt")
    eng.save_tables(got)
    port.save_checkpoint(want, spec.rows, spec.dims, st.ws[0], st.vs[0])
    assert open(got, "rb").read() == open(want, "rb").read()
    fresh = _engine(rows, dims)
    fresh.init_tables(99)
    fresh.load_tables(got)
    w, v = _download(fresh, spec)
    assert np.array_equal(bits(w), bits(st.ws[0])) and np.array_equal(bits(v), bits(st.vs[0]))
    # error paths (std::runtime_error -> RuntimeError)
    other = _engine(rows[:2], dims[:2])
    with pytest.raises(RuntimeError, match="count"):
        other.load_tables(got)
    shape = _engine([300, 5000, 18], dims)
    with pytest.raises(RuntimeError, match="shape"):
        shape.load_tables(got)
    raw = open(got, "rb").read()
    cut = str(tmp_path / "cut.ckpt")
    open(cut, "wb").write(raw[:-9])
    with pytest.raises(RuntimeError, match="truncated"):
        fresh.load_tables(cut)
    tables, _, _ = read_checkpoint(got)
    assert [t[2] for t in tables] == rows


def test_checkpoint_bf16_widen_and_round(tmp_path):
    """bf16 shards: save widens exactly to f32; load rounds f32 to nearest-even."""
    from oracle import read_checkpoint

    rows, dims = [40, 9], [64, 32]
    eng = _engine(rows, dims, dtype="bf16")
    eng.init_tables(5)
    p = str(tmp_path / "bf16.ckpt")
    eng.save_tables(p)
    _, w, v = read_checkpoint(p)
    w16 = np.concatenate([eng.read_rows(f, 0, rows[f])[0].ravel() for f in range(2)])
    assert np.array_equal(bits(w), bits(w16))
    assert np.all(bits(w) & 0xFFFF == 0)  # exactly representable bf16 values
    fresh = _engine(rows, dims, dtype="bf16")
    fresh.init_tables(6)
    fresh.load_tables(p)
    w2 = np.concatenate([fresh.read_rows(f, 0, rows[f])[0].ravel() for f in range(2)])
    assert np.array_equal(bits(w2), bits(w16))


def test_device_gen_batch_bit_exact(port):
    """s2d_gen_batch (device DataGenerator ids, data.cpp:85-136) equals the
    oracle's restatement bit for bit, host and device outputs; the batch
    feeds the step directly; invalid specs raise like FeatureSpec::validate."""
    rows, dims = [100, 3, 5000, 1, 70000], [64, 64, 64, 64, 64]
    zipf, L = [1.0, 1.2, 0.8, 0.0, 1.05], [5, 2, 20, 1, 11]
    eng = _engine(rows, dims)
    B = 96
    for seed, step, rank in ((7, 3, 1), (2024, 0, 0)):
        want = port.gen_batch_ids(seed, step, rank, len(rows), rows, zipf, L, B)
        lengths, ids = eng.gen_batch(seed, step, rank, B, zipf, L)
        assert np.array_equal(lengths.cpu().numpy().view(np.uint32), np.tile(np.array(L, np.uint32), B))
        assert np.array_equal(ids.cpu().numpy().view(np.uint32), want)
        lh, ih = eng.gen_batch(seed, step, rank, B, zipf, L, device=False)
        assert np.array_equal(ih, want) and np.array_equal(lh, np.tile(np.array(L, np.uint32), B))
    eng.init_tables(1)
    pooled = eng.forward(lengths, ids)  # the generated batch is a valid step input
    assert pooled.shape == (B, sum(dims))
    with pytest.raises(ValueError, match="zipf_exponent"):
        eng.gen_batch(1, 0, 0, B, [1.0, -0.5, 1.0, 1.0, 1.0], L)


def test_measured_trace_rows():
    """trace_rows: measured per-collective rows in the reference trace schema
    (topology.hpp:53-61).  At 1x1 nothing crosses ranks (0 bytes) and no
    replica sync runs (no table_allreduce row); the lookup time is measured."""
    import paper_2508_03854_b200 as s2d

    rng = np.random.default_rng(5)
    rows, dims, B = [5000, 300], [64, 32], 256
    eng = _engine(rows, dims)
    eng.init_tables(3)
    eng.set_profiling(True)
    eng.phase_times()
    lengths, ids = make_batch(rng, np.array(rows, np.uint32), B)
    eng.forward(lengths, ids)
    eng.backward_update(upstream(rng, B, sum(dims)))
    eng.synchronize()
    tr = eng.trace_rows(7)
    assert [r["kernel"] for r in tr] == ["lookup_a2a", "grad_a2a"]
    assert all(r["step"] == 7 and r["rank"] == 0 and r["bytes"] == 0 for r in tr)
    assert tr[0]["latency_s"] > 0
    csv = s2d.traces_to_csv(tr, "x").splitlines()
    assert csv[-2].startswith("7,lookup_a2a,0,0,")
    eng.set_profiling(False)


@pytest.mark.parametrize("strategy", ["table-wise", "row-wise"])
def test_apply_row_updates_vs_oracle(port, strategy):
    """s2d_apply_row_updates == apply_row_update (embedding.cpp:108-129)
    called once per listed row in order (oracle), bit-exact, repeated rows
    included; untouched rows bitwise unchanged; errors before any write."""
    rows, dims = [3000, 77], [64, 128]
    eng = _engine(rows, dims, strategy=strategy)
    eng.init_tables(8)
    rng = np.random.default_rng(21)
    for f in range(2):
        lo, hi = eng.owned_range(f)
        w, v = eng.read_rows(f, lo, hi)
        w = np.ascontiguousarray(w, np.float32).reshape(hi - lo, dims[f])
        v = np.ascontiguousarray(v, np.float32)
        n = 500
        rr = rng.integers(lo, hi, size=n).astype(np.uint32)
        rr[1] = rr[0]  # a repeated row: two updates in call order
        delta = rng.standard_normal((n, dims[f])) * 1e-2
        mom = np.abs(rng.standard_normal(n)) * 3
        eng.apply_row_updates(f, rr, delta, mom)
        want_w = np.zeros((hi, dims[f]), np.float32)
        want_w[lo:hi] = w
        want_v = np.zeros(hi, np.float32)
        want_v[lo:] = v
        for i in range(n):
            port.apply_row_update(want_w, want_v, dims[f], (lo, hi), int(rr[i]), delta[i], float(mom[i]))
        gw, gv = eng.read_rows(f, lo, hi)
        assert np.array_equal(bits(np.asarray(gw).ravel()), bits(want_w[lo:hi].ravel()))
        assert np.array_equal(bits(np.asarray(gv)), bits(want_v[lo:hi]))
        with pytest.raises(IndexError):
            eng.apply_row_updates(f, [lo, hi], np.zeros((2, dims[f])), [0.0, 0.0])
        with pytest.raises(ValueError):
            eng.apply_row_updates(f, [lo], np.ones((1, dims[f])), [-1.0])
        gw2, gv2 = eng.read_rows(f, lo, hi)
        assert np.array_equal(bits(np.asarray(gw2).ravel()), bits(np.asarray(gw).ravel()))
        assert np.array_equal(bits(np.asarray(gv2)), bits(np.asarray(gv)))


def test_metrics_row_vs_oracle(port):
    """Device MetricsRow columns (eff_lr_p50 / p99 exact, v_mean within 1e-12)
    against the oracle restatement of trainer.cpp:745-771, after AdaGrad steps
    with hot and cold rows (many moments tie at 0)."""
    from oracle import MeshState

    rng = np.random.default_rng(8)
    rows, dims, B = [500, 3000, 40], [16, 32, 8], 64
    spec = _spec(rows, dims, B, eta=0.07, c=3.0)
    eng = _engine(rows, dims, eta=0.07, c=3.0)
    eng.init_tables(2)
    st = MeshState.init(port, spec, 2)
    for step in range(3):
        lengths, ids = make_batch(rng, spec.rows, B, max_len=12)
        up = upstream(rng, B, spec.sum_dims)
        st.step(port, [lengths], [ids], [up], do_sync=False)
        eng.forward(lengths, ids)
        eng.backward_update(up)
    got = eng.metrics_row()
    want = port.metrics_row(st.vs[0], eta=0.07, eps=1e-8, c=3.0)
    assert got["rows"] == sum(rows)
    assert got["eff_lr_p50"] == want["eff_lr_p50"]
    assert got["eff_lr_p99"] == want["eff_lr_p99"]
    assert abs(got["v_mean"] - want["v_mean"]) <= 1e-12 * abs(want["v_mean"])
