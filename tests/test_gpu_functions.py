"""Function-level forms of the path's reductions on the device
(s2d_pool_ids / s2d_aggregate_group_gradient): the reference's known answers
(tests/test_embedding.cpp:26-121, tests/test_optimizer.cpp:13-48) and
bit-for-bit agreement with the compiled reference functions on random
inputs."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_pool_ids_known_answers():
    import paper_2508_03854_b200 as s2d

    w = np.array([[1.0, 0.0], [0.0, 2.0]], np.float32)  # r0=(1,0), r1=(0,2)
    sh = [(0, 2)]
    assert s2d.pool_ids(w, sh, [1]).tolist() == [0.0, 2.0]
    assert s2d.pool_ids(w, sh, [1, 1])[1] == 4.0
    assert s2d.pool_ids(w, sh, [0, 1]).tolist() == [1.0, 2.0]
    assert s2d.pool_ids(w, sh, []).tolist() == [0.0, 0.0]
    with pytest.raises(IndexError, match=r"7.*\[0,2\)"):
        s2d.pool_ids(w, sh, [7])
    pooled = s2d.lookup_and_pool(w, sh, [[0], [0, 1]])
    assert pooled[0][0] == 1.0 and pooled[1][1] == 2.0
    with pytest.raises(ValueError, match="empty shard set"):
        s2d.pool_ids(w, [], [0])


def test_pool_ids_linear_and_sharded_vs_reference(port):
    import paper_2508_03854_b200 as s2d
    from oracle import Oracle, reference_available

    t = port.init_rows(0, 40, 0, 40, 8, 5).reshape(40, 8)
    ids = [1, 5, 5, 17, 39]
    a = s2d.pool_ids(t, [(0, 40)], ids)
    b = s2d.pool_ids(t * np.float32(2.0), [(0, 40)], ids)
    assert np.array_equal(b, np.float32(2.0) * a)  # linearity x2 exact (test_embedding.cpp:88-98)
    ref = Oracle("reference") if reference_available() else port
    rng = np.random.default_rng(3)
    for trial in range(20):
        rows, dim = int(rng.integers(5, 300)), int(rng.integers(1, 40))
        w = (rng.standard_normal((rows, dim)) * 0.3).astype(np.float32)
        cuts = sorted(set(rng.integers(1, rows, size=int(rng.integers(0, 4))).tolist()))
        bounds = [0] + cuts + [rows]
        shards = [(bounds[i], bounds[i + 1]) for i in range(len(bounds) - 1)]
        rng.shuffle(shards)  # presentation order is part of the contract
        bags = [rng.integers(0, rows, size=int(rng.integers(0, 30))).tolist() for _ in range(17)]
        got = s2d.lookup_and_pool(w, shards, bags)
        for k, bag in enumerate(bags):
            want = ref.pool_ids(w.ravel(), dim, shards, bag)
            assert np.array_equal(got[k].view(np.uint32), want.view(np.uint32)), (trial, k)


def test_aggregate_group_gradient_known_answers():
    import paper_2508_03854_b200 as s2d

    g1, g2 = [1.0, 0.0], [3.0, 0.0]
    out = s2d.aggregate_group_gradient([5], [g1], 4)
    assert len(out) == 1 and out[0]["row"] == 5 and out[0]["g"][0] == 0.25 and out[0]["sample_count"] == 1
    out = s2d.aggregate_group_gradient([7, 7], [g1, g2], 4)
    assert len(out) == 1 and out[0]["g"].tolist() == [1.0, 0.0] and out[0]["sample_count"] == 2
    out = s2d.aggregate_group_gradient([9, 2, 9], [g1, g2, g2], 2)
    assert [o["row"] for o in out] == [2, 9]
    with pytest.raises(ValueError):
        s2d.aggregate_group_gradient([0], [g1], 0)
    assert s2d.aggregate_group_gradient([], np.zeros((0, 2)), 3) == []


def test_aggregate_group_gradient_vs_reference():
    """Random contributions (hot rows with hundreds of contributions
    included) against the compiled reference: rows, counts and every f64
    gradient bit for bit (the device sums each row strictly in arrival
    order)."""
    import paper_2508_03854_b200 as s2d
    from oracle import reference_aggregate, reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(11)
    for trial in range(8):
        n, dim, rows = int(rng.integers(1, 5000)), int(rng.integers(1, 70)), int(rng.integers(1, 3000))
        r = np.minimum(rng.zipf(1.3, size=n) - 1, rows - 1).astype(np.uint32)
        g = (rng.standard_normal((n, dim)) * 1e-3).astype(np.float32).astype(np.float64)
        B = int(rng.integers(1, 5000))
        got = s2d.aggregate_group_gradient(r, g, B)
        wr, wg, wc = reference_aggregate(r, g, B)
        assert [o["row"] for o in got] == wr.tolist(), trial
        assert [o["sample_count"] for o in got] == wc.tolist(), trial
        gg = np.array([o["g"] for o in got])
        assert np.array_equal(gg.view(np.uint64), wg.view(np.uint64)), trial
