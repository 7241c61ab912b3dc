"""BASELINE config 2 at its full size on one GPU (26 Criteo-Kaggle tables,
33.6M x 128 fp32 rows = 17.2 GB, B = 16384, nnz ~ 4.7M, U ~ 0.45M), checked
through properties that do not need the whole-table oracle:

* dedup: the step's unique-row count equals numpy's count of distinct
  (table, row) keys;
* lookup: sampled bags pool bit-exactly to the f64 sum of their rows in item
  order (oracle s2d_oracle.c:362-378 / trainer.cpp pool_and_forward);
* update: sampled touched rows with at most kChunk = 128 contributions are
  bit-exact against the oracle's row step on the f64 item-order gradient sum
  times 1/B (s2d_oracle.c:495-516, optimizer.cpp:31-60); the hottest rows,
  whose sums are re-associated per chunk, within 1e-5 relative;
* untouched rows (weights and moments) are bit-identical after the step.
"""
import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu

SEED = 3
K_CHUNK = 128


def _row(eng, f, r):
    w, v = eng.read_rows(int(f), int(r), int(r) + 1)
    return w[0], v[0]


def test_cfg2_full_size_properties(port):
    import paper_2508_03854_b200 as s2d
    from paper_2508_03854_b200 import workloads

    wl = workloads.get("cfg2")
    F, B, D = wl.F, wl.batch, 128
    assert all(d == D for d in wl.dims)
    tables = [s2d.TableConfig(int(r), D) for r in wl.rows]
    eng = s2d.Sparse2DEmbedding(tables, s2d.Topology(1, 1), rank=0, device=0, strategy="table-wise",
                                optimizer=s2d.OptimizerConfig(eta=wl.eta, eps=1e-8, c=wl.c,
                                                              variant="rowwise-adagrad"))
    eng.init_tables(SEED)
    lengths, ids = wl.batch_for(SEED, 0, 0)
    up = wl.upstream_for(SEED, 0, 0)
    nnz = len(ids)
    assert nnz > 4_000_000

    off = np.concatenate([[0], np.cumsum(lengths, dtype=np.int64)])
    bag_of_item = np.repeat(np.arange(B * F, dtype=np.int64), lengths)
    feat = (bag_of_item % F).astype(np.uint64)
    keys = (feat << np.uint64(32)) | ids.astype(np.uint64)
    order = np.argsort(keys, kind="stable")  # item order within each key
    uniq, first, counts = np.unique(keys[order], return_index=True, return_counts=True)

    rng = np.random.default_rng(0)
    # rows to check after the update: short segments (bit-exact) + the hottest
    short = np.nonzero(counts <= K_CHUNK)[0]
    pick = np.concatenate([rng.choice(short, 96, replace=False), np.argsort(counts)[-4:]])
    # untouched rows
    untouched = []
    touched = set(uniq.tolist())
    while len(untouched) < 32:
        f = int(rng.integers(F))
        r = int(rng.integers(wl.rows[f]))
        if ((f << 32) | r) not in touched:
            untouched.append((f, r))
    bags = rng.choice(np.nonzero(lengths)[0], 48, replace=False)

    # state before the step
    before = {}
    for k in pick:
        f, r = int(uniq[k] >> np.uint64(32)), int(uniq[k] & np.uint64(0xFFFFFFFF))
        before[(f, r)] = _row(eng, f, r)
    bag_rows = {}
    for b in bags:
        f = int(b % F)
        bag_rows[int(b)] = [_row(eng, f, ids[i])[0] for i in range(off[b], off[b + 1])]
    untouched_before = [_row(eng, f, r) for f, r in untouched]

    pooled = eng.forward(lengths, ids)
    for b, rows in bag_rows.items():
        s, f = divmod(b, F)
        acc = np.zeros(D, np.float64)
        for row in rows:
            acc += row.astype(np.float64)
        assert np.array_equal(bits(pooled[s, f * D:(f + 1) * D]), bits(acc.astype(np.float32))), b

    eng.backward_update(up)
    eng.synchronize()
    st = eng.stats()
    assert st["unique_rows"] == len(uniq)

    inv_batch = 1.0 / B
    bit_exact = 0
    for k in pick:
        f, r = int(uniq[k] >> np.uint64(32)), int(uniq[k] & np.uint64(0xFFFFFFFF))
        items = order[first[k]:first[k] + counts[k]]
        g = np.zeros(D, np.float64)
        for i in items:  # item order (stable sort)
            s = int(bag_of_item[i] // F)
            g += up[s, f * D:(f + 1) * D].astype(np.float64)
        g *= inv_batch
        w0, v0 = before[(f, r)]
        want = port.adagrad_row_step(w0, v0, g, eta=wl.eta, eps=1e-8, c=wl.c)
        w1, v1 = _row(eng, f, r)
        if counts[k] <= K_CHUNK:
            assert np.array_equal(bits(w1), bits(want["w"])), (f, r, int(counts[k]))
            assert np.float32(v1) == np.float32(want["v"]), (f, r)
            bit_exact += 1
        else:
            ww = want["w"].astype(np.float64)
            assert np.all(np.abs(w1 - ww) <= 1e-5 * np.maximum(np.abs(ww), 1e-30) + 1e-30), (f, r)
            assert abs(float(v1) - float(want["v"])) <= 1e-5 * abs(float(want["v"])) + 1e-30
    assert bit_exact >= 96

    for (f, r), (w0, v0) in zip(untouched, untouched_before):
        w1, v1 = _row(eng, f, r)
        assert np.array_equal(bits(w1), bits(w0)) and bits(np.float32(v1)) == bits(np.float32(v0)), (f, r)
    eng.close()
