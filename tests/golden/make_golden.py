"""Generates tests/golden/*.npz from the UNMODIFIED reference library
(oracle/_ref/libs2dref.so = /root/reference/proj/src compiled by
oracle/Makefile, driven through its public API by oracle/ref_harness.cpp).

    python tests/golden/make_golden.py        # needs /root/reference (this container)

Cases (small on purpose; inputs are stored with the outputs):
  known_*     the reference's own known-answer tests (test_embedding.cpp,
              test_optimizer.cpp, test_topology.cpp, test_planner.cpp)
  init        init_table rows (embedding.cpp:17-37)
  mesh_*      multi-step 2D steps on T virtual ranks (full replicas per
              group), row-wise / table-wise, AdaGrad c=M / SGD, sync 1 / 3,
              ids from the reference DataGenerator (data.cpp:115-147)
  mixed       per-table dims + variable pooling + empty bags
  cfg1        BASELINE config 1 shapes (8 x 100K x 64, B=512, L=20, Zipf 1.0):
              ids, and sha256 digests of pooled outputs / final replica
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import MeshSpec, MeshState, Oracle, row_wise_plan  # noqa: E402


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def table_wise_plan(ref, rows, n):
    prof = [(f, int(r) * 64, float(len(rows) - f), int(r)) for f, r in enumerate(rows)]
    return ref.plan_greedy(prof, n, "table-wise")


def mesh_case(ref, name, T, M, strategy, c, sgd, sync_interval, steps=4, F=4, R=64, D=8, B=4, L=2):
    N = T // M
    rows = np.full(F, R, np.uint32)
    dims = np.full(F, D, np.uint32)
    plan = row_wise_plan(rows, N) if strategy == "row-wise" else table_wise_plan(ref, rows, N)
    spec = MeshSpec(rows=rows, dims=dims, plan=plan, T=T, M=M, B=B, eta=0.05, c=c, sgd=sgd)
    st = MeshState.init(ref, spec, 22)
    out = dict(T=T, M=M, c=c, sgd=int(sgd), sync_interval=sync_interval, rows=rows, dims=dims, plan=plan, B=B,
               eta=0.05, seed=22)
    for step in range(steps):
        ids = [ref.gen_batch_ids(11, step, r, F, R, 0.9, L, B) for r in range(T)]
        lengths = [np.full(B * F, L, np.uint32) for _ in range(T)]
        up = [(0.01 * np.random.default_rng([step, r]).standard_normal((B, F * D))).astype(np.float32)
              for r in range(T)]
        pooled = st.step(ref, lengths, ids, up, do_sync=(M > 1 and (step + 1) % sync_interval == 0))
        for r in range(T):
            out[f"s{step}_r{r}_ids"] = ids[r]
            out[f"s{step}_r{r}_up"] = up[r]
            out[f"s{step}_r{r}_pooled"] = pooled[r]
    for g in range(M):
        out[f"w{g}"] = st.ws[g]
        out[f"v{g}"] = st.vs[g]
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), steps=steps, **out)


def main():
    ref = Oracle("reference")
    # ---- known answers --------------------------------------------------
    known = {}
    w = np.array([1, 0, 0, 2], np.float32)  # r0=(1,0), r1=(0,2) (test_embedding.cpp:26-33)
    for k, ids in {"single": [1], "dup": [1, 1], "two": [0, 1], "empty": []}.items():
        known[f"pool_{k}"] = ref.pool_ids(w, 2, [(0, 2)], ids)
    t = ref.init_rows(0, 100, 0, 100, 4, 19).ravel()  # sharded == whole (110-121)
    ids = [0, 29, 30, 70, 71, 99, 29]
    known["shard_whole"] = ref.pool_ids(t, 4, [(0, 100)], ids)
    known["shard_split"] = ref.pool_ids(t, 4, [(0, 30), (30, 71), (71, 100)], ids)
    for c in (4.0, 1.0):  # test_optimizer.cpp:50-94
        o = ref.adagrad_row_step([1.0, 1.0], 0.0, [2.0, 0.0], eta=0.1, eps=1e-8, c=c)
        known[f"adagrad_c{int(c)}_w"] = o["w"]
        known[f"adagrad_c{int(c)}_v"] = np.float32(o["v"])
        known[f"adagrad_c{int(c)}_lr"] = np.float64(o["effective_lr"])
    known["lpt_plan"] = ref.plan_greedy([(i, 6400, float(x), 100) for i, x in enumerate([7, 5, 4, 3, 1])], 2)
    known["rowwise_plan"] = ref.plan_greedy([(0, 640, 5.0, 10), (1, 640, 2.0, 10)], 3, "row-wise")
    rng = np.random.default_rng(5)
    rw = rng.standard_normal((64, 16)).astype(np.float32)
    rv = rng.random(64).astype(np.float32)
    rg = rng.standard_normal((64, 16)) * 1e-2
    known["rows_w"], known["rows_v"], known["rows_g"] = rw, rv, rg
    outw, outv = [], []
    for i in range(64):
        o = ref.adagrad_row_step(rw[i], rv[i], rg[i], eta=0.1, eps=1e-8, c=3.0)
        outw.append(o["w"])
        outv.append(o["v"])
    known["rows_w_out"], known["rows_v_out"] = np.array(outw, np.float32), np.array(outv, np.float32)
    np.savez_compressed(os.path.join(HERE, "known.npz"), **known)
    # ---- init_table ------------------------------------------------------
    np.savez_compressed(os.path.join(HERE, "init.npz"),
                        t3=ref.init_rows(3, 100, 0, 100, 16, 11), t0=ref.init_rows(0, 1000, 0, 1000, 64, 2),
                        t7=ref.init_rows(7, 5, 0, 5, 128, 123456789))
    # ---- mesh steps (tiny_options of test_trainer.cpp:19-39) -----------------
    mesh_case(ref, "mesh_8x1_row", 8, 1, "row-wise", 1.0, False, 1)
    mesh_case(ref, "mesh_4x2_row", 8, 2, "row-wise", 2.0, False, 1)
    mesh_case(ref, "mesh_2x4_table", 8, 4, "table-wise", 4.0, False, 1)
    mesh_case(ref, "mesh_2x2_sgd_sync3", 4, 2, "row-wise", 1.0, True, 3, steps=6)
    # ---- mixed dims / variable pooling / empty bags ------------------------------
    rows = np.array([3, 50, 1000, 7], np.uint32)
    dims = np.array([4, 8, 16, 32], np.uint32)
    spec = MeshSpec(rows=rows, dims=dims, plan=row_wise_plan(rows, 2), T=2, M=1, B=16, eta=0.1, c=2.0)
    st = MeshState.init(ref, spec, 4)
    mixed = dict(rows=rows, dims=dims)
    for step in range(3):
        Ls, Is, Us = [], [], []
        for r in range(2):
            g = np.random.default_rng([step, r, 9])
            lengths = g.integers(0, 12, size=16 * 4).astype(np.uint32)
            lengths[::5] = 0
            ids = np.concatenate([g.integers(0, rows[b % 4], size=lengths[b]) for b in range(64)]).astype(np.uint32)
            Ls.append(lengths)
            Is.append(ids)
            Us.append((1e-3 * g.standard_normal((16, int(dims.sum())))).astype(np.float32))
        pooled = st.step(ref, Ls, Is, Us, do_sync=False)
        for r in range(2):
            mixed[f"s{step}_r{r}_len"] = Ls[r]
            mixed[f"s{step}_r{r}_ids"] = Is[r]
            mixed[f"s{step}_r{r}_up"] = Us[r]
            mixed[f"s{step}_r{r}_pooled"] = pooled[r]
    mixed["w"], mixed["v"] = st.ws[0], st.vs[0]
    np.savez_compressed(os.path.join(HERE, "mixed.npz"), **mixed)
    # ---- cfg1 shapes (digests) ------------------------------------------------
    rows = np.full(8, 100_000, np.uint32)
    dims = np.full(8, 64, np.uint32)
    for c in (1.0, 4.0):
        spec = MeshSpec(rows=rows, dims=dims, plan=row_wise_plan(rows, 1), T=1, M=1, B=512, eta=0.1, c=c)
        st = MeshState.init(ref, spec, 2)
        cfg = {}
        for step in range(2):
            ids = ref.gen_batch_ids(7, step, 0, 8, 100_000, 1.0, 20, 512)
            up = (1e-3 * np.random.default_rng([step, 99]).standard_normal((512, 512))).astype(np.float32)
            pooled = st.step(ref, [np.full(512 * 8, 20, np.uint32)], [ids], [up], do_sync=False, threads=8)[0]
            cfg[f"s{step}_ids"] = ids
            cfg[f"s{step}_pooled_sha"] = digest(pooled)
        cfg["w_sha"], cfg["v_sha"] = digest(st.ws[0]), digest(st.vs[0])
        touched = np.nonzero(st.vs[0])[0][:64]
        cfg["sample_rows"] = touched
        cfg["sample_v"] = st.vs[0][touched]
        np.savez_compressed(os.path.join(HERE, f"cfg1_c{int(c)}.npz"), **cfg)
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
