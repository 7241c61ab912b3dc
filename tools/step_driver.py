"""Runs K untimed steps of a workload on one GPU -- the command profiled with
ncu (see profiles/README.md).  Not a benchmark: no timing is reported."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="cfg2")
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--batch", type=int, default=None)
    p.add_argument("--mesh", default=None, help="NxM: run the mesh as virtual ranks on GPU 0 (LocalHub)")
    a = p.parse_args()
    if a.mesh:
        return mesh_main(a)
    import torch

    import paper_2508_03854_b200 as s2d
    from paper_2508_03854_b200 import workloads

    w = workloads.get(a.config)
    if a.batch:
        w.batch = a.batch
    tables = [s2d.TableConfig(int(r), int(d), 1.0) for r, d in zip(w.rows, w.dims)]
    eng = s2d.Sparse2DEmbedding(tables, s2d.Topology(1, 1), strategy=w.strategy,
                                optimizer=s2d.OptimizerConfig(eta=w.eta, c=w.c), weight_dtype=w.dtype, strict=False)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    eng.set_stream(st.cuda_stream)
    eng.init_tables(1)
    lengths, ids = w.batch_for(1, 0, 0)
    up = torch.from_numpy(w.upstream_for(1, 0, 0)).cuda()
    dl = torch.from_numpy(lengths.view(np.int32)).cuda()
    di = torch.from_numpy(ids.view(np.int32)).cuda()
    pooled = torch.empty((w.batch, w.sum_dims), dtype=torch.float32, device="cuda")
    for _ in range(a.steps):
        eng.forward(dl, di, pooled, batch=w.batch)
        eng.backward_update(up)
    eng.synchronize()
    print("steps done", a.steps, eng.stats())


def mesh_main(a):
    """The N>1 kernels (bucketing, fused exchanges, combine, grad gather,
    replica sync) on one GPU: every rank a thread-driven virtual rank."""
    import paper_2508_03854_b200 as s2d
    from paper_2508_03854_b200 import workloads

    n, m = (int(x) for x in a.mesh.lower().split("x"))
    T = n * m
    w = workloads.get(a.config)
    if a.batch:
        w.batch = a.batch
    w.mesh = (n, m)
    tables = [s2d.TableConfig(int(r), int(d), w.plan_cost(f, n)) for f, (r, d) in enumerate(zip(w.rows, w.dims))]
    plan = w.table_plan(n) if (w.strategy == "table-wise" and n > 1) else None
    engs = s2d.local_mesh(tables, s2d.Topology(T, m), strategy=w.strategy, plan=plan,
                          optimizer=s2d.OptimizerConfig(eta=w.eta, c=float(m)), weight_dtype=w.dtype, strict=False)
    s2d.run_ranks(lambda r: engs[r].init_tables(1), T)
    ins = [w.batch_for(1, 0, r) + (w.upstream_for(1, 0, r),) for r in range(T)]

    def go(r):
        for _ in range(a.steps):
            engs[r].forward(ins[r][0], ins[r][1])
            engs[r].backward_update(ins[r][2])
            if m > 1:
                engs[r].sync_replicas()
        engs[r].synchronize()
        return engs[r].stats()

    st = s2d.run_ranks(go, T)
    print("mesh steps done", a.steps, [(x["nnz_owned"], x["unique_rows"], x["dirty_rows"]) for x in st])
    for e in engs:
        e.close()


if __name__ == "__main__":
    main()
