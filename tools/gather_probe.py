"""Probe: how fast can B200 gather cfg2-shaped rows?  Compares torch
embedding_bag / index_select (library kernels, f32 accumulation) with our
lookup kernel, on Zipf ids (cfg2) and on uniform ids.  Diagnostics only."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_03854_b200 as s2d  # noqa: E402
from paper_2508_03854_b200 import workloads  # noqa: E402


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def main():
    w = workloads.get("cfg2")
    lengths, ids = w.batch_for(1, 0, 0)
    F, B = w.F, w.batch
    rows = np.array(w.rows, np.int64)
    base = np.concatenate([[0], np.cumsum(rows)[:-1]])
    feat = np.repeat(np.tile(np.arange(F), B), lengths)
    gids = ids.astype(np.int64) + base[feat]
    total = int(rows.sum())
    weight = torch.randn(total, 128, device="cuda") * 0.01
    offsets = torch.from_numpy(np.concatenate([[0], np.cumsum(lengths)[:-1]]).astype(np.int64)).cuda()
    for name, g in [("zipf", gids), ("uniform", np.random.default_rng(0).integers(0, total, len(gids)))]:
        gi = torch.from_numpy(g).cuda()
        t_eb = timeit(lambda: torch.nn.functional.embedding_bag(gi, weight, offsets, mode="sum"))
        t_is = timeit(lambda: torch.index_select(weight, 0, gi))
        nbytes = len(g) * 512
        print(f"{name:8s} embedding_bag {t_eb*1e3:7.1f} us ({nbytes/t_eb/1e6:6.0f} GB/s)   "
              f"index_select {t_is*1e3:7.1f} us ({2*nbytes/t_is/1e6:6.0f} GB/s rd+wr)")
    # our lookup on zipf and uniform ids (forward only)
    tables = [s2d.TableConfig(int(r), 128) for r in w.rows]
    eng = s2d.Sparse2DEmbedding(tables, s2d.Topology(1, 1), strict=False)
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    eng.set_stream(st.cuda_stream)
    eng.init_tables(1)
    pooled = torch.empty((B, w.sum_dims), device="cuda")
    dl = torch.from_numpy(lengths.view(np.int32)).cuda()
    for name, idv in [("zipf", ids), ("uniform", (np.random.default_rng(1).random(len(ids)) * rows[feat]).astype(np.uint32))]:
        di = torch.from_numpy(idv.view(np.int32)).cuda()
        eng.set_profiling(True)
        t = timeit(lambda: eng.forward(dl, di, pooled, batch=B))
        ph = eng.phase_times()
        eng.set_profiling(False)
        n = ph["lookup"][1]
        print(f"{name:8s} s2d forward {t*1e3:7.1f} us  lookup kernel {ph['lookup'][0]/n*1e3:7.1f} us "
              f"({len(idv)*512/(ph['lookup'][0]/n)/1e6:6.0f} GB/s of rows)")


if __name__ == "__main__":
    main()
