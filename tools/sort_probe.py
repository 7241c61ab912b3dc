"""Writes the (slot, gradient-row) pairs of one config-2 step (N = 1) as the
lookup emits them, plus their dense-rank keys, for tools/sort_probe.cu."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2508_03854_b200 import workloads  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
w = workloads.get("cfg2")
lengths, ids = w.batch_for(7, 0, 0)
F, B = w.F, w.batch
vbase = np.concatenate([[0], np.cumsum(np.array(w.rows, np.uint64))])[:-1]
feat = np.repeat(np.tile(np.arange(F), B), lengths)
bag = np.repeat(np.arange(B * F), lengths)
keys = (vbase[feat] + ids).astype(np.uint32)
vals = ((bag // F) * (w.sum_dims // 4) + feat * 32).astype(np.uint32)
keys.tofile(os.path.join(out, "keys.bin"))
vals.tofile(os.path.join(out, "vals.bin"))
u, dense = np.unique(keys, return_inverse=True)
dense.astype(np.uint32).tofile(os.path.join(out, "dense.bin"))
print("nnz", len(keys), "unique", len(u))
