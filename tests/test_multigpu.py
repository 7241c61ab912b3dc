"""Mesh parity of the 2D step (tests/mp_parity.py).

* test_mesh_parity_local: the T ranks run as virtual ranks (threads of one
  process sharing one GPU over a LocalHub) -- every N > 1 kernel (K1
  bucketing, the fused id / pooled / gradient exchanges, the combine, the
  device barriers, the K5 replica sync) runs on a single B200.
* test_mesh_parity: one process per GPU under torchrun with NCCL + CUDA IPC
  over NVLink; needs >= T GPUs.
"""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


CASES = [
    (2, 1, "row-wise", []),
    (2, 1, "table-wise", []),
    (2, 2, "row-wise", ["--ckpt"]),
    (4, 2, "row-wise", ["--sync-interval", "2", "--steps", "4", "--ckpt"]),
    (4, 1, "table-wise", ["--sgd"]),
    (4, 4, "table-wise", []),
    (2, 1, "table-wise", ["--engine-out", "--ckpt"]),
    (4, 2, "table-wise", ["--engine-out"]),
    (4, 1, "table-wise", ["--mixed-out"]),
    (2, 1, "row-wise", ["--mean"]),
    (4, 2, "table-wise", ["--mean", "--engine-out"]),
    (4, 2, "row-wise", ["--bf16", "--steps", "3"]),
    (2, 1, "row-wise", ["--bf16", "--steps", "3"]),
    (2, 1, "table-wise", ["--bad-id"]),
    (4, 2, "table-wise", ["--sync-interval", "2", "--steps", "4", "ENV:S2D_SYNC_NCCL=1"]),
    (4, 2, "row-wise", ["--sync-interval", "2", "--steps", "4", "ENV:S2D_SYNC_SNAPSHOT=0"]),
    (4, 2, "row-wise", ["--sync-interval", "2", "--steps", "4", "ENV:S2D_SNAP_DENSE=1"]),
    (2, 2, "table-wise", ["--mean", "ENV:S2D_SNAP_DENSE=1"]),
    (2, 2, "row-wise", ["--steps", "4", "ENV:S2D_SYNC_LIST=1"]),
    (4, 2, "table-wise", ["--sync-interval", "2", "--steps", "4", "ENV:S2D_SYNC_LIST=1"]),
    (2, 2, "table-wise", ["--sgd", "--steps", "3"]),
    (3, 3, "row-wise", ["--steps", "3"]),
    (4, 1, "row-wise", ["--bad-id"]),
]


def _case_id(c):
    T, M, strategy, extra = c
    return (f"T{T}-M{M}-{strategy}" + "".join(x.replace("--", "-") for x in extra if x.startswith("--")) +
            "".join("-nccl-sync" for x in extra if x.startswith("ENV:S2D_SYNC_NCCL")) +
            "".join("-slice-sync" for x in extra if x.startswith("ENV:S2D_SYNC_SNAPSHOT")) +
            "".join("-dense-log" for x in extra if x.startswith("ENV:S2D_SNAP_DENSE")) +
            "".join("-dirty-list" for x in extra if x.startswith("ENV:S2D_SYNC_LIST")))


def _env_args(extra):
    env = dict(os.environ)
    for x in extra:  # "ENV:K=V" entries set the environment of the ranks
        if x.startswith("ENV:"):
            k, v = x[4:].split("=", 1)
            env[k] = v
    return env, [x for x in extra if not x.startswith("ENV:")]


@pytest.mark.parametrize("T,M,strategy,extra", CASES, ids=[_case_id(c) for c in CASES])
def test_mesh_parity_local(T, M, strategy, extra):
    if _ngpu() < 1:
        pytest.skip("needs a GPU")
    env, args = _env_args(extra)
    cmd = [sys.executable, os.path.join(ROOT, "tests", "mp_parity.py"), "--local", str(T), "--groups", str(M),
           "--strategy", strategy, *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MP PARITY OK" in r.stdout


@pytest.mark.multigpu
@pytest.mark.parametrize("T,M,strategy,extra", CASES, ids=[_case_id(c) for c in CASES])
def test_mesh_parity(T, M, strategy, extra):
    if _ngpu() < T:
        pytest.skip(f"needs {T} GPUs")
    port = 29500 + 7 * T + M + (0 if strategy == "row-wise" else 50) + (100 if extra else 0)
    env = dict(os.environ)
    for x in extra:  # "ENV:K=V" entries set the environment of the ranks
        if x.startswith("ENV:"):
            k, v = x[4:].split("=", 1)
            env[k] = v
            port += 13
    args = [x for x in extra if not x.startswith("ENV:")]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node", str(T), "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mp_parity.py"), "--groups",
           str(M), "--strategy", strategy, *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MP PARITY OK" in r.stdout
