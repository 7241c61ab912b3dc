"""Builds libsparse2d_b200.so in-tree for sm_100a.

    python -m paper_2508_03854_b200.build        # incremental
    python -m paper_2508_03854_b200.build --force

nvcc compiles every csrc/*.cu / *.cpp for `-gencode arch=compute_100a,
code=sm_100a` with -lineinfo and -fmad=false (the reference's
-ffp-contract=off numerics), links cudart statically and NCCL from the
torch-bundled nvidia-nccl wheel (the same libnccl.so.2 torch loads).
"""
from __future__ import annotations

import concurrent.futures as cf
import fcntl
import glob
import hashlib
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")
LIB = os.path.join(PKG, "libsparse2d_b200.so")
OBJ = os.path.join(PKG, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import importlib.util

    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is None or not spec.submodule_search_locations:
        raise RuntimeError("nvidia-nccl (torch's bundled NCCL) not found")
    return list(spec.submodule_search_locations)[0]


def _flags() -> list[str]:
    nd = nccl_dir()
    return [
        "-O3", "-std=c++17", "-lineinfo", "-fmad=false", *ARCH,
        "-Xcompiler", "-fPIC,-O3,-ffp-contract=off", "--expt-relaxed-constexpr",
        f"-I{INCLUDE}", f"-I{nd}/include", "-Xptxas", "-v",
    ]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers() -> list[str]:
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(INCLUDE, "sparse2d_b200.h")]


def _compile(src: str, flags: list[str], incremental: bool) -> tuple[str, str]:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if incremental and not _stale(obj, [src] + _headers()):
        return obj, ""
    cmd = [NVCC, "-c", src, "-o", obj, *flags]
    if src.endswith(".cpp"):
        cmd += ["-x", "cu"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


STAMP = LIB + ".stamp"


def source_hash() -> str:
    h = hashlib.sha256()
    for p in sorted(sources() + _headers()):
        h.update(os.path.basename(p).encode())
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH).encode())
    return h.hexdigest()


def up_to_date() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return False
    with open(STAMP) as f:
        return f.read().strip() == source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    """Build unless the stamp (sha256 of sources + headers) matches.  A file
    lock serialises concurrent builders (e.g. torchrun ranks)."""
    os.makedirs(OBJ, exist_ok=True)
    with open(os.path.join(OBJ, ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)
        try:
            if not force and up_to_date():
                return LIB
            return _build_locked(force, verbose)
        finally:
            fcntl.flock(lk, fcntl.LOCK_UN)


def _build_locked(force: bool, verbose: bool) -> str:
    srcs = sources()
    flags = _flags()
    # object files are reused only when the previous library is present
    # (a fresh checkout / GPU-box snapshot recompiles everything)
    incremental = not force and os.path.exists(LIB)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, flags, incremental), srcs))
    log = "\n".join(r[1] for r in results if r[1])
    with open(os.path.join(OBJ, "ptxas.log"), "w") as f:
        f.write(log)
    if verbose:
        print(log)
    nd = nccl_dir()
    cmd = [NVCC, "-shared", *ARCH, "-o", LIB + ".tmp", *[r[0] for r in results],
           "-cudart", "static", f"-L{nd}/lib", "-l:libnccl.so.2",
           "-Xlinker", f"-rpath,{nd}/lib"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    with open(STAMP, "w") as f:
        f.write(source_hash())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
