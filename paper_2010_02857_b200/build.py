"""Build libifgf.so in-tree with nvcc for sm_100a (used by __graft_entry__.build)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libifgf.so")
SOURCES = ["plan.cu", "apply.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir() -> str | None:
    """The NCCL that torch loads (nvidia-nccl wheel): libifgf links the same
    libnccl.so.2 so that one NCCL instance serves torch and the library."""
    import site
    for sp in site.getsitepackages() + [site.getusersitepackages()]:
        d = os.path.join(sp, "nvidia", "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    return None


NCCL_DIR = _nccl_dir()
NCCL_INC = ["-I", os.path.join(NCCL_DIR, "include")] if NCCL_DIR else []
NCCL_LINK = (["-L", os.path.join(NCCL_DIR, "lib"), "-Xlinker", "-rpath=" + os.path.join(NCCL_DIR, "lib")]
             if NCCL_DIR else []) + ["-l:libnccl.so.2"]

# IFGF_CHECKS=1: debug build with device-side bounds checks (IFGF_DCHECK).
CHECKS = os.environ.get("IFGF_CHECKS", "0") not in ("", "0")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    *(["-DIFGF_CHECKS"] if CHECKS else []),
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
    *NCCL_INC,
]


def _newest_input_mtime() -> float:
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh", ".h"))]
    files += [os.path.join(ROOT, "include", "ifgf.h"), __file__]
    return max(os.path.getmtime(f) for f in files)


def build(force: bool = False, verbose: bool = False) -> str:
    stamp = LIB + ".checks"
    if CHECKS != os.path.exists(stamp):
        force = True  # switching between the release and the bounds-checked build
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _newest_input_mtime():
        return LIB
    objs = []
    logs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src.replace(".cu", ".o"))
        cmd = [NVCC, *NVCC_FLAGS, "-dc", os.path.join(CSRC, src), "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", tmp, "-lcudart", *NCCL_LINK]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    if CHECKS:
        open(stamp, "w").close()
    elif os.path.exists(stamp):
        os.remove(stamp)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
