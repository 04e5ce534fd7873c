"""Compile the CUDA library (sm_100a) in-tree: paper_1009_2768_b200/libtrmcr.so."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libtrmcr.so")
SRC = os.path.join(HERE, "csrc", "trmcr.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def nccl_dir() -> str:
    """NCCL 2.28 of the Python environment (the one torch.distributed loads)."""
    import nvidia.nccl
    return os.path.dirname(nvidia.nccl.__file__) if getattr(nvidia.nccl, "__file__", None) else list(nvidia.nccl.__path__)[0]


def nccl_flags():
    d = nccl_dir()
    return ["-I", os.path.join(d, "include"), "-L", os.path.join(d, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath=" + os.path.join(d, "lib")]


def sources():
    return [SRC] + glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "trmcr.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    # TRMCR_SPLIT_COMPILE=N: nvcc --split-compile N (development only: ~1 min instead of ~5, but the
    # generated code then depends on N and, measured, on what else the machine is compiling)
    split = ["--split-compile", os.environ["TRMCR_SPLIT_COMPILE"]] if os.environ.get("TRMCR_SPLIT_COMPILE") else []
    cmd = [NVCC, *FLAGS, *split, "-o", tmp, SRC, *nccl_flags()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as f:
        f.write(res.stderr)
    if verbose:
        print(res.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
