"""Build libad2.so (the CUDA path) in-tree for sm_100a.

    python -m paper_1510_00012_b200.build        # nvcc -gencode arch=compute_100a,code=sm_100a

The .so is written next to this file so it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libad2.so")
SO_CHECKED = os.path.join(HERE, "libad2_checked.so")      # device assertions on (-DAD2_CHECKS)
CSRC = os.path.join(HERE, "csrc")
SRCS = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))
DEPS = SRCS + sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))) + \
    [os.path.join(ROOT, "include", "ad2.h"), os.path.abspath(__file__)]
OBJ_DIR = os.path.join(ROOT, "build", "obj")
OBJ_DIR_CHECKED = os.path.join(ROOT, "build", "obj_checked")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-diag-suppress", "128"]


def needs_build(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """nvcc each translation unit for sm_100a (in parallel), then link libad2.so (checked: the
    same sources with device assertions, libad2_checked.so)."""
    so, obj_dir = (SO_CHECKED, OBJ_DIR_CHECKED) if checked else (SO, OBJ_DIR)
    if not (force or needs_build(so)):
        return so
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(obj_dir, exist_ok=True)
    objs = [os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o") for src in SRCS]
    extra = ["-DAD2_CHECKS"] if checked else []

    def cc(pair):
        src, obj = pair
        cmd = [NVCC] + CFLAGS + extra + (["-Xptxas", "-v"] if verbose else []) + ["-c", "-o", obj, src]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
        return r.stderr

    with ThreadPoolExecutor(max_workers=min(len(SRCS), os.cpu_count() or 4)) as ex:
        logs = list(ex.map(cc, zip(SRCS, objs)))
    if verbose:
        print("".join(logs))
    tmp = so + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"])
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
