"""Build the sm_100a C-ABI library in-tree (libensmhd_b200.so).

One nvcc invocation, `-gencode arch=compute_100a,code=sm_100a`, no torch
headers: the library exports only the plain C ABI of include/ensmhd_b200.h.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libensmhd_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


HOST_LIB = os.path.join(HERE, "libensmhd_host.so")
HOST_SRC = os.path.join(HERE, "csrc", "host_symbolic.cpp")


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def build_host(force: bool = False) -> str:
    """The host-side setup helpers (csrc/host_symbolic.cpp): C++ with OpenMP, g++ -O2 -fopenmp."""
    if not force and os.path.exists(HOST_LIB) and os.path.getmtime(HOST_LIB) >= os.path.getmtime(HOST_SRC):
        return HOST_LIB
    cmd = ["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-o", HOST_LIB + ".tmp", HOST_SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("g++ failed building libensmhd_host.so")
    os.replace(HOST_LIB + ".tmp", HOST_LIB)
    return HOST_LIB


def deps():
    return sources() + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
        os.path.join(ROOT, "include", "ensmhd_b200.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    build_host(force)
    if not force and up_to_date():
        return LIB
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-Xcompiler", "-fPIC", "-shared", "-I" + os.path.join(ROOT, "include"),
           "-o", LIB + ".tmp"] + sources() + ["-lcudart"]
    extra = os.environ.get("ENS_NVCC_EXTRA", "").split()   # diagnostic builds only (e.g. -DSG_PROBE)
    cmd[1:1] = extra
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libensmhd_b200.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
