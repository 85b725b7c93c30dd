"""Build libmoe.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2502_06643_b200.build [--force] [--verbose]

The library links against the NCCL that ships with torch's venv (2.28.x), so
one libnccl copy is loaded per process.  The .so is written next to this file
(git-ignored, but it travels to the GPU box with the gpurun snapshot).
"""

import argparse
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmoe.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dir():
    import nvidia.nccl as n  # torch's NCCL wheel
    return list(n.__path__)[0]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "moe.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False, extra=()):
    if not force and not _stale():
        return LIB
    nd = nccl_dir()
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
           *sources(), "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + os.path.join(nd, "lib"), "-o", LIB + ".tmp", *extra]
    if verbose:
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libmoe.so")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas-v", action="store_true")
    ap.add_argument("--define", action="append", default=[], help="extra -D macro (A/B experiments)")
    a = ap.parse_args()
    extra = (["-Xptxas", "-v"] if a.ptxas_v else []) + ["-D" + d for d in a.define]
    print(build(force=a.force or bool(extra), verbose=a.verbose, extra=extra))
