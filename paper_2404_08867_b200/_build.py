"""Build liblq.so in-tree for sm_100a (and the C oracle, which is test-only).

    python -m paper_2404_08867_b200._build
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblq.so")
NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v",
    "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(REPO, "include"),
]


def _sources():
    return [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
            if f.endswith((".cu", ".cuh", ".h"))] + [os.path.join(REPO, "include", "lq.h")]


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def build_native(force=False, verbose=False):
    """Compile csrc/lq_api.cu (which includes the kernels) into liblq.so."""
    if not force and not _stale(LIB, _sources()):
        return LIB
    tmp = LIB + ".tmp"
    cmd = [NVCC, *NVCC_FLAGS, "-o", tmp, os.path.join(CSRC, "lq_api.cu"), os.path.join(CSRC, "lq_jit.cu"), "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    with open(os.path.join(CSRC, "ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


def build_oracle(force=False, verbose=False):
    """Compile the C oracle (test infrastructure) into oracle/build/liblqoracle.so."""
    src = os.path.join(REPO, "oracle", "c", "lq_oracle.c")
    if not os.path.exists(src):
        return None
    out_dir = os.path.join(REPO, "oracle", "build")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "liblqoracle.so")
    if not force and not _stale(out, [src]):
        return out
    cmd = ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off", "-o", out, src, "-lm"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("gcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        print(f"built {out}")
    return out


if __name__ == "__main__":
    build_native(force="--force" in sys.argv, verbose=True)
    build_oracle(force="--force" in sys.argv, verbose=True)
