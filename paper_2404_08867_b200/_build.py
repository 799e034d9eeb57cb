"""Build liblq.so in-tree for sm_100a.

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
    # ptxas register/spill report of the last build (untracked; copies that
    # matter for a profile go to profiles/)
    os.makedirs(os.path.join(REPO, "build"), exist_ok=True)
    with open(os.path.join(REPO, "build", "ptxas.log"), "w") as fh:
        fh.write(res.stderr)
    os.replace(tmp, LIB)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build_native(force="--force" in sys.argv, verbose=True)
