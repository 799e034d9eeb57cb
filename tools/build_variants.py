"""Build liblq variants with extra -D flags (A/B timing of kernel changes):

    python tools/build_variants.py NAME=-DFOO=1,-DBAR=0 NAME2=...

Outputs build/variants/liblq_NAME.so; time them with
    LQ_LIB_PATH=build/variants/liblq_NAME.so python tools/orbit_variant.py 5
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_08867_b200 import _build as B  # noqa: E402

OUT = os.path.join(B.REPO, "build", "variants")


def build(spec):
    name, _, flags = spec.partition("=")
    defs = [f for f in flags.split(",") if f]
    out = os.path.join(OUT, f"liblq_{name}.so")
    cmd = [B.NVCC, *B.NVCC_FLAGS, *defs, "-o", out, os.path.join(B.CSRC, "lq_api.cu"),
           os.path.join(B.CSRC, "lq_jit.cu"), "-ldl"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode:
        raise SystemExit(f"{name}: nvcc failed\n{res.stderr[-3000:]}")
    with open(os.path.join(OUT, f"ptxas_{name}.log"), "w") as fh:
        fh.write(res.stderr)
    return out


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    with ThreadPoolExecutor(4) as ex:
        for out in ex.map(build, sys.argv[1:]):
            print("built", out)
