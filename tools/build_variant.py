"""Experiment builds: recompile one CUDA source with extra -D flags and link a
separate libckv_b200_<tag>.so beside the product library (load it with
CKV_LIB=<path>).  The product build (paper_2412_03213_b200/build.py) is not
touched.

    python tools/build_variant.py ckv_attend.cu t64s3 -DCKV_AT_TILE=64 -DCKV_AT_STAGES=3
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_03213_b200 import build as B  # noqa: E402


def main():
    src, tag, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    B.build()
    objs = [os.path.join(B.BUILD, f + ".o") for f in B.sources()]
    vobj = os.path.join(B.BUILD, f"{src}.{tag}.o")
    cmd = [B.NVCC, *B.ARCH, *B.FLAGS, "-std=c++17", *defs, "-c", os.path.join(B.CSRC, src),
           "-o", vobj]
    subprocess.run(cmd, check=True, capture_output=True)
    objs = [vobj if os.path.basename(o) == src + ".o" else o for o in objs]
    out = os.path.join(B.PKG, f"libckv_b200_{tag}.so")
    subprocess.run([B.NVCC, *B.ARCH, "-shared", "-o", out, *objs, "-lcudart"], check=True)
    print(out)


if __name__ == "__main__":
    main()
