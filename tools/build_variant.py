"""Experiment builds: liblv with extra -D defines on one source (default lv_score.cu; VARIANT_SRC
picks another; the other objects are the main build's), written to
paper_2410_22347_b200/variants/liblv_<name>.so; select with LV_LIB=<path>.

  python tools/build_variant.py spin_mma -DLV_MMA_SPIN
  VARIANT_SRC=lv_rerank.cu python tools/build_variant.py k5g4 -DLV_K5_G4
  VARIANT_SRC=all python tools/build_variant.py checks -DLV_CHECKS      # every source
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_22347_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    B.build()
    out_dir = os.path.join(B.HERE, "variants")
    os.makedirs(out_dir, exist_ok=True)
    src = os.environ.get("VARIANT_SRC", "lv_score.cu")
    srcs = B.SOURCES if src == "all" else [src]
    objs = []
    for sname in srcs:
        obj = os.path.join(out_dir, f"{sname[:-3]}_{name}.o")
        r = subprocess.run([B.NVCC, *B.FLAGS, *defs, "-c", os.path.join(B.CSRC, sname), "-o", obj],
                           capture_output=True, text=True)
        if r.returncode:
            sys.exit(r.stderr)
        objs.append(obj)
    objs += [os.path.join(B.CSRC, s.replace(".cu", ".o")) for s in B.SOURCES if s not in srcs]
    lib = os.path.join(out_dir, f"liblv_{name}.so")
    r = subprocess.run([B.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o", lib],
                       capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr)
    print(lib)


if __name__ == "__main__":
    main()
