"""Build an experimental variant of libmmfhe.so with extra nvcc defines for one source.

    python tools/build_variant.py NAME SOURCE.cu -DFOO=1 [-DBAR=2 ...]

Compiles SOURCE with the defines into build/SOURCE.NAME.o, links it with the regular
objects of the other sources into paper_2603_22437_b200/lib/variants/libmmfhe_NAME.so.
Select it at run time with MMFHE_LIB=<path> (paper_2603_22437_b200/mmfhe.py)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_22437_b200 import build as b  # noqa: E402


def main():
    name, src, defs = sys.argv[1], sys.argv[2], sys.argv[3:]
    b.build()
    srcs, _ = b.sources()
    objs = [os.path.join(b.OBJ_DIR, s + ".o") for s in srcs if s != src]
    vobj = os.path.join(b.OBJ_DIR, f"{src}.{name}.o")
    cmd = [b.NVCC] + b.NVCC_FLAGS + defs + ["-c", os.path.join(b.CSRC, src), "-o", vobj]
    subprocess.run(cmd, check=True)
    out_dir = os.path.join(b.OUT_DIR, "variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"libmmfhe_{name}.so")
    subprocess.run([b.NVCC] + b.ARCH + ["-shared", "-cudart", "shared", "-o", out, vobj] + objs, check=True)
    print(out)


if __name__ == "__main__":
    main()
