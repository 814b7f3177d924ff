"""Build libccdk.so variants with extra -D flags for on-GPU A/B timing.

    python tools/build_variant.py NAME -DCCDK_GEN_MINB=5 -DCCDK_GEN_STAGES=1
    CCDK_LIB=paper_2112_06300_b200/lib/variants/NAME/libccdk.so python bench.py ...
"""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_06300_b200 import build as b

name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(b.LIB, "variants", name)
os.makedirs(out, exist_ok=True)
objs = []
for src in b.CU_SOURCES:
    o = os.path.join(out, src + ".o")
    subprocess.run([b.NVCC, *b.NVCC_FLAGS, *defs, "-I", b.INCLUDE, "-I", b.CSRC, "-c",
                    os.path.join(b.CSRC, src), "-o", o], check=True)
    objs.append(o)
subprocess.run([b.NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs, "-o",
                os.path.join(out, "libccdk.so"), "-cudart", "static"], check=True)
for o in objs:
    os.remove(o)
print(os.path.join(out, "libccdk.so"))
