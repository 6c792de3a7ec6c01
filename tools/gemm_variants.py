"""Build variants of libtally_b200.so that differ only in one source file's
compile-time constants (default kernels_gemm.cu; experiments -- the product
build is build.py):

    python tools/gemm_variants.py NAME [--src=kernels_nn.cu,kernels_tf.cu] -DTALLY_STAGES_BF16_N128=4 ...
    TALLY_LIB_PATH=paper_2410_07381_b200/_lib/variants/NAME.so python tools/gemm_shapes.py
"""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2410_07381_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    srcs = ["kernels_gemm.cu"]
    if defs and defs[0].startswith("--src="):
        srcs, defs = defs[0][6:].split(","), defs[1:]
    B.build()
    vdir = os.path.join(B.HERE, "_lib", "variants")
    os.makedirs(vdir, exist_ok=True)
    objs = {}
    for src in srcs:
        obj = os.path.join(vdir, name + "_" + src + ".o")
        subprocess.run([B.NVCC] + B.CU_FLAGS + defs + ["-c", os.path.join(B.CSRC, src), "-o", obj], check=True)
        objs[src] = obj
    allobjs = [objs.get(s, os.path.join(B.OBJ, s + ".o")) for s in B.SOURCES]
    lib = os.path.join(vdir, name + ".so")
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-o", lib] + allobjs + ["-lcudart", "-lpthread", "-ldl", "-lrt"],
                   check=True)
    print(lib)


if __name__ == "__main__":
    main()
