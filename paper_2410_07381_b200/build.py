"""Build libtally_b200.so in-tree with nvcc for sm_100a.

    python paper_2410_07381_b200/build.py          # incremental
    python paper_2410_07381_b200/build.py --force  (or __graft_entry__.build())

Output: paper_2410_07381_b200/_lib/libtally_b200.so (git-ignored; travels to
the GPU box with the gpurun snapshot).  Cross-compiles without a GPU.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_lib", "obj")
LIB = os.path.join(HERE, "_lib", "libtally_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-Wall,-Wno-format-truncation",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]
CU_FLAGS = ARCH + COMMON + ["-Xptxas", "-warn-spills", "--expt-relaxed-constexpr"]
# experiments only: extra -D flags (e.g. TALLY_NVCC_DEFINES="-DFOO=1"); a
# build with them is a different library -- force a rebuild after changing it
CU_FLAGS += os.environ.get("TALLY_NVCC_DEFINES", "").split()

SOURCES = ["runtime.cu", "kernels_basic.cu", "kernels_gemm.cu", "kernels_nn.cu", "kernels_tf.cu", "runner.cpp", "cuda_device.cpp"]
HEADERS = ["tally_device.cuh", "registry.h", "runtime.h", "runner.h", "epilogue.cuh", "bnfuse.cuh"]


def _deps_mtime():
    paths = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "tally_b200.h")]
    return max(os.path.getmtime(p) for p in paths if os.path.exists(p))


def _compile(src, force):
    path = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src + ".o")
    if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(
            os.path.getmtime(path), _deps_mtime()):
        return obj, None
    flags = CU_FLAGS + (["-x", "cu"] if src.endswith(".cpp") else [])
    cmd = [NVCC] + flags + ["-c", path, "-o", obj]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        return obj, f"$ {' '.join(cmd)}\n{p.stdout}\n{p.stderr}"
    return obj, None


def build(force: bool = False, verbose: bool = False) -> str:
    if shutil.which(NVCC) is None and not os.path.exists(NVCC):
        raise RuntimeError(f"nvcc not found at {NVCC}")
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), SOURCES))
    errs = [e for _, e in results if e]
    if errs:
        raise RuntimeError("libtally_b200 build failed:\n" + "\n".join(errs))
    objs = [o for o, _ in results]
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart", "-lpthread", "-ldl", "-lrt"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError(f"link failed:\n$ {' '.join(cmd)}\n{p.stdout}\n{p.stderr}")
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
