"""Build libh2f.so (sm_100a) in-tree with nvcc.

    python -m paper_2509_11152_b200.build      # or __graft_entry__.build()

Objects go to paper_2509_11152_b200/_build/, the library next to this file,
so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
# development builds: H2F_BUILD_DIR / H2F_LIB_OUT elsewhere, H2F_NVCC_DEFS extra -D flags
OUT = os.environ.get("H2F_BUILD_DIR", os.path.join(HERE, "_build"))
LIB = os.environ.get("H2F_LIB_OUT", os.path.join(HERE, "libh2f.so"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-Wno-deprecated-gpu-targets", "-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3", "-I", CSRC,
          "-I", os.path.join(os.path.dirname(HERE), "include")] + \
    [f"-D{d}" for d in os.environ.get("H2F_NVCC_DEFS", "").split(",") if d]
SOURCES = ["k_gemm.cu", "k_dense.cu", "k_hh.cu", "dense.cpp", "k_solve.cu", "k_top.cu", "runtime.cpp", "h2mat.cpp", "factor.cpp",
           "solve.cpp", "api.cpp", "k_build.cu", "build.cpp"]


def _obj(src):
    return os.path.join(OUT, os.path.splitext(src)[0] + ".o")


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))] + [
        os.path.join(os.path.dirname(HERE), "include", "h2f.h")]


def _compile(src, verbose):
    path = os.path.join(CSRC, src)
    cmd = [NVCC, *ARCH, *COMMON, "-c", path, "-o", _obj(src)]
    if src.endswith(".cu") and verbose:
        cmd += ["-Xptxas", "-v"]
    if src.endswith(".cpp"):
        cmd = [NVCC, *COMMON, "-Xcompiler", "-fopenmp", "-x", "c++", "-c", path, "-o", _obj(src)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{res.stderr}")
    return src, res.stderr


def build(verbose=False, force=False):
    os.makedirs(OUT, exist_ok=True)
    hdrs = _headers()
    todo = [s for s in SOURCES if force or _stale(_obj(s), [os.path.join(CSRC, s), *hdrs])]
    if todo:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(todo))) as ex:
            for src, err in ex.map(lambda s: _compile(s, verbose), todo):
                if verbose and err:
                    print(f"[{src}]\n{err}", file=sys.stderr)
    objs = [_obj(s) for s in SOURCES]
    if force or todo or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart", "-lgomp"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed:\n{res.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
