"""Build libkkrx.so (in-tree) with nvcc for sm_100a.

    python -m paper_2108_07004_b200.build        (or __graft_entry__.build())
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libkkrx.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
         "-Xptxas", "-v", "-I", os.path.join(os.path.dirname(HERE), "include")]
SOURCES = ["kk_rx.cu", "kk_kernels.cu", "kk_constellation.cpp"]
# comparison only (include/kk_cufft_cmp.h): the cuFFT multi-kernel S1-S4 pipeline
CMP_OUT = os.path.join(HERE, "libkkrx_cufft.so")
CMP_SOURCES = ["kk_cufft_cmp.cu"]
CUDA_LIB = os.path.join(os.path.dirname(os.path.dirname(NVCC)), "lib64")


def build_cmp(verbose=False, force=False):
    """libkkrx_cufft.so: the cuFFT comparison pipeline (never the product path)."""
    srcs = [os.path.join(CSRC, s) for s in CMP_SOURCES]
    deps = srcs + [os.path.join(os.path.dirname(HERE), "include", "kk_cufft_cmp.h")]
    if not force and os.path.exists(CMP_OUT) and all(os.path.getmtime(CMP_OUT) >= os.path.getmtime(d) for d in deps):
        return CMP_OUT
    cmd = [NVCC, *ARCH, *FLAGS, "-shared", "-o", CMP_OUT + ".tmp", *srcs, "-cudart", "static",
           "-L", CUDA_LIB, "-lcufft", "-Xlinker", "-rpath=" + CUDA_LIB]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed (%d)" % r.returncode)
    os.replace(CMP_OUT + ".tmp", CMP_OUT)
    return CMP_OUT


def build(verbose=False, force=False, out=None, csrc=None, include=None):
    """out/csrc/include: build another variant (tools/ab_build.py); default = the in-tree library."""
    OUT_ = out or OUT
    CSRC_ = csrc or CSRC
    INC_ = include or os.path.join(os.path.dirname(HERE), "include")
    srcs = [os.path.join(CSRC_, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC_, f) for f in os.listdir(CSRC_) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(INC_, "kk_rx.h"))
    if not force and os.path.exists(OUT_) and all(os.path.getmtime(OUT_) >= os.path.getmtime(d) for d in deps):
        return OUT_
    flags = [f if f != os.path.join(os.path.dirname(HERE), "include") else INC_ for f in FLAGS]
    flags += os.environ.get("KK_EXTRA_NVCC_FLAGS", "").split() if out is not None else []
    cmd = [NVCC, *ARCH, *flags, "-shared", "-o", OUT_ + ".tmp", *srcs, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed (%d)" % r.returncode)
    os.replace(OUT_ + ".tmp", OUT_)
    with open(os.path.join(HERE, "build.log" if out is None else "build_variant.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    return OUT_


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
    print(build_cmp(verbose=True, force="--force" in sys.argv))
