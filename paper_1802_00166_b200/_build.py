"""Build libpcotgpu.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_1802_00166_b200._build     # or __graft_entry__.build()
"""
import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIB = os.path.join(PKG, "libpcotgpu.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + CSRC,
          "-I" + os.path.join(REPO, "include")]
# Stencil bit-exactness: every update is written with __d*_rn intrinsics, and
# -fmad=false additionally forbids contraction anywhere in these units.
CU_FLAGS = {
    "stencil2d.cu": ["-fmad=false"],
    "stencil3d.cu": ["-fmad=false"],
    "gs2d.cu": ["-fmad=false"],
    "misc.cu": ["-fmad=false"],
    "dgemm.cu": [],
    "generic.cu": ["-fmad=false"],
}
CPP = ["spec.cpp", "executor.cpp"]
# headers each unit includes (a kernel unit does not rebuild when the host
# headers change: stencil2d.cu alone takes minutes)
KERNEL_DEPS = ["common.cuh", "kernels.h"]
HOST_DEPS = ["common.cuh", "kernels.h", "spec.h", "generic.h"]


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def _compile(src, flags):
    out = os.path.join(OBJ, os.path.basename(src) + ".o")
    base = os.path.basename(src)
    if base in ("stencil2d.cu", "stencil3d.cu", "gs2d.cu", "dgemm.cu", "misc.cu"):
        deps = [os.path.join(CSRC, d) for d in KERNEL_DEPS] + [src]
    else:
        deps = [os.path.join(CSRC, d) for d in HOST_DEPS] + [src,
                os.path.join(REPO, "include", "pcotgpu.h"), os.path.join(REPO, "include", "pcot_gpu.hpp")]
    if not _stale(out, deps):
        return out, None
    # PCOTGPU_NVCC_EXTRA: development experiments (e.g. -D switches); touch the
    # source to force a rebuild with them
    extra = os.environ.get("PCOTGPU_NVCC_EXTRA", "").split()
    cmd = [NVCC] + ARCH + COMMON + flags + extra + ["-c", src, "-o", out]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        return out, "FAILED: %s\n%s%s" % (" ".join(cmd), p.stdout, p.stderr)
    return out, None


def build(verbose=False):
    os.makedirs(OBJ, exist_ok=True)
    jobs = [(os.path.join(CSRC, f), fl) for f, fl in CU_FLAGS.items()]
    jobs += [(os.path.join(CSRC, f), []) for f in CPP]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        res = list(ex.map(lambda j: _compile(*j), jobs))
    errs = [e for _, e in res if e]
    if errs:
        raise RuntimeError("\n".join(errs))
    objs = [o for o, _ in res]
    if _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart"]
        p = subprocess.run(cmd, capture_output=True, text=True)
        if p.returncode != 0:
            raise RuntimeError("link failed: %s\n%s" % (p.stdout, p.stderr))
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
