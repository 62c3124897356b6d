"""Build libasse.so in-tree for sm_100a (nvcc, static cudart)."""
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libasse.so")
SRCS = [os.path.join(PKG, "csrc", f) for f in ("asse_api.cu", "asse_kernels.cuh", "asse_scan_bin.cuh", "asse_scan_own.cuh", "asse_tma.cuh")] + [
    os.path.join(ROOT, "include", "asse.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-cudart", "static"]


def build(force=False, verbose=False):
    if not force and os.path.exists(LIB) and all(
            os.path.getmtime(s) <= os.path.getmtime(LIB) for s in SRCS):
        return LIB
    cmd = [NVCC, *FLAGS, "-shared", "-I", os.path.join(ROOT, "include"),
           os.path.join(PKG, "csrc", "asse_api.cu"), "-o", LIB + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(out_path, defines=(), verbose=False):
    """Build libasse with extra -D defines into out_path (tools/sweep.py). Never touches
    the product library."""
    extra = os.environ.get("ASSE_NVCC_EXTRA", "").split()   # tools only: compiler-option sweeps
    cmd = [NVCC, *FLAGS, *extra, "-shared", "-I", os.path.join(ROOT, "include"),
           *["-D" + d for d in defines], os.path.join(PKG, "csrc", "asse_api.cu"), "-o", out_path + ".tmp"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    os.replace(out_path + ".tmp", out_path)
    return out_path


if __name__ == "__main__":
    import sys
    print(build(force=True, verbose="-v" in sys.argv))
