"""Build gen/libasse_gen.so: host generator (gcc, OpenMP) + its CUDA twin (nvcc, sm_100a)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libasse_gen.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(out, srcs):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build(force=False):
    srcs = [os.path.join(HERE, f) for f in
            ("asse_gen.h", "gen_internal.h", "asse_gen_host.c", "asse_gen_cuda.cu")]
    if not force and not _stale(LIB, srcs):
        return LIB
    bdir = os.path.join(HERE, "build")
    os.makedirs(bdir, exist_ok=True)
    host_o = os.path.join(bdir, "asse_gen_host.o")
    cu_o = os.path.join(bdir, "asse_gen_cuda.o")
    subprocess.check_call(["gcc", "-O2", "-fPIC", "-fopenmp", "-std=c11", "-c",
                           os.path.join(HERE, "asse_gen_host.c"), "-o", host_o])
    subprocess.check_call([NVCC, *ARCH, "-O3", "-Xcompiler", "-fPIC", "-c",
                           os.path.join(HERE, "asse_gen_cuda.cu"), "-o", cu_o])
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "static", host_o, cu_o,
                           "-Xcompiler", "-fopenmp", "-o", LIB])
    return LIB


if __name__ == "__main__":
    print(build(force=True))
