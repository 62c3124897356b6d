"""Build oracle/liboracle.so (plain C, gcc). Test infrastructure only."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
SRCS = [os.path.join(HERE, f) for f in ("asse_oracle.c", "truth.c")]


def build(force=False):
    if not force and os.path.exists(LIB) and all(
            os.path.getmtime(s) <= os.path.getmtime(LIB) for s in SRCS):
        return LIB
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", *SRCS, "-lm", "-o", LIB])
    return LIB


if __name__ == "__main__":
    print(build(force=True))
