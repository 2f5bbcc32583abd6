"""Build the roofline microbenchmark executable (tools/microbench) for sm_100a."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "microbench.cu")
EXE = os.path.join(HERE, "microbench")


def build(force: bool = False) -> str:
    if force or not os.path.exists(EXE) or os.path.getmtime(EXE) < os.path.getmtime(SRC):
        tmp = EXE + f".tmp{os.getpid()}"
        subprocess.check_call(["nvcc", "-O3", "-std=c++17", "-lineinfo", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-o", tmp, SRC])
        os.replace(tmp, EXE)
    return EXE


if __name__ == "__main__":
    print(build(force=True))
