"""Build the in-tree sm_100a library (nvcc cross-compiles; no GPU needed)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))


def build(jobs: int = 8) -> str:
    subprocess.run(["make", "-s", "-j", str(jobs), "-C", os.path.join(HERE, "csrc")], check=True)
    path = os.path.join(HERE, "lib", "libmoqe_gpu.so")
    if not os.path.exists(path):
        raise RuntimeError("libmoqe_gpu.so was not produced")
    return path


if __name__ == "__main__":
    print(build())
