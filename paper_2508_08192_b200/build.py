"""In-tree build of libspecdec_b200.so for sm_100a (nvcc via make)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")


def build(jobs: int = 8, verbose: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    cmd = ["make", "-C", CSRC, f"-j{jobs}", f"NVCC={nvcc}"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"build failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        print(res.stdout)
    from ._lib import LIB_PATH

    return LIB_PATH


if __name__ == "__main__":
    print(build(verbose=True))
