"""Build the in-tree sm_100a native library (nvcc cross-compiles; no GPU needed).

    python -m paper_2512_02371_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")


def build(verbose: bool = False) -> str:
    os.makedirs(os.path.join(HERE, "_native"), exist_ok=True)
    cmd = ["make", "-j", str(min(16, os.cpu_count() or 1)), "-C", CSRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or r.returncode:
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
    if r.returncode:
        raise RuntimeError("native build failed")
    return os.path.join(HERE, "_native", "libtsb200.so")


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
