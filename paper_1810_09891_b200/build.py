"""Build libnfftk.so in-tree: ``python -m paper_1810_09891_b200.build``."""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def build(jobs=4, verbose=False):
    cmd = ["make", "-C", os.path.join(HERE, "csrc"), f"-j{jobs}"]
    out = subprocess.run(cmd, capture_output=not verbose, text=True)
    if out.returncode != 0:
        sys.stderr.write((out.stdout or "") + (out.stderr or ""))
        raise RuntimeError("libnfftk.so build failed")
    return os.path.join(HERE, "libnfftk.so")


if __name__ == "__main__":
    print(build(verbose=True))
