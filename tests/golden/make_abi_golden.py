"""Fixture: the reference's own ABI description (nfftk.abi.interface_json(),
pkg/src/nfftk/abi.py:131-157), imported from /root/reference in this
container, saved as tests/golden/abi_reference.json for tests/test_abi.py.

    python tests/golden/make_abi_golden.py
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
env = dict(os.environ, PYTHONPATH="/root/reference/pkg/src", PYTHONDONTWRITEBYTECODE="1")
out = subprocess.run([sys.executable, "-c", "from nfftk import abi; print(abi.interface_json(), end='')"],
                     env=env, capture_output=True, text=True, check=True, cwd="/tmp").stdout
with open(os.path.join(HERE, "abi_reference.json"), "w") as fh:
    fh.write(out)
print("wrote", len(out), "bytes")
