"""Golden fixtures for the CLI: run the *reference* CLI (nfftk.cli, imported
from /root/reference in this container; it does not exist on the GPU box)
on small seeded cases and record its CSV rows, result files, exit codes and
error messages under tests/golden/cli/.

    python tests/golden/make_cli_golden.py

Inputs (nodes / coefficient files) are generated here from a seeded PCG64
stream and written next to the outputs, so the GPU-side test replays the
exact same files.
"""

import csv
import io
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
REF = "/root/reference/pkg/src"

CASES = {
    "verify_d1": ["verify", "--bandlimit", "16", "--nodes-count", "64", "--cutoff", "4", "--seed", "3"],
    "verify_d2": ["verify", "--bandlimit", "8,8", "--cutoff", "3", "--seed", "1"],
    "verify_d3_gauss": ["verify", "--bandlimit", "8", "--dim", "3", "--nodes-count", "200", "--cutoff", "2",
                        "--window", "gaussian", "--seed", "2"],
    "verify_fail_tol": ["verify", "--bandlimit", "16", "--nodes-count", "40", "--cutoff", "2",
                        "--tol", "1e-16"],
    "bench_m": ["bench", "--sweep", "m", "--grid", "2,3,5", "--bandlimit", "16", "--nodes-count", "50"],
    "bench_n": ["bench", "--sweep", "n", "--grid", "18,24,32", "--bandlimit", "8,8", "--nodes-count", "60",
                "--cutoff", "3"],
    "usage_no_fhat": ["transform", "--bandlimit", "8,8", "--nodes", "{dir}/nodes_d2.txt", "--out",
                      "{tmp}/x.txt"],
    "usage_dim_mismatch": ["verify", "--bandlimit", "8,8", "--dim", "3"],
    "io_malformed": ["transform", "--bandlimit", "8,8", "--nodes", "{dir}/nodes_bad.txt", "--fhat",
                     "{dir}/fhat_d2.txt", "--out", "{tmp}/x.txt"],
    "transform_d2": ["transform", "--bandlimit", "8,8", "--cutoff", "3", "--nodes", "{dir}/nodes_d2.txt",
                     "--fhat", "{dir}/fhat_d2.txt", "--out", "{tmp}/out_trafo_d2.txt"],
    "transform_d2_adjoint": ["transform", "--bandlimit", "8,8", "--cutoff", "3", "--nodes",
                             "{dir}/nodes_d2.txt", "--adjoint", "--f", "{dir}/f_d2.txt", "--out",
                             "{tmp}/out_adjoint_d2.txt"],
    "transform_d3": ["transform", "--bandlimit", "4,6,8", "--fft-length", "8,12,16", "--nodes",
                     "{dir}/nodes_d3.txt", "--fhat", "{dir}/fhat_d3.txt", "--out", "{tmp}/out_trafo_d3.txt"],
}


def write_inputs():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(2024)

    def vec(path, v):
        with open(path, "w") as fh:
            for z in v:
                fh.write(f"{z.real:.17g} {z.imag:.17g}\n")

    x2 = rng.random((30, 2)) - 0.5
    np.savetxt(os.path.join(OUT, "nodes_d2.txt"), x2, fmt="%.17g")
    vec(os.path.join(OUT, "fhat_d2.txt"), rng.standard_normal(64) + 1j * rng.standard_normal(64))
    vec(os.path.join(OUT, "f_d2.txt"), rng.standard_normal(30) + 1j * rng.standard_normal(30))
    x3 = rng.random((25, 3)) - 0.5
    np.savetxt(os.path.join(OUT, "nodes_d3.txt"), x3, fmt="%.17g")
    vec(os.path.join(OUT, "fhat_d3.txt"), rng.standard_normal(192) + 1j * rng.standard_normal(192))
    with open(os.path.join(OUT, "nodes_bad.txt"), "w") as fh:
        fh.write("0.1 0.2\n\n0.3 zz\n")


def main():
    write_inputs()
    env = dict(os.environ, PYTHONPATH=REF, NUMBA_CACHE_DIR="/tmp/numba_cache", PYTHONDONTWRITEBYTECODE="1")
    record = {}
    for name, template in CASES.items():
        argv = [a.replace("{dir}", OUT).replace("{tmp}", OUT) for a in template]
        r = subprocess.run([sys.executable, "-m", "nfftk.cli"] + argv, env=env, capture_output=True,
                           text=True, cwd="/tmp")
        rows = list(csv.DictReader(io.StringIO(r.stdout))) if r.stdout.startswith("dim,") else []
        record[name] = {
            "argv": list(template),
            "rc": r.returncode,
            "stderr": r.stderr.strip().splitlines()[-1] if r.stderr.strip() else "",
            "rows": [{k: row[k] for k in ("dim", "N", "n", "m", "e2", "einf")} for row in rows],
        }
        print(name, r.returncode, record[name]["stderr"][:80])
    with open(os.path.join(OUT, "cli_golden.json"), "w") as fh:
        json.dump(record, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
