"""Warm set_nodes / precompute wall times for one config (where precompute time goes).
usage: python tools/precompute_probe.py C5 [--single]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1810_09891_b200 as nf  # noqa: E402
from paper_1810_09891_b200 import workloads as wl  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C5"
    prec = "single" if "--single" in sys.argv else "double"
    w = wl.CONFIGS[name]
    p = nf.Plan(w.N, w.M, n=w.n, m=w.m, precision=prec)
    x = torch.from_numpy(wl.nodes(w)).cuda()
    for it in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p.set_nodes(x)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        p.precompute()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"{name} {prec} call {it}: set_nodes {1000 * (t1 - t0):.1f} ms  precompute {1000 * (t2 - t1):.1f} ms",
              flush=True)


if __name__ == "__main__":
    main()
