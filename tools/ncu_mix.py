"""Instruction mix of one kernel in an ncu report: warp-level instructions per
node by opcode, with each opcode's share of the warp-stall samples.

usage: python tools/ncu_mix.py REPORT KERNEL_REGEX CONFIG
"""
import collections
import csv
import io
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_09891_b200 import workloads as wl  # noqa: E402


def num(x):
    try:
        return int(x.replace(",", ""))
    except ValueError:
        return 0


def main():
    rep, kern, cfg = sys.argv[1], sys.argv[2], sys.argv[3]
    M = wl.lookup(cfg).M
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + kern], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    seen, first = set(), []
    for r in rows[hdr + 1:]:
        if len(r) != len(h) or not r[0].startswith("0x"):
            continue
        if r[0] in seen:
            break
        seen.add(r[0])
        first.append(r)
    iex, src = h.index("Instructions Executed"), h.index("Source")
    iss = h.index("Warp Stall Sampling (All Samples)")
    cnt, st = collections.Counter(), collections.Counter()
    for r in first:
        op = r[src].strip().split()
        if not op:
            continue
        o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
        cnt[o] += num(r[iex])
        st[o] += num(r[iss])
    tot, samples = sum(cnt.values()), max(1, sum(st.values()))
    print(f"{kern} at {cfg}: {tot / M:.1f} warp instructions per node ({tot} executed, {len(first)} SASS lines)")
    for k, v in cnt.most_common(28):
        print(f"  {k:12s} {v / M:8.2f} per node   {100.0 * st[k] / samples:5.1f}% of stall samples")


if __name__ == "__main__":
    main()
