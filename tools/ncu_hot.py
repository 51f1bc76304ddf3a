"""Hottest SASS instructions of one kernel in an ncu report (stall samples).

usage: python tools/ncu_hot.py REPORT KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + kern], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    h = rows[hdr]
    data = [r for r in rows[hdr + 1:] if len(r) == len(h)]
    # first kernel instance only
    seen, first = set(), []
    for r in data:
        if r[0] in seen:
            break
        seen.add(r[0])
        first.append(r)
    data = first

    def num(x):
        try:
            return int(x)
        except ValueError:
            return 0

    iss = h.index("Warp Stall Sampling (All Samples)")
    iex = h.index("Instructions Executed")
    src = h.index("Source")
    sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
    tot = sum(num(r[iss]) for r in data)
    print(f"total samples {tot}, instructions {len(data)}, executed {sum(num(r[iex]) for r in data)}")
    top = sorted(range(len(data)), key=lambda i: -num(data[i][iss]))[:n]
    for i in sorted(top):
        r = data[i]
        st = sorted(((num(r[j]), h[j][6:]) for j in sc), reverse=True)[:2]
        print(f"{i:5d} {num(r[iss]):6d} {num(r[iex]):10d}  {r[src].strip()[:58]:58s} {st}")


if __name__ == "__main__":
    main()
