"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of
each kernel in an ncu --set full report, merged into a profiles/*/ncu_traffic.json
under the given config name (bench.py reads it for roofline.traffic).

usage: python tools/ncu_traffic.py REPORT CONFIG OUT_JSON
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys


def main():
    rep, config, out = sys.argv[1:4]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[0]
    kcol = hdr.index("Kernel Name")
    rcol = hdr.index("dram__bytes_read.sum")
    wcol = hdr.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = collections.defaultdict(list)
    for r in rows[2:]:
        name = re.match(r"(?:void )?(?:nfftk::)?(\w+)", r[kcol]).group(1)
        b = float(r[rcol].replace(",", "")) * scale[units[rcol]] + \
            float(r[wcol].replace(",", "")) * scale[units[wcol]]
        acc[name].append(b)
    data = {}
    if os.path.exists(out):
        with open(out) as fh:
            data = json.load(fh)
    data.setdefault(config, {})
    for k, v in acc.items():
        data[config][k] = int(sum(v) / len(v))
    with open(out, "w") as fh:
        json.dump(data, fh, indent=1, sort_keys=True)
    print(json.dumps(data[config]))


if __name__ == "__main__":
    main()
