"""Summarise gpurun_out/bench_*.log lines (local helper)."""
import glob
import json
import os
import sys

os.chdir(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for f in sys.argv[1:] or sorted(glob.glob("gpurun_out/bench_*.log")):
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, open(f).read()[-800:])
        continue
    d = json.loads(lines[-1])
    ph = {k: round(v, 4) for k, v in d.get("phases_ms_per_step", {}).items()}
    print(f"{f}: {d['value']:.3g} nodes/s  {d['ms_per_step']:.3f} ms/step  e2e {d['e2e']['value']:.3g}  {ph}")
