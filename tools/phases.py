"""Print value / e2e / phase times from bench logs: python tools/phases.py LOG..."""
import json
import sys

for p in sys.argv[1:]:
    try:
        d = json.loads(open(p).read().strip().splitlines()[-1])
    except Exception as e:  # noqa: BLE001
        print(p, "unreadable", e)
        continue
    ph = d.get("phases_ms_per_step", {})
    print(f"{p}: value {d['value']:.3e} e2e {d['e2e']['value']:.3e} step {d['ms_per_step']:.3f} ms | "
          f"interp {ph.get('interp', 0):.3f} spread {ph.get('spread', 0):.3f} | "
          + " ".join(f"{k} {v:.3f}" for k, v in ph.items() if k not in ('interp', 'spread')))
