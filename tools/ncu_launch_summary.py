"""Per-kernel share of an ncu --metrics gpu__time_duration.sum launch list."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
for i, r in enumerate(rows):
    if "Kernel Name" in r and "Metric Value" in r:
        hdr, rows = r, rows[i + 1:]
        break
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot = collections.Counter()
cnt = collections.Counter()
for r in rows:
    if len(r) != len(hdr):
        continue
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
             "second": 1e6, "s": 1e6}.get(unit, 1.0)
    name = r[ki].split("(")[0].replace("void ", "")
    tot[name] += v * scale
    cnt[name] += 1
SETUP = ("k_fma_peak", "k_build_psi", "Radix", "Scan", "k_bin_keys", "k_sum_widths", "k_gather_sorted",
         "k_check_range", "k_fill_subs", "k_count_subs", "k_lex_keys", "FillFunctor")
step = {k: v for k, v in tot.items() if not any(t in k for t in SETUP)}
all_us = sum(tot.values())
step_us = sum(step.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s} {'step%':>7s}")
for k, v in tot.most_common():
    st = f"{100 * v / step_us:6.1f}%" if k in step else "  setup"
    print(f"{k[:60]:60s} {cnt[k]:8d} {v:12.1f} {v / cnt[k]:10.2f} {100 * v / all_us:6.1f}% {st}")
print("(durations are ncu-serialised, cold-cache; compare shares, not absolutes)")
