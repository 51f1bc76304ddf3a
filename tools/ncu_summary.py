"""Summarise an ncu report: key throughput metrics + instruction mix per
execution-count class (per-node / per-row / per-CTA costs)."""
import collections
import csv
import io
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "lts__t_sectors_op_red.sum", "launch__registers_per_thread",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units, rows = r[0], r[1], r[2:]
    for row in rows:
        name = row[hdr.index("Kernel Name")]
        print("=====", name[:60])
        for k in WANT:
            if k in hdr:
                print(f"  {k:80s} {row[hdr.index(k)]} {units[hdr.index(k)]}")


def mix(rep, kernel, nodes):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kernel}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    seen, uniq = set(), []
    for r in data:
        if r[0] not in seen:
            seen.add(r[0])
            uniq.append(r)
    ie = hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    f = lambda v: float(v.replace(",", "") or 0)
    cls, cnt, st, ex = collections.Counter(), collections.Counter(), collections.Counter(), {}
    for r in uniq:
        e = f(r[ie])
        cls[e] += e
        cnt[e] += 1
        st[e] += f(r[si])
        ex.setdefault(e, r[1].strip()[:60])
    tot, stot = sum(cls.values()), sum(st.values()) or 1
    print(f"--- {kernel}: {tot:.3g} warp-instr, {tot / nodes:.1f} per node")
    for e, v in sorted(cls.items(), key=lambda x: -x[1])[:10]:
        print(f"  exec={e:>12.0f} n={cnt[e]:4d} instr={v / tot * 100:5.1f}% stall={st[e] / stot * 100:5.1f}% "
              f"per_node={v / nodes:6.1f}  e.g. {ex[e]}")
    top = sorted(uniq, key=lambda r: -f(r[si]))[:12]
    print("  top stall instructions:")
    for r in top:
        print(f"    {f(r[si]) / stot * 100:5.1f}%  {r[1].strip()[:70]}")


if __name__ == "__main__":
    rep = sys.argv[1]
    raw(rep)
    if len(sys.argv) > 2:
        nodes = float(sys.argv[2])
        for k in (sys.argv[3:] or ["k_interp", "k_spread"]):
            try:
                mix(rep, k, nodes)
            except (IndexError, ValueError):
                pass
