"""Instruction histogram of the hot kernels from the built objects (cuobjdump
-sass): the mnemonics that show TMA / bulk copies / bulk reductions /
mbarriers (UTMALDG, UBLKCP, UBLKRED, SYNCS) next to the FP64 work.

usage: python tools/sass_hist.py OUTDIR
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BUILD = os.path.join(ROOT, "paper_1810_09891_b200", "csrc", "build")
KERNELS = [("residue.o", "k_spread_res"), ("gridding.o", "k_interp_pipe"), ("gridding.o", "k_spread_pipe"),
           ("gridding.o", "k_spread2_pipe"), ("fft.o", "k_fft_pass")]
KEY = ("UTMALDG", "UTMAPF", "UBLKCP", "UBLKRED", "UBLKPF", "SYNCS", "DFMA", "DMUL", "FFMA", "LDS", "STS",
       "SHFL", "ATOMS", "ATOMG", "RED", "BAR", "LDG", "STG", "LDGSTS", "ARRIVES", "DADD")


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles")
    os.makedirs(out, exist_ok=True)
    for obj, kern in KERNELS:
        txt = subprocess.run(["cuobjdump", "-sass", os.path.join(BUILD, obj)], capture_output=True, text=True).stdout
        fn, hist = None, {}
        for line in txt.splitlines():
            m = re.search(r"Function : (\S+)", line)
            if m:
                fn = m.group(1) if kern in m.group(1) else None
                if fn:
                    hist[fn] = collections.Counter()
                continue
            if fn:
                m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\d\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]+)?", line)
                if m:
                    hist[fn][m.group(2) + (m.group(3) or "")] += 1
        with open(os.path.join(out, f"sass_{kern}.txt"), "w") as fh:
            for fn, h in hist.items():
                demangled = subprocess.run(["cu++filt", fn], capture_output=True, text=True).stdout.strip() or fn
                total = sum(h.values())
                fh.write(f"== {demangled[:120]}\n   {total} instructions\n")
                groups = collections.Counter()
                for op, n in h.items():
                    groups[op.split(".")[0]] += n
                fh.write("   key mnemonics: " + ", ".join(f"{k} x{groups[k]}" for k in KEY if groups.get(k)) + "\n")
                for op, n in h.most_common():
                    if op.split(".")[0] in ("UTMALDG", "UTMAPF", "UBLKCP", "UBLKRED", "UBLKPF", "SYNCS", "ATOMS"):
                        fh.write(f"      {op:44s} {n}\n")
        print("wrote", os.path.join(out, f"sass_{kern}.txt"))


if __name__ == "__main__":
    main()
