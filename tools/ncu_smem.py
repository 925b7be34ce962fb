#!/usr/bin/env python
"""Shared-memory wavefronts (actual vs ideal) per CUDA source line of one
kernel, from an ncu --set full report (source page) + nvdisasm line info.

    python tools/ncu_smem.py REPORT.ncu-rep KERNEL_REGEX LIB.so [--top N]
Profiling aid only."""
import collections
import csv
import io
import subprocess
import sys

sys.path.insert(0, __import__("os").path.dirname(__file__))
from ncu_lines import line_map  # noqa: E402


def main():
    rep, kre, lib = sys.argv[1:4]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kre}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    iw = hdr.index("L1 Wavefronts Shared")
    ii = hdr.index("L1 Wavefronts Shared Ideal")
    lm = line_map(lib, kre.strip(".*"))
    act = collections.Counter()
    ide = collections.Counter()
    base = None
    for r in rows[2:]:
        try:
            addr = int(r[0], 16)
        except ValueError:
            continue
        if base is None:
            base = addr
        f, ln, topl = lm.get(addr - base, ("?", 0, None))
        key = topl if topl else (f, ln)
        try:
            act[key] += int(float(r[iw] or 0))
            ide[key] += int(float(r[ii] or 0))
        except ValueError:
            pass
    tot = sum(act.values()) or 1
    print(f"total smem wavefronts {tot}, ideal {sum(ide.values())}")
    for key, a in act.most_common(top):
        print(f"{100 * a / tot:5.1f}%  {a:10d}  ideal {ide[key]:10d}  {key[0]}:{key[1]}")


if __name__ == "__main__":
    main()
