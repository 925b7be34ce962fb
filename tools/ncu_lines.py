#!/usr/bin/env python
"""Attribute ncu warp-stall samples of one kernel to CUDA source lines.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX LIB.so [--top N]

Joins `ncu --page source --csv` (per-SASS-instruction samples) with
`nvdisasm --print-line-info-inline` of the kernel's cubin (offset -> file:line,
including the call site of inlined helpers).  Profiling aid only.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile


def sass_samples(rep, kregex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kregex}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    res = []
    base = None
    for r in rows[2:]:
        try:
            addr = int(r[0], 16)
            s = int(r[si])
        except (ValueError, IndexError):
            continue
        if base is None:
            base = addr
        res.append((addr - base, s, r[1].strip()))
    return res


def line_map(lib, kname_part):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d,
                   capture_output=True)
    m = {}
    for cub in glob.glob(os.path.join(d, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "-gi", cub], capture_output=True, text=True).stdout
        cur_fn = None
        loc = ("?", 0, "")
        for line in txt.splitlines():
            fm = re.match(r"\s*\.text\.(\S+):", line)
            if fm:
                cur_fn = fm.group(1)
                continue
            lm = re.search(r'//## File "([^"]+)", line (\d+)(.*)', line)
            if lm:
                inl = re.search(r'inlined at "([^"]+)", line (\d+)', lm.group(3))
                top = (os.path.basename(inl.group(1)), int(inl.group(2))) if inl else None
                loc = (os.path.basename(lm.group(1)), int(lm.group(2)), top)
                continue
            om = re.match(r"\s*/\*([0-9a-f]{4,})\*/", line)
            if om and cur_fn and kname_part in cur_fn:
                m[int(om.group(1), 16)] = loc
    return m


def main():
    rep, kre, lib = sys.argv[1:4]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    samples = sass_samples(rep, kre)
    lm = line_map(lib, kre.strip(".*"))
    tot = sum(s for _, s, _ in samples) or 1
    by_line = collections.Counter()
    by_top = collections.Counter()
    for off, s, ins in samples:
        f, ln, topl = lm.get(off, ("?", 0, None))
        by_line[(f, ln)] += s
        by_top[topl if topl else (f, ln)] += s
    print(f"total samples {tot}")
    print("-- by innermost source line")
    for (f, ln), s in by_line.most_common(top):
        print(f"{100 * s / tot:5.1f}%  {f}:{ln}")
    print("-- by outermost (call-site) line")
    for (f, ln), s in by_top.most_common(top):
        print(f"{100 * s / tot:5.1f}%  {f}:{ln}")


if __name__ == "__main__":
    main()
