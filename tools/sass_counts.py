#!/usr/bin/env python
"""Per-kernel SASS instruction counts of libdeltanet.so that prove the
Blackwell paths (B200_PROFILING.md SASS mnemonics): UTCHMMA / UTCQMMA
(tcgen05.mma), UTMALDG / UTMASTG (TMA tensor load / store), UBLKCP (bulk
copy), LDTM / STTM (TMEM load / store), UTCBAR (tcgen05.commit), HMMA
(warp-level mma.sync), FFMA.  Static counts (instructions in the binary,
not executed counts).  Profiling aid.

    python tools/sass_counts.py [--md profiles/r02_sass_counts.md]
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2406_06484_b200", "libdeltanet.so")
OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "LDTM", "STTM",
       "HMMA", "FFMA", "SYNCS"]


def main():
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                         check=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(2)
            for o in OPS:
                if op == o:
                    counts[cur][o] += 1
            counts[cur]["_total"] += 1
    demangle = lambda n: subprocess.run(["c++filt", n], capture_output=True,
                                        text=True).stdout.strip() or n
    rows = []
    for fn, c in counts.items():
        if not any(c[o] for o in ("UTCHMMA", "UTMALDG", "LDTM", "HMMA", "FFMA")):
            continue
        name = demangle(fn)
        name = name.replace("(anonymous namespace)::", "")
        name = re.sub(r"\(.*", "", name).replace("dn::", "")
        rows.append((name, c))
    hdr = "| kernel | " + " | ".join(OPS) + " | total SASS |"
    lines = [hdr, "|---" * (len(OPS) + 2) + "|"]
    for name, c in rows:
        lines.append(f"| `{name}` | " + " | ".join(str(c[o]) for o in OPS) +
                     f" | {c['_total']} |")
    text = "\n".join(lines)
    print(text)
    if "--md" in sys.argv:
        sys.path.insert(0, ROOT)
        from paper_2406_06484_b200.build import sources_sha
        md = sys.argv[sys.argv.index("--md") + 1]
        with open(md, "w") as f:
            f.write("# Static SASS instruction counts per kernel (cuobjdump -sass libdeltanet.so)\n\n")
            f.write(f"Kernel sources sha16 `{sources_sha()}` "
                    "(paper_2406_06484_b200.build.sources_sha). Static counts: instructions "
                    "present in the binary, not executed counts. UTCHMMA = tcgen05.mma "
                    "(kind::f16), UTMALDG/UTMASTG = TMA tensor load/store, UBLKCP = "
                    "cp.async.bulk, LDTM/STTM = tcgen05.ld/st, UTCBAR = tcgen05.commit, "
                    "HMMA = warp-level mma.sync (the tf32 UT-inverse merges), SYNCS = "
                    "mbarrier ops.\n\n")
            f.write(text + "\n")


if __name__ == "__main__":
    main()
