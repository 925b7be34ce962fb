#!/usr/bin/env python
"""Key metrics of the tcgen05 kernels from an ncu --set full report, as a
markdown table row per kernel plus profiles/ncu_traffic.json.  Profiling aid.

    python tools/ncu_summary.py REPORT.ncu-rep [--json profiles/ncu_traffic.json]
                                [--sha FILE] [--kernels a,b]

--sha FILE: the kernel-sources hash (paper_2406_06484_b200.build.sources_sha)
written by the capture command on the GPU box; default: the current tree.
bench.py marks `traffic` stale when it differs from the benched sources.
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("duration us", "gpu__time_duration.sum", 1e-3),
    ("DRAM read MB", "dram__bytes_read.sum", None),
    ("DRAM write MB", "dram__bytes_write.sum", None),
    ("DRAM thr %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("tensor pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("SM thr %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("smem wavefronts M", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1e-6),
    ("regs", "launch__registers_per_thread", 1),
]
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def raw(rep, k):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name",
                          f"regex:{k}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main():
    rep = sys.argv[1]
    out_json = sys.argv[sys.argv.index("--json") + 1] if "--json" in sys.argv else None
    print("| kernel | " + " | ".join(m[0] for m in METRICS) + " |")
    print("|---" * (len(METRICS) + 1) + "|")
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2406_06484_b200.build import sources_sha
    sha = open(sys.argv[sys.argv.index("--sha") + 1]).read().strip() if "--sha" in sys.argv \
        else sources_sha()
    kernels = (sys.argv[sys.argv.index("--kernels") + 1].split(",") if "--kernels" in sys.argv
               else ["tc_fwd_kernel", "tc_bwd_kernel"])
    head = subprocess.run(["git", "rev-parse", "--short=12", "HEAD"], capture_output=True,
                          text=True).stdout.strip()
    js = {"_source": f"ncu --set full --clock-control none, report {rep}; "
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch",
          "workload": "B=8 H=16 L=4096 d=128 C=64 bf16",
          "sources_sha16": sha, "git_head_at_summary": head}
    for k in kernels:
        h, u, v = raw(rep, k)
        cells, vals = [], {}
        for name, m, sc in METRICS:
            i = h.index(m)
            x = float(v[i].replace(",", ""))
            if m == "gpu__time_duration.sum":
                x *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                      "msecond": 1e3}[u[i]]
            elif sc is None:
                x *= SCALE[u[i]]
            else:
                x *= sc
            vals[name] = x
            cells.append(f"{x:.1f}")
        print(f"| {k} | " + " | ".join(cells) + " |")
        js[k] = {"dram_read_bytes": int(vals["DRAM read MB"] * 1e6),
                 "dram_write_bytes": int(vals["DRAM write MB"] * 1e6),
                 "duration_us": vals["duration us"]}
    if out_json:
        json.dump(js, open(out_json, "w"), indent=1)


if __name__ == "__main__":
    main()
