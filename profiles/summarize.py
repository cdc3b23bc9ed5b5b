"""Turns ncu outputs from gpurun_out/ into the committed summaries here.

    python profiles/summarize.py launches <launches.csv> > profiles/rN_launches.md
    python profiles/summarize.py full <report.ncu-rep>   > profiles/rN_ncu_full.md
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict, defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[i], rows[i + 1:]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = OrderedDict()
    for r in data:
        if r[mi] == "gpu__time_duration.sum":
            per[r[ii]] = (r[ki].split("(")[0].replace("void ", "").strip(), float(r[vi].replace(",", "")))
    items = list(per.values())
    # one step = the launches between consecutive plan_mark kernels; use the last full step
    starts = [k for k, (n, _) in enumerate(items) if "k_plan_mark" in n or "k_fplan" in n]
    step = items[starts[-2]:starts[-1]] if len(starts) >= 2 else items
    tot = sum(t for _, t in step)
    agg = defaultdict(lambda: [0.0, 0])
    for n, t in step:
        agg[n][0] += t
        agg[n][1] += 1
    print(f"# ncu launch list (gpu__time_duration.sum, --clock-control none), one step of {len(step)} launches")
    print()
    print("Cold-cache and serialised by ncu: compare shares, not absolutes.")
    print()
    print("| kernel | launches | ns | share |")
    print("|---|---|---|---|")
    for n, (t, c) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        print(f"| `{n}` | {c} | {t:,.0f} | {100 * t / tot:.1f}% |")
    print(f"| **total** | {len(step)} | {tot:,.0f} | 100% |")


METRICS = [
    ("gpu__time_duration.sum", "duration (ns)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    print("# ncu --set full (--clock-control none), one launch per kernel")
    print()
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
        print(f"## `{name}`")
        print()
        for m, label in METRICS:
            if m in hdr:
                j = hdr.index(m)
                print(f"- {label}: {r[j]} {units[j]}")
        vals = sorted([(float(r[i] or 0), hdr[i].replace("smsp__pcsamp_warps_issue_stalled_", "")) for i in stall],
                      reverse=True)
        tot = sum(v for v, _ in vals) or 1
        print("- stall samples: " + ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in vals[:6]))
        print()


def traffic(path):
    """{kernel: dram read + write bytes per launch} for bench.py's roofline.traffic."""
    import json
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {}
    for r in data:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0].strip()
        base = name.split("::")[-1]
        fast = {"k_fplan": "f_plan", "k_fwd": "f_fwd", "k_bwd": "f_bwd", "k_coreimg": "f_sgd"}
        key = fast[base] if base in fast else base.replace("k_", "", 1)
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            j = hdr.index(m)
            tot += float(r[j].replace(",", "")) * scale.get(units[j], 1)
        res.setdefault(key, tot)
    print(json.dumps({"source": path, "bytes_per_launch": res}, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](sys.argv[2])
