"""Per-kernel mean duration / DRAM bytes from an ncu --csv launch list: python tools/launch_table.py <csv>"""
import csv
import sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[i], rows[i + 1:]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: defaultdict(list))
for r in data:
    agg[r[ki].split("(")[0].replace("void ", "")][r[mi]].append(float(r[vi].replace(",", "")))
for k, m in agg.items():
    t = m["gpu__time_duration.sum"]
    rd, wr = m.get("dram__bytes_read.sum", [0]), m.get("dram__bytes_write.sum", [0])
    print(f"{k:40s} n={len(t):3d} mean {sum(t) / len(t) / 1e3:8.2f} us  last {t[-1] / 1e3:8.2f} us  "
          f"dram rd {rd[-1] / 1e6:7.2f} MB wr {wr[-1] / 1e6:7.2f} MB")
