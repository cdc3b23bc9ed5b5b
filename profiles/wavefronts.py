"""Shared-memory (L1 data pipe) wavefronts per source line of one kernel from
an ncu report: python profiles/wavefronts.py <report> <kernel regex> [top]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
f, line, src, hdr = "", 0, "", None
agg = collections.defaultdict(lambda: [0.0, 0.0, ""])


def num(v):
    try:
        return float(v)
    except ValueError:
        return 0.0


for x in csv.reader(io.StringIO(out)):
    if not x:
        continue
    if x[0] == "File Path":
        f = x[1].split("/")[-1]
        continue
    if x[0] == "Line No":
        hdr = x
        wi, di = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
        continue
    if hdr is None or len(x) < len(hdr):
        continue
    if x[0]:
        line, src = int(x[0]), x[1]
        continue
    a = agg[(f, line)]
    a[0] += num(x[wi])
    a[1] += num(x[di])
    a[2] = src.strip()[:70]
tot = sum(v[0] for v in agg.values())
print(f"total shared wavefronts {tot:.0f}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / tot * 100:5.1f}%  ideal/actual {v[1] / max(v[0], 1):4.2f}  {k[0]}:{k[1]}  {v[2]}")
