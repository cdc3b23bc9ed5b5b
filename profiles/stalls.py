"""Per-source-line warp-stall samples of one kernel from an ncu report
(`--import-source on`): python profiles/stalls.py <report> <kernel regex> [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, line, src = "", None, ""
agg = defaultdict(lambda: defaultdict(float))
texts = {}
hdr = None
total = 0.0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:
        line, src = r[0], r[1]
        continue
    key = (fname, int(line) if line else 0)
    texts[key] = src.strip()[:70]
    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    s = num(r[hdr.index("Warp Stall Sampling (All Samples)")])
    agg[key]["samples"] += s
    agg[key]["inst"] += num(r[hdr.index("Instructions Executed")])
    total += s
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            agg[key][h[6:]] += num(r[i])
tinst = sum(d["inst"] for d in agg.values())
print(f"total samples {total:.0f}, instructions {tinst:.0f}")
sortkey = "inst" if "--inst" in sys.argv else "samples"
for key, d in sorted(agg.items(), key=lambda kv: -kv[1][sortkey])[:top]:
    st = sorted(((v, k) for k, v in d.items() if k not in ("samples", "inst")), reverse=True)[:3]
    print(f"{d['samples'] / total * 100:5.1f}% inst {d['inst'] / tinst * 100:5.1f}% {key[0]}:{key[1]:<5} {texts[key]:60s} " +
          " ".join(f"{k}={v / max(d['samples'], 1) * 100:.0f}%" for v, k in st))
