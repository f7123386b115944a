"""Aggregate an ncu SASS source-page CSV (--page source --print-source sass)
by CUDA source line, using the line info of the library's own disassembly
(nvdisasm -g).  usage: sass_line_stalls.py page.csv all.sass kernel_substr [top]"""
import csv
import re
import sys
from collections import defaultdict

page, sass, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(page)))
hdr = rows[1]
data = rows[2:]
ia, isrc, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
# line info from nvdisasm -g: "//## File ..., line N" comments precede instructions
lines = {}
cur = None
inside = False
for l in open(sass):
    if l.startswith("//----") and ".text." in l:
        inside = kname in l
        continue
    if not inside:
        continue
    m = re.search(r'line (\d+)', l)
    if l.strip().startswith("//##") and m:
        cur = int(m.group(1))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        lines[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: defaultdict(int))
tot = 0
for r in data:
    off = int(r[ia], 16) - base
    ln = lines.get(off)
    s = int(r[isamp] or 0)
    tot += s
    agg[ln]["samples"] += s
    for i in stall_cols:
        v = int(r[i] or 0)
        if v:
            agg[ln][hdr[i]] += v
print(f"total samples {tot}")
for ln, d in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = sorted(((k, v) for k, v in d.items() if k != "samples"), key=lambda kv: -kv[1])[:4]
    print(f"line {ln}: {d['samples']} ({100*d['samples']/max(tot,1):.1f}%)  " + ", ".join(f"{k[6:]}={v}" for k, v in st))
