#!/usr/bin/env python3
"""Executed warp instructions and stall samples per CUDA source line: joins an
`ncu --page source --print-source sass --csv` export (gzip ok) with an
`nvdisasm -g -c` listing of the same kernel by instruction offset.

    python tools/ncu_lines.py sass.csv.gz kernel.dis [N]
"""
import collections
import csv
import gzip
import re
import sys

sass, dis = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
op = gzip.open if sass.endswith(".gz") else open
rows = [r for r in csv.reader(op(sass, "rt")) if len(r) >= 6]
hdr = next(i for i, r in enumerate(rows) if r[0] == "Address")
data = rows[hdr + 1:]
base = int(data[0][0], 16)
by_off = {int(r[0], 16) - base: (int(r[5] or 0), int(r[4] or 0), r[1].strip()) for r in data}
line_of = {}
cur = None
for l in open(dis):
    m = re.search(r'line (\d+)', l) if "//## File" in l else None
    if m:
        cur = int(m.group(1))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,6})\*/", l)
    if m:
        line_of[int(m.group(1), 16)] = cur
ex = collections.Counter()
st = collections.Counter()
n = collections.Counter()
for off, (e, s, _) in by_off.items():
    ln = line_of.get(off)
    ex[ln] += e
    st[ln] += s
    n[ln] += 1
tot_e, tot_s = sum(ex.values()) or 1, sum(st.values()) or 1
print("total executed %d, samples %d" % (tot_e, tot_s))
print("  line   exec%  stall%  static")
for ln, e in ex.most_common(top):
    print("%6s  %5.1f%%  %5.1f%%  %5d" % (ln, 100.0 * e / tot_e, 100.0 * st[ln] / tot_s, n[ln]))
