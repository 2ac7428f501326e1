"""Tabulate a tools/cfg0_sweep.sh log: one row per (variant, chunks), GUpd/s per depth."""
import re
import sys

path, bts = sys.argv[1], sys.argv[2].split(",")
rows, cur, vals = [], None, []
for line in open(path):
    if line.startswith("=="):
        if cur:
            rows.append((cur, vals))
        cur, vals = (line.split()[2], line.split()[4]), []
    else:
        m = re.search(r"GUpd/s ([\d.]+)", line)
        if m:
            vals.append(float(m.group(1)))
if cur:
    rows.append((cur, vals))
print("var  ch  " + " ".join("%6s" % ("bt" + b) for b in bts))
for (v, c), vs in rows:
    print("%3s %3s  " % (v, c) + " ".join("%6.0f" % x for x in vs))
