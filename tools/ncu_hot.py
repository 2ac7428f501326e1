#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from an ncu report (source page).

    python tools/ncu_hot.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
for i, r in enumerate(rows):
    if "Source" in r and any("Sampling" in c for c in r):
        hdr = i
        break
if hdr is None:
    print(out[:2000])
    sys.exit(1)
h = rows[hdr]
isrc = h.index("Source")
isamp = [j for j, c in enumerate(h) if c.startswith("# Samples") or c == "Warp Stall Sampling (All Samples)"]
isamp = isamp[0] if isamp else [j for j, c in enumerate(h) if "Sampling" in c][0]
iexec = h.index("Instructions Executed") if "Instructions Executed" in h else None
data = []
for k, r in enumerate(rows[hdr + 1:]):
    try:
        data.append((int(r[isamp] or 0), k, r[isrc], int(r[iexec] or 0) if iexec is not None else 0))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot, "instructions", len(data))
for s, k, src, ex in sorted(data, reverse=True)[:top]:
    print("%6d %5.1f%%  #%5d  exec %9d  %s" % (s, 100.0 * s / tot, k, ex, src[:90]))
