#!/usr/bin/env python3
"""Summarise an ncu --set full report (one kernel launch) into profiles/.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/ncu_x_r01 [--cells N --bt B]

Writes <out>.json (key counters) and <out>.md (human summary incl. top stall
reasons and instruction mix from the source page)."""
import argparse
import collections
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed.sum": "inst_executed",
    "smsp__inst_executed.sum": "inst_executed_smsp",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
              "usecond": 1e-6, "msecond": 1e-3, "second": 1, "%": 1, "": 1,
              "register/thread": 1, "inst": 1, "hz": 1, "Mhz": 1e6, "Ghz": 1e9}


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--cells", type=float, default=0, help="cells per launch (2-D stencil)")
    ap.add_argument("--bt", type=int, default=0)
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    raw = ncu_csv(a.rep, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    d = {"kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                d[KEYS[h]] = float(v.replace(",", "")) * UNIT_SCALE.get(u, 1)
            except ValueError:
                d[KEYS[h]] = v
    if "dram_read" in d and "dram_write" in d:
        d["dram_bytes"] = d["dram_read"] + d["dram_write"]
    if a.cells:
        d["algorithmic_bytes"] = 16.0 * a.cells
        d["traffic_over_algorithmic"] = d.get("dram_bytes", 0) / d["algorithmic_bytes"]
        if a.bt:
            d["updates"] = a.cells * a.bt
            d["dram_bytes_per_update"] = d.get("dram_bytes", 0) / d["updates"]
            inst = d.get("inst_executed") or d.get("inst_executed_smsp", 0)
            d["thread_inst_per_update"] = inst * 32 / d["updates"]
    # stall reasons + instruction mix from the source page
    src = ncu_csv(a.rep, "source")
    stalls, mix = collections.Counter(), collections.Counter()
    if len(src) > 2:
        h = src[1]
        ix = {n: i for i, n in enumerate(h)}
        sc = [n for n in h if n.startswith("stall_") and "(Not" not in n]
        for r in src[2:]:
            if len(r) < len(h):
                continue
            op = r[ix["Source"]].strip().split()
            if not op:
                continue
            o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
            mix[o.split(".")[0]] += int(r[ix["Instructions Executed"]] or 0)
            for n in sc:
                stalls[n] += int(r[ix[n]] or 0)
    tot = sum(stalls.values()) or 1
    d["stall_top"] = [[k, round(v / tot, 3)] for k, v in stalls.most_common(6)]
    mt = sum(mix.values()) or 1
    d["inst_mix_top"] = [[k, round(v / mt, 3)] for k, v in mix.most_common(10)]
    with open(a.out + ".json", "w") as f:
        json.dump(d, f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write("# %s\n\nSource report: `%s` (ncu --set full, one launch)\n\n" % (a.title or d["kernel"], a.rep))
        f.write("| counter | value |\n|---|---|\n")
        for k, v in d.items():
            if k in ("stall_top", "inst_mix_top", "kernel"):
                continue
            f.write("| %s | %s |\n" % (k, ("%.4g" % v) if isinstance(v, float) else v))
        f.write("\nKernel: `%s`\n\nTop stall reasons (share of samples): %s\n\nInstruction mix (share of executed): %s\n"
                % (d["kernel"], ", ".join("%s %.1f%%" % (k, 100 * v) for k, v in d["stall_top"]),
                   ", ".join("%s %.1f%%" % (k, 100 * v) for k, v in d["inst_mix_top"])))
    print(json.dumps({k: d[k] for k in d if k not in ("stall_top", "inst_mix_top")}, indent=0)[:2000])


if __name__ == "__main__":
    main()
