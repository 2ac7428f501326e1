"""SLT-vs-COT sweep driver on the GPU.

GPU analogue of the reference's `run_sweep` (reference core/src/sweep.cpp:35-141,
CSV schema docs/formats.md "sweep CSV"): for every (scheme x tile) cell, run the
kernel `samples` times through the executor and report device time; with
`ncu=True` each cell is re-run once under Nsight Compute and the simulated
off-chip accesses of the reference (CacheSim OCA, cachesim.cpp:91-127) are
replaced by measured DRAM bytes and the L2 hit rate — the paper's question
(does the recursive tile order cut off-chip traffic?) asked of the B200.

    python -m paper_1802_00166_b200.sweep jacobi2d -p T=64,N=8192 \
        --tiles 4x64x256,6x64x256 --schemes slt,cot --samples 3 [--ncu] [--csv out.csv]
"""
import argparse
import csv
import io
import json
import os
import statistics
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
if REPO not in sys.path:
    sys.path.insert(0, REPO)

CSV_HEADER = ("scheme,tile,samples,ms_mean,ms_stddev,ms_cov,launches,dram_bytes,l2_hit_pct,"
              "checksum,parity")


def parse_params(s):
    out = {}
    for kv in s.split(","):
        k, v = kv.split("=")
        out[k.strip()] = int(v)
    return out


def parse_tiles(s):
    return [[int(v) for v in t.split("x")] for t in s.split(",") if t]


def _ncu_cell(kernel, params, scheme, tile):
    """DRAM bytes + L2 hit rate summed over the cell's launches (one run)."""
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,"
           "lts__t_sectors.sum", "--clock-control", "none", "--csv",
           sys.executable, "-m", "paper_1802_00166_b200.sweep", kernel,
           "-p", ",".join("%s=%d" % kv for kv in params.items()), "--tiles",
           "x".join(map(str, tile)), "--schemes", scheme, "--samples", "1", "--quiet",
           "--no-warmup", "--no-verify"]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=REPO)
    return parse_ncu_csv(p.stdout)


def parse_ncu_csv(text):
    """(DRAM bytes, sector-weighted L2 hit %) summed over the launches of an
    `ncu --metrics ... --csv` listing (also used on captures made one cell per
    process: `ncu ... python -m paper_1802_00166_b200.sweep ... --samples 1
    --quiet --no-warmup > cell.csv`)."""
    rows = [r for r in csv.reader(io.StringIO(text)) if len(r) > 10]
    if not rows:
        return None, None
    h = rows[0]
    iname, ival, iunit = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    dram, hit_w, sect = 0.0, 0.0, 0.0
    per_launch_sect = {}
    per_launch_hit = {}
    for i, r in enumerate(rows[1:]):
        key = r[h.index("ID")] if "ID" in h else i
        v = float(r[ival].replace(",", ""))
        if r[iname].startswith("dram__bytes"):
            dram += v * scale.get(r[iunit], 1)
        elif r[iname] == "lts__t_sectors.sum":
            per_launch_sect[key] = v
        elif r[iname] == "lts__t_sector_hit_rate.pct":
            per_launch_hit[key] = v
    for k, s in per_launch_sect.items():
        sect += s
        hit_w += s * per_launch_hit.get(k, 0.0)
    return dram, (hit_w / sect if sect else None)


def run_sweep(kernel, params, tiles, schemes=("slt", "cot"), samples=3, device=0, ncu=False,
              warmup=True, want=None, verify=True):
    """One result dict per (scheme, tile) cell, reference run_sweep order.

    Every timed sample also yields the output's FNV-1a checksum (computed on
    the host after the device timing); a cell's `parity` is "ok" only if all
    of its samples equal `want` (default: the untiled run's checksum, itself
    compared with the reference golden by the test suite) — every order must
    reproduce the same bits (reference tests/acceptance.cpp:345-392)."""
    import paper_1802_00166_b200 as P

    cells = []
    with P.GpuExecutor(kernel, params, device=device) as ex:
        if verify and want is None:
            want = ex.run_untiled().checksum_hex
        for scheme in schemes:
            for tile in tiles if scheme != "untiled" else [[]]:
                if warmup:
                    ex.run(scheme, tile, skip_checksum=True)  # warm-up / plan build
                rs = [ex.run(scheme, tile, skip_checksum=not verify) for _ in range(samples)]
                ms = [r.device_ms for r in rs]
                mean = statistics.fmean(ms)
                sd = statistics.pstdev(ms) if len(ms) > 1 else 0.0
                sums = sorted({r.checksum_hex for r in rs}) if verify else []
                cell = {"scheme": scheme, "tile": tile, "samples": samples, "ms_mean": mean,
                        "ms_stddev": sd, "ms_cov": sd / mean if mean else 0.0, "ms": ms,
                        "launches": rs[0].launches, "bt": rs[0].bt, "dram_bytes": None,
                        "l2_hit_pct": None, "checksum": "|".join(sums),
                        "parity": (None if not verify else "ok" if sums == [want] else "MISMATCH")}
                cells.append(cell)
    if ncu:
        for c in cells:
            c["dram_bytes"], c["l2_hit_pct"] = _ncu_cell(kernel, params, c["scheme"], c["tile"])
    return cells


def sweep_csv(cells):
    """CSV in the spirit of the reference sweep CSV (formats.md), OCA -> DRAM bytes."""
    out = [CSV_HEADER]
    for c in cells:
        out.append("%s,%s,%d,%.4f,%.4f,%.6f,%d,%s,%s,%s,%s" % (
            c["scheme"], "x".join(map(str, c["tile"])) or "-", c["samples"], c["ms_mean"],
            c["ms_stddev"], c["ms_cov"], c["launches"],
            "" if c["dram_bytes"] is None else "%.0f" % c["dram_bytes"],
            "" if c["l2_hit_pct"] is None else "%.2f" % c["l2_hit_pct"],
            c.get("checksum", ""), c.get("parity") or ""))
    return "\n".join(out) + "\n"


def summary_lines(cells):
    """Per scheme, pooled over every sample of every cell (reference
    formats.md "sweep CSV": `summary scheme=... cells=... mean=... stddev=...
    cov=...`), here in device milliseconds."""
    lines = []
    for scheme in dict.fromkeys(c["scheme"] for c in cells):
        ms = [v for c in cells if c["scheme"] == scheme for v in c.get("ms", [c["ms_mean"]])]
        mean = statistics.fmean(ms)
        sd = statistics.pstdev(ms) if len(ms) > 1 else 0.0
        n = sum(1 for c in cells if c["scheme"] == scheme)
        lines.append("summary scheme=%s cells=%d mean=%.4f stddev=%.4f cov=%.6f"
                     % (scheme, n, mean, sd, sd / mean if mean else 0.0))
    return lines


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("kernel")
    ap.add_argument("-p", "--params", required=True)
    ap.add_argument("--tiles", required=True)
    ap.add_argument("--schemes", default="slt,cot")
    ap.add_argument("--samples", type=int, default=3)
    ap.add_argument("--ncu", action="store_true")
    ap.add_argument("--csv")
    ap.add_argument("--quiet", action="store_true")
    ap.add_argument("--no-warmup", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the per-sample checksums")
    ap.add_argument("--want", help="expected checksum (default: the untiled run's)")
    a = ap.parse_args(argv)
    cells = run_sweep(a.kernel, parse_params(a.params), parse_tiles(a.tiles),
                      a.schemes.split(","), a.samples, ncu=a.ncu, warmup=not a.no_warmup,
                      want=a.want, verify=not a.no_verify)
    text = sweep_csv(cells)
    if a.csv:
        with open(a.csv, "w") as f:
            f.write(text)
    if not a.quiet:
        sys.stdout.write(text)
        for line in summary_lines(cells):
            print(line)
    bad = [c for c in cells if c["parity"] == "MISMATCH"]
    if bad:
        sys.stderr.write("sweep: %d cell(s) differ from the expected checksum\n" % len(bad))
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
