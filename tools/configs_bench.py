#!/usr/bin/env python3
"""The five BASELINE configs on one B200 through the executor's default
schedule: throughput, bytes/update, roofline fraction and reference parity.

    python tools/configs_bench.py [--reps 3] > profiles/configs_r01.json

One JSON line per config.  Stencils: GUpd/s = N^d * T / device time of one
`run_untiled` (copy-in of F included), roofline = GUpd/s * 16/bt B against
the measured HBM copy bandwidth (MEASURED_PEAKS.json).  GEMM: TFLOP/s =
2N^3 / time against the measured DMMA peak (profiles/fp64_peaks_r01.json).
Parity: the run's FNV-1a checksum against the reference golden where one is
pinned (tests/golden/golden.json); GEMM is checked by the test-suite's
normwise/componentwise 1e-12 bound instead (reordered sums).
"""
import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_1802_00166_b200 as P  # noqa: E402

CONFIGS = [
    ("cfg0", "jacobi2d", {"T": 256, "N": 2048}, 2),
    ("cfg1", "heat3d_b", {"T": 100, "N": 384}, 3),
    ("cfg2", "gs2d", {"T": 64, "N": 4096}, 2),
    ("cfg3", "gemm", {"N": 4096}, 2),
    ("cfg4", "jacobi2d", {"T": 512, "N": 32768}, 2),
]


def peaks():
    hbm = 6552.3
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        hbm = float(d.get("hbm_gbs", hbm))
    except (OSError, ValueError):
        pass
    dmma = 37.1
    try:
        with open(os.path.join(REPO, "profiles", "fp64_peaks_r01.json")) as f:
            d = json.load(f)
        dmma = max(r["TFLOPs"] for r in d["results"] if r["probe"].startswith("dmma"))
    except (OSError, ValueError, KeyError):
        pass
    return hbm, dmma


def golden(kernel, params):
    with open(os.path.join(REPO, "tests", "golden", "golden.json")) as f:
        g = json.load(f)
    for e in g["entries"]:
        if e["kernel"] == kernel and e["params"] == params:
            return e["checksum"]
    return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    hbm, dmma = peaks()
    for name, kernel, params, reps in CONFIGS:
        if a.only and name not in a.only.split(","):
            continue
        big = params.get("N", 0) >= 32768
        with P.GpuExecutor(kernel, params) as ex:
            first = ex.run_untiled(skip_checksum=big)
            times = [ex.run_untiled(skip_checksum=True).device_ms for _ in range(max(1, min(reps, a.reps)))]
            ms = sorted(times)[len(times) // 2]
            line = {"config": name, "kernel": kernel, "params": params, "ms": round(ms, 3),
                    "bt": first.bt, "launches": first.launches}
            if kernel == "gemm":
                tf = 2 * params["N"] ** 3 / (ms / 1e3) / 1e12
                line.update({"TFLOP/s": round(tf, 2), "roofline": {"bound": "fp64 DMMA", "peak_TFLOPs": dmma,
                                                                    "frac": round(tf / dmma, 3)},
                             "parity": "normwise/componentwise <= 1e-12 (tests/test_gpu_parity.py)"})
            else:
                nd = 3 if kernel.startswith("heat3d") else 2
                upd = params["N"] ** nd * params["T"]
                gu = upd / (ms / 1e3) / 1e9
                line["GUpd/s"] = round(gu, 1)
                if kernel == "gs2d":
                    line["roofline"] = {"bound": "fp64 dependence latency (in-place wavefront)",
                                        "note": "HBM traffic ~1 B/update: F in, Out back, one wrap "
                                                "buffer round trip per 16 sweeps"}
                else:
                    bpu = 16.0 / max(first.bt, 1)
                    line["roofline"] = {"bound": "hbm", "bytes_per_update": bpu, "peak_GBs": hbm,
                                        "achieved_GBs": round(gu * bpu, 1), "frac": round(gu * bpu / hbm, 3)}
                want = golden(kernel, params)
                if want and not big:
                    line["parity"] = {"golden": want, "got": first.checksum_hex,
                                      "match": first.checksum_hex == want}
                elif big:
                    line["parity"] = "full-size windows/ring/scaling (tests/test_gpu_parity.py::test_config4...)"
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
