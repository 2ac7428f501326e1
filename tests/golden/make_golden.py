#!/usr/bin/env python3
"""Generate tests/golden/golden.json by running the UNMODIFIED reference.

TEST INFRASTRUCTURE.  Runs in the build container only (needs
/root/reference, compiled by `make -C oracle`):

* small sizes: the reference interpreter (`Executor`, reference
  core/src/exec.cpp) under `allocate()` maps AND single-assignment maps, with
  the shadow-version dependence oracle on, untiled + SLT + COT orders
  (the parity template of reference tests/acceptance.cpp:345-392);
* BASELINE config sizes: the reference's emitted recursive C (emit_c,
  use_alloc, OpenMP tasks), compiled with the reference build line
  `cc -std=c99 -O2 -ffp-contract=off -fopenmp` (tools/pcot.cpp:489-493),
  which the reference asserts is bit-identical to the interpreter
  (tests/acceptance.cpp:662-711).

Every entry records the FNV-1a checksum of the output array (reference
formats.md "CHECKSUM").  Tiny cases also record the output cells as hex bit
patterns.

    python tests/golden/make_golden.py [--big]
"""
import argparse
import json
import os
import re
import subprocess
import sys
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_BIN = os.path.join(REPO, "oracle", "_ref", "pcot_ref")
CORPUS = "/root/reference/proj/kernels"
KDIR = os.path.join(REPO, "kernels")
OUT = os.path.join(REPO, "tests", "golden", "golden.json")
GCC = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"


def kernel_path(name):
    p = os.path.join(KDIR, name + ".kernel")
    return p if os.path.exists(p) else name  # corpus kernels via PCOT_KERNEL_PATH


def env():
    e = dict(os.environ)
    e["PCOT_KERNEL_PATH"] = CORPUS
    return e


def pstr(params):
    return ",".join("%s=%d" % kv for kv in params.items())


def run_interp(name, params, scheme="untiled", tile=None, alloc=True, dump=None):
    cmd = [REF_BIN, "run", kernel_path(name), pstr(params), "--scheme", scheme]
    if tile:
        cmd += ["--tile", ",".join(map(str, tile))]
    if alloc:
        cmd.append("--alloc")
    if dump:
        cmd += ["--dump", dump]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env())
    if out.returncode != 0:
        raise RuntimeError("%s failed: %s %s" % (cmd, out.stdout, out.stderr))
    kv = dict(l.split(" ", 1) for l in out.stdout.strip().splitlines())
    return kv


def run_emitted(name, params, leaf, threads=8):
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "k.c")
        b = os.path.join(d, "k")
        subprocess.run([REF_BIN, "emit", kernel_path(name), pstr(params), "--openmp",
                        "--leaf", ",".join(map(str, leaf)), "-o", c], check=True, env=env())
        subprocess.run([GCC, "-std=c99", "-O2", "-ffp-contract=off", "-fopenmp", c, "-lm",
                        "-o", b], check=True)
        e = env()
        e["OMP_NUM_THREADS"] = str(threads)
        out = subprocess.run([b], capture_output=True, text=True, env=e, check=True)
        m = re.search(r"CHECKSUM ([0-9a-f]{16})", out.stdout)
        return m.group(1)


SMALL = [
    # (kernel, params, tiles for SLT/COT, dump cells)
    ("jacobi2d", {"T": 0, "N": 8}, [(1, 4, 4)], True),
    ("jacobi2d", {"T": 1, "N": 3}, [(1, 2, 2)], True),
    ("jacobi2d", {"T": 4, "N": 8}, [(2, 4, 4)], True),
    ("jacobi2d", {"T": 16, "N": 64}, [(8, 32, 32), (4, 16, 64)], False),
    ("jacobi2d", {"T": 13, "N": 37}, [(4, 8, 16)], False),
    ("jacobi2d", {"T": 32, "N": 130}, [(8, 32, 32)], False),
    ("heat2d", {"T": 16, "N": 64}, [(8, 32, 32)], False),
    ("heat2d", {"T": 9, "N": 23}, [(4, 8, 8)], False),
    ("heat2d", {"T": 32, "N": 256}, [], False),
    ("heat3d_b", {"T": 3, "N": 8}, [(2, 4, 4, 4)], True),
    ("heat3d_b", {"T": 8, "N": 24}, [(4, 8, 8, 8)], False),
    ("heat3d_b", {"T": 5, "N": 19}, [(2, 8, 8, 8)], False),
    ("heat3d_b", {"T": 12, "N": 40}, [], False),
    ("heat3d", {"T": 8, "N": 24}, [(4, 8, 8, 8)], False),
    ("heat3d", {"T": 5, "N": 17}, [], False),
    ("gs2d", {"T": 4, "N": 12}, [(2, 4, 8)], True),
    ("gs2d", {"T": 1, "N": 3}, [], True),
    ("gs2d", {"T": 8, "N": 33}, [(4, 8, 16)], False),
    ("gs2d", {"T": 16, "N": 64}, [(8, 16, 32)], False),
    ("gs2d", {"T": 6, "N": 101}, [], False),
    ("gemm", {"N": 1}, [], True),
    ("gemm", {"N": 16}, [(4, 4, 4)], True),
    ("gemm", {"N": 33}, [(8, 8, 8)], False),
    ("gemm", {"N": 64}, [(16, 16, 16)], False),
]

BIG = [
    # BASELINE configs 0-3 (config 4 is pinned through size-independent
    # properties + the config-0 golden; its oracle needs ~34 GB and ~1 h).
    ("jacobi2d", {"T": 256, "N": 2048}, (32, 128, 512)),
    ("heat3d_b", {"T": 100, "N": 384}, (16, 32, 32, 128)),
    ("gs2d", {"T": 64, "N": 4096}, (16, 64, 1024)),
    ("gemm", {"N": 4096}, (64, 64, 64)),
    # mid sizes used by the GPU parity tests
    ("jacobi2d", {"T": 64, "N": 1024}, (16, 64, 256)),
    ("jacobi2d", {"T": 40, "N": 1000}, (16, 64, 256)),
    ("heat2d", {"T": 64, "N": 1024}, (16, 64, 256)),
    ("heat3d_b", {"T": 20, "N": 130}, (8, 16, 16, 64)),
    ("heat3d", {"T": 20, "N": 130}, (8, 16, 16, 64)),
    ("gs2d", {"T": 16, "N": 1024}, (8, 32, 512)),
    ("gs2d", {"T": 5, "N": 1000}, (4, 32, 512)),
    ("gemm", {"N": 512}, (32, 32, 32)),
    ("gemm", {"N": 1000}, (32, 32, 32)),
]

# BASELINE config 4 at full size (32768^2, T=512): the emitted C needs ~34 GB of
# host RAM and ~20-30 min on 8 cores, so it runs only on request (--cfg4).
HUGE = [
    ("jacobi2d", {"T": 512, "N": 32768}, (16, 128, 1024)),
]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also run the emitted-C goldens")
    ap.add_argument("--cfg4", action="store_true", help="also run config 4 at full size (~34 GB RAM)")
    args = ap.parse_args()
    if not os.path.exists(REF_BIN):
        sys.exit("build the reference first: make -C oracle")
    old = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            for e in json.load(f)["entries"]:
                old[(e["kernel"], pstr(e["params"]))] = e
    entries = []
    for name, params, tiles, dump in SMALL:
        with tempfile.TemporaryDirectory() as d:
            dp = os.path.join(d, "out.bin")
            base = run_interp(name, params, dump=dp if dump else None)
            cells = None
            if dump:
                raw = open(dp, "rb").read()
                cells = [raw[i:i + 8][::-1].hex() for i in range(0, len(raw), 8)]
        checks = ["untiled+alloc"]
        sa = run_interp(name, params, alloc=False)
        assert sa["CHECKSUM"] == base["CHECKSUM"], (name, params, "single-assignment")
        checks.append("untiled+single")
        for tile in tiles:
            for scheme in ("slt", "cot"):
                r = run_interp(name, params, scheme, tile)
                assert r["CHECKSUM"] == base["CHECKSUM"], (name, params, scheme, tile)
                assert r["violation"] == "0", (name, params, scheme, tile)
                checks.append("%s%s" % (scheme, list(tile)))
        assert base["violation"] == "0"
        if name in ("heat2d", "heat3d"):  # this repo's restatement of the corpus kernel
            mine = run_interp(os.path.join(KDIR, name + "_hold.kernel"), params)
            assert mine["CHECKSUM"] == base["CHECKSUM"], (name, params, "hold restatement")
            checks.append("%s_hold.kernel" % name)
        e = {"kernel": name, "params": params, "checksum": base["CHECKSUM"],
             "source": "reference interpreter (Executor, check_oracle=on)",
             "points": int(base["points"]), "schemes_agree": checks}
        if cells is not None:
            e["out_hex"] = cells
        entries.append(e)
        print(name, params, base["CHECKSUM"], checks, flush=True)
    for name, params, leaf in BIG:
        key = (name, pstr(params))
        if not args.big and key in old:
            entries.append(old[key])
            continue
        if not args.big:
            continue
        chk = run_emitted(name, params, leaf)
        entries.append({"kernel": name, "params": params, "checksum": chk,
                        "source": "reference emitted C (emit_c use_alloc, -O2 "
                                  "-ffp-contract=off -fopenmp), leaf %s" % list(leaf)})
        print(name, params, chk, flush=True)
    for name, params, leaf in HUGE:
        key = (name, pstr(params))
        if not args.cfg4:
            if key in old:
                entries.append(old[key])
            continue
        chk = run_emitted(name, params, leaf, threads=os.cpu_count() or 8)
        entries.append({"kernel": name, "params": params, "checksum": chk,
                        "source": "reference emitted C (emit_c use_alloc, -O2 "
                                  "-ffp-contract=off -fopenmp), leaf %s" % list(leaf)})
        print(name, params, chk, flush=True)
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "/root/reference/proj (compiled by oracle/Makefile)",
                   "entries": entries}, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
