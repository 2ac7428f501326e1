#!/usr/bin/env python3
"""Generate tests/golden/corpus.json: the reference corpus kernels outside the
hot-path registry (triangle, lud, osp, heat1d-fig7), run by the UNMODIFIED
reference interpreter (oracle/_ref/pcot_ref, single-assignment storage,
dependence oracle on).

TEST INFRASTRUCTURE.  Runs in the build container only (needs /root/reference
and `make -C oracle`).  Records the FNV-1a output checksum, the ExecResult
counters (points / reads / writes, reference exec.cpp:404-407) and, for tiny
cases, the output cells as hex bit patterns.

    python tests/golden/make_corpus_golden.py
"""
import json
import os
import struct
import subprocess
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
REF_BIN = os.path.join(REPO, "oracle", "_ref", "pcot_ref")
CORPUS = "/root/reference/proj/kernels"
OUT = os.path.join(REPO, "tests", "golden", "corpus.json")

CASES = [
    ("triangle", {"N": 1}), ("triangle", {"N": 2}), ("triangle", {"N": 12}), ("triangle", {"N": 100}),
    ("lud", {"N": 1}), ("lud", {"N": 2}), ("lud", {"N": 8}), ("lud", {"N": 40}),
    ("osp", {"N": 2}), ("osp", {"N": 3}), ("osp", {"N": 9}), ("osp", {"N": 30}),
    ("heat1d-fig7", {"T": 1, "N": 3}), ("heat1d-fig7", {"T": 10, "N": 20}),
    ("heat1d-fig7", {"T": 50, "N": 200}),
]


# Large sizes under allocate()'s memory maps (the folded storage the
# reference's CLI uses with --alloc): the reference's emitted C (emit_c
# use_alloc, -O2 -ffp-contract=off -fopenmp), which the reference asserts is
# bit-identical to its interpreter (tests/acceptance.cpp:662-711).
MAPPED = [("lud", {"N": 512}), ("osp", {"N": 256}), ("triangle", {"N": 4096}),
          ("heat1d-fig7", {"T": 256, "N": 2048})]


def run_emitted(name, params):
    import re

    env = dict(os.environ, PCOT_KERNEL_PATH=CORPUS, OMP_NUM_THREADS=str(os.cpu_count() or 8))
    ps = ",".join("%s=%d" % kv for kv in params.items())
    with tempfile.TemporaryDirectory() as d:
        c, b = os.path.join(d, "k.c"), os.path.join(d, "k")
        subprocess.run([REF_BIN, "emit", name, ps, "--openmp", "-o", c], check=True, env=env)
        gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
        subprocess.run([gcc, "-std=c99", "-O2", "-ffp-contract=off", "-fopenmp", c, "-lm", "-o", b],
                       check=True)
        out = subprocess.run([b], capture_output=True, text=True, env=env, check=True).stdout
    return re.search(r"CHECKSUM ([0-9a-f]{16})", out).group(1)


def run(name, params, dump):
    env = dict(os.environ, PCOT_KERNEL_PATH=CORPUS)
    ps = ",".join("%s=%d" % kv for kv in params.items())
    cmd = [REF_BIN, "run", name, ps, "--scheme", "untiled", "--dump", dump]  # oracle on
    p = subprocess.run(cmd, capture_output=True, text=True, env=env)
    if p.returncode != 0:  # the driver's --dump handles square outputs only
        p = subprocess.run(cmd[:-2], capture_output=True, text=True, env=env, check=True)
    return dict(l.split(" ", 1) for l in p.stdout.strip().splitlines())


def main():
    entries = []
    for name, params in CASES:
        with tempfile.TemporaryDirectory() as d:
            dump = os.path.join(d, "out.bin")
            kv = run(name, params, dump)
            e = {"kernel": name, "params": params, "checksum": kv["CHECKSUM"],
                 "points": int(kv["points"]), "reads": int(kv["reads"]),
                 "writes": int(kv["writes"]), "violation": int(kv["violation"])}
            if os.path.exists(dump) and os.path.getsize(dump) <= 8 * 64:
                raw = open(dump, "rb").read()
                e["out_hex"] = ["%016x" % v for v in struct.unpack("<%dQ" % (len(raw) // 8), raw)]
            entries.append(e)
            print(name, params, e["checksum"], e["points"])
    mapped = []
    for name, params in MAPPED:
        chk = run_emitted(name, params)
        mapped.append({"kernel": name, "params": params, "checksum": chk, "maps": "allocate",
                       "source": "reference emitted C (emit_c use_alloc, OpenMP)"})
        print(name, params, chk, "(allocate maps)")
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_corpus_golden.py",
                   "reference": "oracle/_ref/pcot_ref run <kernel> --scheme untiled (single-assignment "
                                "storage; /root/reference/proj/kernels)",
                   "entries": entries, "mapped": mapped}, f, indent=1)


if __name__ == "__main__":
    main()
