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
    with open(OUT, "w") as f:
        json.dump({"generator": "tests/golden/make_corpus_golden.py",
                   "reference": "oracle/_ref/pcot_ref run <kernel> --scheme untiled (single-assignment "
                                "storage; /root/reference/proj/kernels)",
                   "entries": entries}, f, indent=1)


if __name__ == "__main__":
    main()
