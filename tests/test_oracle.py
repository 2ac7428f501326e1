"""CPU: pin the oracle (C restatement) against the reference's own outputs.

tests/golden/golden.json was produced by running the UNMODIFIED reference
(interpreter at small sizes, its emitted C at config sizes); see
tests/golden/make_golden.py.  The oracle must reproduce every checksum bit
for bit before any GPU parity claim rests on it.
"""
import os

import numpy as np
import pytest

from tests import oracle_ctypes as O

SMALL = [e for e in O.goldens() if "interpreter" in e["source"]]
BIG = [e for e in O.goldens() if "emitted" in e["source"]]


def _ids(entries):
    return ["%s-%s" % (e["kernel"], "-".join("%s%d" % kv for kv in e["params"].items()))
            for e in entries]


def test_fnv1a_known_answers():
    # reference tests/test_exec.cpp:20-24
    assert O.fnv1a(np.frombuffer(b"", dtype=np.uint8)) == 0xcbf29ce484222325
    assert O.fnv1a(np.frombuffer(b"a", dtype=np.uint8)) == 0xaf63dc4c8601ec8c


def test_init_value_range_and_determinism():
    # reference tests/test_exec.cpp:10-18
    a = O.init_array("F", 10000)
    b = O.init_array("F", 10000)
    assert np.array_equal(a, b)
    assert a.min() >= 0.0 and a.max() < 1.0
    assert not np.array_equal(a, O.init_array("G", 10000))
    assert O.lib().oracle_init_value(b"F", 1234) == a[1234]
    w = O.init_window("F", 100, 7, 11, 5, 9)
    assert np.array_equal(w, a.reshape(100, 100)[7:12, 11:20])


@pytest.mark.parametrize("e", SMALL, ids=_ids(SMALL))
def test_oracle_matches_reference_interpreter(e):
    out = O.reference_output(e["kernel"], e["params"])
    assert "%016x" % O.fnv1a(out) == e["checksum"]
    if "out_hex" in e:
        want = np.array([int(h, 16) for h in e["out_hex"]], dtype=np.uint64)
        assert np.array_equal(out.view(np.uint64), want)


@pytest.mark.parametrize("e", BIG, ids=_ids(BIG))
def test_oracle_matches_reference_emitted_c(e):
    if e["kernel"] == "gemm" and e["params"]["N"] > 1024:
        pytest.skip("N=4096 oracle GEMM is exercised on the GPU box (rows subset)")
    if e["params"].get("N", 0) >= 32768 and not os.environ.get("PCOT_FULL_ORACLE"):
        # config 4 at full size: 5.5e11 updates, ~5 min on 16 cores and 24 GiB; run with
        # PCOT_FULL_ORACLE=1 (passes: the oracle reproduces the reference's 2d0b3eb672343d76)
        pytest.skip("full-size config 4 oracle run: set PCOT_FULL_ORACLE=1")
    out = O.reference_output(e["kernel"], e["params"])
    assert "%016x" % O.fnv1a(out) == e["checksum"]


def test_oracle_gemm_matches_reference_config3_samples():
    """Config 3 (N=4096): the oracle's sequential-k GEMM reproduces the
    reference's emitted-C result bit for bit on 32 of its sampled cells
    (tests/golden/gemm4096_samples.json, generated from the reference's dump;
    its checksum equals the full-output golden)."""
    import json
    import os

    with open(os.path.join(O.REPO, "tests", "golden", "gemm4096_samples.json")) as f:
        g = json.load(f)
    N = g["params"]["N"]
    gold = [e["checksum"] for e in O.goldens() if e["kernel"] == "gemm" and e["params"] == {"N": N}]
    assert gold == [g["checksum"]]
    A = O.init_array("A", N * N)
    B = O.init_array("B", N * N)
    for i in range(0, N, N // 32):
        row = O.gemm(N, A, B, (i, i + 1)).reshape(N, N)[i]
        j = (i * 2654435761 + 12345) % N
        assert "%016x" % row[j:j + 1].view(np.uint64)[0] == g["out_hex"][i], (i, j)
