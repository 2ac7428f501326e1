"""Corpus kernels outside the hot-path registry (triangle, lud, osp,
heat1d-fig7) on the device interpreter (csrc/generic.cu), against the
reference interpreter's checksums and ExecResult counters
(tests/golden/corpus.json, made by tests/golden/make_corpus_golden.py from the
reference corpus files).  The restated specs in kernels/ are pinned to those
same goldens through the compiled reference when it is present.
"""
import json
import os
import subprocess

import numpy as np
import pytest

import paper_1802_00166_b200 as P
from tests import oracle_ctypes as O

with open(os.path.join(O.REPO, "tests", "golden", "corpus.json")) as _f:
    CORPUS = json.load(_f)["entries"]
REF_BIN = os.path.join(O.REPO, "oracle", "_ref", "pcot_ref")


def _id(e):
    return "%s-%s" % (e["kernel"], "-".join("%s%d" % kv for kv in e["params"].items()))


def _kpath(name):
    return os.path.join(O.REPO, "kernels", name + ".kernel")


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="reference driver not built (oracle/_ref)")
@pytest.mark.parametrize("e", CORPUS, ids=[_id(e) for e in CORPUS])
def test_restated_corpus_specs_match_reference(e):
    """kernels/<name>.kernel run by the compiled reference == the corpus file's golden."""
    ps = ",".join("%s=%d" % kv for kv in e["params"].items())
    out = subprocess.run([REF_BIN, "run", _kpath(e["kernel"]), ps, "--scheme", "untiled"],
                         capture_output=True, text=True, timeout=300)
    kv = dict(l.split(" ", 1) for l in out.stdout.strip().splitlines())
    assert kv["CHECKSUM"] == e["checksum"]
    assert (int(kv["points"]), int(kv["reads"]), int(kv["writes"])) == (e["points"], e["reads"], e["writes"])


def test_generic_kernels_are_outside_the_registry():
    for name in ("triangle", "lud", "osp", "heat1d-fig7"):
        with pytest.raises(P.PcotError) as ex:
            P.recognize(_kpath(name), json.load(open(_kpath(name)))["check_params"])
        assert ex.value.kind in ("Unsupported", "Validation")


@pytest.mark.gpu
@pytest.mark.parametrize("e", CORPUS, ids=[_id(e) for e in CORPUS])
def test_corpus_kernel_on_device_matches_reference(e):
    with P.GpuExecutor(_kpath(e["kernel"]), e["params"]) as ex:
        assert ex.info.family == 5  # generic interpreter
        r = ex.run_untiled()
        assert r.checksum_hex == e["checksum"]
        assert (r.points, r.reads, r.writes) == (e["points"], e["reads"], e["writes"])
        assert r.launches > 0
        if "out_hex" in e:
            out = ex.array_data("Out")
            want = np.array([int(h, 16) for h in e["out_hex"]], dtype=np.uint64)
            assert np.array_equal(out.view(np.uint64), want)
        assert ex.run_untiled().checksum_hex == e["checksum"]  # rerun: same storage reset


SMALL = [e for e in O.goldens() if "out_hex" in e and "points" in e]


@pytest.mark.gpu
@pytest.mark.parametrize("e", SMALL, ids=[_id(e) for e in SMALL])
def test_registry_kernels_through_the_interpreter(monkeypatch, e):
    """PCOTGPU_FORCE_GENERIC: the hot-path kernels' specs through the generic
    interpreter reproduce the same goldens (an independent device path)."""
    monkeypatch.setenv("PCOTGPU_FORCE_GENERIC", "1")
    with P.GpuExecutor(O.kernel_path(e["kernel"]), e["params"]) as ex:
        assert ex.info.family == 5
        r = ex.run_untiled()
        assert r.points == e["points"]
        out = ex.array_data("Out")
        want = np.array([int(h, 16) for h in e["out_hex"]], dtype=np.uint64)
        if e["kernel"] == "gemm":  # the interpreter runs the spec's sequential-k order: exact
            assert np.array_equal(out.view(np.uint64), want)
        assert r.checksum_hex == e["checksum"]


@pytest.mark.gpu
def test_interpreter_input_from_host_and_errors():
    with P.GpuExecutor(_kpath("triangle"), {"N": 12}) as ex:
        B = ex.array_data("B")
        ex.write_array("B", 2.0 * B)
        r2 = ex.run_untiled()
        out2 = ex.array_data("Out")
        ex.reset()
        ex.run_untiled()
        assert np.array_equal(out2, 2.0 * ex.array_data("Out"))  # linear recurrence, power of 2
        assert r2.points == 90
    spec = json.load(open(_kpath("triangle")))
    spec["statements"][1]["body"] = "C[i - 1, j - 1] + C[i, j + 5]"  # reads past the extent
    with P.GpuExecutor(json.dumps(spec), {"N": 12}) as ex:
        with pytest.raises(P.PcotError) as err:
            ex.run_untiled()
        assert err.value.kind == "Validation"


# Reads that the reference's order serves from a cell's OLD value (the reading
# statement's own write, or a write by a later point).  Checksums from the
# unmodified reference (`pcot_ref run <k> N=8 --scheme untiled`; its shadow
# oracle also flags the kernels as violating, which the reference reports
# instead of rejecting).  The dataflow grid would wait for those writes; the
# interpreter must detect the order and run them sequentially.
ORDER_CASES = [("selfread", "84f9cec8af7cb928"), ("futureread", "de90f9ad18f16e28")]


@pytest.mark.gpu
@pytest.mark.parametrize("name,want", ORDER_CASES)
def test_interpreter_read_before_write_runs_in_reference_order(name, want):
    import time

    path = os.path.join(O.REPO, "tests", "kernels_extra", name + ".kernel")
    with P.GpuExecutor(path, {"N": 8}) as ex:
        t0 = time.perf_counter()
        r = ex.run_untiled()
        assert time.perf_counter() - t0 < 5.0  # no dependence wait until a spin cap
        assert r.checksum_hex == want
        assert (r.points, r.reads, r.writes) == (8, 16, 8)


@pytest.mark.skipif(not os.path.exists(REF_BIN), reason="reference driver not built (oracle/_ref)")
@pytest.mark.parametrize("name,want", ORDER_CASES)
def test_read_before_write_goldens_match_reference(name, want):
    path = os.path.join(O.REPO, "tests", "kernels_extra", name + ".kernel")
    out = subprocess.run([REF_BIN, "run", path, "N=8", "--scheme", "untiled"],
                         capture_output=True, text=True, timeout=60)
    kv = dict(l.split(" ", 1) for l in out.stdout.strip().splitlines())
    assert kv["CHECKSUM"] == want
