"""PRDG -> CUDA emitter (the GPU analogue of the reference's
emit_c, emit_c.cpp:191-262): the device interpreter's kernels emitted as
straight-line CUDA per statement — constant domain rows, one IEEE-rounded
intrinsic per body operation in the reference's postfix order — and compiled
by NVRTC for sm_100a.  CPU: the emitted source of every corpus kernel and of a
hot-path spec compiles; GPU: compiled and interpreted runs give the
reference's bits."""
import json
import os

import numpy as np
import pytest

import paper_1802_00166_b200 as P
from tests import oracle_ctypes as O

KDIR = os.path.join(O.REPO, "kernels")
CASES = [("lud", {"N": 8}), ("osp", {"N": 9}), ("triangle", {"N": 12}),
         ("heat1d-fig7", {"T": 10, "N": 20}), ("jacobi2d", {"T": 4, "N": 8}), ("gs2d", {"T": 4, "N": 12})]


def _kp(name):
    return os.path.join(KDIR, name + ".kernel")


@pytest.mark.parametrize("name,params", CASES, ids=[c[0] for c in CASES])
def test_emitted_source_compiles_for_sm100a(name, params):
    src = P.generic_source(_kp(name), params, compile=True)
    spec = json.load(open(_kp(name)))
    # one guarded block and one write per statement, rounding intrinsics only
    assert src.count("if (!gwrite<MODE>") == len(spec["statements"])
    body = src.split("struct JitPE")[1]
    assert "fma" not in body  # one rounding per operation, never contracted
    assert "__dadd_rn" in body or "__dsub_rn" in body or name == "osp"


def test_emitted_body_keeps_the_reference_operand_order():
    src = P.generic_source(_kp("jacobi2d"), {"T": 4, "N": 8})
    body = src.split("struct JitPE")[1]
    # 0.2 * ((((c + N) + S) + W) + E): four chained adds, then the multiply by the literal
    i = body.index("__dmul_rn(")
    adds = body[:i].count("__dadd_rn(")
    assert adds >= 4 and "0x1.999999999999ap-3" in body


GPU_CASES = [e for e in json.load(open(os.path.join(O.REPO, "tests", "golden", "corpus.json")))["entries"]
             if e["points"] > 50]


@pytest.mark.gpu
@pytest.mark.parametrize("e", GPU_CASES, ids=["%s-%s" % (e["kernel"], "-".join("%s%d" % kv for kv in e["params"].items()))
                                              for e in GPU_CASES])
def test_compiled_and_interpreted_runs_agree_with_reference(monkeypatch, e):
    got = {}
    for jit in ("1", "0"):
        monkeypatch.setenv("PCOTGPU_GENERIC_JIT", jit)
        with P.GpuExecutor(_kp(e["kernel"]), e["params"]) as ex:
            r = ex.run_untiled()
            mode, compiled, why = ex.generic_info()
            assert compiled == (jit == "1"), why
            got[jit] = (r.checksum_hex, r.points, r.reads, r.writes, mode)
    assert got["1"] == got["0"]
    assert got["1"][0] == e["checksum"]
    assert got["1"][1:4] == (e["points"], e["reads"], e["writes"])
