"""CPU: the drop-in boundary — C-ABI library loads, exports every declared
symbol, and the host-side registration path (kernel JSON parse + recognizer)
behaves like the reference's (names, counters, error kinds)."""
import json
import os
import re

import pytest

import paper_1802_00166_b200 as P
from tests import oracle_ctypes as O

HEADER = os.path.join(O.REPO, "include", "pcotgpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(pcotgpu_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = P.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    bound = {name for name, _, _ in P._SIGS}
    assert set(syms) <= bound, set(syms) - bound
    assert L.pcotgpu_abi_version() == 1


def test_fnv1a_through_abi():
    assert P.fnv1a(b"") == 0xcbf29ce484222325
    assert P.fnv1a(b"a") == 0xaf63dc4c8601ec8c


@pytest.mark.parametrize("e", [e for e in O.goldens() if "points" in e],
                         ids=lambda e: "%s-%s" % (e["kernel"], e["params"]))
def test_recognizer_counters_match_reference(e):
    info = P.recognize(O.kernel_path(e["kernel"]), e["params"])
    # ExecResult.points of the reference interpreter run (closed form here)
    assert info.points == e["points"]
    fam = {"jacobi2d": "stencil2d5", "heat2d": "stencil2d5", "heat3d_b": "stencil3d7",
           "heat3d": "stencil3d7", "gs2d": "gs2d9", "gemm": "gemm"}[e["kernel"]]
    assert info.family_name == fam


def test_recognizer_fields():
    i = P.recognize("jacobi2d", {"T": 256, "N": 2048})
    assert (i.family_name, i.ring_hold, i.T, i.N) == ("stencil2d5", 0, 256, 2048)
    i = P.recognize(O.kernel_path("heat2d"), {"T": 5, "N": 9})
    assert i.ring_hold == 1
    i = P.recognize("heat3d_b", {"T": 100, "N": 384})
    assert (i.family_name, i.rule, i.ring_hold) == ("stencil3d7", 0, 0)
    i = P.recognize(O.kernel_path("heat3d"), {"T": 3, "N": 7})
    assert (i.rule, i.ring_hold) == (1, 1)
    i = P.recognize("gemm", {"N": 4096})
    assert (i.family_name, i.N) == ("gemm", 4096)
    # huge sizes recognise in closed form (no enumeration)
    i = P.recognize("jacobi2d", {"T": 512, "N": 32768})
    assert i.points == (32768 - 2) ** 2 + 513 * (4 * 32768 - 4) + 512 * (32768 - 2) ** 2 + 32768 ** 2


def _spec(name):
    with open(O.kernel_path(name)) as f:
        return json.load(f)


def test_error_kinds_mirror_reference():
    with pytest.raises(P.PcotError) as ex:
        P.recognize("{ not json", [1, 2])
    assert ex.value.kind == "Parse"
    k = _spec("jacobi2d")
    with pytest.raises(P.PcotError) as ex:  # wrong parameter count -> DimMismatch
        P.recognize(json.dumps(k), [4])
    assert ex.value.kind == "DimMismatch"
    bad = json.loads(json.dumps(k))
    bad["statements"][5]["body"] = bad["statements"][5]["body"].replace("0.2", "0.25")
    with pytest.raises(P.PcotError) as ex:  # not a registered update body
        P.recognize(json.dumps(bad), [4, 8])
    assert ex.value.kind == "Unsupported"
    bad = json.loads(json.dumps(k))
    bad["statements"][5]["body"] = "0.2 * (X[t - 1, x - 1, y - 1] + Q[t, x])"
    with pytest.raises(P.PcotError) as ex:  # read of an undeclared array (kernel_io.cpp:75)
        P.recognize(json.dumps(bad), [4, 8])
    assert ex.value.kind == "Validation"
    bad["statements"][5]["body"] = "0.2 * (X[t - 1, x - 1, y - 1] + q)"
    with pytest.raises(P.PcotError) as ex:  # unknown name in the body grammar
        P.recognize(json.dumps(bad), [4, 8])
    assert ex.value.kind == "Parse"
    bad = json.loads(json.dumps(k))
    bad["statements"][1]["domain"] = bad["statements"][1]["domain"][2:]  # ring piece loses t bounds
    with pytest.raises(P.PcotError) as ex:
        P.recognize(json.dumps(bad), [4, 8])
    assert ex.value.kind in ("Unbounded", "Unsupported")
    bad = json.loads(json.dumps(k))
    del bad["statements"][2]  # ring no longer covered
    with pytest.raises(P.PcotError) as ex:
        P.recognize(json.dumps(bad), [4, 8])
    assert ex.value.kind == "Unsupported"
    bad = json.loads(json.dumps(k))
    bad["statements"][0]["depth"] = 2
    bad["statements"][0]["domain"] = [r[:2] + r[3:] for r in bad["statements"][0]["domain"]]
    bad["statements"][0]["writes"]["subscripts"] = ["0", "x", "x"]
    bad["statements"][0]["body"] = "F[x, x]"
    with pytest.raises(P.PcotError) as ex:  # reference: "kernel must be embedded"
        P.recognize(json.dumps(bad), [4, 8])
    assert ex.value.kind == "Validation"


def test_find_kernel_file_search_order(tmp_path, monkeypatch):
    d = tmp_path / "kdir"
    d.mkdir()
    (d / "mine.kernel").write_text(open(O.kernel_path("jacobi2d")).read())
    monkeypatch.setenv("PCOT_KERNEL_PATH", "/nonexistent:" + str(d))
    assert P.find_kernel_file("mine") == str(d / "mine.kernel")
    assert P.find_kernel_file("mine.kernel") == str(d / "mine.kernel")
    assert P.find_kernel_file(O.kernel_path("gs2d")) == O.kernel_path("gs2d")
    assert P.find_kernel_file("no-such-kernel") == ""


def test_gpu_path_fails_loudly_without_device():
    n = P.ctypes.c_int()
    P.lib().pcotgpu_device_count(P.ctypes.byref(n))
    if n.value > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(P.PcotError) as ex:
        P.GpuExecutor("jacobi2d", {"T": 2, "N": 8})
    assert ex.value.kind == "Cuda"
