"""The drop-in boundary from plain C (tests/c/abi_demo.c against
include/pcotgpu.h and libpcotgpu.so): builds on CPU, runs on the GPU."""
import os
import subprocess

import pytest

from tests import oracle_ctypes as O

SRC = os.path.join(O.REPO, "tests", "c", "abi_demo.c")
LIBDIR = os.path.join(O.REPO, "paper_1802_00166_b200")
GCC = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"


def build(tmp_path):
    exe = str(tmp_path / "abi_demo")
    subprocess.run([GCC, "-std=c99", "-O2", "-I", os.path.join(O.REPO, "include"), SRC, "-L", LIBDIR,
                    "-lpcotgpu", "-Wl,-rpath," + LIBDIR, "-o", exe], check=True)
    return exe


def test_c_consumer_compiles_and_links(tmp_path):
    exe = build(tmp_path)
    assert os.path.exists(exe)


def _golden(kernel, **params):
    for e in O.goldens():
        if e["kernel"] == kernel and e["params"] == params:
            return e
    raise KeyError(kernel)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel,params,scheme,leaf", [
    ("jacobi2d", {"T": 40, "N": 1000}, 1, 5),
    ("gs2d", {"T": 16, "N": 1024}, 0, 0),
    ("heat3d_b", {"T": 20, "N": 130}, 2, 2),
])
def test_c_consumer_runs_and_matches_reference(tmp_path, kernel, params, scheme, leaf):
    exe = build(tmp_path)
    args = [exe, O.kernel_path(kernel)] + [str(v) for v in params.values()] + [str(scheme), str(leaf)]
    out = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    kv = dict(l.split(" ", 1) for l in out.stdout.strip().splitlines())
    assert kv["CHECKSUM"] == _golden(kernel, **params)["checksum"]
