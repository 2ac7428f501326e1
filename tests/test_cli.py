"""`pcot run --executor gpu`: integration/pcot_run_gpu.cpp, the
reference CLI's cmd_run (tools/pcot.cpp:238-336) with the executor switch,
built against the unmodified reference front end (oracle/Makefile ->
oracle/_ref/pcot_run).  The GPU run must print the same points / reads /
writes / leaves / nodes / CHECKSUM lines as the reference's CPU executor."""
import os
import subprocess

import pytest

from tests import oracle_ctypes as O

CLI = os.path.join(O.REPO, "oracle", "_ref", "pcot_run")
KDIR = os.path.join(O.REPO, "kernels")
pytestmark = pytest.mark.skipif(not os.path.exists(CLI), reason="pcot_run not built (needs /root/reference)")


def _run(args):
    p = subprocess.run([CLI] + args, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, PCOT_KERNEL_PATH=KDIR))
    kv = dict(l.split(" ", 1) for l in p.stdout.strip().splitlines() if " " in l)
    return p.returncode, kv, p.stdout + p.stderr


def test_cpu_executor_is_the_reference():
    rc, kv, txt = _run(["jacobi2d", "-p", "T=16,N=64", "--scheme", "cot", "--tile", "8,32,32",
                        "--executor", "cpu"])
    assert rc == 0, txt
    assert kv["CHECKSUM"] == "8ac68aaa5f994860" and kv["executor"] == "cpu"
    assert kv["tile"] == "8x32x32" and int(kv["OCA"]) > 0


def test_usage_and_io_exit_codes():
    assert _run(["jacobi2d", "-p", "T=16"])[0] == 2            # N not set
    assert _run(["jacobi2d", "-p", "T=4,N=8", "--scheme", "zig"])[0] == 2
    assert _run(["jacobi2d", "-p", "T=4,N=8", "--scheme", "slt"])[0] == 2  # --tile required
    assert _run(["jacobi2d", "-p", "T=4,N=8", "--executor", "tpu"])[0] == 2
    assert _run(["no_such_kernel", "-p", "N=4"])[0] == 3


CASES = [
    ["jacobi2d", "-p", "T=16,N=64", "--scheme", "cot", "--tile", "8,32,32"],
    ["jacobi2d", "-p", "T=13,N=37", "--scheme", "slt", "--tile", "4,8,16", "--alloc"],
    ["heat3d_b", "-p", "T=5,N=19", "--alloc"],
    ["gs2d", "-p", "T=8,N=33", "--scheme", "cot", "--tile", "4,8,16", "--alloc"],
    ["lud", "-p", "N=40", "--alloc"],
    ["osp", "-p", "N=30", "--scheme", "slt", "--tile", "4,4"],
    ["heat1d-fig7", "-p", "T=10,N=20", "--alloc"],
]


@pytest.mark.gpu
@pytest.mark.parametrize("args", CASES, ids=["-".join(a[:1] + a[2:3] + a[3:5]) for a in CASES])
def test_gpu_executor_prints_the_references_results(args):
    rc, cpu, txt = _run(args + ["--executor", "cpu", "--no-check"])
    assert rc == 0, txt
    rc, gpu, txt = _run(args + ["--executor", "gpu"])
    assert rc == 0, txt
    for k in ("kernel", "params", "scheme", "tile", "points", "reads", "writes", "leaves", "nodes", "CHECKSUM"):
        assert gpu[k] == cpu[k], (k, gpu[k], cpu[k])
    assert gpu["executor"] == "gpu" and gpu["OCA"] == "-"
