"""COT tile order (reference cot_order / split_orthants, tiler.cpp:98-117,
150-203) as launched on the GPU: the compact Morton rank (csrc/common.cuh
morton_compact) walks a W x H rectangle of CTAs in the recursive Z order with
no idle CTAs.  Host-only check (nvcc compiles the header for the CPU)."""
import os
import subprocess
import tempfile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_compact_morton_rank_is_a_monotone_bijection():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "m")
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-std=c++17", "-I",
                        os.path.join(REPO, "paper_1802_00166_b200", "csrc"),
                        os.path.join(REPO, "tests", "c", "morton_check.cu"), "-o", exe],
                       check=True, capture_output=True)
        out = subprocess.run([exe], capture_output=True, text=True)
        assert out.returncode == 0 and "MORTON_BAD 0" in out.stdout
