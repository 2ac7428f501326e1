"""SLT-vs-COT sweep driver (reference core/src/sweep.cpp:35-141).
CPU: CSV / pooled summary / ncu parsing.  GPU: every cell of a {scheme x tile}
grid is timed AND reproduces the reference golden checksum."""
import pytest

from paper_1802_00166_b200 import sweep as SW
from tests import oracle_ctypes as O


def _cells():
    return [
        {"scheme": "slt", "tile": [4, 64, 256], "samples": 2, "ms_mean": 1.0, "ms_stddev": 0.0,
         "ms_cov": 0.0, "ms": [1.0, 1.0], "launches": 10, "dram_bytes": 1e9, "l2_hit_pct": 50.0,
         "checksum": "00000000000000aa", "parity": "ok"},
        {"scheme": "cot", "tile": [4, 64, 256], "samples": 2, "ms_mean": 3.0, "ms_stddev": 1.0,
         "ms_cov": 1 / 3, "ms": [2.0, 4.0], "launches": 10, "dram_bytes": None, "l2_hit_pct": None,
         "checksum": "00000000000000aa", "parity": "ok"},
    ]


def test_sweep_csv_schema_and_pooled_summary():
    text = SW.sweep_csv(_cells())
    lines = text.strip().splitlines()
    assert lines[0] == SW.CSV_HEADER
    assert lines[1].split(",")[:3] == ["slt", "4x64x256", "2"]
    assert lines[1].endswith("00000000000000aa,ok")
    assert lines[2].split(",")[7:9] == ["", ""]  # no ncu numbers -> empty fields
    summ = SW.summary_lines(_cells())
    assert summ[0] == "summary scheme=slt cells=1 mean=1.0000 stddev=0.0000 cov=0.000000"
    assert summ[1].startswith("summary scheme=cot cells=1 mean=3.0000 stddev=1.0000")


def test_parse_ncu_csv_weights_l2_hit_by_sectors():
    hdr = '"ID","Process ID","Process Name","Host Name","Kernel Name","Context","Stream","Block Size","Grid Size","Device","CC","Section Name","Metric Name","Metric Unit","Metric Value"'
    def row(i, name, unit, v):
        return '"%d","1","p","h","k","1","7","(1,1,1)","(1,1,1)","0","10.0","Command line profiler metrics","%s","%s","%s"' % (i, name, unit, v)
    text = "\n".join([hdr,
                      row(0, "dram__bytes_read.sum", "Mbyte", "2"), row(0, "dram__bytes_write.sum", "Kbyte", "500"),
                      row(0, "lts__t_sector_hit_rate.pct", "%", "80"), row(0, "lts__t_sectors.sum", "sector", "100"),
                      row(1, "dram__bytes_read.sum", "byte", "1000"), row(1, "lts__t_sector_hit_rate.pct", "%", "20"),
                      row(1, "lts__t_sectors.sum", "sector", "300")])
    dram, hit = SW.parse_ncu_csv(text)
    assert dram == pytest.approx(2e6 + 5e5 + 1000)
    assert hit == pytest.approx((80 * 100 + 20 * 300) / 400)


@pytest.mark.gpu
def test_sweep_every_cell_reproduces_the_golden():
    want = [e["checksum"] for e in O.goldens()
            if e["kernel"] == "jacobi2d" and e["params"] == {"T": 40, "N": 1000}][0]
    cells = SW.run_sweep("jacobi2d", {"T": 40, "N": 1000}, [[2, 64, 256], [5, 32, 128], [8, 64, 512]],
                         ("untiled", "slt", "cot"), samples=2, want=want)
    assert len(cells) == 1 + 3 + 3
    assert all(c["parity"] == "ok" for c in cells), [(c["scheme"], c["tile"], c["checksum"]) for c in cells]
    assert {c["bt"] for c in cells if c["scheme"] != "untiled"} == {2, 5, 8}


@pytest.mark.gpu
def test_sweep_cli_fails_on_a_wrong_expected_checksum(capsys):
    rc = SW.main(["gs2d", "-p", "T=4,N=40", "--tiles", "2x8x16", "--schemes", "slt,cot",
                  "--samples", "1", "--want", "0000000000000000", "--quiet"])
    assert rc == 1
