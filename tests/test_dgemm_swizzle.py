"""Host check of the DGEMM fragment addressing under the TMA 128-byte swizzle
(paper_1802_00166_b200/csrc/dgemm_tma.cu): the permuted DMMA row / column
mapping must (a) cover every tile element exactly once and (b) make every
64-bit fragment load bank-conflict free per half-warp (16 lanes x 8 B = the
128 B a shared-memory wavefront serves)."""
import itertools

A_BOX = 128 * 128  # bytes: 128 rows x 16 doubles
B_BOX = 32 * 128   # bytes: 32 rows x 16 doubles (BK = 32)


def swz(row, dbl):
    """Byte offset of double `dbl` (0..15) of box row `row` under SWIZZLE_128B."""
    chunk = (dbl >> 1) ^ (row & 7)
    return row * 128 + chunk * 16 + (dbl & 1) * 8


def a_addr(wm, i, ks, lane):
    g, q = lane >> 2, lane & 3
    pg = (g & 3) * 2 + (g >> 2)
    a_base = (wm * 32 + pg) * 128 + (q & 1) * 8
    off = (((ks & 3) * 2 + (q >> 1)) ^ pg) << 4
    return (ks >> 2) * A_BOX + i * 1024 + a_base + off, (wm * 32 + i * 8 + pg, ks * 4 + q)


def b_addr(wn, j, ks, lane):
    g, q = lane >> 2, lane & 3
    b_base = wn * 2 * B_BOX + q * 128 + (g & 1) * 8
    off = (((j & 1) * 2 + (g >> 2) + ((g >> 1) & 1) * 4) ^ ((ks & 1) * 4 + q)) << 4
    n = wn * 32 + (j >> 1) * 16 + (j & 1) * 4 + (g >> 2) * 2 + ((g >> 1) & 1) * 8 + (g & 1)
    return b_base + off + (j >> 1) * B_BOX + ks * 512, (ks * 4 + q, n)


def test_a_fragment_addresses_match_the_swizzled_box():
    seen = set()
    for wm, i, ks, lane in itertools.product(range(4), range(4), range(8), range(32)):
        addr, (m, k) = a_addr(wm, i, ks, lane)
        assert addr == (k >> 4) * A_BOX + swz(m, k & 15)
        seen.add((m, k))
    assert len(seen) == 128 * 32  # every A element of the stage is read by some lane


def test_b_fragment_addresses_match_the_swizzled_box():
    seen = set()
    for wn, j, ks, lane in itertools.product(range(4), range(4), range(8), range(32)):
        addr, (k, n) = b_addr(wn, j, ks, lane)
        assert addr == (n >> 4) * B_BOX + swz(k, n & 15)
        seen.add((k, n))
    assert len(seen) == 32 * 128


def test_fragment_loads_are_bank_conflict_free_per_half_warp():
    for f, ranges in ((a_addr, (range(4), range(4), range(8))), (b_addr, (range(4), range(4), range(8)))):
        for x, y, ks in itertools.product(*ranges):
            for half in (range(0, 16), range(16, 32)):
                banks = {(f(x, y, ks, lane)[0] % 128) // 8 for lane in half}
                assert len(banks) == 16


def test_c_columns_of_a_lane_are_adjacent():
    # DMMA columns 2q, 2q+1 (C fragment) map to adjacent tile columns: double2 stores
    for q in range(4):
        cols = []
        for e in (0, 1):
            c = 2 * q + e
            cols.append((c >> 2) * 2 + ((c >> 1) & 1) * 8 + (c & 1))
        assert cols[1] == cols[0] + 1 and cols[0] == (q >> 1) * 2 + (q & 1) * 8
