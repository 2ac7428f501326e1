#!/usr/bin/env python3
"""Generate the four kernel specs the BASELINE configs need, in the reference's
kernel-spec JSON format (reference proj/docs/formats.md:7-85).

The reference corpus has no zero-ring Jacobi-2D, no BASELINE-rule Heat-3D, no
Gauss-Seidel and no GEMM (reference SPEC.md:161), so they are
written here as data and loaded through the reference's own parser
(`parse_kernel`, kernel_io.cpp:118-197).  Domain rows use the reference row
encoding: row . (indices ++ params ++ [1]) >= 0.

    python kernels/gen_kernels.py        # rewrites kernels/*.kernel
"""
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))


class Space:
    """Index/param naming for one kernel; builds domain rows from dicts."""

    def __init__(self, indices, params):
        self.indices = list(indices)
        self.params = list(params)
        self.cols = self.indices + self.params + ["1"]

    def row(self, coeffs):
        for k in coeffs:
            if k not in self.cols:
                raise KeyError(k)
        return [int(coeffs.get(c, 0)) for c in self.cols]

    # helpers: every affine form is a dict {name: coeff, "1": const}
    def ge(self, a, b=None):
        """a >= b  (b defaults to 0)."""
        d = dict(a)
        for k, v in (b or {}).items():
            d[k] = d.get(k, 0) - v
        return self.row(d)

    def between(self, form, lo, hi):
        """lo <= form <= hi, lo/hi are affine dicts."""
        return [self.ge(form, lo), self.ge(hi, form)]

    def eq(self, form, val):
        return self.between(form, val, val)


def C(v):
    return {"1": v}


def lin(*terms, const=0):
    d = {"1": const}
    for coef, name in terms:
        d[name] = d.get(name, 0) + coef
    return d


def stmt(sid, depth, rows, arr, subs, body):
    return {"id": sid, "depth": depth, "domain": rows,
            "writes": {"array": arr, "subscripts": subs}, "body": body}


def spec(name, params, indices, check, arrays, statements):
    return {"name": name, "params": params, "indices": indices,
            "check_params": check, "arrays": arrays, "statements": statements,
            "edges": [], "tilable_band": list(range(len(indices)))}


# ---------------------------------------------------------------- jacobi2d
def jacobi2d():
    """Jacobi-2D 5-point, zero Dirichlet ring at every t (BASELINE cfg 0/4).

    Same time-skew as the corpus heat2d (x = i + t, y = j + t) and exactly the
    corpus update body (reference kernels/heat2d.kernel:32), but the ring is
    the literal 0.0 at all 0 <= t <= T instead of being copied from F.
    """
    s = Space(["t", "x", "y"], ["T", "N"])
    i = lin((1, "x"), (-1, "t"))          # un-skewed row
    j = lin((1, "y"), (-1, "t"))          # un-skewed column
    N1, N2 = lin((1, "N"), const=-1), lin((1, "N"), const=-2)
    t_all = s.between(lin((1, "t")), C(0), lin((1, "T")))
    t_up = s.between(lin((1, "t")), C(1), lin((1, "T")))
    t0 = s.eq(lin((1, "t")), C(0))
    i_in, j_in = s.between(i, C(1), N2), s.between(j, C(1), N2)
    i_all, j_all = s.between(i, C(0), N1), s.between(j, C(0), N1)
    W = "X[t, x, y]"
    sts = [
        stmt("S0", 3, t0 + i_in + j_in, "X", ["t", "x", "y"], "F[x, y]"),
        stmt("R0", 3, t_all + s.eq(i, C(0)) + j_all, "X", ["t", "x", "y"], "0.0"),
        stmt("R1", 3, t_all + s.eq(i, N1) + j_all, "X", ["t", "x", "y"], "0.0"),
        stmt("R2", 3, t_all + i_in + s.eq(j, C(0)), "X", ["t", "x", "y"], "0.0"),
        stmt("R3", 3, t_all + i_in + s.eq(j, N1), "X", ["t", "x", "y"], "0.0"),
        stmt("S1", 3, t_up + i_in + j_in, "X", ["t", "x", "y"],
             "0.2 * (X[t - 1, x - 1, y - 1] + X[t - 1, x - 2, y - 1] + "
             "X[t - 1, x, y - 1] + X[t - 1, x - 1, y - 2] + X[t - 1, x - 1, y])"),
        stmt("Sfin", 3, s.eq(lin((1, "t")), lin((1, "T"))) + i_all + j_all, "Out",
             ["x - T", "y - T"], W),
    ]
    arrays = [
        {"name": "F", "rank": 2, "extents": ["N", "N"], "kind": "input"},
        {"name": "X", "rank": 3, "extents": ["T + 1", "N + T", "N + T"], "kind": "temp"},
        {"name": "Out", "rank": 2, "extents": ["N", "N"], "kind": "output"},
    ]
    return spec("jacobi2d", ["T", "N"], ["t", "x", "y"], {"T": 3, "N": 6}, arrays, sts)


def heat2d_hold():
    """Same semantics as the reference corpus heat2d (kernels/heat2d.kernel):
    t=0 copies all of F, the ring is copied forward from step t-1 (so it keeps
    F's values), interior gets the 5-point body.  Written independently here
    so the GPU test-suite does not need the reference tree; make_golden.py
    checks that the reference interpreter gives both specs the same checksum.
    """
    s = Space(["t", "x", "y"], ["T", "N"])
    i = lin((1, "x"), (-1, "t"))
    j = lin((1, "y"), (-1, "t"))
    N1, N2 = lin((1, "N"), const=-1), lin((1, "N"), const=-2)
    t_up = s.between(lin((1, "t")), C(1), lin((1, "T")))
    t0 = s.eq(lin((1, "t")), C(0))
    i_in, j_in = s.between(i, C(1), N2), s.between(j, C(1), N2)
    i_all, j_all = s.between(i, C(0), N1), s.between(j, C(0), N1)
    subs = ["t", "x", "y"]
    cp = "X[t - 1, x - 1, y - 1]"
    sts = [
        stmt("S0", 3, t0 + i_all + j_all, "X", subs, "F[x, y]"),
        stmt("S1", 3, t_up + i_in + j_in, "X", subs,
             "0.2 * (X[t - 1, x - 1, y - 1] + X[t - 1, x - 2, y - 1] + "
             "X[t - 1, x, y - 1] + X[t - 1, x - 1, y - 2] + X[t - 1, x - 1, y])"),
        stmt("C0", 3, t_up + s.eq(i, C(0)) + j_all, "X", subs, cp),
        stmt("C1", 3, t_up + s.eq(i, N1) + j_all, "X", subs, cp),
        stmt("C2", 3, t_up + i_in + s.eq(j, C(0)), "X", subs, cp),
        stmt("C3", 3, t_up + i_in + s.eq(j, N1), "X", subs, cp),
        stmt("Sfin", 3, s.eq(lin((1, "t")), lin((1, "T"))) + i_all + j_all, "Out",
             ["x - T", "y - T"], "X[t, x, y]"),
    ]
    arrays = [
        {"name": "F", "rank": 2, "extents": ["N", "N"], "kind": "input"},
        {"name": "X", "rank": 3, "extents": ["T + 1", "N + T", "N + T"], "kind": "temp"},
        {"name": "Out", "rank": 2, "extents": ["N", "N"], "kind": "output"},
    ]
    return spec("heat2d_hold", ["T", "N"], ["t", "x", "y"], {"T": 3, "N": 6}, arrays, sts)


def heat3d_hold():
    """Same semantics as the reference corpus heat3d (kernels/heat3d.kernel:34):
    0.1 * (c + 6 neighbours), ring copied forward from step t-1."""
    s = Space(["t", "x", "y", "w"], ["T", "N"])
    i = lin((1, "x"), (-1, "t"))
    j = lin((1, "y"), (-1, "t"))
    k = lin((1, "w"), (-1, "t"))
    N1, N2 = lin((1, "N"), const=-1), lin((1, "N"), const=-2)
    t_up = s.between(lin((1, "t")), C(1), lin((1, "T")))
    t0 = s.eq(lin((1, "t")), C(0))
    inn = [s.between(v, C(1), N2) for v in (i, j, k)]
    alll = [s.between(v, C(0), N1) for v in (i, j, k)]
    subs = ["t", "x", "y", "w"]
    c = "X[t - 1, x - 1, y - 1, w - 1]"
    body = ("0.1 * (" + c + " + X[t - 1, x - 2, y - 1, w - 1] + X[t - 1, x, y - 1, w - 1] + "
            "X[t - 1, x - 1, y - 2, w - 1] + X[t - 1, x - 1, y, w - 1] + "
            "X[t - 1, x - 1, y - 1, w - 2] + X[t - 1, x - 1, y - 1, w])")
    sts = [stmt("S0", 4, t0 + alll[0] + alll[1] + alll[2], "X", subs, "F[x, y, w]"),
           stmt("S1", 4, t_up + inn[0] + inn[1] + inn[2], "X", subs, body)]
    n = 0
    for v, rest in ((i, alll[1] + alll[2]), (j, inn[0] + alll[2]), (k, inn[0] + inn[1])):
        for val in (C(0), N1):
            sts.append(stmt("C%d" % n, 4, t_up + s.eq(v, val) + rest, "X", subs, c))
            n += 1
    sts.append(stmt("Sfin", 4, s.eq(lin((1, "t")), lin((1, "T"))) + alll[0] + alll[1] + alll[2],
                    "Out", ["x - T", "y - T", "w - T"], "X[t, x, y, w]"))
    arrays = [
        {"name": "F", "rank": 3, "extents": ["N", "N", "N"], "kind": "input"},
        {"name": "X", "rank": 4, "extents": ["T + 1", "N + T", "N + T", "N + T"],
         "kind": "temp"},
        {"name": "Out", "rank": 3, "extents": ["N", "N", "N"], "kind": "output"},
    ]
    return spec("heat3d_hold", ["T", "N"], ["t", "x", "y", "w"], {"T": 2, "N": 5}, arrays, sts)


# ---------------------------------------------------------------- heat3d_b
def heat3d_b():
    """Heat-3D 7-point with the BASELINE rule c + 0.125*(sum6 - 6c), zero ring.

    Skew x,y,w = i,j,k + t as in the corpus heat3d (reference
    kernels/heat3d.kernel), body operand order fixed per SURVEY.md §B.
    """
    s = Space(["t", "x", "y", "w"], ["T", "N"])
    i = lin((1, "x"), (-1, "t"))
    j = lin((1, "y"), (-1, "t"))
    k = lin((1, "w"), (-1, "t"))
    N1, N2 = lin((1, "N"), const=-1), lin((1, "N"), const=-2)
    t_all = s.between(lin((1, "t")), C(0), lin((1, "T")))
    t_up = s.between(lin((1, "t")), C(1), lin((1, "T")))
    t0 = s.eq(lin((1, "t")), C(0))
    inn = [s.between(v, C(1), N2) for v in (i, j, k)]
    alll = [s.between(v, C(0), N1) for v in (i, j, k)]
    subs = ["t", "x", "y", "w"]
    c = "X[t - 1, x - 1, y - 1, w - 1]"
    body = (c + " + 0.125 * (X[t - 1, x - 2, y - 1, w - 1] + X[t - 1, x, y - 1, w - 1] + "
            "X[t - 1, x - 1, y - 2, w - 1] + X[t - 1, x - 1, y, w - 1] + "
            "X[t - 1, x - 1, y - 1, w - 2] + X[t - 1, x - 1, y - 1, w] - 6.0 * " + c + ")")
    sts = [stmt("S0", 4, t0 + inn[0] + inn[1] + inn[2], "X", subs, "F[x, y, w]")]
    # ring: faces i in {0,N-1}; j in {0,N-1} (interior i); k in {0,N-1} (interior i,j)
    n = 0
    for v, rest in ((i, alll[1] + alll[2]), (j, inn[0] + alll[2]), (k, inn[0] + inn[1])):
        for val in (C(0), N1):
            sts.append(stmt("R%d" % n, 4, t_all + s.eq(v, val) + rest, "X", subs, "0.0"))
            n += 1
    sts.append(stmt("S1", 4, t_up + inn[0] + inn[1] + inn[2], "X", subs, body))
    sts.append(stmt("Sfin", 4, s.eq(lin((1, "t")), lin((1, "T"))) + alll[0] + alll[1] + alll[2],
                    "Out", ["x - T", "y - T", "w - T"], "X[t, x, y, w]"))
    arrays = [
        {"name": "F", "rank": 3, "extents": ["N", "N", "N"], "kind": "input"},
        {"name": "X", "rank": 4, "extents": ["T + 1", "N + T", "N + T", "N + T"],
         "kind": "temp"},
        {"name": "Out", "rank": 3, "extents": ["N", "N", "N"], "kind": "output"},
    ]
    return spec("heat3d_b", ["T", "N"], ["t", "x", "y", "w"], {"T": 2, "N": 5}, arrays, sts)


# ---------------------------------------------------------------- gs2d
def gs2d():
    """In-place Gauss-Seidel 9-point (BASELINE cfg 2), lexicographic order.

    Skew x = t + i, y = 2t + i + j makes every dependence non-negative
    (SURVEY.md §B): new values for the 4 lexicographic predecessors, old values
    for the rest, summed in row-major 3x3 order, then IEEE-divided by 9.0.
    """
    s = Space(["t", "x", "y"], ["T", "N"])
    i = lin((1, "x"), (-1, "t"))
    j = lin((1, "y"), (-1, "x"), (-1, "t"))
    N1, N2 = lin((1, "N"), const=-1), lin((1, "N"), const=-2)
    t_all = s.between(lin((1, "t")), C(0), lin((1, "T")))
    t_up = s.between(lin((1, "t")), C(1), lin((1, "T")))
    t0 = s.eq(lin((1, "t")), C(0))
    i_in, j_in = s.between(i, C(1), N2), s.between(j, C(1), N2)
    i_all, j_all = s.between(i, C(0), N1), s.between(j, C(0), N1)
    subs = ["t", "x", "y"]
    body = ("(X[t, x - 1, y - 2] + X[t, x - 1, y - 1] + X[t, x - 1, y] + X[t, x, y - 1] + "
            "X[t - 1, x - 1, y - 2] + X[t - 1, x - 1, y - 1] + X[t - 1, x, y - 2] + "
            "X[t - 1, x, y - 1] + X[t - 1, x, y]) / 9.0")
    sts = [
        stmt("S0", 3, t0 + i_in + j_in, "X", subs, "F[x - t, y - x - t]"),
        stmt("R0", 3, t_all + s.eq(i, C(0)) + j_all, "X", subs, "0.0"),
        stmt("R1", 3, t_all + s.eq(i, N1) + j_all, "X", subs, "0.0"),
        stmt("R2", 3, t_all + i_in + s.eq(j, C(0)), "X", subs, "0.0"),
        stmt("R3", 3, t_all + i_in + s.eq(j, N1), "X", subs, "0.0"),
        stmt("S1", 3, t_up + i_in + j_in, "X", subs, body),
        stmt("Sfin", 3, s.eq(lin((1, "t")), lin((1, "T"))) + i_all + j_all, "Out",
             ["x - t", "y - x - t"], "X[t, x, y]"),
    ]
    arrays = [
        {"name": "F", "rank": 2, "extents": ["N", "N"], "kind": "input"},
        {"name": "X", "rank": 3, "extents": ["T + 1", "N + T", "2 * N + 2 * T"],
         "kind": "temp"},
        {"name": "Out", "rank": 2, "extents": ["N", "N"], "kind": "output"},
    ]
    return spec("gs2d", ["T", "N"], ["t", "x", "y"], {"T": 3, "N": 6}, arrays, sts)


# ---------------------------------------------------------------- gemm
def gemm():
    """C += A*B, fp64, sequential-k reduction; A, B mapped to [-1,1) by 2u-1.

    The [-1,1) inputs are written as (2.0*A - 1.0) of the [0,1) init values
    (reference exec.cpp:21-28), which is exact in fp64.
    """
    s = Space(["i", "j", "k"], ["N"])
    N1 = lin((1, "N"), const=-1)
    ij = s.between(lin((1, "i")), C(0), N1) + s.between(lin((1, "j")), C(0), N1)
    sts = [
        stmt("S0", 3, ij + s.eq(lin((1, "k")), C(0)), "C", ["i", "j", "k"], "0.0"),
        stmt("S1", 3, ij + s.between(lin((1, "k")), C(1), lin((1, "N"))), "C",
             ["i", "j", "k"],
             "C[i, j, k - 1] + (2.0 * A[i, k - 1] - 1.0) * (2.0 * B[k - 1, j] - 1.0)"),
        stmt("Sfin", 3, ij + s.eq(lin((1, "k")), lin((1, "N"))), "Out", ["i", "j"],
             "C[i, j, k]"),
    ]
    arrays = [
        {"name": "A", "rank": 2, "extents": ["N", "N"], "kind": "input"},
        {"name": "B", "rank": 2, "extents": ["N", "N"], "kind": "input"},
        {"name": "C", "rank": 3, "extents": ["N", "N", "N + 1"], "kind": "temp"},
        {"name": "Out", "rank": 2, "extents": ["N", "N"], "kind": "output"},
    ]
    return spec("gemm", ["N"], ["i", "j", "k"], {"N": 3}, arrays, sts)


# ------------------------------------------------------- corpus restatements
# The reference corpus kernels outside the hot-path registry, restated from
# their documented semantics so the device interpreter (csrc/generic.cu) can
# be tested without /root/reference (tests/golden/corpus.json pins each one to
# the reference interpreter's checksum on the corpus file itself).

def triangle():
    """Prefix-style triangle recurrence: C[i, 0] = B[i]; C[i, j] = C[i-1, j-1]
    + C[i, j-1] for 1 <= j <= i < N; Out[i] = C[i, i]."""
    s = Space(["i", "j"], ["N"])
    N1 = lin((1, "N"), const=-1)
    i_all = s.between(lin((1, "i")), C(0), N1)
    sts = [
        stmt("S0", 2, i_all + s.eq(lin((1, "j")), C(0)), "C", ["i", "j"], "B[i]"),
        stmt("S1", 2, [s.ge(lin((1, "j")), C(1)), s.ge(lin((1, "i")), lin((1, "j"))),
                       s.ge(N1, lin((1, "i")))], "C", ["i", "j"], "C[i - 1, j - 1] + C[i, j - 1]"),
        stmt("Sfin", 2, s.eq(lin((1, "i"), (-1, "j")), C(0)) + i_all, "Out", ["i"], "C[i, j]"),
    ]
    arrays = [
        {"name": "B", "rank": 1, "extents": ["N"], "kind": "input"},
        {"name": "C", "rank": 2, "extents": ["N", "N"], "kind": "temp"},
        {"name": "Out", "rank": 1, "extents": ["N"], "kind": "output"},
    ]
    return spec("triangle", ["N"], ["i", "j"], {"N": 8}, arrays, sts)


def heat1d_fig7():
    """1-D heat with a coupling term to the left boundary cell (the paper's
    figure-7 example): X[0, i] = F[i]; interior X[t, i] = 0.25*(X[t-1, i-1] +
    X[t-1, i] + X[t-1, i+1] + X[t-1, 0]); both boundary cells copied forward
    (the left one by a depth-1 statement over t only); Out = X[T, .]."""
    s = Space(["t", "i"], ["T", "N"])
    N1, N2 = lin((1, "N"), const=-1), lin((1, "N"), const=-2)
    t_up = s.between(lin((1, "t")), C(1), lin((1, "T")))
    s1 = Space(["t"], ["T", "N"])  # the depth-1 statement's own space
    sts = [
        stmt("S0", 2, s.eq(lin((1, "t")), C(0)) + s.between(lin((1, "i")), C(0), N1), "X",
             ["t", "i"], "F[i]"),
        stmt("S1", 2, t_up + s.between(lin((1, "i")), C(1), N2), "X", ["t", "i"],
             "0.25 * (X[t - 1, i - 1] + X[t - 1, i] + X[t - 1, i + 1] + X[t - 1, 0])"),
        stmt("S2", 1, s1.between(lin((1, "t")), C(1), lin((1, "T"))), "X", ["t", "0"],
             "X[t - 1, 0]"),
        stmt("S3", 2, t_up + s.eq(lin((1, "i")), N1), "X", ["t", "i"], "X[t - 1, i]"),
        stmt("Sfin", 2, s.eq(lin((1, "t")), lin((1, "T"))) + s.between(lin((1, "i")), C(0), N1),
             "Out", ["i"], "X[t, i]"),
    ]
    arrays = [
        {"name": "F", "rank": 1, "extents": ["N"], "kind": "input"},
        {"name": "X", "rank": 2, "extents": ["T + 1", "N"], "kind": "temp"},
        {"name": "Out", "rank": 1, "extents": ["N"], "kind": "output"},
    ]
    k = spec("heat1d-fig7", ["T", "N"], ["t", "i"], {"T": 8, "N": 8}, arrays, sts)
    k["tilable_band"] = [0]
    return k


def lud():
    """LU decomposition without pivoting, single-assignment over k: level 0
    copies M (diagonal + N), level k eliminates the trailing block, Out takes
    U from level i (j >= i) and L from level j (i > j)."""
    s = Space(["k", "i", "j"], ["N"])
    N1 = lin((1, "N"), const=-1)
    k0 = s.eq(lin((1, "k")), C(0))
    upd = "A[k - 1, i, j] - A[k - 1, i, k - 1] * A[k - 1, k - 1, j] / A[k - 1, k - 1, k - 1]"
    sts = [
        stmt("S0d", 3, k0 + s.eq(lin((1, "i"), (-1, "j")), C(0)) + s.between(lin((1, "i")), C(0), N1),
             "A", ["k", "i", "j"], "M[i, j] + N"),
        stmt("S0l", 3, k0 + [s.ge(lin((1, "j"))), s.ge(lin((1, "i"), (-1, "j")), C(1)),
                             s.ge(N1, lin((1, "i")))], "A", ["k", "i", "j"], "M[i, j]"),
        stmt("S0u", 3, k0 + [s.ge(lin((1, "i"))), s.ge(lin((1, "j"), (-1, "i")), C(1)),
                             s.ge(N1, lin((1, "j")))], "A", ["k", "i", "j"], "M[i, j]"),
        stmt("S", 3, s.between(lin((1, "k")), C(1), N1) + s.between(lin((1, "i")), lin((1, "k")), N1)
             + s.between(lin((1, "j")), lin((1, "k")), N1), "A", ["k", "i", "j"], upd),
        stmt("SfU", 3, s.eq(lin((1, "k"), (-1, "i")), C(0)) + s.between(lin((1, "j")), lin((1, "i")), N1)
             + [s.ge(lin((1, "i")))], "Out", ["i", "j"], "A[k, i, j]"),
        stmt("SfL", 3, s.eq(lin((1, "k"), (-1, "j")), C(0)) + [s.ge(lin((1, "i"), (-1, "j")), C(1)),
                                                              s.ge(N1, lin((1, "i"))), s.ge(lin((1, "j")))],
             "Out", ["i", "j"], "A[k, i, j]"),
    ]
    arrays = [
        {"name": "M", "rank": 2, "extents": ["N", "N"], "kind": "input"},
        {"name": "A", "rank": 3, "extents": ["N", "N", "N"], "kind": "temp"},
        {"name": "Out", "rank": 2, "extents": ["N", "N"], "kind": "output"},
    ]
    return spec("lud", ["N"], ["k", "i", "j"], {"N": 6}, arrays, sts)


def osp():
    """Optimal-split dynamic programme over interval length u and right end v:
    C[v-1, v] = W[v-1]*W[v] (u = 1); for u >= 2 the running minimum Acc over
    split points m, then C[v-u, v] = min + W[v-u]*W[v] (C is overwritten: the
    interpreter runs it in the reference's order); Out[0] = C[0, N-1]."""
    s = Space(["u", "v", "m"], ["N"])
    s2 = Space(["u", "v"], ["N"])
    N1 = lin((1, "N"), const=-1)
    uv = s.between(lin((1, "u")), C(2), N1) + s.between(lin((1, "v")), lin((1, "u")), N1)
    sts = [
        stmt("Sb", 2, s2.eq(lin((1, "u")), C(1)) + s2.between(lin((1, "v")), C(1), N1), "C",
             ["v - u", "v"], "W[v - u] * W[v]"),
        stmt("Sa0", 3, uv + s.eq(lin((1, "m"), (-1, "v"), (1, "u")), C(1)), "Acc", ["u", "v", "m"],
             "C[v - u, m] + C[m, v]"),
        stmt("Sa", 3, uv + [s.ge(lin((1, "m"), (-1, "v"), (1, "u")), C(2)),
                            s.ge(lin((1, "v"), (-1, "m")), C(1))], "Acc", ["u", "v", "m"],
             "min(Acc[u, v, m - 1], C[v - u, m] + C[m, v])"),
        stmt("Sc", 3, uv + s.eq(lin((1, "m"), (-1, "v")), C(-1)), "C", ["v - u", "v"],
             "Acc[u, v, m] + W[v - u] * W[v]"),
        stmt("Sfin", 3, s.eq(lin((1, "u")), N1) + s.eq(lin((1, "v")), N1)
             + s.eq(lin((1, "m"), (-1, "v")), C(-1)), "Out", ["0"], "C[v - u, v]"),
    ]
    arrays = [
        {"name": "W", "rank": 1, "extents": ["N"], "kind": "input"},
        {"name": "C", "rank": 2, "extents": ["N", "N"], "kind": "temp"},
        {"name": "Acc", "rank": 3, "extents": ["N", "N", "N"], "kind": "temp"},
        {"name": "Out", "rank": 1, "extents": ["1"], "kind": "output"},
    ]
    k = spec("osp", ["N"], ["u", "v", "m"], {"N": 8}, arrays, sts)
    k["tilable_band"] = [0, 1]
    return k


def dump(obj):
    """Compact rows, one statement field per line."""
    return json.dumps(obj, indent=1) + "\n"


def main():
    for fn in (jacobi2d, heat2d_hold, heat3d_hold, heat3d_b, gs2d, gemm, triangle, heat1d_fig7,
               lud, osp):
        k = fn()
        path = os.path.join(HERE, k["name"] + ".kernel")
        with open(path, "w") as f:
            f.write(dump(k))
        print("wrote", path)


if __name__ == "__main__":
    main()
