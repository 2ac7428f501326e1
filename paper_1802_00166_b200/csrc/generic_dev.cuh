// Device runtime of the generic executor (generic.h), shared by the
// interpreter (generic.cu, nvcc) and the kernels the PRDG -> CUDA emitter
// compiles at run time (generic_jit.cpp, NVRTC): the plan tables, storage
// addressing under memory maps, and the read / write protocols of the three
// schedules.  Self-contained (no includes): the NVRTC prelude defines PCOT_DEV
// and the fixed-width integer types.
#pragma once

constexpr int kMaxIdx = 6, kMaxRank = 6, kMaxStack = 32;
constexpr long long kSpinCapG = 200000000LL;

struct GAff {
  int64_t c[kMaxIdx];
  int64_t k;
};
// One array reference: storage dims (map composed with the subscripts, params
// folded) with their modulus / extent / stride, and the logical cell id
// (row-major over the declared extents, the reference's logical_flat).
struct GRef {
  int array, rank, aff0, laff;
  int64_t ext[kMaxRank], stride[kMaxRank], mod[kMaxRank];
};
enum GOpKind { OLit, OAff, ORead, OAdd, OSub, OMul, ODiv, OMin, OMax, ONeg, OSqrt };
struct GOp {
  int kind, arg;
  double lit;
};
struct GStmt {
  int row0, nrows, op0, nops, wref, nreads;
};
struct GDev {
  int nidx, nstmt;
  int64_t lo[kMaxIdx], ext[kMaxIdx], npoints;
  const GStmt* st;
  const GAff* rows;
  const GAff* affs;
  const GRef* refs;
  const GOp* ops;
  double* const* arr;
  const int64_t* fbase;  // first flag of each array (logical cells)
  unsigned* flags;       // dense dataflow: 1 = cell holds its final value; count pass: writes
  unsigned long long* writer;  // count pass: min over writes of (point * nstmt + statement)
  unsigned* bad;               // order pass: 1 if a read precedes (or is) its cell's write
  const int64_t* sbase;  // first shadow of each array (storage cells)
  long long* shadow;     // mapped dataflow: logical id held by each storage cell
  const int64_t* lsize;  // logical cells per array
  int never_ok;          // dense storage: reads of never-written cells see their initial value
  const int* is_input;   // per array
  unsigned long long* next;
  unsigned long long* cnt;  // points, reads, writes
  int* err;                 // 0 ok; s+1: out-of-extent in statement s; -1: wait cap
};

PCOT_DEV int64_t aff_eval(const GAff& a, const int64_t* z, int n) {
  int64_t v = a.k;
  for (int i = 0; i < n; ++i) v += a.c[i] * z[i];
  return v;
}

PCOT_DEV bool in_domain(const GDev& g, const GStmt& s, const int64_t* z) {
  for (int r = 0; r < s.nrows; ++r)
    if (aff_eval(g.rows[s.row0 + r], z, g.nidx) < 0) return false;
  return true;
}

// Storage cell (reference phys_flat, exec.cpp:310-325): modulo dims wrap,
// the others must lie inside the map's extents.
PCOT_DEV bool cell_of(const GDev& g, const GRef& r, const int64_t* z, int64_t* flat) {
  int64_t f = 0;
  for (int d = 0; d < r.rank; ++d) {
    int64_t comp = aff_eval(g.affs[r.aff0 + d], z, g.nidx);
    if (r.mod[d] > 0) {
      comp %= r.mod[d];
      if (comp < 0) comp += r.mod[d];
    } else if (comp < 0 || comp >= r.ext[d]) {
      return false;
    }
    f += comp * r.stride[d];
  }
  *flat = f;
  return true;
}

// Logical cell id (reference logical_flat, exec.cpp:327-331); -1 if outside
// the declared extents (the run then cannot be checked cell by cell).
PCOT_DEV int64_t logical_of(const GDev& g, const GRef& r, const int64_t* z) {
  const int64_t l = aff_eval(g.affs[r.laff], z, g.nidx);
  return l >= 0 && l < g.lsize[r.array] ? l : -1;
}

PCOT_DEV void decode(const GDev& g, unsigned long long p, int64_t* z) {
  for (int i = g.nidx - 1; i >= 0; --i) {
    const unsigned long long e = (unsigned long long)g.ext[i];
    z[i] = g.lo[i] + int64_t(p % e);
    p /= e;
  }
}

PCOT_DEV unsigned ld_acq_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PCOT_DEV void st_rel_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

PCOT_DEV long long ld_acq_s64(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
PCOT_DEV void st_rel_s64(long long* p, long long v) {
  asm volatile("st.release.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
PCOT_DEV void st_rlx_s64(long long* p, long long v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
PCOT_DEV double ld_acq_f64(const double* p) {
  double v;
  asm volatile("ld.acquire.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
PCOT_DEV void st_rel_f64(double* p, double v) {
  asm volatile("st.release.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// Plain L2 (cg) load / store without the intrinsic headers (NVRTC).
PCOT_DEV double ld_cg_f64(const double* p) {
  double v;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
PCOT_DEV void st_cg_f64(double* p, double v) { asm volatile("st.global.cg.f64 [%0], %1;" ::"l"(p), "d"(v)); }

// One read of statement `si` at point z through reference `ri`, under the
// schedule's protocol (0 sequential; 1 dense storage, per-cell ready flags;
// 2 mapped storage, per-storage-cell shadows holding the logical id of the
// value they hold — the reference's shadow array, exec.cpp:360-368, used as
// the wait).  On an error it records it and clears `ok`.
template <int MODE>
PCOT_DEV double gread(const GDev& g, int ri, const int64_t* z, int si, bool& ok) {
  const GRef& r = g.refs[ri];
  int64_t f = 0;
  if (!cell_of(g, r, z, &f)) {
    atomicCAS(g.err, 0, si + 1);
    ok = false;
    return 0.0;
  }
  if (MODE == 1) {
    const unsigned* fl = g.flags + g.fbase[r.array] + f;
    long long it = 0;
    while (ld_acq_u32(fl) == 0) {
      if (++it > kSpinCapG) {
        atomicCAS(g.err, 0, -1);
        ok = false;
        return 0.0;
      }
      // a failed point never publishes its cell: stop waiting on error
      if ((it & 255) == 0 && *reinterpret_cast<volatile int*>(g.err) != 0) {
        ok = false;
        return 0.0;
      }
      __nanosleep(64);
    }
  }
  if (MODE == 2) {
    // wait until the storage cell holds this logical cell's value ...
    const long long want = logical_of(g, r, z);
    const long long* sh = g.shadow + g.sbase[r.array] + f;
    const unsigned long long* wk = g.writer + g.fbase[r.array];
    long long it = 0;
    for (long long held; (held = ld_acq_s64(sh)) != want;) {
      // the cell holds a LATER occupant (its write comes after ours in the
      // reference's order): our value was overwritten before this read — the
      // fold is not universal for this kernel
      if (held >= 0 && wk[held] > wk[want]) {
        atomicCAS(g.err, 0, -2);
        ok = false;
        return 0.0;
      }
      if (++it > kSpinCapG) {
        atomicCAS(g.err, 0, -1);
        ok = false;
        return 0.0;
      }
      if ((it & 255) == 0 && *reinterpret_cast<volatile int*>(g.err) != 0) {
        ok = false;
        return 0.0;
      }
      __nanosleep(64);
    }
    // (seqlock: a writer invalidates the shadow before its data store, so a
    // load that saw new data also sees the changed shadow)
    const double v = ld_acq_f64(g.arr[r.array] + f);
    // ... and still does after the load: a map that is not a universal
    // occupancy vector could let a later write reuse the cell early
    if (ld_acq_s64(sh) != want) {
      atomicCAS(g.err, 0, -2);
      ok = false;
    }
    return v;
  }
  return ld_cg_f64(g.arr[r.array] + f);
}

// The write of statement `si` at point z through reference `ri`.
template <int MODE>
PCOT_DEV bool gwrite(const GDev& g, int ri, const int64_t* z, int si, double v) {
  const GRef& w = g.refs[ri];
  int64_t f = 0;
  if (!cell_of(g, w, z, &f)) {
    atomicCAS(g.err, 0, si + 1);
    return false;
  }
  if (MODE == 2) {  // invalidate, data, publish (see the reader's seqlock)
    long long* sh = g.shadow + g.sbase[w.array] + f;
    st_rlx_s64(sh, -2);
    st_rel_f64(g.arr[w.array] + f, v);
    st_rel_s64(sh, logical_of(g, w, z));
  } else {
    st_cg_f64(g.arr[w.array] + f, v);
  }
  if (MODE == 1) st_rel_u32(g.flags + g.fbase[w.array] + f, 1u);
  return true;
}

// Persistent dataflow grid: warps take 32 consecutive points in the
// reference's order; reads wait for their cell's flag (dense) or shadow
// (mapped).  PE::run<MODE>(g, z, c3) executes the statements of one point.
template <int MODE, class PE>
PCOT_DEV void dataflow_loop(const GDev& g) {
  const int lane = threadIdx.x & 31;
  unsigned long long c3[3] = {0, 0, 0};
  int64_t z[kMaxIdx];
  bool ok = true;
  for (;;) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(g.next, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (base >= (unsigned long long)g.npoints) break;
    const unsigned long long p = base + lane;
    if (ok && p < (unsigned long long)g.npoints) {
      decode(g, p, z);
      ok = PE::template run<MODE>(g, z, c3);
    }
  }
  atomicAdd(&g.cnt[0], c3[0]);
  atomicAdd(&g.cnt[1], c3[1]);
  atomicAdd(&g.cnt[2], c3[2]);
}

// One thread, the reference's exact order (odometer: no 64-bit divisions).
template <class PE>
PCOT_DEV void sequential_loop(const GDev& g) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long c3[3] = {0, 0, 0};
  int64_t z[kMaxIdx];
  if (g.npoints > 0) decode(g, 0, z);
  for (unsigned long long p = 0; p < (unsigned long long)g.npoints; ++p) {
    if (!PE::template run<0>(g, z, c3)) break;
    for (int i = g.nidx - 1; i >= 0; --i) {
      if (++z[i] < g.lo[i] + g.ext[i]) break;
      z[i] = g.lo[i];
    }
  }
  g.cnt[0] = c3[0];
  g.cnt[1] = c3[1];
  g.cnt[2] = c3[2];
}
