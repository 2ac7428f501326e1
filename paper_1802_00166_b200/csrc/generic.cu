// Generic device executor: see generic.h.  Follows the reference's
// Executor::exec_stmt / run_level semantics (core/src/exec.cpp:347-472): the
// union of the statement domains is walked in lexicographic index order, each
// point runs the statements that contain it in declaration order, and each
// body is the postfix program of the reference's flatten (exec.cpp:187-224).
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <numeric>

#include "common.cuh"
#include "generic.h"
#include "kernels.h"

namespace pcotgpu {

namespace {

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

// Run every statement of point z.  Returns false on an error (recorded).
// DATAFLOW: 0 sequential; 1 dense storage, per-cell ready flags; 2 mapped
// storage, per-storage-cell shadows holding the logical id of the value they
// hold (the reference's shadow array, exec.cpp:360-368, used as the wait).
template <int DATAFLOW>
PCOT_DEV bool exec_point(const GDev& g, const int64_t* z, unsigned long long* c3) {
  for (int si = 0; si < g.nstmt; ++si) {
    const GStmt s = g.st[si];
    if (!in_domain(g, s, z)) continue;
    double stk[kMaxStack];
    int sp = 0;
    for (int o = 0; o < s.nops; ++o) {
      const GOp op = g.ops[s.op0 + o];
      switch (op.kind) {
        case OLit: stk[sp++] = op.lit; break;
        case OAff: stk[sp++] = double(aff_eval(g.affs[op.arg], z, g.nidx)); break;
        case ORead: {
          const GRef& r = g.refs[op.arg];
          int64_t f = 0;
          if (!cell_of(g, r, z, &f)) {
            atomicCAS(g.err, 0, si + 1);
            return false;
          }
          if (DATAFLOW == 1) {
            const unsigned* fl = g.flags + g.fbase[r.array] + f;
            long long it = 0;
            while (ld_acq_u32(fl) == 0) {
              if (++it > kSpinCapG) {
                atomicCAS(g.err, 0, -1);
                return false;
              }
              // a failed point never publishes its cell: stop waiting on error
              if ((it & 255) == 0 && *reinterpret_cast<volatile int*>(g.err) != 0) return false;
              __nanosleep(64);
            }
          }
          if (DATAFLOW == 2) {
            // wait until the storage cell holds this logical cell's value ...
            const long long want = logical_of(g, r, z);
            const long long* sh = g.shadow + g.sbase[r.array] + f;
            const unsigned long long* wk = g.writer + g.fbase[r.array];
            long long it = 0;
            for (long long held; (held = ld_acq_s64(sh)) != want;) {
              // the cell holds a LATER occupant (its write comes after ours in
              // the reference's order): our value was overwritten before this
              // read — the fold is not universal for this kernel
              if (held >= 0 && wk[held] > wk[want]) {
                atomicCAS(g.err, 0, -2);
                return false;
              }
              if (++it > kSpinCapG) {
                atomicCAS(g.err, 0, -1);
                return false;
              }
              if ((it & 255) == 0 && *reinterpret_cast<volatile int*>(g.err) != 0) return false;
              __nanosleep(64);
            }
            // (seqlock: a writer invalidates the shadow before its data store,
            // so a load that saw new data also sees the changed shadow)
            const double v = ld_acq_f64(g.arr[r.array] + f);
            // ... and still does after the load: a map that is not a universal
            // occupancy vector could let a later write reuse the cell early
            if (ld_acq_s64(sh) != want) {
              atomicCAS(g.err, 0, -2);
              return false;
            }
            stk[sp++] = v;
            break;
          }
          stk[sp++] = __ldcg(g.arr[r.array] + f);
          break;
        }
        case OAdd: --sp, stk[sp - 1] = __dadd_rn(stk[sp - 1], stk[sp]); break;
        case OSub: --sp, stk[sp - 1] = __dsub_rn(stk[sp - 1], stk[sp]); break;
        case OMul: --sp, stk[sp - 1] = __dmul_rn(stk[sp - 1], stk[sp]); break;
        case ODiv: --sp, stk[sp - 1] = __ddiv_rn(stk[sp - 1], stk[sp]); break;
        case OMin: {  // reference exec.cpp: b < a ? b : a
          const double b = stk[--sp], a = stk[sp - 1];
          stk[sp - 1] = b < a ? b : a;
          break;
        }
        case OMax: {  // a < b ? b : a
          const double b = stk[--sp], a = stk[sp - 1];
          stk[sp - 1] = a < b ? b : a;
          break;
        }
        case ONeg: stk[sp - 1] = -stk[sp - 1]; break;
        case OSqrt: stk[sp - 1] = __dsqrt_rn(stk[sp - 1]); break;
      }
    }
    const GRef& w = g.refs[s.wref];
    int64_t f = 0;
    if (!cell_of(g, w, z, &f)) {
      atomicCAS(g.err, 0, si + 1);
      return false;
    }
    if (DATAFLOW == 2) {  // invalidate, data, publish (see the reader's seqlock)
      long long* sh = g.shadow + g.sbase[w.array] + f;
      st_rlx_s64(sh, -2);
      st_rel_f64(g.arr[w.array] + f, stk[sp - 1]);
      st_rel_s64(sh, logical_of(g, w, z));
    } else {
      __stcg(g.arr[w.array] + f, stk[sp - 1]);
    }
    if (DATAFLOW == 1) st_rel_u32(g.flags + g.fbase[w.array] + f, 1u);
    c3[0] += 1;
    c3[1] += unsigned(s.nreads);
    c3[2] += 1;
  }
  return true;
}

__global__ void generic_count_kernel(GDev g) {
  int64_t z[kMaxIdx];
  for (unsigned long long p = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       p < (unsigned long long)g.npoints; p += (unsigned long long)gridDim.x * blockDim.x) {
    decode(g, p, z);
    for (int si = 0; si < g.nstmt; ++si) {
      const GStmt s = g.st[si];
      if (!in_domain(g, s, z)) continue;
      const GRef& w = g.refs[s.wref];
      int64_t f = 0;
      if (!cell_of(g, w, z, &f)) {
        atomicCAS(g.err, 0, si + 1);
        continue;
      }
      const int64_t l = logical_of(g, w, z);
      if (l < 0) {  // written outside its declared extents: no per-cell check possible
        atomicOr(g.bad, 4u);
        continue;
      }
      atomicAdd(g.flags + g.fbase[w.array] + l, 1u);
      atomicMin(g.writer + g.fbase[w.array] + l, p * (unsigned long long)g.nstmt + si);
    }
  }
}

// The dataflow grid makes every read wait for its cell's (single) write.  That
// reproduces the reference only if, in the reference's order, the write comes
// strictly before the read: a read of a cell written later (or by the reading
// statement itself, whose write follows its body) sees the old value there.
// Flags such kernels so they run in the reference's sequential order instead.
__global__ void generic_order_kernel(GDev g) {
  int64_t z[kMaxIdx];
  for (unsigned long long p = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       p < (unsigned long long)g.npoints; p += (unsigned long long)gridDim.x * blockDim.x) {
    decode(g, p, z);
    for (int si = 0; si < g.nstmt; ++si) {
      const GStmt s = g.st[si];
      if (!in_domain(g, s, z)) continue;
      const unsigned long long me = p * (unsigned long long)g.nstmt + si;
      for (int o = 0; o < s.nops; ++o) {
        const GOp op = g.ops[s.op0 + o];
        if (op.kind != ORead) continue;
        const GRef& r = g.refs[op.arg];
        int64_t f = 0;
        if (!cell_of(g, r, z, &f)) continue;  // reported by the run itself
        const int64_t l = logical_of(g, r, z);
        if (l < 0) {
          atomicOr(g.bad, 8u);
          continue;
        }
        const unsigned long long w = g.writer[g.fbase[r.array] + l];
        // a never-written cell holds its initial value: fine in dense storage
        // (ready flag set up front) and for inputs (their shadows hold their
        // own ids), but a folded temp's slot is shared
        if (w == ~0ull) {
          if (!g.never_ok && !g.is_input[r.array]) atomicOr(g.bad, 2u);
        } else if (w >= me) {
          atomicOr(g.bad, 1u);
        }
      }
    }
  }
}

// flags <- (written at most... never written) ? ready : pending; max count
__global__ void generic_flags_kernel(unsigned* flags, int64_t n, unsigned* maxc) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const unsigned c = flags[i];
    if (c > 1) atomicMax(maxc, c);
    flags[i] = c == 0 ? 1u : 0u;
  }
}

// mapped dataflow: shadows <- inputs hold their own cells (reference
// init_storage: shadow[f] = f), everything else -1 (nothing written yet)
__global__ void generic_shadow_init_kernel(long long* sh, int64_t n, int64_t base, int is_input) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    sh[base + i] = is_input ? i : -1;
}

// Persistent dataflow grid: warps take 32 consecutive points in the
// reference's order; reads wait for their cell's flag (dense) or shadow (mapped).
template <int MODE>
__global__ void generic_dataflow_kernel(GDev g) {
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
      ok = exec_point<MODE>(g, z, c3);
    }
  }
  atomicAdd(&g.cnt[0], c3[0]);
  atomicAdd(&g.cnt[1], c3[1]);
  atomicAdd(&g.cnt[2], c3[2]);
}

// One thread, the reference's exact order (kernels that overwrite cells).
__global__ void generic_sequential_kernel(GDev g) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long c3[3] = {0, 0, 0};
  int64_t z[kMaxIdx];
  if (g.npoints > 0) decode(g, 0, z);
  for (unsigned long long p = 0; p < (unsigned long long)g.npoints; ++p) {
    if (!exec_point<0>(g, z, c3)) break;
    // next point in lexicographic order (odometer: no 64-bit divisions)
    for (int i = g.nidx - 1; i >= 0; --i) {
      if (++z[i] < g.lo[i] + g.ext[i]) break;
      z[i] = g.lo[i];
    }
  }
  g.cnt[0] = c3[0];
  g.cnt[1] = c3[1];
  g.cnt[2] = c3[2];
}

// ---------------------------------------------------------------- host side
int64_t floor_div(int64_t a, int64_t b) {  // b > 0
  return a >= 0 ? a / b : -((-a + b - 1) / b);
}
int64_t ceil_div(int64_t a, int64_t b) { return -floor_div(-a, b); }

using Row = std::vector<int64_t>;  // coefficients over n indices, then constant

void normalize(Row& r) {
  int64_t g = 0;
  for (size_t i = 0; i + 1 < r.size(); ++i) g = std::gcd(g, r[i] < 0 ? -r[i] : r[i]);
  if (g > 1) {
    for (size_t i = 0; i + 1 < r.size(); ++i) r[i] /= g;
    r.back() = floor_div(r.back(), g);  // integer tightening: a.z + k >= 0, a = g a'
  }
}

// Bounds of index q over the integer points of {rows >= 0} (rational
// Fourier-Motzkin relaxation, tightened).  Returns false if empty.
bool project_bounds(std::vector<Row> rows, size_t n, size_t q, int64_t* lo, int64_t* hi,
                    bool* bounded) {
  for (size_t e = 0; e < n; ++e) {
    if (e == q) continue;
    std::vector<Row> pos, neg, keep;
    for (auto& r : rows) (r[e] > 0 ? pos : r[e] < 0 ? neg : keep).push_back(r);
    for (const auto& p : pos)
      for (const auto& m : neg) {
        Row c(n + 1);
        const int64_t a = p[e], b = -m[e];
        for (size_t i = 0; i <= n; ++i) c[i] = b * p[i] + a * m[i];
        normalize(c);
        keep.push_back(c);
      }
    std::sort(keep.begin(), keep.end());
    keep.erase(std::unique(keep.begin(), keep.end()), keep.end());
    if (keep.size() > 4000) fail(ErrorKind::Overflow, "GpuExecutor: domain projection too large");
    rows.swap(keep);
  }
  int64_t L = INT64_MIN, H = INT64_MAX;
  for (const auto& r : rows) {
    if (r[q] > 0) L = std::max(L, ceil_div(-r.back(), r[q]));
    else if (r[q] < 0) H = std::min(H, floor_div(r.back(), -r[q]));
    else if (r.back() < 0) return false;
  }
  *bounded = L != INT64_MIN && H != INT64_MAX;
  *lo = L;
  *hi = H;
  return L <= H;
}

}  // namespace

struct GenericPlan {
  int device = 0;
  int nidx = 0;
  std::vector<std::string> names;
  std::vector<ArrayKind> kinds;
  std::vector<uint64_t> words;
  std::vector<double*> ptrs;
  std::vector<int64_t> fbase;   // logical cells: flags / writer base per array
  std::vector<int64_t> lsizes;  // logical cells per array (declared extents)
  std::vector<int64_t> sbase;   // storage cells: shadow base per array
  int64_t nflags = 0, nshadow = 0;
  bool mapped = false;          // some map is not the identity at the declared extents
  std::vector<GStmt> st;
  std::vector<GAff> rows, affs;
  std::vector<GRef> refs;
  std::vector<GOp> ops;
  std::vector<std::string> stmt_ids;
  int64_t lo[kMaxIdx] = {0}, ext[kMaxIdx] = {0};
  int64_t npoints = 0;
  // device copies
  GStmt* d_st = nullptr;
  GAff *d_rows = nullptr, *d_affs = nullptr;
  GRef* d_refs = nullptr;
  GOp* d_ops = nullptr;
  double** d_arr = nullptr;
  int64_t* d_fbase = nullptr;
  int64_t* d_sbase = nullptr;
  int64_t* d_lsize = nullptr;
  int* d_is_input = nullptr;
  unsigned bad = 0;  // why the dataflow grid was declined (order-check bits)
  long long* d_shadow = nullptr;
  unsigned* d_flags = nullptr;
  unsigned* d_flags0 = nullptr;  // initial flags (dataflow)
  unsigned long long* d_misc = nullptr;  // next, points, reads, writes
  int* d_err = nullptr;
  unsigned* d_maxc = nullptr;  // [0] max writes per cell, [1] order violation
  unsigned long long* d_writer = nullptr;
  bool dataflow = false;
  bool counted = false;
};

namespace {

void ckc(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(ErrorKind::Cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class T>
T* upload(const std::vector<T>& v) {
  T* d = nullptr;
  if (v.empty()) return nullptr;
  ckc(cudaMalloc(&d, v.size() * sizeof(T)), "cudaMalloc");
  ckc(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "H2D");
  // pageable H2D on the legacy stream may still be in flight on return, and the
  // executor's non-blocking stream does not wait for the legacy stream
  ckc(cudaStreamSynchronize(0), "H2D");
  return d;
}

// Affine over (depth indices ++ params) -> GAff over full indices with the
// params folded into the constant (embedding: missing indices get 0).
GAff fold(const Affine& a, size_t depth, size_t full, const IntVec& prm) {
  GAff g;
  std::memset(&g, 0, sizeof(g));
  for (size_t i = 0; i < depth && i < a.c.size(); ++i) g.c[i] = a.c[i];
  g.k = a.k;
  for (size_t j = 0; j < prm.size(); ++j)
    if (depth + j < a.c.size()) g.k += a.c[depth + j] * prm[j];
  (void)full;
  return g;
}

int64_t eval_extent(const Affine& a, size_t nidx, const IntVec& prm) {
  int64_t v = a.k;
  const size_t off = a.c.size() >= nidx + prm.size() ? nidx : 0;
  for (size_t j = 0; j < prm.size(); ++j)
    if (off + j < a.c.size()) v += a.c[off + j] * prm[j];
  return v;
}

}  // namespace

GenericPlan* generic_plan_create(const KernelSpec& k, const IntVec& prm,
                                 const std::vector<MemoryMap>& maps, int device) {
  if (prm.size() != k.params.size()) fail(ErrorKind::DimMismatch, "GpuExecutor: parameter count");
  const size_t full = k.indices.size();
  if (full == 0 || full > size_t(kMaxIdx)) fail(ErrorKind::Unsupported, "generic executor: 1..6 indices");
  auto P = std::make_unique<GenericPlan>();
  P->device = device;
  P->nidx = int(full);
  ckc(cudaSetDevice(device), "cudaSetDevice");
  // ---- arrays: storage by the caller's memory map (reference exec.cpp:
  // 234-245, MemoryMap::words), else dense at the declared extents
  auto map_of = [&](const std::string& name) -> const MemoryMap* {
    for (const auto& m : maps)
      if (m.array == name) return &m;
    return nullptr;
  };
  std::map<std::string, int> aid;
  int64_t fb = 0, sb = 0;
  for (const auto& a : k.arrays) {
    if (a.rank > size_t(kMaxRank)) fail(ErrorKind::Unsupported, "generic executor: rank > 6");
    uint64_t lw = 1;
    IntVec decl;
    for (const auto& e : a.extents) {
      const int64_t v = eval_extent(e, full, prm);
      if (v < 0) fail(ErrorKind::Validation, "array " + a.name + ": negative extent");
      lw *= uint64_t(v);
      decl.push_back(v);
    }
    uint64_t w = lw;
    if (const MemoryMap* m = map_of(a.name)) {
      if (m->extents.size() > size_t(kMaxRank)) fail(ErrorKind::Unsupported, "generic executor: storage rank > 6");
      w = 1;
      for (int64_t e : m->extents) w *= uint64_t(e);
      bool identity = m->extents == decl;
      for (size_t q = 0; identity && q < m->extents.size(); ++q) {
        identity = m->constant[q] == 0 && m->moduli[q] == 0;
        for (size_t c = 0; c < a.rank; ++c) identity = identity && m->linear[q][c] == (q == c ? 1 : 0);
      }
      if (!identity) P->mapped = true;
    }
    if (w > (uint64_t(1) << 33)) fail(ErrorKind::Unsupported, "generic executor: array " + a.name + " storage too large");
    aid[a.name] = int(P->names.size());
    P->names.push_back(a.name);
    P->kinds.push_back(a.kind);
    P->words.push_back(w);
    P->fbase.push_back(fb);
    P->lsizes.push_back(int64_t(lw));
    P->sbase.push_back(sb);
    fb += int64_t(lw);
    sb += int64_t(w);
    double* d = nullptr;
    ckc(cudaMalloc(&d, std::max<uint64_t>(w, 1) * 8), "cudaMalloc");
    P->ptrs.push_back(d);
  }
  P->nflags = fb;
  P->nshadow = sb;
  auto make_ref = [&](const std::string& arr, const std::vector<Affine>& subs, size_t depth) {
    const ArrayDecl* ad = k.find_array(arr);
    if (subs.size() != ad->rank) fail(ErrorKind::Validation, "Executor: subscript arity for " + arr);
    GRef r;
    std::memset(&r, 0, sizeof(r));
    r.array = aid.at(arr);
    std::vector<GAff> cell;
    for (const auto& s : subs) cell.push_back(fold(s, depth, full, prm));
    // logical id over the declared extents
    GAff l;
    std::memset(&l, 0, sizeof(l));
    int64_t lstride = 1;
    for (int d = int(ad->rank) - 1; d >= 0; --d) {
      for (size_t t = 0; t < full; ++t) l.c[t] += lstride * cell[size_t(d)].c[t];
      l.k += lstride * cell[size_t(d)].k;
      lstride *= eval_extent(ad->extents[size_t(d)], full, prm);
    }
    r.laff = int(P->affs.size());
    P->affs.push_back(l);
    r.aff0 = int(P->affs.size());
    const MemoryMap* m = map_of(arr);
    if (m) {  // storage_k = map_k(cell): compose (reference build_ref, exec.cpp:150-163)
      r.rank = int(m->extents.size());
      for (int q = 0; q < r.rank; ++q) {
        GAff a;
        std::memset(&a, 0, sizeof(a));
        a.k = m->constant[size_t(q)];
        for (size_t j = 0; j < ad->rank; ++j) {
          const int64_t wgt = m->linear[size_t(q)][j];
          a.k += wgt * cell[j].k;
          for (size_t t = 0; t < full; ++t) a.c[t] += wgt * cell[j].c[t];
        }
        P->affs.push_back(a);
        r.ext[q] = m->extents[size_t(q)];
        r.mod[q] = m->moduli[size_t(q)];
      }
    } else {
      r.rank = int(ad->rank);
      for (int q = 0; q < r.rank; ++q) {
        P->affs.push_back(cell[size_t(q)]);
        r.ext[q] = eval_extent(ad->extents[size_t(q)], full, prm);
      }
    }
    int64_t stride = 1;
    for (int d = r.rank - 1; d >= 0; --d) {
      r.stride[d] = stride;
      stride *= r.ext[d];
    }
    P->refs.push_back(r);
    return int(P->refs.size() - 1);
  };
  // ---- statements: embed, fold params, compile bodies
  std::vector<int64_t> lo(full, INT64_MAX), hi(full, INT64_MIN);
  bool any = false;
  for (const auto& s : k.statements) {
    GStmt g;
    std::memset(&g, 0, sizeof(g));
    g.row0 = int(P->rows.size());
    std::vector<Row> frows;
    for (const auto& r : s.domain) {
      Affine a;
      a.c.assign(r.begin(), r.end() - 1);
      a.k = r.back();
      GAff ga = fold(a, s.depth, full, prm);
      P->rows.push_back(ga);
      Row fr(ga.c, ga.c + full);
      fr.push_back(ga.k);
      frows.push_back(fr);
    }
    for (size_t q = s.depth; q < full; ++q) {  // embed: z_q = 0
      for (int sg : {1, -1}) {
        GAff ga;
        std::memset(&ga, 0, sizeof(ga));
        ga.c[q] = sg;
        P->rows.push_back(ga);
        Row fr(full + 1, 0);
        fr[q] = sg;
        frows.push_back(fr);
      }
    }
    g.nrows = int(P->rows.size()) - g.row0;
    // point box: project the statement's domain on every index
    bool empty = false;
    std::vector<int64_t> slo(full), shi(full);
    for (size_t q = 0; q < full && !empty; ++q) {
      bool bounded = true;
      if (!project_bounds(frows, full, q, &slo[q], &shi[q], &bounded)) empty = true;
      else if (!bounded) fail(ErrorKind::Unbounded, "Executor: unbounded loop level in " + s.id);
    }
    if (!empty) {
      any = true;
      for (size_t q = 0; q < full; ++q) lo[q] = std::min(lo[q], slo[q]), hi[q] = std::max(hi[q], shi[q]);
    }
    // body -> postfix (left, right, op), reads counted statically
    g.op0 = int(P->ops.size());
    int nreads = 0;
    std::function<void(const ExprPtr&)> emit = [&](const ExprPtr& e) {
      GOp op;
      op.arg = 0;
      op.lit = 0.0;
      switch (e->kind) {
        case Expr::Kind::Lit: op.kind = OLit; op.lit = e->lit; break;
        case Expr::Kind::Aff:
          op.kind = OAff;
          op.arg = int(P->affs.size());
          P->affs.push_back(fold(e->aff, s.depth, full, prm));
          break;
        case Expr::Kind::Read:
          op.kind = ORead;
          op.arg = make_ref(e->array, e->subs, s.depth);
          ++nreads;
          break;
        case Expr::Kind::Neg: emit(e->l); op.kind = ONeg; break;
        case Expr::Kind::Sqrt: emit(e->l); op.kind = OSqrt; break;
        default:
          emit(e->l);
          emit(e->r);
          op.kind = e->kind == Expr::Kind::Add ? OAdd : e->kind == Expr::Kind::Sub ? OSub
                  : e->kind == Expr::Kind::Mul ? OMul : e->kind == Expr::Kind::Div ? ODiv
                  : e->kind == Expr::Kind::Min ? OMin : OMax;
          break;
      }
      P->ops.push_back(op);
    };
    emit(s.body);
    g.nops = int(P->ops.size()) - g.op0;
    g.nreads = nreads;
    // stack depth bound (postfix: pushes minus pops)
    int sp = 0, mx = 0;
    for (int o = g.op0; o < g.op0 + g.nops; ++o) {
      const int kd = P->ops[size_t(o)].kind;
      sp += (kd == OLit || kd == OAff || kd == ORead) ? 1 : (kd == ONeg || kd == OSqrt) ? 0 : -1;
      mx = std::max(mx, sp);
    }
    if (mx > kMaxStack) fail(ErrorKind::Unsupported, "generic executor: expression too deep in " + s.id);
    g.wref = make_ref(s.write_array, s.write_subs, s.depth);
    P->st.push_back(g);
    P->stmt_ids.push_back(s.id);
  }
  P->npoints = 0;
  if (any) {
    P->npoints = 1;
    for (size_t q = 0; q < full; ++q) {
      P->lo[q] = lo[q];
      P->ext[q] = hi[q] - lo[q] + 1;
      if (P->ext[q] <= 0 || P->npoints > (int64_t(1) << 50) / P->ext[q])
        fail(ErrorKind::Overflow, "generic executor: iteration box too large");
      P->npoints *= P->ext[q];
    }
  }
  P->d_st = upload(P->st);
  P->d_rows = upload(P->rows);
  P->d_affs = upload(P->affs);
  P->d_refs = upload(P->refs);
  P->d_ops = upload(P->ops);
  P->d_arr = upload(P->ptrs);
  P->d_fbase = upload(P->fbase);
  P->d_sbase = upload(P->sbase);
  P->d_lsize = upload(P->lsizes);
  {
    std::vector<int> inp;
    for (auto kd : P->kinds) inp.push_back(kd == ArrayKind::Input ? 1 : 0);
    P->d_is_input = upload(inp);
  }
  if (P->mapped)
    ckc(cudaMalloc(&P->d_shadow, std::max<int64_t>(P->nshadow, 1) * sizeof(long long)), "cudaMalloc");
  ckc(cudaMalloc(&P->d_flags, std::max<int64_t>(P->nflags, 1) * sizeof(unsigned)), "cudaMalloc");
  ckc(cudaMalloc(&P->d_flags0, std::max<int64_t>(P->nflags, 1) * sizeof(unsigned)), "cudaMalloc");
  ckc(cudaMalloc(&P->d_misc, 4 * sizeof(unsigned long long)), "cudaMalloc");
  ckc(cudaMalloc(&P->d_err, sizeof(int)), "cudaMalloc");
  ckc(cudaMalloc(&P->d_maxc, 2 * sizeof(unsigned)), "cudaMalloc");
  return P.release();
}

void generic_plan_destroy(GenericPlan* p) {
  if (!p) return;
  for (double* d : p->ptrs) cudaFree(d);
  cudaFree(p->d_st);
  cudaFree(p->d_rows);
  cudaFree(p->d_affs);
  cudaFree(p->d_refs);
  cudaFree(p->d_ops);
  cudaFree(p->d_arr);
  cudaFree(p->d_fbase);
  cudaFree(p->d_sbase);
  cudaFree(p->d_lsize);
  cudaFree(p->d_is_input);
  cudaFree(p->d_shadow);
  cudaFree(p->d_flags);
  cudaFree(p->d_flags0);
  cudaFree(p->d_misc);
  cudaFree(p->d_err);
  cudaFree(p->d_maxc);
  cudaFree(p->d_writer);
  delete p;
}

size_t generic_array_count(const GenericPlan* p) { return p->names.size(); }
const std::string& generic_array_name(const GenericPlan* p, size_t i) { return p->names[i]; }
ArrayKind generic_array_kind(const GenericPlan* p, size_t i) { return p->kinds[i]; }
uint64_t generic_array_words(const GenericPlan* p, size_t i) { return p->words[i]; }
double* generic_array_ptr(GenericPlan* p, size_t i) { return p->ptrs[i]; }

cudaError_t generic_init_inputs(GenericPlan* p, cudaStream_t s) {
  cudaError_t e;
  for (size_t i = 0; i < p->names.size(); ++i) {
    if (p->kinds[i] != ArrayKind::Input || p->words[i] == 0) continue;
    const uint64_t h = fnv1a(p->names[i].data(), p->names[i].size());
    if ((e = fill_init_value(p->ptrs[i], int64_t(p->words[i]), 1, int64_t(p->words[i]), h, 0, s)) !=
        cudaSuccess)
      return e;
  }
  return cudaSuccess;
}

static GDev dev_args(GenericPlan* p) {
  GDev g;
  std::memset(&g, 0, sizeof(g));
  g.nidx = p->nidx;
  g.nstmt = int(p->st.size());
  for (int i = 0; i < p->nidx; ++i) g.lo[i] = p->lo[i], g.ext[i] = p->ext[i];
  g.npoints = p->npoints;
  g.st = p->d_st;
  g.rows = p->d_rows;
  g.affs = p->d_affs;
  g.refs = p->d_refs;
  g.ops = p->d_ops;
  g.arr = p->d_arr;
  g.fbase = p->d_fbase;
  g.sbase = p->d_sbase;
  g.lsize = p->d_lsize;
  g.shadow = p->d_shadow;
  g.never_ok = p->mapped ? 0 : 1;
  g.is_input = p->d_is_input;
  g.writer = p->d_writer;  // mapped dataflow: writer keys of the logical cells
  g.flags = p->d_flags;
  g.next = p->d_misc;
  g.cnt = p->d_misc + 1;
  g.err = p->d_err;
  return g;
}

cudaError_t generic_run(GenericPlan* p, cudaStream_t s, GenericCounts* counts, std::string* err_msg) {
  cudaError_t e;
  GDev g = dev_args(p);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, p->device);
  // temps and outputs start at 0.0 every run (inputs persist)
  for (size_t i = 0; i < p->names.size(); ++i)
    if (p->kinds[i] != ArrayKind::Input && p->words[i])
      if ((e = cudaMemsetAsync(p->ptrs[i], 0, p->words[i] * 8, s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p->d_err, 0, sizeof(int), s)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(p->d_misc, 0, 4 * sizeof(unsigned long long), s)) != cudaSuccess) return e;
  // the per-cell checks index the logical cells (flags 4 B + writer 8 B each)
  const bool checkable = p->nflags <= (int64_t(1) << 31);
  if (!p->counted && !checkable) {
    p->dataflow = false;  // too large to verify: the reference's sequential order
    p->counted = true;
  }
  if (!p->counted) {  // write counts once per plan: single assignment -> dataflow grid
    if ((e = cudaMemsetAsync(p->d_flags, 0, std::max<int64_t>(p->nflags, 1) * sizeof(unsigned), s)) != cudaSuccess)
      return e;
    if ((e = cudaMemsetAsync(p->d_maxc, 0, 2 * sizeof(unsigned), s)) != cudaSuccess) return e;
    const size_t wbytes = size_t(std::max<int64_t>(p->nflags, 1)) * sizeof(unsigned long long);
    if ((e = cudaMalloc(&p->d_writer, wbytes)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(p->d_writer, 0xff, wbytes, s)) != cudaSuccess) return e;
    g.writer = p->d_writer;
    g.bad = p->d_maxc + 1;
    if (p->npoints > 0) {
      generic_count_kernel<<<sms * 8, 256, 0, s>>>(g);
      count_launch();
      generic_order_kernel<<<sms * 8, 256, 0, s>>>(g);
      count_launch();
    }
    if (p->nflags > 0) {
      generic_flags_kernel<<<sms * 4, 256, 0, s>>>(p->d_flags, p->nflags, p->d_maxc);
      count_launch();
    }
    unsigned maxc[2] = {0, 0};
    int err = 0;
    if ((e = cudaMemcpyAsync(maxc, p->d_maxc, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(&err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if (err > 0) {
      if (err_msg) *err_msg = "out-of-extent write in statement " + p->stmt_ids[size_t(err - 1)];
      return cudaErrorInvalidValue;
    }
    if (!p->mapped) {  // dense storage: only the counting pass needs the writer keys
      cudaFree(p->d_writer);
      p->d_writer = nullptr;
    }
    p->dataflow = maxc[0] <= 1 && maxc[1] == 0;
    p->bad = maxc[1] | (maxc[0] > 1 ? 16u : 0u);
    if (env_int("PCOTGPU_GENERIC_DEBUG", 0))
      std::fprintf(stderr, "generic: mapped=%d logical=%lld storage=%lld max_writes=%u order_bits=%u -> %s\n",
                   int(p->mapped), (long long)p->nflags, (long long)p->nshadow, maxc[0], maxc[1],
                   p->dataflow ? (p->mapped ? "dataflow (shadows)" : "dataflow (flags)") : "sequential");
    if ((e = cudaMemcpyAsync(p->d_flags0, p->d_flags, std::max<int64_t>(p->nflags, 1) * sizeof(unsigned),
                             cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return e;
    p->counted = true;
  } else if (p->dataflow && !p->mapped) {
    if ((e = cudaMemcpyAsync(p->d_flags, p->d_flags0, std::max<int64_t>(p->nflags, 1) * sizeof(unsigned),
                             cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return e;
  }
  if (p->dataflow && p->mapped) {  // storage reset: shadows say what each cell holds
    for (size_t i = 0; i < p->names.size(); ++i) {
      if (!p->words[i]) continue;
      generic_shadow_init_kernel<<<sms * 2, 256, 0, s>>>(p->d_shadow, int64_t(p->words[i]), p->sbase[i],
                                                         p->kinds[i] == ArrayKind::Input ? 1 : 0);
      count_launch();
    }
  }
  if (p->npoints > 0) {
    if (p->dataflow && p->mapped) {
      generic_dataflow_kernel<2><<<sms * 4, 128, 0, s>>>(g);
      count_launch();
      // a storage cell reused under a waiting reader (the map folds along a
      // vector that is not universal for this kernel's dependences): this run
      // is void; the plan switches to the reference's sequential order for
      // good and the run is repeated from the initial storage
      int e2 = 0;
      if ((e = cudaMemcpyAsync(&e2, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      if (e2 == -2) {
        p->dataflow = false;
        if (env_int("PCOTGPU_GENERIC_DEBUG", 0))
          std::fprintf(stderr, "generic: storage reuse race detected -> sequential\n");
        return generic_run(p, s, counts, err_msg);
      }
    } else if (p->dataflow) {
      generic_dataflow_kernel<1><<<sms * 4, 128, 0, s>>>(g);
    } else {
      generic_sequential_kernel<<<1, 32, 0, s>>>(g);
    }
    if (!(p->dataflow && p->mapped)) count_launch();
  }
  unsigned long long c[3] = {0, 0, 0};
  int err = 0;
  if ((e = cudaMemcpyAsync(c, p->d_misc + 1, sizeof(c), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(&err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  if (err != 0) {
    if (err_msg)
      *err_msg = err > 0 ? "out-of-extent access in statement " + p->stmt_ids[size_t(err - 1)]
                 : err == -2 ? std::string("dependence violation: a storage cell was reused before its "
                                           "value was read (the memory map is not a universal occupancy vector)")
                             : std::string("dataflow wait exceeded its bound (kernel not legal in lexicographic order)");
    return cudaErrorInvalidValue;
  }
  if (counts) {
    counts->points = c[0];
    counts->reads = c[1];
    counts->writes = c[2];
    counts->parallel = p->dataflow;
    counts->mode = !p->dataflow ? 0 : p->mapped ? 2 : 1;
  }
  return cudaSuccess;
}

}  // namespace pcotgpu
