// Generic device executor: see generic.h.  Follows the reference's
// Executor::exec_stmt / run_level semantics (core/src/exec.cpp:347-472): the
// union of the statement domains is walked in lexicographic index order, each
// point runs the statements that contain it in declaration order, and each
// body is the postfix program of the reference's flatten (exec.cpp:187-224).
#include <algorithm>
#include <cuda.h>
#include <dlfcn.h>
#include <climits>
#include <cstdio>
#include <cmath>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>

#include "common.cuh"
#include "generic.h"
#include "kernels.h"

namespace pcotgpu {

namespace {

#include "generic_dev.cuh"

// Run every statement of point z (interpreter: the reference's postfix
// program, exec.cpp:187-224, one rounding per operation).  Returns false on an
// error (recorded).
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
          bool ok = true;
          const double v = gread<DATAFLOW>(g, op.arg, z, si, ok);
          if (!ok) return false;
          stk[sp++] = v;
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
    if (!gwrite<DATAFLOW>(g, s.wref, z, si, stk[sp - 1])) return false;
    c3[0] += 1;
    c3[1] += unsigned(s.nreads);
    c3[2] += 1;
  }
  return true;
}

struct InterpPE {
  template <int MODE>
  static PCOT_DEV bool run(const GDev& g, const int64_t* z, unsigned long long* c3) {
    return exec_point<MODE>(g, z, c3);
  }
};

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

template <int MODE>
__global__ void generic_dataflow_kernel(GDev g) {
  dataflow_loop<MODE, InterpPE>(g);
}

__global__ void generic_sequential_kernel(GDev g) { sequential_loop<InterpPE>(g); }

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
  // PRDG -> CUDA emitter: the plan's statements as straight-line device code,
  // compiled at run time (NVRTC); null when unavailable (interpreter then)
  std::string jit_src, jit_why;
  void* jit_module = nullptr;  // CUmodule
  void* jit_fn[3] = {nullptr, nullptr, nullptr};  // sequential, dataflow flags, dataflow shadows
  bool jit_tried = false;
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
                                 const std::vector<MemoryMap>& maps, int device, bool host_only) {
  if (prm.size() != k.params.size()) fail(ErrorKind::DimMismatch, "GpuExecutor: parameter count");
  const size_t full = k.indices.size();
  if (full == 0 || full > size_t(kMaxIdx)) fail(ErrorKind::Unsupported, "generic executor: 1..6 indices");
  auto P = std::make_unique<GenericPlan>();
  P->device = device;
  P->nidx = int(full);
  if (!host_only) ckc(cudaSetDevice(device), "cudaSetDevice");
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
    if (!host_only) ckc(cudaMalloc(&d, std::max<uint64_t>(w, 1) * 8), "cudaMalloc");
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
  if (host_only) return P.release();  // tables only (the emitter's source)
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

// ---------------------------------------------------------------- PRDG -> CUDA emitter
// The GPU analogue of the reference's emit_c (emit_c.cpp:191-262): every
// statement of the plan becomes straight-line device code — its domain rows
// as constant affine tests, its body as one IEEE-rounded intrinsic per
// operation in the reference's postfix order (exec.cpp:187-224), its reads
// and write through the shared runtime (generic_dev.cuh: map addressing and
// the schedule's wait / publish protocol).  Compiled at run time with NVRTC
// for sm_100a and launched in place of the interpreter kernels; no operand
// stack, no per-operation dispatch.

static const char kGenericDevSrc[] =
#include "generic_dev_src.inc"
    ;

namespace {

std::string aff_src(const GAff& a, int nidx) {
  std::string e;
  for (int i = 0; i < nidx; ++i)
    if (a.c[i]) e += " + (" + std::to_string((long long)a.c[i]) + "LL * z[" + std::to_string(i) + "])";
  e += " + (" + std::to_string((long long)a.k) + "LL)";
  return "(0LL" + e + ")";
}

std::string lit_src(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%a", v);
  return std::string("(") + b + ")";
}

struct NvrtcApi {
  void* h = nullptr;
  int (*create)(void**, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
  int (*compile)(void*, int, const char* const*) = nullptr;
  int (*log_size)(void*, size_t*) = nullptr;
  int (*log)(void*, char*) = nullptr;
  int (*cubin_size)(void*, size_t*) = nullptr;
  int (*cubin)(void*, char*) = nullptr;
  int (*destroy)(void**) = nullptr;
  bool ok = false;
};

const NvrtcApi& nvrtc() {
  static const NvrtcApi api = [] {
    NvrtcApi a;
    a.h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_LOCAL);
    if (!a.h) a.h = dlopen("libnvrtc.so", RTLD_NOW | RTLD_LOCAL);
    if (!a.h) return a;
    a.create = reinterpret_cast<decltype(a.create)>(dlsym(a.h, "nvrtcCreateProgram"));
    a.compile = reinterpret_cast<decltype(a.compile)>(dlsym(a.h, "nvrtcCompileProgram"));
    a.log_size = reinterpret_cast<decltype(a.log_size)>(dlsym(a.h, "nvrtcGetProgramLogSize"));
    a.log = reinterpret_cast<decltype(a.log)>(dlsym(a.h, "nvrtcGetProgramLog"));
    a.cubin_size = reinterpret_cast<decltype(a.cubin_size)>(dlsym(a.h, "nvrtcGetCUBINSize"));
    a.cubin = reinterpret_cast<decltype(a.cubin)>(dlsym(a.h, "nvrtcGetCUBIN"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(a.h, "nvrtcDestroyProgram"));
    a.ok = a.create && a.compile && a.log_size && a.log && a.cubin_size && a.cubin && a.destroy;
    return a;
  }();
  return api;
}

struct DriverApi {
  CUresult (*load)(CUmodule*, const void*) = nullptr;
  CUresult (*get)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                     CUstream, void**, void**) = nullptr;
  CUresult (*unload)(CUmodule) = nullptr;
  bool ok = false;
};

const DriverApi& driver() {
  static const DriverApi api = [] {
    DriverApi a;
    auto sym = [](const char* n) -> void* {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(n, &fn, cudaEnableDefault, &q) != cudaSuccess ||
          q != cudaDriverEntryPointSuccess)
        return nullptr;
      return fn;
    };
    a.load = reinterpret_cast<decltype(a.load)>(sym("cuModuleLoadData"));
    a.get = reinterpret_cast<decltype(a.get)>(sym("cuModuleGetFunction"));
    a.launch = reinterpret_cast<decltype(a.launch)>(sym("cuLaunchKernel"));
    a.unload = reinterpret_cast<decltype(a.unload)>(sym("cuModuleUnload"));
    a.ok = a.load && a.get && a.launch && a.unload;
    return a;
  }();
  return api;
}

// compiled modules by (device, source): kept for the process (a module is a
// few tens of KB; plans of the same kernel and binding reuse it)
std::mutex& jit_cache_mu() {
  static std::mutex m;
  return m;
}
std::map<std::pair<int, std::string>, CUmodule>& jit_cache() {
  static std::map<std::pair<int, std::string>, CUmodule> c;
  return c;
}

}  // namespace

// Source of the plan's kernels (host only: no device needed).
std::string generic_emit_source(const GenericPlan* P) {
  std::string o;
  o += "#define PCOT_DEV __device__ __forceinline__\n";
  o += "typedef long long int64_t;\n";
  o += kGenericDevSrc;
  o += "\nstruct JitPE {\n  template <int MODE>\n"
       "  static PCOT_DEV bool run(const GDev& g, const int64_t* z, unsigned long long* c3) {\n";
  for (size_t si = 0; si < P->st.size(); ++si) {
    const GStmt& st = P->st[si];
    o += "    // statement " + P->stmt_ids[si] + "\n    if (1";
    for (int r = 0; r < st.nrows; ++r) o += "\n        && " + aff_src(P->rows[size_t(st.row0 + r)], P->nidx) + " >= 0LL";
    o += ") {\n      bool ok = true;\n";
    std::vector<std::string> stk;
    int t = 0;
    for (int q = st.op0; q < st.op0 + st.nops; ++q) {
      const GOp& op = P->ops[size_t(q)];
      const std::string v = "t" + std::to_string(t++);
      std::string e;
      auto pop = [&]() { std::string x = stk.back(); stk.pop_back(); return x; };
      switch (op.kind) {
        case OLit: e = lit_src(op.lit); break;
        case OAff: e = "(double)" + aff_src(P->affs[size_t(op.arg)], P->nidx); break;
        case ORead:
          o += "      const double " + v + " = gread<MODE>(g, " + std::to_string(op.arg) + ", z, " +
               std::to_string(si) + ", ok);\n      if (!ok) return false;\n";
          stk.push_back(v);
          continue;
        case OAdd: { const std::string b = pop(), a = pop(); e = "__dadd_rn(" + a + ", " + b + ")"; break; }
        case OSub: { const std::string b = pop(), a = pop(); e = "__dsub_rn(" + a + ", " + b + ")"; break; }
        case OMul: { const std::string b = pop(), a = pop(); e = "__dmul_rn(" + a + ", " + b + ")"; break; }
        case ODiv: { const std::string b = pop(), a = pop(); e = "__ddiv_rn(" + a + ", " + b + ")"; break; }
        case OMin: { const std::string b = pop(), a = pop(); e = "(" + b + " < " + a + " ? " + b + " : " + a + ")"; break; }
        case OMax: { const std::string b = pop(), a = pop(); e = "(" + a + " < " + b + " ? " + b + " : " + a + ")"; break; }
        case ONeg: e = "(-" + pop() + ")"; break;
        case OSqrt: e = "__dsqrt_rn(" + pop() + ")"; break;
      }
      o += "      const double " + v + " = " + e + ";\n";
      stk.push_back(v);
    }
    o += "      if (!gwrite<MODE>(g, " + std::to_string(st.wref) + ", z, " + std::to_string(si) + ", " +
         stk.back() + ")) return false;\n";
    o += "      c3[0] += 1; c3[1] += " + std::to_string(st.nreads) + "; c3[2] += 1;\n    }\n";
  }
  o += "    return true;\n  }\n};\n";
  o += "extern \"C\" __global__ void pcot_jit_seq(GDev g) { sequential_loop<JitPE>(g); }\n";
  o += "extern \"C\" __global__ void pcot_jit_df1(GDev g) { dataflow_loop<1, JitPE>(g); }\n";
  o += "extern \"C\" __global__ void pcot_jit_df2(GDev g) { dataflow_loop<2, JitPE>(g); }\n";
  return o;
}

// Compile + load the plan's kernels once; false (with the reason) when NVRTC
// or the driver entry points are unavailable or compilation fails.
bool generic_jit_build(GenericPlan* P) {
  if (P->jit_tried) return P->jit_module != nullptr;
  P->jit_tried = true;
  if (env_int("PCOTGPU_GENERIC_JIT", 1) == 0) {
    P->jit_why = "disabled (PCOTGPU_GENERIC_JIT=0)";
    return false;
  }
  const NvrtcApi& nv = nvrtc();
  const DriverApi& dr = driver();
  if (!nv.ok || !dr.ok) {
    P->jit_why = !nv.ok ? "libnvrtc not loadable" : "driver entry points unavailable";
    return false;
  }
  P->jit_src = generic_emit_source(P);
  CUmodule cached = nullptr;
  {  // one compile per (device, source) and process: plans of the same kernel share it
    std::lock_guard<std::mutex> lk(jit_cache_mu());
    auto it = jit_cache().find({P->device, P->jit_src});
    if (it != jit_cache().end()) cached = it->second;
  }
  if (cached) {
    const char* names[3] = {"pcot_jit_seq", "pcot_jit_df1", "pcot_jit_df2"};
    for (int q = 0; q < 3; ++q) {
      CUfunction f = nullptr;
      if (dr.get(&f, cached, names[q]) != CUDA_SUCCESS) {
        P->jit_why = std::string("cuModuleGetFunction ") + names[q];
        return false;
      }
      P->jit_fn[q] = f;
    }
    P->jit_module = cached;
    P->jit_why = "compiled (cached)";
    return true;
  }
  void* prog = nullptr;
  if (nv.create(&prog, P->jit_src.c_str(), "pcot_generic.cu", 0, nullptr, nullptr) != 0) {
    P->jit_why = "nvrtcCreateProgram failed";
    return false;
  }
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false", "-lineinfo"};
  const int rc = nv.compile(prog, 4, opts);
  if (rc != 0) {
    size_t n = 0;
    nv.log_size(prog, &n);
    std::string lg(n, '\0');
    nv.log(prog, &lg[0]);
    P->jit_why = "NVRTC: " + lg.substr(0, 2000);
    nv.destroy(&prog);
    return false;
  }
  size_t n = 0;
  nv.cubin_size(prog, &n);
  std::vector<char> cubin(n);
  nv.cubin(prog, cubin.data());
  nv.destroy(&prog);
  cudaSetDevice(P->device);
  cudaFree(nullptr);  // the runtime's primary context is current
  CUmodule m = nullptr;
  if (dr.load(&m, cubin.data()) != CUDA_SUCCESS) {
    P->jit_why = "cuModuleLoadData failed";
    return false;
  }
  {
    std::lock_guard<std::mutex> lk(jit_cache_mu());
    jit_cache()[{P->device, P->jit_src}] = m;
  }
  const char* names[3] = {"pcot_jit_seq", "pcot_jit_df1", "pcot_jit_df2"};
  for (int q = 0; q < 3; ++q) {
    CUfunction f = nullptr;
    if (dr.get(&f, m, names[q]) != CUDA_SUCCESS) {
      dr.unload(m);
      P->jit_why = std::string("cuModuleGetFunction ") + names[q];
      return false;
    }
    P->jit_fn[q] = f;
  }
  P->jit_module = m;
  P->jit_why = "compiled";
  return true;
}

const std::string& generic_jit_status(const GenericPlan* p) { return p->jit_why; }

// Host only: emit and NVRTC-compile the plan's kernels (no module load).
bool generic_jit_compile_check(const GenericPlan* P, std::string* log) {
  const NvrtcApi& nv = nvrtc();
  if (!nv.ok) {
    if (log) *log = "libnvrtc not loadable";
    return false;
  }
  const std::string src = generic_emit_source(P);
  void* prog = nullptr;
  if (nv.create(&prog, src.c_str(), "pcot_generic.cu", 0, nullptr, nullptr) != 0) return false;
  const char* opts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false"};
  const int rc = nv.compile(prog, 3, opts);
  size_t n = 0;
  nv.log_size(prog, &n);
  std::string lg(n, '\0');
  if (n) nv.log(prog, &lg[0]);
  size_t cb = 0;
  if (rc == 0) nv.cubin_size(prog, &cb);
  nv.destroy(&prog);
  if (log) *log = lg;
  return rc == 0 && cb > 0;
}

static cudaError_t jit_launch(GenericPlan* P, int q, unsigned grid, unsigned block, GDev g, cudaStream_t s) {
  void* args[] = {&g};
  const CUresult r = driver().launch(static_cast<CUfunction>(P->jit_fn[q]), grid, 1, 1, block, 1, 1, 0,
                                     reinterpret_cast<CUstream>(s), args, nullptr);
  count_launch();
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

void generic_plan_destroy(GenericPlan* p) {
  if (!p) return;
  // (compiled modules stay in the process-wide cache)
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
  const bool jit = p->npoints > 0 && generic_jit_build(p);
  if (p->npoints > 0) {
    if (p->dataflow && p->mapped) {
      if (jit) {
        if ((e = jit_launch(p, 2, unsigned(sms * 4), 128, g, s)) != cudaSuccess) return e;
      } else {
        generic_dataflow_kernel<2><<<sms * 4, 128, 0, s>>>(g);
        count_launch();
      }
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
      if (jit) {
        if ((e = jit_launch(p, 1, unsigned(sms * 4), 128, g, s)) != cudaSuccess) return e;
      } else {
        generic_dataflow_kernel<1><<<sms * 4, 128, 0, s>>>(g);
        count_launch();
      }
    } else {
      if (jit) {
        if ((e = jit_launch(p, 0, 1, 32, g, s)) != cudaSuccess) return e;
      } else {
        generic_sequential_kernel<<<1, 32, 0, s>>>(g);
        count_launch();
      }
    }
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
    counts->compiled = p->jit_module != nullptr;
  }
  return cudaSuccess;
}

}  // namespace pcotgpu
