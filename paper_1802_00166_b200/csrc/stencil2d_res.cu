// 2-D 5-point stencil, grid resident on chip for the whole run (sm_100a).
//
// Small grids (BASELINE config 0: 2048^2, T=256; both ping-pong slabs sit in L2)
// are launch- and latency-bound under the streaming kernel of stencil2d.cu: 32
// launches of ~37 us, 1.6x redundant halo work.  Here the grid is loaded ONCE:
// one persistent CTA per SM owns a band of consecutive rows (2048 rows / 147
// bands = 14 rows x 16 KB = 224 KB of shared memory), steps it T times in
// place, and stores it once.  Same arithmetic as the reference body
// (core/src/exec.cpp:347-428 over kernels/jacobi2d.kernel / heat2d.kernel):
//   0.2 * ((((c + (i-1,j)) + (i+1,j)) + (i,j-1)) + (i,j+1)), one rounding per
// operation, ring cells never updated (zeroed or held by the caller).
//
// In-place step: every thread owns 4 adjacent columns and walks its rows top to
// bottom with the old rows r-1, r, r+1 in registers; W/E neighbours by warp
// shuffle.  Across warps the neighbour column is foreign shared memory that
// its owner overwrites during the sweep, so lanes 0 / 31 copy their foreign
// edge column (all rows, old values) into registers at the start of the step:
// two CTA barriers per step (after the previous step's writes, before this
// step's), none per row, and the warps drift through the sweep independently.
// The band's last row is computed first (published early, kept in registers
// until the sweep is over).  A thread's 4 columns sit in shared memory as two
// 16-byte halves 512 B apart (lane-contiguous), so every 128-bit access is
// bank-conflict free.
//
// Band-to-band: a step needs the neighbours' boundary rows of the previous
// step.  Each band stores its new first/last row into a double-buffered global
// exchange line as soon as they exist (first thing in the step); every double
// travels as two 64-bit words {step tag, low half} / {step tag, high half}, so a
// word is valid by itself (aligned 64-bit accesses are single-copy atomic) and
// the reader needs no flag, no fence and no barrier: each thread loads its own
// four columns of the neighbours' rows in the middle of the sweep (the store ->
// L2 -> load latency runs under the remaining rows) and re-polls at the start
// of the next step only if a tag is still old.  A slot written at step t is
// overwritten at step t+2, which the writer reaches only after it has consumed
// the reader's step t+1 rows, which were computed from the slot's content: the
// data dependence orders the reuse.  Cooperative launch guarantees
// co-residency; a capped spin raises a fault word instead of hanging.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

struct S2ResPlan {
  int device = 0, n = 0, npad = 0, nt = 0, nbands = 0, rmax = 0;
  size_t smem = 0;
  unsigned long long* xbuf = nullptr;  // [2][nbands][2][2 * npad] tagged words
  int* d_err = nullptr;                // fault word
  int* h_err = nullptr;                // pinned
  unsigned epoch = 0;                  // step tags of a run: epoch + t
};

namespace {

constexpr int kSpinCapR = 1 << 22;  // polls (each an L2 round trip) before a fault is raised

struct ResArgs {
  const double* in;
  double* out;
  int64_t ld_in, ld_out;
  int n, T, npad, nbands, rwait, nosync;
  unsigned epoch;
  unsigned long long* xbuf;
  int* err;
};

PCOT_DEV int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Four doubles -> eight self-validating words {tag:32 | half:32} (64 B).
PCOT_DEV void xput(unsigned long long* p, const double (&v)[4], unsigned tag) {
  const unsigned long long hi = static_cast<unsigned long long>(tag) << 32;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v[c]));
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p + 2 * c),
                 "l"(hi | (u & 0xffffffffull)), "l"(hi | (u >> 32))
                 : "memory");
  }
}
PCOT_DEV void xload(unsigned long long (&w)[8], const unsigned long long* p) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];"
                 : "=l"(w[2 * c]), "=l"(w[2 * c + 1])
                 : "l"(p + 2 * c)
                 : "memory");
}
PCOT_DEV bool xvalid(const unsigned long long (&w)[8], unsigned tag) {
  bool ok = true;
#pragma unroll
  for (int i = 0; i < 8; ++i) ok = ok && unsigned(w[i] >> 32) == tag;
  return ok;
}
PCOT_DEV void xvalue(double (&v)[4], const unsigned long long (&w)[8]) {
#pragma unroll
  for (int c = 0; c < 4; ++c)
    v[c] = __longlong_as_double(
        static_cast<long long>((w[2 * c + 1] << 32) | (w[2 * c] & 0xffffffffull)));
}

PCOT_DEV void ld4(double (&v)[4], const double* p) {  // 32-B aligned
  const double2 a = *reinterpret_cast<const double2*>(p);
  const double2 b = *reinterpret_cast<const double2*>(p + 2);
  v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
}
PCOT_DEV void st4(double* p, const double (&v)[4]) {
  *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
  *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
}
// New values of 4 adjacent cells from the old rows (up, mid, dn); eW / eE are
// the cross-warp neighbours (used by lanes 0 / 31); columns outside cmask keep.
PCOT_DEV void upd4(double (&nv)[4], const double (&mid)[4], const double (&up)[4],
                   const double (&dn)[4], double eW, double eE, int lane, unsigned cmask) {
#ifdef PCOT_RES_NOSHFL  // timing probe: wrong results
  double W = mid[3], E = mid[0];
#else
  double W = __shfl_up_sync(0xffffffffu, mid[3], 1);
  double E = __shfl_down_sync(0xffffffffu, mid[0], 1);
#endif
  if (lane == 0) W = eW;
  if (lane == 31) E = eE;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double left = c > 0 ? mid[c > 0 ? c - 1 : 0] : W;
    const double right = c < 3 ? mid[c < 3 ? c + 1 : 0] : E;
    double s = add(mid[c], up[c]);
    s = add(s, dn[c]);
    s = add(s, left);
    s = add(s, right);
    nv[c] = mul(0.2, s);
  }
  if (cmask != 0xFu) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (!((cmask >> c) & 1u)) nv[c] = mid[c];
  }
}

#ifndef PCOT_RES_PF
#define PCOT_RES_PF 2  // rows ahead of use the sweep loads its own columns
#endif
constexpr int kResRows = 14;  // most rows per band (one instantiation per band height)

PCOT_DEV void lds4(double (&v)[4], uint32_t addr) {  // halves at addr and addr + 512
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(addr) : "memory");
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2+512];" : "=d"(v[2]), "=d"(v[3]) : "r"(addr) : "memory");
}
PCOT_DEV void sts4(uint32_t addr, const double (&v)[4]) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(v[0]), "d"(v[1]) : "memory");
  asm volatile("st.shared.v2.f64 [%0+512], {%1, %2};" ::"r"(addr), "d"(v[2]), "d"(v[3]) : "memory");
}
PCOT_DEV double lds1_if(uint32_t addr, bool p) {  // predicated load, 0.0 otherwise (no select after it)
  double v = 0.0;
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.shared.f64 %0, [%1];\n}\n"
               : "+d"(v)
               : "r"(addr), "r"(uint32_t(p))
               : "memory");
  return v;
}

// The whole run of one band of R rows (R is a template parameter so that the
// row loops unroll with static register names: no rotation moves, no guards).
template <int R>
PCOT_DEV void res_run(const ResArgs& a, int g0) {
  extern __shared__ __align__(16) double sm[];  // R rows x npad
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NT = a.npad >> 2;
  const int b = blockIdx.x;
  const bool has_up = b > 0, has_dn = b + 1 < a.nbands;
  const int c0 = tid * 4;
  const uint32_t rs = uint32_t(a.npad) * 8;  // row pitch in bytes
  // shared-memory home of this thread's columns: {c0, c0+1} at sp, {c0+2, c0+3} 512 B on
  const uint32_t sp = smem_u32(sm) + uint32_t(warp * 128 + lane * 2) * 8;
  unsigned cmask = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (c0 + c >= 1 && c0 + c <= a.n - 2) cmask |= 1u << c;
  auto gload = [&](double (&v)[4], int64_t grow) {  // input slab row, zero beyond column n-1
    const double* p = a.in + grow * a.ld_in + c0;
    if (c0 + 3 < a.n) {
      ld4(v, p);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = c0 + c < a.n ? p[c] : 0.0;
    }
  };
  double top[4] = {0, 0, 0, 0}, bot[4] = {0, 0, 0, 0};
  {
    double v[4];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      gload(v, g0 + r);
      sts4(sp + r * rs, v);
    }
    if (has_up) gload(top, g0 - 1);
    if (has_dn) gload(bot, g0 + R);
  }

  // exchange lines: slot (parity, band, first=0 / last=1), 2 * npad words each
  const size_t xrow = size_t(2) * a.npad;
  unsigned long long* const xmine = a.xbuf + size_t(b) * 2 * xrow + 2 * c0;
  const unsigned long long* const xup = a.xbuf + (size_t(b - 1) * 2 + 1) * xrow + 2 * c0;
  const unsigned long long* const xdn = a.xbuf + (size_t(b + 1) * 2) * xrow + 2 * c0;
  const size_t xpar = size_t(a.nbands) * 2 * xrow;  // parity stride
  unsigned long long wtop[8], wbot[8];
  // foreign edge column: lane 0 reads column c0-1 (the previous warp's lane 31,
  // its column 3), lane 31 column c0+4 (the next warp's lane 0, its column 0)
  const bool edgeW = lane == 0 && tid > 0, edgeE = lane == 31 && tid < NT - 1;
  const bool edge = edgeW || edgeE;
  const uint32_t epos =
      smem_u32(sm) + uint32_t(edgeW ? (warp - 1) * 128 + 64 + 31 * 2 + 1 : (edgeE ? (warp + 1) * 128 : 0)) * 8;
  const bool keep_first = g0 == 0, keep_last = g0 + R == a.n;
  constexpr int RW = R >= 4 ? R / 2 : 0;  // sweep row after which the neighbours' rows are requested
  for (int t = 1; t <= a.T; ++t) {
    __syncthreads();  // the previous step's rows are written
    double ecol[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
#ifdef PCOT_RES_NOEDGE  // timing probe: wrong results
      ecol[r] = 0.0;
#else
      ecol[r] = lds1_if(epos + r * rs, edge);
#endif
    }
    if (t > 1) {  // the neighbours' rows of step t-1, requested during the last sweep
      const unsigned tag = a.epoch + unsigned(t - 1);
      const size_t par = ((t - 1) & 1) ? xpar : 0;
      int spins = 0;
      if (has_up) {
        while (!xvalid(wtop, tag) && !a.nosync) {
          if (++spins > kSpinCapR || ((spins & 255) == 0 && ld_relaxed(a.err) != 0)) {
            atomicExch(a.err, 1);
            break;
          }
          xload(wtop, xup + par);
        }
        xvalue(top, wtop);
      }
      if (has_dn) {
        while (!xvalid(wbot, tag) && !a.nosync) {
          if (++spins > kSpinCapR || ((spins & 255) == 0 && ld_relaxed(a.err) != 0)) {
            atomicExch(a.err, 1);
            break;
          }
          xload(wbot, xdn + par);
        }
        xvalue(bot, wbot);
      }
    }
    const unsigned tag = a.epoch + unsigned(t);
    const size_t par = (t & 1) ? xpar : 0;
    // ---- the band's last row first (kept in registers until the sweep is over)
    double lastnew[4];
    {
      double rl[4], rl1[4];
      lds4(rl, sp + (R - 1) * rs);
      lds4(rl1, sp + (R - 2) * rs);
      upd4(lastnew, rl, rl1, bot, ecol[R - 1], ecol[R - 1], lane, keep_last ? 0u : cmask);
#if !defined(PCOT_RES_NOX) && !defined(PCOT_RES_NOPUT)
      if (has_dn) xput(xmine + par + xrow, lastnew, tag);
#endif
    }
    double rows[R][4];  // old rows, own columns; static indices, live for three iterations each
    lds4(rows[0], sp);
    if (PCOT_RES_PF == 2) lds4(rows[1], sp + rs);
    __syncthreads();  // every foreign edge column is in registers: rows may be overwritten
    // ---- rows 0 .. R-2, top to bottom, in place
#pragma unroll
    for (int r = 0; r < R - 1; ++r) {
      double nv[4];
      if (r + PCOT_RES_PF < R) lds4(rows[r + PCOT_RES_PF], sp + (r + PCOT_RES_PF) * rs);
      if (r == 0)
        upd4(nv, rows[0], top, rows[1], ecol[0], ecol[0], lane, keep_first ? 0u : cmask);
      else
        upd4(nv, rows[r], rows[r - 1], rows[r + 1], ecol[r], ecol[r], lane, cmask);
#if !defined(PCOT_RES_NOX) && !defined(PCOT_RES_NOPUT)
      if (r == 0 && has_up) xput(xmine + par, nv, tag);
#endif
      sts4(sp + r * rs, nv);
#if defined(PCOT_RES_NOX) || defined(PCOT_RES_NOLOAD)  // timing probe: wrong results
      if (false) {
#else
      if (r == RW && t < a.T) {
#endif  // the neighbours' rows of step t, for step t+1
        if (has_up) xload(wtop, xup + par);
        if (has_dn) xload(wbot, xdn + par);
      }
    }
    sts4(sp + (R - 1) * rs, lastnew);
  }
  __syncthreads();
  // ---- the band back to the output slab
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double v[4];
    lds4(v, sp + r * rs);
    double* p = a.out + int64_t(g0 + r) * a.ld_out + c0;
    if (c0 + 3 < a.n) {
      st4(p, v);
    } else {
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c0 + c < a.n) p[c] = v[c];
    }
  }
}

__global__ void __launch_bounds__(512, 1) s2d5_res_kernel(ResArgs a) {
  const int b = blockIdx.x;
  const int g0 = int(int64_t(b) * a.n / a.nbands), g1 = int(int64_t(b + 1) * a.n / a.nbands);
  switch (g1 - g0) {
    case 2: res_run<2>(a, g0); break;
    case 3: res_run<3>(a, g0); break;
    case 4: res_run<4>(a, g0); break;
    case 5: res_run<5>(a, g0); break;
    case 6: res_run<6>(a, g0); break;
    case 7: res_run<7>(a, g0); break;
    case 8: res_run<8>(a, g0); break;
    case 9: res_run<9>(a, g0); break;
    case 10: res_run<10>(a, g0); break;
    case 11: res_run<11>(a, g0); break;
    case 12: res_run<12>(a, g0); break;
    case 13: res_run<13>(a, g0); break;
    case 14: res_run<14>(a, g0); break;
    default: break;  // the plan never creates other heights
  }
}

}  // namespace

// The resident kernel applies when every band (>= 2 rows, one per SM) fits in
// shared memory and the launch can be cooperative.
S2ResPlan* s2d5_res_create(int64_t n, int device) {
  if (n < 64 || n > 2048) return nullptr;
  if (cudaSetDevice(device) != cudaSuccess) return nullptr;
  int sms = 0, coop = 0, smem_max = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess ||
      cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device) != cudaSuccess ||
      cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess ||
      !coop)
    return nullptr;
  S2ResPlan p;
  p.device = device;
  p.n = int(n);
  p.npad = int((n + 127) / 128 * 128);
  p.nt = p.npad / 4;
  p.nbands = int(std::min<int64_t>(sms, n / 2));
  p.rmax = int((n + p.nbands - 1) / p.nbands);
  p.smem = size_t(p.rmax) * p.npad * 8;
  if (p.rmax > kResRows || p.smem > size_t(smem_max)) return nullptr;
  int slots = 0;
  if (kernel_slots(reinterpret_cast<const void*>(s2d5_res_kernel), p.nt, p.smem, &slots) != cudaSuccess ||
      slots < p.nbands)
    return nullptr;
  const size_t xbytes = size_t(2) * p.nbands * 2 * 2 * p.npad * 8;
  if (cudaMalloc(&p.xbuf, xbytes) != cudaSuccess) return nullptr;
  if (cudaMalloc(&p.d_err, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&p.h_err, sizeof(int)) != cudaSuccess ||
      cudaMemset(p.xbuf, 0, xbytes) != cudaSuccess || cudaMemset(p.d_err, 0, sizeof(int)) != cudaSuccess) {
    cudaFree(p.xbuf);
    cudaFree(p.d_err);
    return nullptr;
  }
  *p.h_err = 0;
  p.epoch = 1;  // tag 0 is the cleared buffer
  return new S2ResPlan(p);
}

void s2d5_res_destroy(S2ResPlan* p) {
  if (!p) return;
  cudaFree(p->xbuf);
  cudaFree(p->d_err);
  if (p->h_err) cudaFreeHost(p->h_err);
  delete p;
}

cudaError_t s2d5_res_run(S2ResPlan* p, const Slab2D& in, const Slab2D& out, int64_t T,
                         cudaStream_t stream) {
  if (!p || T < 1 || in.cols != p->n || in.rows != p->n) return cudaErrorInvalidValue;
  cudaError_t e;
  if ((e = kernel_slots(reinterpret_cast<const void*>(s2d5_res_kernel), p->nt, p->smem, nullptr)) !=
      cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(p->d_err, 0, sizeof(int), stream)) != cudaSuccess) return e;
  ResArgs a;
  a.in = in.origin;
  a.out = out.origin;
  a.ld_in = in.ld;
  a.ld_out = out.ld;
  a.n = p->n;
  a.T = int(T);
  a.npad = p->npad;
  a.nbands = p->nbands;
  a.rwait = 0;
  a.nosync = env_int("PCOTGPU_RES_NOSYNC", 0);  // timing experiments only: wrong results
  a.epoch = p->epoch;
  p->epoch += unsigned(T) + 1;  // tags never repeat across runs (mod 2^32)
  a.xbuf = p->xbuf;
  a.err = p->d_err;
  void* args[] = {&a};
  e = cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(s2d5_res_kernel), dim3(p->nbands),
                                  dim3(p->nt), args, p->smem, stream);
  count_launch();
  if (e != cudaSuccess) return e;
  return cudaMemcpyAsync(p->h_err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, stream);
}

int s2d5_res_fault(S2ResPlan* p) {
  if (!p) return 0;
  const int f = *p->h_err;
  *p->h_err = 0;
  return f;
}

}  // namespace pcotgpu
