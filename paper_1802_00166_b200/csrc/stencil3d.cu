// 3-D 7-point temporally blocked 2.5-D streaming stencil for sm_100a.
//
// Replaces exec_stmt over the heat3d kernels (reference core/src/exec.cpp:
// 347-428; kernels/heat3d.kernel:34 and this repo's kernels/heat3d_b.kernel).
//
// Tile = a (j,k) plane window of KW x JW input cells streamed along i:
//   * lane -> C consecutive k columns, warp -> RJ consecutive j rows;
//   * input planes arrive through a PF-deep shared-memory ring (one TMA bulk
//     copy per j row, issued by warp 0, mbarrier complete_tx);
//   * level L keeps planes rho-1, rho, rho+1 (slot = plane mod 3) in
//     registers; k-neighbours come by warp shuffle, j-neighbours inside the
//     thread or, at warp edges, through a double-buffered shared-memory row
//     exchange (one __syncthreads per input plane).
// The (j,k) window shrinks by one cell per level: output KW-2BT x JW-2BT.
// Per-point order = the kernel body's parse tree (neighbours (i-1),(i+1),
// (j-1),(j+1),(k-1),(k+1)); explicit _rn intrinsics, no FMA.
#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

namespace {

constexpr int kC3 = 2;               // k columns per thread
constexpr int kRJ = 4;               // j rows per thread
constexpr int kNW3 = 8;              // warps per CTA
constexpr int kNT3 = kNW3 * 32;
constexpr int kKW = 32 * kC3;        // 64 input k columns
constexpr int kJW = kNW3 * kRJ;      // 32 input j rows
constexpr int kKL = kKW + 2;         // loaded row length (alignment slack)
constexpr int kPF3 = 4;              // planes in flight

struct S3Args {
  const double* in;
  double* out;
  int64_t n;
  int64_t pj_in, pi_in, pj_out, pi_out;
  int64_t halo;
  int kout, jout;
  int nk, nj, nchunks, H;
  int order;
};

template <int BT>
struct Regs3 {
  double v[BT][3][kRJ][kC3];
};

template <int RULE>
PCOT_DEV double update7(double c, double im, double ip, double jm, double jp, double km,
                        double kp) {
  if (RULE == 0) {  // heat3d_b: c + 0.125 * ((((((im+ip)+jm)+jp)+km)+kp) - 6.0*c)
    double s = add(im, ip);
    s = add(s, jm);
    s = add(s, jp);
    s = add(s, km);
    s = add(s, kp);
    s = sub(s, mul(6.0, c));
    return add(c, mul(0.125, s));
  } else {  // heat3d: 0.1 * ((((((c+im)+ip)+jm)+jp)+km)+kp)
    double s = add(c, im);
    s = add(s, ip);
    s = add(s, jm);
    s = add(s, jp);
    s = add(s, km);
    s = add(s, kp);
    return mul(0.1, s);
  }
}

template <int BT, int RULE, bool MASK, bool HOLD, int P>
PCOT_DEV void s3_iter(Regs3<BT>& R, const double* __restrict__ plane, int shift, int64_t k,
                      int par, double* __restrict__ edge, int warp, int lane, const S3Args& a,
                      int64_t jb, int64_t kb, int64_t i0, int64_t i1, int64_t j0, int64_t jend,
                      int64_t k0, int64_t kend) {
  // edge layout: [par][warp][top/bottom][L][lane][C]
  constexpr int EW = 2 * BT * 32 * kC3;  // doubles per warp
  {
    constexpr int s = P % 3;
#pragma unroll
    for (int r = 0; r < kRJ; ++r)
#pragma unroll
      for (int c = 0; c < kC3; ++c)
        R.v[0][s][r][c] = plane[(warp * kRJ + r) * kKL + shift + lane * kC3 + c];
  }
  const double* eprev = edge + (par ^ 1) * (kNW3 * EW);
#pragma unroll
  for (int L = 0; L < BT; ++L) {
    const int rel = P - L - 1;
    const int sm = ((rel % 3) + 3) % 3;
    const int st = (((rel - 1) % 3) + 3) % 3;
    const int sb = (((rel + 1) % 3) + 3) % 3;
    const int64_t rho = k - L - 1;
    // j-neighbours beyond this warp's rows
    double up[kC3], dn[kC3];
#pragma unroll
    for (int c = 0; c < kC3; ++c) {
      up[c] = R.v[L][sm][0][c];
      dn[c] = R.v[L][sm][kRJ - 1][c];
    }
    if (warp > 0) {
#pragma unroll
      for (int c = 0; c < kC3; ++c)
        up[c] = eprev[(warp - 1) * EW + ((1 * BT + L) * 32 + lane) * kC3 + c];
    }
    if (warp + 1 < kNW3) {
#pragma unroll
      for (int c = 0; c < kC3; ++c)
        dn[c] = eprev[(warp + 1) * EW + ((0 * BT + L) * 32 + lane) * kC3 + c];
    }
    double nv[kRJ][kC3];
#pragma unroll
    for (int r = 0; r < kRJ; ++r) {
      const double* mid = R.v[L][sm][r];
      double W = __shfl_up_sync(0xffffffffu, mid[kC3 - 1], 1);
      double E = __shfl_down_sync(0xffffffffu, mid[0], 1);
#pragma unroll
      for (int c = 0; c < kC3; ++c) {
        const double jm = r > 0 ? R.v[L][sm][r > 0 ? r - 1 : 0][c] : up[c];
        const double jp = r < kRJ - 1 ? R.v[L][sm][r < kRJ - 1 ? r + 1 : 0][c] : dn[c];
        const double km = c > 0 ? mid[c > 0 ? c - 1 : 0] : W;
        const double kp = c < kC3 - 1 ? mid[c < kC3 - 1 ? c + 1 : 0] : E;
        nv[r][c] = update7<RULE>(mid[c], R.v[L][st][r][c], R.v[L][sb][r][c], jm, jp, km, kp);
      }
    }
    if (MASK) {
      const bool iin = rho >= 1 && rho <= a.n - 2;
#pragma unroll
      for (int r = 0; r < kRJ; ++r) {
        const int64_t j = jb + r;
        const bool jin = iin && j >= 1 && j <= a.n - 2;
#pragma unroll
        for (int c = 0; c < kC3; ++c) {
          const int64_t kk = kb + c;
          if (!(jin && kk >= 1 && kk <= a.n - 2)) nv[r][c] = HOLD ? R.v[L][sm][r][c] : 0.0;
        }
      }
    }
    if (L + 1 < BT) {
#pragma unroll
      for (int r = 0; r < kRJ; ++r)
#pragma unroll
        for (int c = 0; c < kC3; ++c) R.v[L + 1 < BT ? L + 1 : 0][sm][r][c] = nv[r][c];
    } else if (rho >= i0 && rho < i1) {
#pragma unroll
      for (int r = 0; r < kRJ; ++r) {
        const int64_t j = jb + r;
        if (j < j0 || j >= jend) continue;
        double* dst = a.out + rho * a.pi_out + j * a.pj_out;
#pragma unroll
        for (int c = 0; c < kC3; ++c) {
          const int64_t kk = kb + c;
          if (kk >= k0 && kk < kend) __stcs(dst + kk, nv[r][c]);
        }
      }
    }
  }
  // publish top/bottom rows of the newest plane (k-L) of every level
  double* ecur = edge + par * (kNW3 * EW);
#pragma unroll
  for (int L = 0; L < BT; ++L) {
    const int s = (((P - L) % 3) + 3) % 3;
#pragma unroll
    for (int c = 0; c < kC3; ++c) {
      ecur[warp * EW + ((0 * BT + L) * 32 + lane) * kC3 + c] = R.v[L][s][0][c];
      ecur[warp * EW + ((1 * BT + L) * 32 + lane) * kC3 + c] = R.v[L][s][kRJ - 1][c];
    }
  }
}

template <int BT, int RULE, bool MASK, bool HOLD>
PCOT_DEV void s3_tile(const S3Args& a, int tk, int tj, int chunk, double* ring, uint64_t* bars,
                      double* edge) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t k0 = int64_t(tk) * a.kout, j0 = int64_t(tj) * a.jout;
  const int64_t kend = k0 + a.kout < a.n ? k0 + a.kout : a.n;
  const int64_t jend = j0 + a.jout < a.n ? j0 + a.jout : a.n;
  const int64_t i0 = int64_t(chunk) * a.H;
  const int64_t i1 = i0 + a.H < a.n ? i0 + a.H : a.n;
  const int64_t kstart = i0 - BT;
  const int64_t niter = ((i1 + BT - kstart) + 2) / 3 * 3;
  const int64_t kfirst = k0 - BT, jfirst = j0 - BT;
  const int64_t cs = kfirst >= 0 ? (kfirst & ~int64_t(1)) : -((-kfirst + 1) & ~int64_t(1));
  const int shift = int(kfirst - cs);
  const int64_t kb = kfirst + lane * kC3;
  const int64_t jb = jfirst + warp * kRJ;
  const int64_t lo = -a.halo, hi = a.n + a.halo - 1;

  auto issue = [&](int64_t it) {  // warp 0, all lanes
    int64_t pl = kstart + it;
    pl = pl < lo ? lo : (pl > hi ? hi : pl);
    const int slot = int(it % kPF3);
    if (lane == 0) mbar_arrive_expect_tx(&bars[slot], kJW * kKL * 8);
    __syncwarp();
    int64_t jr = jfirst + lane;
    jr = jr < lo ? lo : (jr > hi ? hi : jr);
    bulk_g2s(ring + (slot * kJW + lane) * kKL, a.in + pl * a.pi_in + jr * a.pj_in + cs, kKL * 8,
             &bars[slot]);
  };
  if (warp == 0) {
    for (int it = 0; it < kPF3 && it < niter; ++it) issue(it);
  }
  Regs3<BT> R;
#pragma unroll
  for (int L = 0; L < BT; ++L)
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
      for (int r = 0; r < kRJ; ++r)
#pragma unroll
        for (int c = 0; c < kC3; ++c) R.v[L][s][r][c] = 0.0;

  for (int64_t it = 0; it < niter; it += 3) {
#define PCOT_S3_STEP(P)                                                                        \
  {                                                                                            \
    const int64_t itp = it + P;                                                                \
    const int slot = int(itp % kPF3);                                                          \
    mbar_wait(&bars[slot], uint32_t((itp / kPF3) & 1));                                        \
    s3_iter<BT, RULE, MASK, HOLD, P>(R, ring + slot * kJW * kKL, shift, kstart + itp,          \
                                     int(itp & 1), edge, warp, lane, a, jb, kb, i0, i1, j0,    \
                                     jend, k0, kend);                                          \
    __syncthreads();                                                                           \
    if (warp == 0 && itp + kPF3 < niter) issue(itp + kPF3);                                    \
  }
    PCOT_S3_STEP(0)
    PCOT_S3_STEP(1)
    PCOT_S3_STEP(2)
#undef PCOT_S3_STEP
  }
}

template <int BT, int RULE, bool HOLD>
__global__ void __launch_bounds__(kNT3, 1) s3d7_kernel(S3Args a) {
  extern __shared__ __align__(128) double smem3[];
  double* ring = smem3;
  double* edge = ring + kPF3 * kJW * kKL;
  uint64_t* bars = reinterpret_cast<uint64_t*>(edge + 2 * kNW3 * 2 * BT * 32 * kC3);
  const int ntile = a.nk * a.nj;
  int tile = blockIdx.x % ntile, chunk = blockIdx.x / ntile;
  int tk, tj;
  if (a.order == kOrderLex) {
    tj = tile / a.nk;
    tk = tile - tj * a.nk;
  } else {  // Morton over (tk, tj)
    int side = 1;
    while (side < a.nk || side < a.nj) side <<= 1;
    int x = 0, y = 0, id = blockIdx.x % (side * side);
    chunk = blockIdx.x / (side * side);
    for (int b = 0; b < 12; ++b) {
      x |= ((id >> (2 * b)) & 1) << b;
      y |= ((id >> (2 * b + 1)) & 1) << b;
    }
    tk = x;
    tj = y;
    if (tk >= a.nk || tj >= a.nj) return;
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPF3; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t k0 = int64_t(tk) * a.kout, j0 = int64_t(tj) * a.jout;
  const int64_t i0 = int64_t(chunk) * a.H;
  const int64_t i1 = i0 + a.H < a.n ? i0 + a.H : a.n;
  const bool edge_tile = (k0 - BT <= 0) || (k0 + a.kout + BT >= a.n - 1) || (j0 - BT <= 0) ||
                         (j0 + a.jout + BT >= a.n - 1) || (i0 - BT <= 0) ||
                         (i1 + BT >= a.n - 1);
  if (edge_tile)
    s3_tile<BT, RULE, true, HOLD>(a, tk, tj, chunk, ring, bars, edge);
  else
    s3_tile<BT, RULE, false, HOLD>(a, tk, tj, chunk, ring, bars, edge);
}

template <int BT, int RULE, bool HOLD>
cudaError_t launch3(const S3Args& a, cudaStream_t stream) {
  const size_t smem = size_t(kPF3) * kJW * kKL * 8 + size_t(2) * kNW3 * 2 * BT * 32 * kC3 * 8 +
                      kPF3 * 8;
  auto fn = s3d7_kernel<BT, RULE, HOLD>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  int grid;
  if (a.order == kOrderLex) {
    grid = a.nk * a.nj * a.nchunks;
  } else {
    int side = 1;
    while (side < a.nk || side < a.nj) side <<= 1;
    grid = side * side * a.nchunks;
  }
  fn<<<grid, kNT3, smem, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int BT>
cudaError_t launch3_bt(const S3Args& a, int rule, int hold, cudaStream_t s) {
  if (rule == 0)
    return hold ? launch3<BT, 0, true>(a, s) : launch3<BT, 0, false>(a, s);
  return hold ? launch3<BT, 1, true>(a, s) : launch3<BT, 1, false>(a, s);
}

}  // namespace

int s3d7_max_bt() { return 4; }

cudaError_t s3d7_advance(const Grid3D& in, const Grid3D& out, int bt, int rule, int ring_hold,
                         int order, cudaStream_t stream) {
  if (bt < 1 || bt > 4) return cudaErrorInvalidValue;
  if (in.halo < bt + 3 || (in.pitch_j & 1) || (in.pitch_i & 1) ||
      (reinterpret_cast<uintptr_t>(in.origin) & 15))
    return cudaErrorInvalidValue;
  S3Args a;
  a.in = in.origin;
  a.out = out.origin;
  a.n = in.n;
  a.pj_in = in.pitch_j;
  a.pi_in = in.pitch_i;
  a.pj_out = out.pitch_j;
  a.pi_out = out.pitch_i;
  a.halo = in.halo;
  a.kout = kKW - 2 * bt;
  a.jout = kJW - 2 * bt;
  a.nk = int((a.n + a.kout - 1) / a.kout);
  a.nj = int((a.n + a.jout - 1) / a.jout);
  const int64_t tiles = int64_t(a.nk) * a.nj;
  int64_t want = (2 * 148 * 2 + tiles - 1) / tiles;  // ~2 waves of 2 CTAs/SM
  int64_t H = (a.n + want - 1) / want;
  if (H < 8 * bt) H = 8 * bt;
  if (H > a.n) H = a.n;
  a.H = int(H);
  a.nchunks = int((a.n + H - 1) / H);
  a.order = order;
  switch (bt) {
    case 1: return launch3_bt<1>(a, rule, ring_hold, stream);
    case 2: return launch3_bt<2>(a, rule, ring_hold, stream);
    case 3: return launch3_bt<3>(a, rule, ring_hold, stream);
    default: return launch3_bt<4>(a, rule, ring_hold, stream);
  }
}

}  // namespace pcotgpu
