// 3-D 7-point temporally blocked 2.5-D streaming stencil for sm_100a.
//
// Replaces exec_stmt over the heat3d kernels (reference core/src/exec.cpp:
// 347-428; kernels/heat3d.kernel:34 and this repo's kernels/heat3d_b.kernel).
//
// Tile = a (j,k) plane window of KW x JW input cells streamed along i:
//   * lane -> C consecutive k columns, warp -> RJ consecutive j rows; a warp
//     spans the whole window width, so k-neighbours come by warp shuffle with
//     no cross-warp traffic (lanes 0/31 read the shrinking halo);
//   * input planes arrive through a PF-deep shared-memory ring (one TMA bulk
//     copy per j row, issued by warp 0, mbarrier complete_tx);
//   * level L keeps planes rho-1, rho, rho+1 (slot = plane mod 3) in
//     registers; j-neighbours inside the thread or, at warp edges, through a
//     double-buffered shared-memory row exchange (one __syncthreads per plane).
// The (j,k) window shrinks by one cell per level: output KW-2BT x JW-2BT.
// Ring handling: tiles whose window stays inside the interior in (j,k) run
// the unmasked body; planes at i = 0 / N-1 (or outside) are handled by a
// warp-uniform branch; only (j,k)-edge tiles pay per-element selects.
// Per-point order = the kernel body's parse tree (neighbours (i-1),(i+1),
// (j-1),(j+1),(k-1),(k+1)); explicit _rn intrinsics, no FMA.
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

namespace {

template <int C_, int RJ_, int NW_, int MINB_, int PF_>
struct Geo {
  static constexpr int C = C_, RJ = RJ_, NW = NW_, MINB = MINB_, PF = PF_;
  static constexpr int NT = NW * 32;
  static constexpr int KW = 32 * C;   // input k columns
  static constexpr int JW = NW * RJ;  // input j rows
  static constexpr int KL = KW + 2;   // loaded row length (alignment slack)
};

struct S3Args {
  const double* in;
  double* out;
  int n;
  int64_t pj_in, pi_in, pj_out, pi_out;
  int halo;
  int kout, jout;
  int nk, nj, nchunks, H;
  int order;
};

__host__ __device__ constexpr int m3(int v) { return ((v % 3) + 3) % 3; }

template <int BT, class G>
struct Regs3 {
  double v[BT][3][G::RJ][G::C];
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

// edge layout per parity: [warp][top=0/bottom=1][L][lane][C]
template <int BT, class G>
struct Edge3 {
  static constexpr int EW = 2 * BT * 32 * G::C;  // doubles per warp
  static constexpr int kPerPar = G::NW * EW;
};

template <int BT, int RULE, bool MASKJK, bool HOLD, class G, int P>
PCOT_DEV void s3_iter(Regs3<BT, G>& R, const double* __restrict__ plane, int shift, int k, int par,
                      double* __restrict__ edge, int warp, int lane, const S3Args& a, int jb,
                      int kb, unsigned jkmask, int i0, int i1, int j0, int jend, int k0, int kend) {
  constexpr int C = G::C, RJ = G::RJ, NW = G::NW;
  constexpr int EW = Edge3<BT, G>::EW;
  {
    constexpr int s = m3(P);
#pragma unroll
    for (int r = 0; r < RJ; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c)
        R.v[0][s][r][c] = plane[(warp * RJ + r) * G::KL + shift + lane * C + c];
  }
  const double* eprev = edge + (par ^ 1) * Edge3<BT, G>::kPerPar;
#pragma unroll
  for (int L = 0; L < BT; ++L) {
    const int sm = m3(P - L - 1), st = m3(P - L - 2), sb = m3(P - L);
    const int rho = k - L - 1;
    double up[C], dn[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      up[c] = warp > 0 ? eprev[(warp - 1) * EW + ((1 * BT + L) * 32 + lane) * C + c]
                       : R.v[L][sm][0][c];
      dn[c] = warp + 1 < NW ? eprev[(warp + 1) * EW + ((0 * BT + L) * 32 + lane) * C + c]
                            : R.v[L][sm][RJ - 1][c];
    }
    double nv[RJ][C];
#pragma unroll
    for (int r = 0; r < RJ; ++r) {
      const double* mid = R.v[L][sm][r];
      const double W = __shfl_up_sync(0xffffffffu, mid[C - 1], 1);
      const double E = __shfl_down_sync(0xffffffffu, mid[0], 1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double jm = r > 0 ? R.v[L][sm][r > 0 ? r - 1 : 0][c] : up[c];
        const double jp = r < RJ - 1 ? R.v[L][sm][r < RJ - 1 ? r + 1 : 0][c] : dn[c];
        const double km = c > 0 ? mid[c > 0 ? c - 1 : 0] : W;
        const double kp = c < C - 1 ? mid[c < C - 1 ? c + 1 : 0] : E;
        nv[r][c] = update7<RULE>(mid[c], R.v[L][st][r][c], R.v[L][sb][r][c], jm, jp, km, kp);
      }
    }
    if (MASKJK) {
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (!((jkmask >> (r * C + c)) & 1u)) nv[r][c] = HOLD ? R.v[L][sm][r][c] : 0.0;
    }
    if (rho < 1 || rho > a.n - 2) {  // ring / outside plane: warp-uniform
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) nv[r][c] = HOLD ? R.v[L][sm][r][c] : 0.0;
    }
    if (L + 1 < BT) {
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) R.v[L + 1 < BT ? L + 1 : 0][sm][r][c] = nv[r][c];
    } else if (rho >= i0 && rho < i1) {
#pragma unroll
      for (int r = 0; r < RJ; ++r) {
        const int j = jb + r;
        if (j < j0 || j >= jend) continue;
        double* dst = a.out + int64_t(rho) * a.pi_out + int64_t(j) * a.pj_out;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const int kk = kb + c;
          if (kk >= k0 && kk < kend) __stcs(dst + kk, nv[r][c]);
        }
      }
    }
  }
  // publish top/bottom rows of the newest plane (k-L) of every level
  double* ecur = edge + par * Edge3<BT, G>::kPerPar;
#pragma unroll
  for (int L = 0; L < BT; ++L) {
    const int s = m3(P - L);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      ecur[warp * EW + ((0 * BT + L) * 32 + lane) * C + c] = R.v[L][s][0][c];
      ecur[warp * EW + ((1 * BT + L) * 32 + lane) * C + c] = R.v[L][s][RJ - 1][c];
    }
  }
}

template <int BT, int RULE, bool MASKJK, bool HOLD, class G>
PCOT_DEV void s3_tile(const S3Args& a, int tk, int tj, int chunk, double* ring, uint64_t* bars,
                      double* edge) {
  constexpr int C = G::C, RJ = G::RJ, JW = G::JW, KL = G::KL, PF = G::PF;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int k0 = tk * a.kout, j0 = tj * a.jout;
  const int kend = k0 + a.kout < a.n ? k0 + a.kout : a.n;
  const int jend = j0 + a.jout < a.n ? j0 + a.jout : a.n;
  const int i0 = chunk * a.H;
  const int i1 = i0 + a.H < a.n ? i0 + a.H : a.n;
  const int kstart = i0 - BT;
  const int niter = ((i1 + BT - kstart) + 2) / 3 * 3;
  const int kfirst = k0 - BT, jfirst = j0 - BT;
  const int cs = kfirst >= 0 ? (kfirst & ~1) : -((-kfirst + 1) & ~1);
  const int shift = kfirst - cs;
  const int kb = kfirst + lane * C;
  const int jb = jfirst + warp * RJ;
  const int lo = -a.halo, hi = a.n + a.halo - 1;
  unsigned jkmask = 0;  // interior (j,k) cells of this thread's patch
#pragma unroll
  for (int r = 0; r < RJ; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int j = jb + r, kk = kb + c;
      if (j >= 1 && j <= a.n - 2 && kk >= 1 && kk <= a.n - 2) jkmask |= 1u << (r * C + c);
    }

  auto issue = [&](int it) {  // warp 0, all lanes
    int pl = kstart + it;
    pl = pl < lo ? lo : (pl > hi ? hi : pl);
    const int slot = it % PF;
    if (lane == 0) mbar_arrive_expect_tx(&bars[slot], JW * KL * 8);
    __syncwarp();
    for (int row = lane; row < JW; row += 32) {
      int jr = jfirst + row;
      jr = jr < lo ? lo : (jr > hi ? hi : jr);
      bulk_g2s(ring + (slot * JW + row) * KL,
               a.in + int64_t(pl) * a.pi_in + int64_t(jr) * a.pj_in + cs, KL * 8, &bars[slot]);
    }
  };
  if (warp == 0) {
    for (int it = 0; it < PF && it < niter; ++it) issue(it);
  }
  Regs3<BT, G> R;
#pragma unroll
  for (int L = 0; L < BT; ++L)
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) R.v[L][s][r][c] = 0.0;

  for (int it = 0; it < niter; it += 3) {
#define PCOT_S3_STEP(P)                                                                     \
  {                                                                                         \
    const int itp = it + P;                                                                 \
    const int slot = itp % PF;                                                              \
    mbar_wait(&bars[slot], uint32_t((itp / PF) & 1));                                       \
    s3_iter<BT, RULE, MASKJK, HOLD, G, P>(R, ring + slot * JW * KL, shift, kstart + itp,     \
                                          itp & 1, edge, warp, lane, a, jb, kb, jkmask, i0,  \
                                          i1, j0, jend, k0, kend);                           \
    __syncthreads();                                                                        \
    if (warp == 0 && itp + PF < niter) issue(itp + PF);                                     \
  }
    PCOT_S3_STEP(0)
    PCOT_S3_STEP(1)
    PCOT_S3_STEP(2)
#undef PCOT_S3_STEP
  }
}

template <int BT, int RULE, bool HOLD, class G>
__global__ void __launch_bounds__(G::NT, G::MINB) s3d7_kernel(S3Args a) {
  extern __shared__ __align__(128) double smem3[];
  double* ring = smem3;
  double* edge = ring + G::PF * G::JW * G::KL;
  uint64_t* bars = reinterpret_cast<uint64_t*>(edge + 2 * Edge3<BT, G>::kPerPar);
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
    for (int i = 0; i < G::PF; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int k0 = tk * a.kout, j0 = tj * a.jout;
  const bool edge_jk = (k0 - BT <= 0) || (k0 + a.kout + BT >= a.n - 1) || (j0 - BT <= 0) ||
                       (j0 + a.jout + BT >= a.n - 1);
  if (edge_jk)
    s3_tile<BT, RULE, true, HOLD, G>(a, tk, tj, chunk, ring, bars, edge);
  else
    s3_tile<BT, RULE, false, HOLD, G>(a, tk, tj, chunk, ring, bars, edge);
}

template <int BT, int RULE, bool HOLD, class G>
cudaError_t launch3(S3Args a, cudaStream_t stream) {
  constexpr size_t smem = size_t(G::PF) * G::JW * G::KL * 8 +
                          size_t(2) * Edge3<BT, G>::kPerPar * 8 + G::PF * 8;
  auto fn = s3d7_kernel<BT, RULE, HOLD, G>;
  static int slots = 0;
  if (slots == 0) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    int occ = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, G::NT, smem);
    slots = (occ > 0 ? occ : 1) * (sms > 0 ? sms : 148);
  }
  a.kout = G::KW - 2 * BT;
  a.jout = G::JW - 2 * BT;
  a.nk = (a.n + a.kout - 1) / a.kout;
  a.nj = (a.n + a.jout - 1) / a.jout;
  // chunk height: whole waves of resident CTAs, minimise waves * (H + 2*BT + 2)
  const int64_t tiles = int64_t(a.nk) * a.nj;
  int best = 1;
  double bestc = 1e300;
  for (int nc = 1; nc <= (a.n / (4 * BT) > 1 ? a.n / (4 * BT) : 1); ++nc) {
    const int H = (a.n + nc - 1) / nc;
    const int64_t waves = (tiles * nc + slots - 1) / slots;
    const double cost = double(waves) * (H + 2 * BT + 2);
    if (cost < bestc * 0.999) bestc = cost, best = nc;
  }
  a.nchunks = best;
  a.H = (a.n + best - 1) / best;
  int grid;
  if (a.order == kOrderLex) {
    grid = a.nk * a.nj * a.nchunks;
  } else {
    int side = 1;
    while (side < a.nk || side < a.nj) side <<= 1;
    grid = side * side * a.nchunks;
  }
  fn<<<grid, G::NT, smem, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int BT, class G>
cudaError_t launch3_rule(const S3Args& a, int rule, int hold, cudaStream_t s) {
  if (rule == 0) return hold ? launch3<BT, 0, true, G>(a, s) : launch3<BT, 0, false, G>(a, s);
  return hold ? launch3<BT, 1, true, G>(a, s) : launch3<BT, 1, false, G>(a, s);
}

// Variant table (C, RJ, NW, MINB, PF); PCOTGPU_S3D7_VARIANT selects one.
template <int BT>
cudaError_t launch3_bt(const S3Args& a, int rule, int hold, int variant, cudaStream_t s) {
  if (variant < 0)  // measured best per depth (profiles/kbench_r01.md)
    variant = BT <= 2 ? 3 : BT == 3 ? 1 : 0;
  switch (variant) {
    case 0: return launch3_rule<BT, Geo<2, 4, 8, 1, 4>>(a, rule, hold, s);
    case 2: return launch3_rule<BT, Geo<2, 2, 8, 2, 4>>(a, rule, hold, s);
    case 3: return launch3_rule<BT, Geo<2, 4, 4, 2, 4>>(a, rule, hold, s);
    case 4: return launch3_rule<BT, Geo<1, 4, 8, 2, 4>>(a, rule, hold, s);
    default: return launch3_rule<BT, Geo<2, 2, 16, 1, 4>>(a, rule, hold, s);
  }
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
  a.n = int(in.n);
  a.pj_in = in.pitch_j;
  a.pi_in = in.pitch_i;
  a.pj_out = out.pitch_j;
  a.pi_out = out.pitch_i;
  a.halo = int(in.halo);
  a.order = order;
  static int variant = -2;
  if (variant == -2) {
    const char* v = std::getenv("PCOTGPU_S3D7_VARIANT");
    variant = v ? std::atoi(v) : -1;
  }
  switch (bt) {
    case 1: return launch3_bt<1>(a, rule, ring_hold, variant, stream);
    case 2: return launch3_bt<2>(a, rule, ring_hold, variant, stream);
    case 3: return launch3_bt<3>(a, rule, ring_hold, variant, stream);
    default: return launch3_bt<4>(a, rule, ring_hold, variant, stream);
  }
}

}  // namespace pcotgpu
