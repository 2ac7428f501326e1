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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

namespace {

// PCOTGPU_S3D7_CHUNKS: tuning override of the plane chunking (tools/kbench.py s3d7)
int forced_chunks() { return env_int("PCOTGPU_S3D7_CHUNKS", 0); }

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
  } else {  // Morton over (tk, tj), compact rank
    morton_compact(tile, a.nk, a.nj, tk, tj);
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
  int slots = 0;
  if (cudaError_t e = kernel_slots(reinterpret_cast<const void*>(fn), G::NT, smem, &slots)) return e;
  if (slots <= 0) return cudaErrorInvalidConfiguration;
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
  if (const int fc = forced_chunks(); fc > 0 && fc <= a.n) {
    a.nchunks = fc;
    a.H = (a.n + fc - 1) / fc;
  }
  const int grid = a.nk * a.nj * a.nchunks;  // both orders
  fn<<<grid, G::NT, smem, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int BT, class G>
cudaError_t launch3_rule(const S3Args& a, int rule, int hold, cudaStream_t s) {
  if (rule == 0) return hold ? launch3<BT, 0, true, G>(a, s) : launch3<BT, 0, false, G>(a, s);
  return hold ? launch3<BT, 1, true, G>(a, s) : launch3<BT, 1, false, G>(a, s);
}

// ---------------------------------------------------------------------------
// Version 2: level 0 straight from the TMA plane ring.  The input planes
// rho-1, rho, rho+1 and the j/k halo are all in shared memory, so the first
// level needs no register window and no neighbour exchange (its 7 operands
// are vector shared loads); levels 1..BT-1 keep the 3-plane register window
// with k-neighbours by shuffle and warp-edge rows through shared memory.
// Windows start at even k (16-B aligned rows, double2 loads/stores), edge
// arrays are padded so no thread selects between sources, and ring planes
// (i = 0 / N-1) take a warp-uniform branch instead of per-element selects.
template <int C_, int RJ_, int NW_, int MINB_, int PF_, bool RC_ = false>
struct Geo2 {
  static constexpr int C = C_, RJ = RJ_, NW = NW_, MINB = MINB_, PF = PF_;
  static constexpr bool RC = RC_;     // level-0 rows cached in registers (3 planes)
  static constexpr int NT = NW * 32;
  static constexpr int KW = 32 * C;   // window k columns
  static constexpr int JW = NW * RJ;  // window j rows
  static constexpr int KL = KW + 4;   // ring row: columns kfirst-2 .. kfirst+KW+1
  static constexpr int JL = JW + 2;   // ring rows: jfirst-1 .. jfirst+JW
  static constexpr int SLOT = (JL * KL + 15) / 16 * 16;  // ring slot (128-B aligned)
  static_assert(C % 2 == 0, "double2 rows");
};

template <int BT, class G>
struct Regs3v2 {
  double v[BT > 1 ? BT - 1 : 1][3][G::RJ][G::C];  // levels 1..BT-1
  double z[G::RC ? 3 : 1][G::RJ][G::C];           // level-0 rows 0..RJ-1 (RC)
};

// edges per parity: [warp + 1][top=0 / bottom=1][level 1..BT-1][lane][C]
template <int BT, class G>
struct Edge3v2 {
  static constexpr int LV = BT > 1 ? BT - 1 : 1;
  static constexpr int EW = 2 * LV * 32 * G::C;  // doubles per warp
  static constexpr int kPerPar = (G::NW + 2) * EW;
};

template <int BT, int RULE, bool MASKJK, bool HOLD, class G, int P>
PCOT_DEV void s3v2_iter(Regs3v2<BT, G>& R, const double* __restrict__ ring, int k, int s0, int s1,
                        int s2, int par,
                        double* __restrict__ edge, int warp, int lane, const S3Args& a,
                        unsigned jkmask, int i0, int i1, double* __restrict__ oplane,
                        unsigned smask, unsigned rmask) {
  constexpr int C = G::C, RJ = G::RJ, KL = G::KL, SLOT = G::SLOT;
  constexpr int EW = Edge3v2<BT, G>::EW;
  // ring slots of input planes k-2, k-1, k; this thread's cell (r, c) of
  // plane slot s sits at s*SLOT + (warp*RJ + r + 1)*KL + lane*C + c + 2
  const int tb = (warp * RJ + 1) * KL + lane * C + 2;
  // (s0, s1, s2 = their slots, kept as running counters by the caller: no
  // modulo per plane)
  const double* p0 = ring + s0 * SLOT + tb;
  const double* p1 = ring + s1 * SLOT + tb;
  const double* p2 = ring + s2 * SLOT + tb;
  const double* eprev = edge + (par ^ 1) * Edge3v2<BT, G>::kPerPar;
  double* ecur = edge + par * Edge3v2<BT, G>::kPerPar;
  // Warp-edge rows of levels >= 1 were published in the previous iteration:
  // load them kPFE levels ahead of use (the first ones before level 0), so the
  // shared-memory latency is off the level chain (the compiler cannot hoist an
  // eprev load above this iteration's ecur stores itself).
  constexpr int LVp = Edge3v2<BT, G>::LV;
  constexpr int kPFE = 2;
  double upP[LVp][C], dnP[LVp][C];
  auto prefetch = [&](const int L) {  // level L >= 1
    if (L >= 1 && L < BT) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        upP[L >= 1 && L < BT ? L - 1 : 0][c] =
            eprev[(warp + 0) * EW + ((1 * LVp + (L - 1)) * 32 + lane) * C + c];
        dnP[L >= 1 && L < BT ? L - 1 : 0][c] =
            eprev[(warp + 2) * EW + ((0 * LVp + (L - 1)) * 32 + lane) * C + c];
      }
    }
  };
#pragma unroll
  for (int L = 1; L <= kPFE; ++L) prefetch(L);
  // ---- level 0 -> 1, plane k-1
  {
    const int rho = k - 1;
    double nv[RJ][C];
    double row[RJ + 2][C];  // plane k-1, rows r-1 .. RJ
    if constexpr (G::RC) {
      // plane k's rows stay in registers for its next two uses (centre, i-1)
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; c += 2) {
          const double2 v = *reinterpret_cast<const double2*>(p2 + r * KL + c);
          R.z[G::RC ? m3(P) : 0][r][c] = v.x;
          R.z[G::RC ? m3(P) : 0][r][c + 1] = v.y;
        }
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) row[r + 1][c] = R.z[G::RC ? m3(P - 1) : 0][r][c];
#pragma unroll
      for (int c = 0; c < C; c += 2) {
        const double2 u = *reinterpret_cast<const double2*>(p1 - KL + c);
        const double2 w = *reinterpret_cast<const double2*>(p1 + RJ * KL + c);
        row[0][c] = u.x, row[0][c + 1] = u.y, row[RJ + 1][c] = w.x, row[RJ + 1][c + 1] = w.y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < RJ + 2; ++r)
#pragma unroll
        for (int c = 0; c < C; c += 2) {
          const double2 v = *reinterpret_cast<const double2*>(p1 + (r - 1) * KL + c);
          row[r][c] = v.x;
          row[r][c + 1] = v.y;
        }
    }
    const bool ringp = rho < 1 || rho > a.n - 2;
    // computed on every plane, then overridden on the two ring planes (a
    // warp-uniform, almost never taken branch; an if/else diamond around the
    // update made the compiler pre-zero all of nv on every plane)
#pragma unroll
    for (int r = 0; r < RJ; ++r) {
      double im[C], ip[C];
      if constexpr (G::RC) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          im[c] = R.z[G::RC ? m3(P - 2) : 0][r][c];
          ip[c] = R.z[G::RC ? m3(P) : 0][r][c];
        }
      } else {
#pragma unroll
        for (int c = 0; c < C; c += 2) {
          const double2 u = *reinterpret_cast<const double2*>(p0 + r * KL + c);
          const double2 w = *reinterpret_cast<const double2*>(p2 + r * KL + c);
          im[c] = u.x, im[c + 1] = u.y, ip[c] = w.x, ip[c + 1] = w.y;
        }
      }
      const double W = p1[r * KL - 1], E = p1[r * KL + C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double km = c > 0 ? row[r + 1][c > 0 ? c - 1 : 0] : W;
        const double kp = c < C - 1 ? row[r + 1][c < C - 1 ? c + 1 : 0] : E;
        nv[r][c] = update7<RULE>(row[r + 1][c], im[c], ip[c], row[r][c], row[r + 2][c], km, kp);
      }
    }
    if (MASKJK && jkmask != (1u << (RJ * C)) - 1u) {  // only threads with ring cells
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (!((jkmask >> (r * C + c)) & 1u)) nv[r][c] = HOLD ? row[r + 1][c] : 0.0;
    }
    if (ringp) {
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) nv[r][c] = HOLD ? row[r + 1][c] : 0.0;
    }
    if (BT > 1) {
      constexpr int s = m3(P);  // level 1's newest plane (k-1) -> slot P
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) R.v[0][s][r][c] = nv[r][c];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        ecur[(warp + 1) * EW + ((0 * Edge3v2<BT, G>::LV + 0) * 32 + lane) * C + c] = nv[0][c];
        ecur[(warp + 1) * EW + ((1 * Edge3v2<BT, G>::LV + 0) * 32 + lane) * C + c] = nv[RJ - 1][c];
      }
    } else if (rho >= i0 && rho < i1 && smask != 0u) {
#pragma unroll
      for (int r = 0; r < RJ; ++r) {
        if (!((rmask >> r) & 1u)) continue;
        double* dst = oplane + r * a.pj_out;
        if (smask == (1u << C) - 1u) {
#pragma unroll
          for (int c = 0; c < C; c += 2)
            __stcs(reinterpret_cast<double2*>(dst + c), make_double2(nv[r][c], nv[r][c + 1]));
        } else {  // grid-edge tiles only
#pragma unroll
          for (int c = 0; c < C; ++c)
            if ((smask >> c) & 1u) __stcs(dst + c, nv[r][c]);
        }
      }
    }
  }
  // ---- levels 1..BT-1 (register window; level index L, R.v[L-1])
#pragma unroll
  for (int L = 1; L < BT; ++L) {
    constexpr int LV = Edge3v2<BT, G>::LV;
    const int sm = m3(P - L), st = m3(P - L - 1), sb = m3(P - L + 1);
    const int rho = k - L - 1;
    const double(*mid)[C] = R.v[L - 1][sm];
    double nv[RJ][C];
    const bool ringp = rho < 1 || rho > a.n - 2;
    prefetch(L + kPFE);
    // padded: warp 0 / NW-1 read pad rows (halo cells)
    const double* up = upP[L - 1];
    const double* dn = dnP[L - 1];
#pragma unroll
    for (int r = 0; r < RJ; ++r) {
      const double W = __shfl_up_sync(0xffffffffu, mid[r][C - 1], 1);
      const double E = __shfl_down_sync(0xffffffffu, mid[r][0], 1);
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double jm = r > 0 ? mid[r > 0 ? r - 1 : 0][c] : up[c];
        const double jp = r < RJ - 1 ? mid[r < RJ - 1 ? r + 1 : 0][c] : dn[c];
        const double km = c > 0 ? mid[r][c > 0 ? c - 1 : 0] : W;
        const double kp = c < C - 1 ? mid[r][c < C - 1 ? c + 1 : 0] : E;
        nv[r][c] = update7<RULE>(mid[r][c], R.v[L - 1][st][r][c], R.v[L - 1][sb][r][c], jm, jp,
                                 km, kp);
      }
    }
    if (MASKJK && jkmask != (1u << (RJ * C)) - 1u) {  // only threads with ring cells
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c)
          if (!((jkmask >> (r * C + c)) & 1u)) nv[r][c] = HOLD ? mid[r][c] : 0.0;
    }
    if (ringp) {
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) nv[r][c] = HOLD ? mid[r][c] : 0.0;
    }
    if (L + 1 < BT) {
      constexpr int dummy = 0;
      (void)dummy;
      const int sn = m3(P - L);  // level L+1's newest plane k-L-1 -> its slot
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) R.v[L < BT - 1 ? L : 0][sn][r][c] = nv[r][c];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        ecur[(warp + 1) * EW + ((0 * LV + L) * 32 + lane) * C + c] = nv[0][c];
        ecur[(warp + 1) * EW + ((1 * LV + L) * 32 + lane) * C + c] = nv[RJ - 1][c];
      }
    } else if (rho >= i0 && rho < i1 && smask != 0u) {
#pragma unroll
      for (int r = 0; r < RJ; ++r) {
        if (!((rmask >> r) & 1u)) continue;
        double* dst = oplane + r * a.pj_out;
        if (smask == (1u << C) - 1u) {
#pragma unroll
          for (int c = 0; c < C; c += 2)
            __stcs(reinterpret_cast<double2*>(dst + c), make_double2(nv[r][c], nv[r][c + 1]));
        } else {  // grid-edge tiles only
#pragma unroll
          for (int c = 0; c < C; ++c)
            if ((smask >> c) & 1u) __stcs(dst + c, nv[r][c]);
        }
      }
    }
  }
}

template <int BT, int RULE, bool MASKJK, bool HOLD, class G>
PCOT_DEV void s3v2_tile(const S3Args& a, const CUtensorMap* tmap, int tk, int tj, int chunk,
                        double* ring, uint64_t* bars, double* edge) {
  constexpr int C = G::C, RJ = G::RJ, JL = G::JL, KL = G::KL, PF = G::PF, SLOT = G::SLOT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // windows start at even k: k0 = tk*kout - (BT&1) makes kfirst = k0 - BT even
  const int k0u = tk * a.kout - (BT & 1), j0 = tj * a.jout;
  const int k0 = k0u < 0 ? 0 : k0u;
  const int kend = k0u + a.kout < a.n ? k0u + a.kout : a.n;
  const int jend = j0 + a.jout < a.n ? j0 + a.jout : a.n;
  const int i0 = chunk * a.H;
  const int i1 = i0 + a.H < a.n ? i0 + a.H : a.n;
  const int kstart = i0 - BT;
  const int niter = ((i1 + BT - kstart) + 2) / 3 * 3;
  const int kfirst = k0u - BT, jfirst = j0 - BT;
  const int kb = kfirst + lane * C;
  const int jrow0 = jfirst + warp * RJ;
  unsigned smask = 0;  // columns this thread stores
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (kb + c >= k0 && kb + c < kend) smask |= 1u << c;
  const int lo = -a.halo, hi = a.n + a.halo - 1;
  unsigned jkmask = 0;
#pragma unroll
  for (int r = 0; r < RJ; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int j = jrow0 + r, kk = kb + c;
      if (j >= 1 && j <= a.n - 2 && kk >= 1 && kk <= a.n - 2) jkmask |= 1u << (r * C + c);
    }
  // rows this thread stores, and the output plane pointer of the current
  // iteration's last level (plane k - BT), advanced by one plane per iteration
  unsigned rmask = 0;
#pragma unroll
  for (int r = 0; r < RJ; ++r)
    if (jrow0 + r >= j0 && jrow0 + r < jend) rmask |= 1u << r;
  if (rmask == 0u) smask = 0u;
  double* oplane = a.out + kb + int64_t(kstart - BT) * a.pi_out + int64_t(jrow0) * a.pj_out;
  // plane `pl` into slot pl mod PF: one tensor-TMA box (KL x JL) starting at
  // (column kfirst-2, row jfirst-1); the map's origin is the halo corner
  (void)lo;
  (void)hi;
  auto issue = [&](int pl, int slot) {  // warp 0, lane 0; slot = pl mod PF
    if (lane == 0) {
      mbar_arrive_expect_tx(&bars[slot], JL * KL * 8);
      tma_load_3d(ring + slot * SLOT, tmap, kfirst - 2 + a.halo, jfirst - 1 + a.halo, pl + a.halo,
                  &bars[slot]);
    }
  };
  // prefetch distance PF-2: slot of plane k+PF-2 held plane k-2, last read at k
  // running ring state: slots of planes k-2, k-1, k and the phase of plane k's
  // barrier (a slot is used once every PF iterations).  Depths >= 3 run
  // 512-thread CTAs at the 128-register cap, where the per-plane modulo
  // arithmetic cost registers (bt=3: 478 -> 550 GUpd/s with running counters);
  // the shallower kernels are faster with the modulo in uniform registers
  // (bt=1: 305 vs 272), so they keep it (profiles/s3d7_r02.md).
  constexpr bool kRun = BT >= 3;
  const int sl0 = ((kstart % PF) + PF) % PF;
  int s2 = sl0, s1 = (sl0 + PF - 1) % PF, s0 = (sl0 + PF - 2) % PF, wrap = 0;
  uint32_t phase = 0;
  if (warp == 0)
    for (int it = 0; it < PF - 2 && it < niter; ++it) issue(kstart + it, (sl0 + it) % PF);
  Regs3v2<BT, G> R;
#pragma unroll
  for (int L = 0; L < Edge3v2<BT, G>::LV; ++L)
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
      for (int r = 0; r < RJ; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) R.v[L][s][r][c] = 0.0;
#pragma unroll
  for (int s = 0; s < (G::RC ? 3 : 1); ++s)
#pragma unroll
    for (int r = 0; r < RJ; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c) R.z[s][r][c] = 0.0;
  for (int it = 0; it < niter; it += 3) {
#define PCOT_S3V2_STEP(P)                                                                    \
  {                                                                                          \
    const int itp = it + P;                                                                  \
    const int k = kstart + itp;                                                              \
    int q0, q1, q2;                                                                          \
    uint32_t ph;                                                                             \
    if constexpr (kRun) {                                                                    \
      q0 = s0, q1 = s1, q2 = s2, ph = phase;                                                 \
    } else {                                                                                 \
      q0 = (((k - 2) % PF) + PF) % PF, q1 = (((k - 1) % PF) + PF) % PF;                      \
      q2 = ((k % PF) + PF) % PF, ph = uint32_t((itp / PF) & 1);                              \
    }                                                                                        \
    mbar_wait(&bars[q2], ph);                                                                \
    s3v2_iter<BT, RULE, MASKJK, HOLD, G, P>(R, ring, k, q0, q1, q2, itp & 1, edge, warp, lane, a, \
                                            jkmask, i0, i1, oplane, smask, rmask);             \
    oplane += a.pi_out;                                                                      \
    __syncthreads();                                                                         \
    /* plane k+PF-2 goes into the slot that held plane k-2 */                                \
    if (warp == 0 && itp + PF - 2 < niter) issue(k + PF - 2, q0);                            \
    if constexpr (kRun) {                                                                    \
      s0 = s1;                                                                               \
      s1 = s2;                                                                               \
      s2 = s2 + 1 == PF ? 0 : s2 + 1;                                                        \
      if (++wrap == PF) wrap = 0, phase ^= 1u;                                               \
    }                                                                                        \
  }
    PCOT_S3V2_STEP(0)
    PCOT_S3V2_STEP(1)
    PCOT_S3V2_STEP(2)
#undef PCOT_S3V2_STEP
  }
}

template <int BT, int RULE, bool HOLD, class G>
__global__ void __launch_bounds__(G::NT, G::MINB)
    s3d7v2_kernel(S3Args a, const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) double smem3[];
  double* ring = smem3;
  double* edge = ring + G::PF * G::SLOT;
  uint64_t* bars = reinterpret_cast<uint64_t*>(edge + 2 * Edge3v2<BT, G>::kPerPar);
  const int ntile = a.nk * a.nj;
  int tile = blockIdx.x % ntile, chunk = blockIdx.x / ntile;
  int tk, tj;
  if (a.order == kOrderLex) {
    tj = tile / a.nk;
    tk = tile - tj * a.nk;
  } else {  // Morton over (tk, tj), compact rank
    morton_compact(tile, a.nk, a.nj, tk, tj);
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < G::PF; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();  // PDL: no global access before the previous depth block completes
  griddep_launch_dependents();
  const int k0 = tk * a.kout - (BT & 1), j0 = tj * a.jout;
  const bool edge_jk = (k0 - BT <= 0) || (k0 + a.kout + BT >= a.n - 1) || (j0 - BT <= 0) ||
                       (j0 + a.jout + BT >= a.n - 1);
  if (edge_jk)
    s3v2_tile<BT, RULE, true, HOLD, G>(a, &tmap, tk, tj, chunk, ring, bars, edge);
  else
    s3v2_tile<BT, RULE, false, HOLD, G>(a, &tmap, tk, tj, chunk, ring, bars, edge);
}

// 3-D tensor map over the whole padded input cube (halo included), box KL x JL x 1.
cudaError_t encode_plane_map(CUtensorMap* m, const S3Args& a, int kl, int jl) {
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {  // thread-safe one-time lookup
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return (e == cudaSuccess && q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)
               : nullptr;
  }();
  if (!encode) return cudaErrorNotSupported;
  const double* base = a.in - int64_t(a.halo) * (a.pi_in + a.pj_in + 1);
  const cuuint64_t dims[3] = {cuuint64_t(a.pj_in), cuuint64_t(a.pi_in / a.pj_in),
                              cuuint64_t(a.n + 2 * a.halo)};
  const cuuint64_t strides[2] = {cuuint64_t(a.pj_in) * 8, cuuint64_t(a.pi_in) * 8};
  const cuuint32_t box[3] = {cuuint32_t(kl), cuuint32_t(jl), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int BT, int RULE, bool HOLD, class G>
cudaError_t launch3v2(S3Args a, cudaStream_t stream) {
  constexpr size_t smem = size_t(G::PF) * G::SLOT * 8 +
                          size_t(2) * Edge3v2<BT, G>::kPerPar * 8 + G::PF * 8;
  auto fn = s3d7v2_kernel<BT, RULE, HOLD, G>;
  int slots = 0;
  if (cudaError_t e = kernel_slots(reinterpret_cast<const void*>(fn), G::NT, smem, &slots)) return e;
  if (slots <= 0) return cudaErrorInvalidConfiguration;
  a.kout = G::KW - 2 * BT;
  a.jout = G::JW - 2 * BT;
  a.nk = (a.n + (BT & 1) + a.kout - 1) / a.kout;
  a.nj = (a.n + a.jout - 1) / a.jout;
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
  if (const int fc = forced_chunks(); fc > 0 && fc <= a.n) {
    a.nchunks = fc;
    a.H = (a.n + fc - 1) / fc;
  }
  const int grid = a.nk * a.nj * a.nchunks;  // both orders
  CUtensorMap tmap;
  cudaError_t e = encode_plane_map(&tmap, a, G::KL, G::JL);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};  // programmatic dependent launch (see stencil2d.cu)
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(G::NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, fn, a, tmap);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int BT, class G>
cudaError_t launch3v2_rule(const S3Args& a, int rule, int hold, cudaStream_t s) {
  if (rule == 0) return hold ? launch3v2<BT, 0, true, G>(a, s) : launch3v2<BT, 0, false, G>(a, s);
  return hold ? launch3v2<BT, 1, true, G>(a, s) : launch3v2<BT, 1, false, G>(a, s);
}

// Variant table (C, RJ, NW, MINB, PF); PCOTGPU_S3D7_VARIANT selects one.
template <int BT>
cudaError_t launch3_bt(const S3Args& a, int rule, int hold, int variant, cudaStream_t s) {
  if (variant < 0)  // measured best per depth (profiles/s3d7_r01.md)
    variant = BT == 1 ? 29 : BT == 2 ? 28 : BT == 3 ? 15 : 0;
  if (variant >= 10 && BT > 3) variant = 0;  // version 2 holds at most 2 register levels
  switch (variant) {
    case 0: return launch3_rule<BT, Geo<2, 4, 8, 1, 4>>(a, rule, hold, s);
    case 2: return launch3_rule<BT, Geo<2, 2, 8, 2, 4>>(a, rule, hold, s);
    case 3: return launch3_rule<BT, Geo<2, 4, 4, 2, 4>>(a, rule, hold, s);
    case 4: return launch3_rule<BT, Geo<1, 4, 8, 2, 4>>(a, rule, hold, s);
    // version 2 (level 0 from the plane ring), BT <= 3
    case 10: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 8, 1, 6>>(a, rule, hold, s);
    case 11: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 4, 2, 4>>(a, rule, hold, s);
    case 12: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 2, 8, 2, 4>>(a, rule, hold, s);
    case 13: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<4, 2, 8, 1, 4>>(a, rule, hold, s);
    case 14: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 8, 1, 4>>(a, rule, hold, s);
    case 15: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 16, 1, 4>>(a, rule, hold, s);
    case 16: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 2, 16, 1, 4>>(a, rule, hold, s);
    case 17: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 12, 1, 4>>(a, rule, hold, s);
    case 18: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 3, 16, 1, 4>>(a, rule, hold, s);
    case 19: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 8, 1, 8>>(a, rule, hold, s);
    case 20: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 3, 16, 1, 5>>(a, rule, hold, s);
    case 21: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 4, 2, 6>>(a, rule, hold, s);
    case 22: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 8, 2, 4>>(a, rule, hold, s);
    case 23: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 6, 2, 4>>(a, rule, hold, s);
    case 24: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 12, 1, 4>>(a, rule, hold, s);
    case 25: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 8, 1, 4, true>>(a, rule, hold, s);
    case 26: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 16, 1, 4, true>>(a, rule, hold, s);
    case 27: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 8, 2, 4, true>>(a, rule, hold, s);
    case 28: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 8, 2, 5, true>>(a, rule, hold, s);
    case 29: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 6, 2, 4, true>>(a, rule, hold, s);
    case 30: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 3, 8, 2, 4, true>>(a, rule, hold, s);
    case 31: return launch3v2_rule<BT <= 3 ? BT : 1, Geo2<2, 4, 6, 2, 5, true>>(a, rule, hold, s);
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
  const int variant = env_int("PCOTGPU_S3D7_VARIANT", -1);
  switch (bt) {
    case 1: return launch3_bt<1>(a, rule, ring_hold, variant, stream);
    case 2: return launch3_bt<2>(a, rule, ring_hold, variant, stream);
    case 3: return launch3_bt<3>(a, rule, ring_hold, variant, stream);
    default: return launch3_bt<4>(a, rule, ring_hold, variant, stream);
  }
}

}  // namespace pcotgpu
