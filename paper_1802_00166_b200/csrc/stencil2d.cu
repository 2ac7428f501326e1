// 2-D 5-point temporally blocked streaming stencil for sm_100a.
//
// Replaces the reference's interpreted hot loop for heat2d/jacobi2d
// (reference core/src/exec.cpp:347-428 exec_stmt over kernels/heat2d.kernel:32)
// and the tile order that feeds it (tiler.cpp:189-243): one launch advances the
// grid `BT` time steps per HBM round trip (16/BT algorithmic bytes per update).
//
// Tile = column strip (W_IN = NT*C input columns, W_OUT = W_IN - 2*BT output
// columns) x row chunk [r0, r1).  The CTA streams input rows r0-BT .. r1+BT-1:
//   * rows arrive in a PF-deep shared-memory ring through the TMA engine
//     (cp.async.bulk, mbarrier complete_tx), issued by one thread;
//   * each thread owns C adjacent columns; level L (0..BT-1) keeps its last
//     three rows in registers (slot = row mod 3, loop unrolled by 3 so every
//     register index is static);
//   * level L+1 row rho needs level L rows rho-1..rho+1 of its own columns
//     (registers) and the west/east neighbours at row rho, produced one
//     iteration earlier: warp shuffles inside a warp, a double-buffered
//     shared-memory edge exchange across warps (one __syncthreads per row).
// Operation order per point is the reference body's parse tree:
//   0.2 * ((((c + (i-1,j)) + (i+1,j)) + (i,j-1)) + (i,j+1)), no FMA.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

// PCOTGPU_PDL=0 turns programmatic dependent launch off (A/B measurements).
bool pdl_enabled() { return env_int("PCOTGPU_PDL", 1) != 0; }

namespace {

constexpr int kPF = 8;  // TMA ring depth (rows in flight)

#ifndef PCOT_S2_PFE
#define PCOT_S2_PFE 2  // edge-exchange loads issued this many levels ahead of use
#endif

struct S2Args {
  const double* in;
  double* out;
  int64_t ld_in, ld_out;
  int64_t cols;              // N
  int64_t g0;                // global row of local row 0
  int64_t nrows;             // global rows
  int64_t row_lo, row_hi;    // local rows produced
  int64_t load_lo, load_hi;  // clamp range for input rows
  int H;                     // chunk height
  int nstrips, nchunks;
  int order;
  int w_out;
  // In-kernel halo exchange (row-sharded grids, P2P over NVLink): output rows
  // [row_lo, mir_lo) are also stored at mir_up + row*ld_out + col (the upper
  // neighbour's ghost rows below its slab), rows [mir_hi, row_hi) at mir_dn
  // + row*ld_out + col (the lower neighbour's ghost rows); null = no mirror.
  double* mir_up;
  double* mir_dn;
  int64_t mir_lo, mir_hi;
};

// Tile id -> (strip, chunk): lexicographic (SLT-like) or Morton/Z order of the
// strips x chunks rectangle (the COT recursive order, reference
// tiler.cpp:150-203), ranked compactly: no idle CTAs.
PCOT_DEV bool tile_coords(int id, int nstrips, int nchunks, int order, int& strip, int& chunk) {
  if (order == kOrderLex) {
    chunk = id / nstrips;
    strip = id - chunk * nstrips;
    return true;
  }
  morton_compact(id, nstrips, nchunks, strip, chunk);
  return true;
}

__host__ __device__ constexpr int smod3(int v) { return ((v % 3) + 3) % 3; }

template <int BT, int C>
struct Regs {
  double v[BT][3][C];
};

// Edge exchange: XS = false -> warp shuffles + smem only across warps;
// XS = true -> every thread publishes its first/last column of every level's
// newest row in shared memory (2 STS) and reads its neighbours' (2 LDS): no
// shuffles, no selects, no predicates (measured: fewer instructions/update).
template <int BT, int NT, bool XS>
struct EdgeLayout {
  static constexpr int kPerPar = XS ? BT * 2 * (NT + 2) : (NT / 32) * 2 * BT;
  static constexpr int kDoubles = 2 * kPerPar;
};

template <int BT, int C, int NT, int MASK, bool HOLD, bool XS, int P>
PCOT_DEV void s2d5_iter(Regs<BT, C>& R, const double* __restrict__ ring_row, uint64_t* bar,
                        uint32_t phase, int k, int par, double* __restrict__ edge, int warp,
                        int lane, const S2Args& a, int64_t cb, int r0, int r1, unsigned smask,
                        unsigned cmask) {
  constexpr int NW = NT / 32;
  constexpr int SHIFT = 0;  // window start is even for every depth (see s2d5_tile)
  constexpr int EP = EdgeLayout<BT, NT, XS>::kPerPar;
  const double* eprev = edge + (par ^ 1) * EP;  // written at k-1
  double* ecur = edge + par * EP;
  const int tid = threadIdx.x;
  // XS layout: [level][L=0 / R=1][NT+2], thread t at index t+1
  auto xs_l = [&](double* base, int L) { return base + (L * 2 + 0) * (NT + 2); };
  auto xs_r = [&](double* base, int L) { return base + (L * 2 + 1) * (NT + 2); };
  // XS: the neighbours' edges were published in the previous iteration, so
  // their loads need not wait for this row's TMA, nor sit on the level chain:
  // they are issued kPFE levels ahead of use (levels 0..kPFE-1 before the wait).
  constexpr int kPFE = PCOT_S2_PFE;
  double Wp[BT], Ep[BT];
  if constexpr (XS) {
#pragma unroll
    for (int L = 0; L < (kPFE < BT ? kPFE : BT); ++L) {
      Wp[L] = xs_r(const_cast<double*>(eprev), L)[tid];
      Ep[L] = xs_l(const_cast<double*>(eprev), L)[tid + 2];
    }
  }
  mbar_wait(bar, phase);
  // ---- level 0: input row k
  {
    constexpr int s = smod3(P);
    const double* src = ring_row + SHIFT + tid * C;
    if constexpr (SHIFT == 0 && C % 2 == 0) {
#pragma unroll
      for (int c = 0; c < C; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(src + c);
        R.v[0][s][c] = v.x;
        R.v[0][s][c + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) R.v[0][s][c] = src[c];
    }
    if constexpr (XS) {
      xs_l(ecur, 0)[tid + 1] = R.v[0][s][0];
      xs_r(ecur, 0)[tid + 1] = R.v[0][s][C - 1];
    }
  }
#pragma unroll
  for (int L = 0; L < BT; ++L) {
    const int sm = smod3(P - L - 1);
    const int st = smod3(P - L - 2);
    const int sb = smod3(P - L);
    const double* top = R.v[L][st];
    const double* mid = R.v[L][sm];
    const double* bot = R.v[L][sb];
    double W, E;
    if constexpr (XS) {
      if (L + kPFE < BT) {
        Wp[L + kPFE < BT ? L + kPFE : 0] = xs_r(const_cast<double*>(eprev), L + kPFE)[tid];
        Ep[L + kPFE < BT ? L + kPFE : 0] = xs_l(const_cast<double*>(eprev), L + kPFE)[tid + 2];
      }
      W = Wp[L];
      E = Ep[L];
    } else {
      W = __shfl_up_sync(0xffffffffu, mid[C - 1], 1);
      E = __shfl_down_sync(0xffffffffu, mid[0], 1);
      if (lane == 0 && warp > 0) W = eprev[((warp - 1) * 2 + 1) * BT + L];
      if (lane == 31 && warp + 1 < NW) E = eprev[((warp + 1) * 2 + 0) * BT + L];
    }
    const int rho = k - L - 1;
    double nv[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double left = c > 0 ? mid[c > 0 ? c - 1 : 0] : W;
      const double right = c < C - 1 ? mid[c < C - 1 ? c + 1 : 0] : E;
      double s = add(mid[c], top[c]);
      s = add(s, bot[c]);
      s = add(s, left);
      s = add(s, right);
      nv[c] = mul(0.2, s);
    }
    // MASK bit 1: the strip touches column 0/N-1 -> per-thread column mask;
    // MASK bit 2: the chunk touches row 0/N-1 -> warp-uniform row test.
    if (MASK & 1) {
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (!((cmask >> c) & 1u)) nv[c] = HOLD ? mid[c] : 0.0;
    }
    if (MASK & 2) {
      const int64_t gr = a.g0 + rho;
      if (gr < 1 || gr > a.nrows - 2) {
#pragma unroll
        for (int c = 0; c < C; ++c) nv[c] = HOLD ? mid[c] : 0.0;
      }
    }
    if (L + 1 < BT) {
#pragma unroll
      for (int c = 0; c < C; ++c) R.v[L + 1 < BT ? L + 1 : 0][sm][c] = nv[c];
      if constexpr (XS) {
        xs_l(ecur, L + 1)[tid + 1] = nv[0];
        xs_r(ecur, L + 1)[tid + 1] = nv[C - 1];
      }
    } else if (rho >= r0 && rho < r1) {
      // smask: this thread's output columns.  Halo threads (mask 0) skip the
      // store without a divergent scalar path; only grid-edge strips have
      // partially covered threads.
      const int64_t off = int64_t(rho) * a.ld_out + cb;
      double* dst = a.out + off;
      if (SHIFT == 0 && C % 2 == 0 && smask == (1u << C) - 1u) {
#pragma unroll
        for (int c = 0; c < C; c += 2)
#ifdef PCOT_S2_EXP_NOSTORE  // experiment: store only when the result is NaN
          if (nv[c] != nv[c])
#endif
          __stcs(reinterpret_cast<double2*>(dst + c), make_double2(nv[c], nv[c + 1]));
      } else if (smask != 0u && smask != (1u << C) - 1u) {
#pragma unroll
        for (int c = 0; c < C; ++c)
          if ((smask >> c) & 1u) __stcs(dst + c, nv[c]);
      }
      // P2P halo: the same values into the neighbour's ghost row.  Compiled
      // only into the row-edge body (MASK bit 2), which the tiles holding a
      // shard's first/last bt rows run for those rows; the interior body —
      // nearly all of the work — carries no extra code or registers.
      double* md = nullptr;
      if constexpr ((MASK & 2) != 0)
        md = rho < a.mir_lo ? a.mir_up : (rho >= a.mir_hi ? a.mir_dn : nullptr);
      if (md != nullptr) {
        md += off;
        if (SHIFT == 0 && C % 2 == 0 && smask == (1u << C) - 1u) {
#pragma unroll
          for (int c = 0; c < C; c += 2)
            *reinterpret_cast<double2*>(md + c) = make_double2(nv[c], nv[c + 1]);
        } else if (smask != 0u && smask != (1u << C) - 1u) {
#pragma unroll
          for (int c = 0; c < C; ++c)
            if ((smask >> c) & 1u) md[c] = nv[c];
        }
      }
    }
  }
  // ---- publish this iteration's newest row edges of every level (rows k-L)
  if constexpr (!XS) {
    if (lane == 0) {
#pragma unroll
      for (int L = 0; L < BT; ++L) ecur[(warp * 2 + 0) * BT + L] = R.v[L][smod3(P - L)][0];
    }
    if (lane == 31) {
#pragma unroll
      for (int L = 0; L < BT; ++L) ecur[(warp * 2 + 1) * BT + L] = R.v[L][smod3(P - L)][C - 1];
    }
  }
}

template <int BT, int C, int NT, int MASK, bool HOLD, bool XS, int kPF>
PCOT_DEV void s2d5_tile(const S2Args& a, int strip, int chunk, double* ring, uint64_t* bars,
                        double* edge) {
  constexpr int W_LOAD = NT * C + 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Strips start at s*W_OUT - (BT&1) so the window start (strip - BT) is even
  // for every depth: 16-B aligned TMA source, vector LDS/STG per thread.
  const int64_t cstrip = int64_t(strip) * a.w_out - (BT & 1);
  const int64_t c0 = cstrip < 0 ? 0 : cstrip;
  const int64_t cend = cstrip + a.w_out < a.cols ? cstrip + a.w_out : a.cols;
  const int r0 = int(a.row_lo) + chunk * a.H;
  const int r1 = r0 + a.H < int(a.row_hi) ? r0 + a.H : int(a.row_hi);
  const int kstart = r0 - BT;
  const int niter = ((r1 + BT - kstart) + 2) / 3 * 3;
  const int64_t cfirst = cstrip - BT;
  const int64_t cs = cfirst;  // even
  const int64_t cb = cfirst + tid * C;
  unsigned smask = 0;  // columns this thread stores
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (cb + c >= c0 && cb + c < cend) smask |= 1u << c;
  unsigned cmask = 0;  // interior columns of this thread
#pragma unroll
  for (int c = 0; c < C; ++c)
    if (cb + c >= 1 && cb + c <= a.cols - 2) cmask |= 1u << c;

  auto issue = [&](int64_t it) {
#ifdef PCOT_S2_EXP_NOLOAD  // experiment: every row from one L2-resident row
    int64_t row = kstart + (it & 1);
#else
    int64_t row = kstart + it;
#endif
    row = row < a.load_lo ? a.load_lo : (row > a.load_hi ? a.load_hi : row);
    const int slot = int(it % kPF);
    mbar_arrive_expect_tx(&bars[slot], W_LOAD * 8);
    bulk_g2s(ring + slot * W_LOAD, a.in + row * a.ld_in + cs, W_LOAD * 8, &bars[slot]);
  };
  if (tid == 0) {
    for (int it = 0; it < kPF && it < niter; ++it) issue(it);
  }
  Regs<BT, C> R;
#pragma unroll
  for (int L = 0; L < BT; ++L)
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
      for (int c = 0; c < C; ++c) R.v[L][s][c] = 0.0;

  // Row-edge chunks need the row mask only while some level's row is on or
  // outside the ring: input rows k with every level's row k-1-L (L < BT) in
  // [1, nrows-2] (global) run the unmasked body.
  // The same holds for the rows whose last level is mirrored to a neighbour
  // (rho = k - BT in [0, mir_lo) or [mir_hi, rows)).
  int64_t k_safe_lo = 1 - a.g0 + BT, k_safe_hi = a.nrows - 1 - a.g0;
  if (a.mir_up != nullptr && a.mir_lo + BT > k_safe_lo) k_safe_lo = a.mir_lo + BT;
  if (a.mir_dn != nullptr && a.mir_hi - 1 + BT < k_safe_hi) k_safe_hi = a.mir_hi - 1 + BT;
  // The TMA refill rotates over the warps (lane 0): the ~30 issue
  // instructions would otherwise make warp 0 the last to reach every barrier.
  constexpr int NW = NT / 32;
  // Every warp waits on the row's mbarrier itself (measured faster than one
  // waiter + the barrier: the try_wait latency then overlaps across warps).
#define PCOT_S2_STEP(M, P)                                                                       \
  {                                                                                              \
    const int itp = it + P;                                                                      \
    const int slot = itp % kPF;                                                                  \
    s2d5_iter<BT, C, NT, M, HOLD, XS, P>(R, ring + slot * W_LOAD, &bars[slot],                   \
                                         uint32_t((itp / kPF) & 1), kstart + itp, itp & 1, edge, \
                                         warp, lane, a, cb, r0, r1, smask, cmask);               \
    __syncthreads();                                                                             \
    if (lane == 0 && warp == itp % NW && itp + kPF < niter) issue(itp + kPF);                    \
  }
  for (int it = 0; it < niter; it += 3) {
    if ((MASK & 2) && !(kstart + it >= k_safe_lo && kstart + it + 2 <= k_safe_hi)) {
      PCOT_S2_STEP(MASK, 0)
      PCOT_S2_STEP(MASK, 1)
      PCOT_S2_STEP(MASK, 2)
    } else {
      PCOT_S2_STEP(MASK & 1, 0)
      PCOT_S2_STEP(MASK & 1, 1)
      PCOT_S2_STEP(MASK & 1, 2)
    }
  }
#undef PCOT_S2_STEP
}

template <int MINB>
__host__ __device__ constexpr int ring_depth() {
  return MINB >= 4 ? 4 : 8;  // rows in flight; 4 CTAs/SM must fit in 228 KB
}

template <int BT, int C, int NT, int MINB, bool HOLD, bool XS>
__global__ void __launch_bounds__(NT, MINB) s2d5_kernel(S2Args a) {
  constexpr int W_LOAD = NT * C + 2;
  constexpr int kPF = ring_depth<MINB>();
  extern __shared__ __align__(128) double smem2[];
  double* ring = smem2;
  double* edge = ring + kPF * W_LOAD;
  uint64_t* bars = reinterpret_cast<uint64_t*>(edge + EdgeLayout<BT, NT, XS>::kDoubles);
  int strip, chunk;
  if (!tile_coords(blockIdx.x, a.nstrips, a.nchunks, a.order, strip, chunk)) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPF; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  // PDL: the prologue above overlaps the previous launch's tail; its output
  // (this launch's input) and its input (this launch's output) are safe after
  // the wait.  Dependents may then start launching into freed slots.
  griddep_wait();
  griddep_launch_dependents();
  const int64_t c0 = int64_t(strip) * a.w_out - (BT & 1);
  const int64_t r0 = a.row_lo + int64_t(chunk) * a.H;
  const int64_t r1 = r0 + a.H < a.row_hi ? r0 + a.H : a.row_hi;
  // Tiles whose dependence cone touches the ring (or the outside) need masks:
  // column-edge strips per element, row-edge chunks by a uniform row test.
  const bool edge_c = (c0 - BT <= 0) || (c0 + a.w_out + BT >= a.cols - 1);
  const bool edge_r = (a.g0 + r0 - BT <= 0) || (a.g0 + r1 + BT >= a.nrows - 1) ||
                      (a.mir_up != nullptr && r0 < a.mir_lo) ||
                      (a.mir_dn != nullptr && r1 > a.mir_hi);
  const int mk = (edge_c ? 1 : 0) | (edge_r ? 2 : 0);
  if (mk == 0)
    s2d5_tile<BT, C, NT, 0, HOLD, XS, kPF>(a, strip, chunk, ring, bars, edge);
  else if (mk == 2)
    s2d5_tile<BT, C, NT, 2, HOLD, XS, kPF>(a, strip, chunk, ring, bars, edge);
  else
    s2d5_tile<BT, C, NT, 3, HOLD, XS, kPF>(a, strip, chunk, ring, bars, edge);
}

// Pick the chunk height so the grid fills whole waves of resident CTAs:
// minimise waves * (H + 2*BT + 2) (time ~ rounds x rows streamed per tile).
// Tall tiles in few waves measured up to 1.6x slower than many waves of
// ~250-500-row tiles on the 32768^2 grid (profiles/s2d5_r01b.md), so chunks
// taller than 512 rows are re-chosen around 384 rows.  Grids that cannot fill
// every resident slot with one wave of such tiles (L2-resident grids, e.g.
// 2048^2) are latency-bound per row, so there the chunks shrink down to
// 2*BT+16 rows until the wave is full (2048^2, bt=4: 64-row -> 32-row tiles,
// 597 -> 731 GUpd/s, tools/cfg0_sweep.sh).
void size_grid(S2Args& a, int bt, int rows, int slots) {
  const int hmin = 2 * bt + 16;
  auto pick = [&](int lo, int hi) {
    int best_n = lo;
    double best = 1e300;
    for (int nc = lo; nc <= hi; ++nc) {
      const int H = (rows + nc - 1) / nc;
      const int64_t tiles = int64_t(a.nstrips) * nc;
      const int64_t waves = (tiles + slots - 1) / slots;
      const double cost = double(waves) * (H + 2 * bt + 2);
      if (cost < best * 0.999) best = cost, best_n = nc;
    }
    return best_n;
  };
  const int maxc = rows / hmin > 1 ? rows / hmin : 1;
  int nc = pick(1, maxc);
  if ((rows + nc - 1) / nc > 512) {
    const int mid = rows / 384 > 1 ? rows / 384 : 1;
    const int lo = mid * 3 / 4 > 1 ? mid * 3 / 4 : 1;
    const int hi = mid * 4 / 3 < maxc ? mid * 4 / 3 : maxc;
    nc = pick(lo, hi > lo ? hi : lo);
  }
  a.nchunks = nc;
  a.H = (rows + nc - 1) / nc;
}

template <int BT, int C, int NT, int MINB, bool XS>
cudaError_t launch_cfg(S2Args a, int ring_hold, int rows, cudaStream_t stream) {
  auto kern = ring_hold ? s2d5_kernel<BT, C, NT, MINB, true, XS>
                        : s2d5_kernel<BT, C, NT, MINB, false, XS>;
  constexpr int kPF = ring_depth<MINB>();
  constexpr size_t smem = size_t(kPF) * (NT * C + 2) * 8 +
                          size_t(EdgeLayout<BT, NT, XS>::kDoubles) * 8 + size_t(kPF) * 8;
  int sl = 0;
  if (cudaError_t e = kernel_slots(reinterpret_cast<const void*>(kern), NT, smem, &sl)) return e;
  if (sl <= 0) return cudaErrorInvalidConfiguration;
  a.w_out = NT * C - 2 * BT;
  a.nstrips = int((a.cols + (BT & 1) + a.w_out - 1) / a.w_out);
  size_grid(a, BT, rows, sl);
  const int force_chunks = env_int("PCOTGPU_S2D5_CHUNKS", 0);  // tuning override of the row chunking
  if (force_chunks > 0 && force_chunks <= rows) {
    a.nchunks = force_chunks;
    a.H = (rows + force_chunks - 1) / force_chunks;
  }
  const int grid = a.nstrips * a.nchunks;  // both orders (compact Morton rank for COT)
  if (env_int("PCOTGPU_S2D5_DEBUG", 0))
    std::fprintf(stderr, "s2d5 bt=%d C=%d NT=%d slots=%d strips=%d chunks=%d H=%d grid=%d\n", BT, C,
                 NT, sl, a.nstrips, a.nchunks, a.H, grid);
  // Programmatic dependent launch: back-to-back depth blocks overlap one
  // launch's drain with the next one's CTA launch and prologue.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Variant table: (C, NT, MINB).  Variant 0 is the default; PCOTGPU_S2D5_VARIANT
// selects another for tuning.
template <int BT>
cudaError_t launch_bt(const S2Args& a, int ring_hold, int rows, int variant, cudaStream_t s) {
  if (variant < 0) {  // measured best per depth (tools/kbench.py s2d5; profiles/kbench_r01.md)
    if (int64_t(rows) * a.cols <= (int64_t(1) << 24))
      variant = 8;  // small (L2-resident) grids: 128-thread strips, 4 CTAs/SM, short chunks
                    // (2048^2 T=256 at bt=8: 907 GUpd/s; profiles/cfg0_r01.txt)
    else
      variant = BT <= 4 ? 6 : BT == 6 ? 12 : 4;
  }
  switch (variant) {
    case 1: return launch_cfg<BT, 2, 256, 2, false>(a, ring_hold, rows, s);
    case 2: return launch_cfg<BT, 4, 256, 1, false>(a, ring_hold, rows, s);
    case 3: return launch_cfg<BT, 4, 128, 3, false>(a, ring_hold, rows, s);
    case 4: return launch_cfg<BT, 4, 128, 2, true>(a, ring_hold, rows, s);
    case 5: return launch_cfg<BT, 4, 128, 3, true>(a, ring_hold, rows, s);
    case 6: return launch_cfg<BT, 4, 128, 4, true>(a, ring_hold, rows, s);
    case 7: return launch_cfg<BT, 2, 256, 2, true>(a, ring_hold, rows, s);
    case 8: return launch_cfg<BT, 2, 128, 4, true>(a, ring_hold, rows, s);
    case 9: return launch_cfg<BT, 2, 64, 8, true>(a, ring_hold, rows, s);
    case 10: return launch_cfg<BT, 4, 64, 6, true>(a, ring_hold, rows, s);
    case 11: return launch_cfg<BT, 4, 96, 4, true>(a, ring_hold, rows, s);
    // six columns per thread: 1/3 less edge exchange per update, and the
    // 48-B per-thread stride makes the level-0 LDS.128 bank-conflict free
    case 12: return launch_cfg<BT, 6, 64, 3, true>(a, ring_hold, rows, s);
    case 13: return launch_cfg<BT, 6, 64, 4, true>(a, ring_hold, rows, s);
    case 14: return launch_cfg<BT, 6, 128, 2, true>(a, ring_hold, rows, s);
    case 15: return launch_cfg<BT, 6, 32, 8, true>(a, ring_hold, rows, s);

    default: return launch_cfg<BT, 4, 128, 2, false>(a, ring_hold, rows, s);
  }
}

}  // namespace

int s2d5_max_bt() { return 8; }

int s2d5_window_cols() { return 1024 + 2; }

cudaError_t s2d5_advance(const Slab2D& in, const Slab2D& out, int64_t g0, int64_t nrows,
                         int bt, int ring_hold, int order, int row_lo, int row_hi,
                         cudaStream_t stream) {
  return s2d5_advance_p2p(in, out, g0, nrows, bt, ring_hold, order, row_lo, row_hi, nullptr,
                          nullptr, 0, stream);
}

cudaError_t s2d5_advance_p2p(const Slab2D& in, const Slab2D& out, int64_t g0, int64_t nrows,
                             int bt, int ring_hold, int order, int row_lo, int row_hi,
                             double* mirror_up, double* mirror_dn, int mirror_rows,
                             cudaStream_t stream) {
  if (mirror_rows < 0 || mirror_rows > out.rows) return cudaErrorInvalidValue;
  if (bt < 1 || bt > 8) return cudaErrorInvalidValue;
  if (row_hi <= row_lo) return cudaSuccess;
  if (in.ghost < bt + 3 || in.padl < bt + 1) return cudaErrorInvalidValue;
  if ((in.ld & 1) || (reinterpret_cast<uintptr_t>(in.origin) & 15)) return cudaErrorInvalidValue;
  S2Args a;
  a.in = in.origin;
  a.out = out.origin;
  a.ld_in = in.ld;
  a.ld_out = out.ld;
  a.cols = in.cols;
  a.g0 = g0;
  a.nrows = nrows;
  a.row_lo = row_lo;
  a.row_hi = row_hi;
  a.load_lo = -in.ghost;
  a.load_hi = in.rows + in.ghost - 1;
  a.order = order;
  a.mir_up = mirror_rows > 0 ? mirror_up : nullptr;
  a.mir_dn = mirror_rows > 0 ? mirror_dn : nullptr;
  a.mir_lo = mirror_rows;
  a.mir_hi = out.rows - mirror_rows;
  const int variant = env_int("PCOTGPU_S2D5_VARIANT", -1);  // -1: automatic per depth
  const int rows = row_hi - row_lo;
#ifdef PCOT_S2_DEV_BT  // development: instantiate one depth only (fast SASS checks)
  return bt == PCOT_S2_DEV_BT ? launch_bt<PCOT_S2_DEV_BT>(a, ring_hold, rows, variant, stream)
                              : cudaErrorInvalidValue;
#else
  switch (bt) {
    case 1: return launch_bt<1>(a, ring_hold, rows, variant, stream);
    case 2: return launch_bt<2>(a, ring_hold, rows, variant, stream);
    case 3: return launch_bt<3>(a, ring_hold, rows, variant, stream);
    case 4: return launch_bt<4>(a, ring_hold, rows, variant, stream);
    case 5: return launch_bt<5>(a, ring_hold, rows, variant, stream);
    case 6: return launch_bt<6>(a, ring_hold, rows, variant, stream);
    case 7: return launch_bt<7>(a, ring_hold, rows, variant, stream);
    default: return launch_bt<8>(a, ring_hold, rows, variant, stream);
  }
#endif
}

}  // namespace pcotgpu
