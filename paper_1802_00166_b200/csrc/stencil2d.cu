// 2-D 5-point temporally blocked streaming stencil for sm_100a.
//
// Replaces the reference's interpreted hot loop for heat2d/jacobi2d
// (reference core/src/exec.cpp:347-428 exec_stmt over kernels/heat2d.kernel:32)
// and the tile order that feeds it (tiler.cpp:189-243): one launch advances the
// grid `BT` time steps per HBM round trip.
//
// Tile = column strip (W_IN = NT*C input columns, W_OUT = W_IN - 2*BT output
// columns) x row chunk [r0, r1).  The CTA streams input rows r0-BT .. r1+BT-1:
//   * rows arrive in a PF-deep shared-memory ring through the TMA engine
//     (cp.async.bulk, mbarrier complete_tx), issued by one thread;
//   * each thread owns C adjacent columns; level L (0..BT-1) keeps its last
//     three rows in registers (slot = row mod 3, loop unrolled by 3 so every
//     register index is static);
//   * level L+1 row rho needs level L rows rho-1..rho+1 of its own columns
//     (registers) and the west/east neighbours at row rho: warp shuffles
//     inside a warp, a double-buffered shared-memory edge exchange across
//     warps (one __syncthreads per input row).
// Operation order per point is the reference body's parse tree:
//   0.2 * ((((c + (i-1,j)) + (i+1,j)) + (i,j-1)) + (i,j+1)), no FMA.
#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

namespace {

constexpr int kC = 2;      // columns per thread
constexpr int kNT = 256;   // threads per CTA
constexpr int kPF = 8;     // TMA ring depth (rows in flight)

struct S2Args {
  const double* in;
  double* out;
  int64_t ld_in, ld_out;
  int64_t cols;      // N
  int64_t g0;        // global row of local row 0
  int64_t nrows;     // global rows
  int64_t row_lo, row_hi;  // local rows produced
  int64_t load_lo, load_hi;  // clamp range for input rows
  int H;             // chunk height
  int nstrips, nchunks;
  int order;
  int w_out;
};

PCOT_DEV int pmod3(int v) { return ((v % 3) + 3) % 3; }

// Morton (Z-order) decode of a linear tile id over a 2^k x 2^k covering grid
// (COT-style recursive order, reference tiler.cpp:150-203); ids landing outside
// the real grid are skipped by the caller via the returned flag.
PCOT_DEV bool tile_coords(int id, int nstrips, int nchunks, int order, int& strip, int& chunk) {
  if (order == kOrderLex) {
    chunk = id / nstrips;
    strip = id - chunk * nstrips;
    return true;
  }
  int x = 0, y = 0;
  for (int b = 0; b < 16; ++b) {
    x |= ((id >> (2 * b)) & 1) << b;
    y |= ((id >> (2 * b + 1)) & 1) << b;
  }
  chunk = y;
  strip = x;
  return strip < nstrips && chunk < nchunks;
}

template <int BT>
struct Regs {
  double v[BT][3][kC];
};

template <int BT, bool MASK, bool HOLD, int P>
PCOT_DEV void s2d5_iter(Regs<BT>& R, const double* __restrict__ ring_row, int shift, int64_t k,
                        int par, double* __restrict__ edge, int warp, int lane,
                        int nwarps, const S2Args& a, int64_t cb, int64_t r0, int64_t r1,
                        int64_t c0, int64_t cend) {
  // ---- level 0: input row k
  {
    constexpr int s = ((P % 3) + 3) % 3;
    const double* src = ring_row + shift + threadIdx.x * kC;
#pragma unroll
    for (int c = 0; c < kC; ++c) R.v[0][s][c] = src[c];
  }
  const double* eprev = edge + (par ^ 1) * (nwarps * 2 * BT);  // written at k-1
#pragma unroll
  for (int L = 0; L < BT; ++L) {
    const int rho_rel = P - L - 1;  // (rho - kstart) mod 3 basis, static
    const int sm = ((rho_rel % 3) + 3) % 3;
    const int st = (((rho_rel - 1) % 3) + 3) % 3;
    const int sb = (((rho_rel + 1) % 3) + 3) % 3;
    const double* top = R.v[L][st];
    const double* mid = R.v[L][sm];
    const double* bot = R.v[L][sb];
    double W = __shfl_up_sync(0xffffffffu, mid[kC - 1], 1);
    double E = __shfl_down_sync(0xffffffffu, mid[0], 1);
    if (lane == 0 && warp > 0) W = eprev[((warp - 1) * 2 + 1) * BT + L];
    if (lane == 31 && warp + 1 < nwarps) E = eprev[((warp + 1) * 2 + 0) * BT + L];
    const int64_t rho = k - L - 1;
    double nv[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) {
      double left = c > 0 ? mid[c - 1] : W;
      double right = c < kC - 1 ? mid[c + 1] : E;
      double s = add(mid[c], top[c]);
      s = add(s, bot[c]);
      s = add(s, left);
      s = add(s, right);
      nv[c] = mul(0.2, s);
    }
    if (MASK) {
      const int64_t gr = a.g0 + rho;
      const bool row_in = gr >= 1 && gr <= a.nrows - 2;
#pragma unroll
      for (int c = 0; c < kC; ++c) {
        const int64_t col = cb + c;
        const bool in = row_in && col >= 1 && col <= a.cols - 2;
        if (!in) nv[c] = HOLD ? mid[c] : 0.0;
      }
    }
    if (L + 1 < BT) {
#pragma unroll
      for (int c = 0; c < kC; ++c) R.v[(L + 1) < BT ? L + 1 : 0][sm][c] = nv[c];
    } else {
      if (rho >= r0 && rho < r1) {
        double* dst = a.out + rho * a.ld_out;
#pragma unroll
        for (int c = 0; c < kC; ++c) {
          const int64_t col = cb + c;
          if (col >= c0 && col < cend) __stcs(dst + col, nv[c]);
        }
      }
    }
  }
  // ---- publish this iteration's newest row edges of every level (rows k-L)
  double* ecur = edge + par * (nwarps * 2 * BT);
  if (lane == 0) {
#pragma unroll
    for (int L = 0; L < BT; ++L) {
      const int s = (((P - L) % 3) + 3) % 3;
      ecur[(warp * 2 + 0) * BT + L] = R.v[L][s][0];
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int L = 0; L < BT; ++L) {
      const int s = (((P - L) % 3) + 3) % 3;
      ecur[(warp * 2 + 1) * BT + L] = R.v[L][s][kC - 1];
    }
  }
}

template <int BT, bool MASK, bool HOLD>
PCOT_DEV void s2d5_tile(const S2Args& a, int strip, int chunk, double* ring, uint64_t* bars,
                        double* edge) {
  constexpr int W_IN = kNT * kC;
  constexpr int W_LOAD = W_IN + 2;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = kNT / 32;
  const int64_t c0 = int64_t(strip) * a.w_out;
  const int64_t cend = c0 + a.w_out < a.cols ? c0 + a.w_out : a.cols;
  const int64_t r0 = a.row_lo + int64_t(chunk) * a.H;
  const int64_t r1 = r0 + a.H < a.row_hi ? r0 + a.H : a.row_hi;
  const int64_t kstart = r0 - BT;
  const int64_t niter = ((r1 + BT - kstart) + 2) / 3 * 3;
  const int64_t cfirst = c0 - BT;
  const int64_t cs = cfirst >= 0 ? (cfirst & ~int64_t(1)) : -((-cfirst + 1) & ~int64_t(1));
  const int shift = int(cfirst - cs);
  const int64_t cb = cfirst + tid * kC;

  auto issue = [&](int64_t it) {
    int64_t row = kstart + it;
    row = row < a.load_lo ? a.load_lo : (row > a.load_hi ? a.load_hi : row);
    const int slot = int(it % kPF);
    mbar_arrive_expect_tx(&bars[slot], W_LOAD * 8);
    bulk_g2s(ring + slot * W_LOAD, a.in + row * a.ld_in + cs, W_LOAD * 8, &bars[slot]);
  };
  if (tid == 0) {
    for (int it = 0; it < kPF && it < niter; ++it) issue(it);
  }
  Regs<BT> R;
#pragma unroll
  for (int L = 0; L < BT; ++L)
#pragma unroll
    for (int s = 0; s < 3; ++s)
#pragma unroll
      for (int c = 0; c < kC; ++c) R.v[L][s][c] = 0.0;

  for (int64_t it = 0; it < niter; it += 3) {
#define PCOT_S2_STEP(P)                                                                    \
  {                                                                                        \
    const int64_t itp = it + P;                                                            \
    const int slot = int(itp % kPF);                                                       \
    mbar_wait(&bars[slot], uint32_t((itp / kPF) & 1));                                     \
    s2d5_iter<BT, MASK, HOLD, P>(R, ring + slot * W_LOAD, shift, kstart + itp, int(itp & 1),  \
                                 edge, warp, lane, nwarps, a, cb, r0, r1, c0, cend);        \
    __syncthreads();                                                                       \
    if (tid == 0 && itp + kPF < niter) issue(itp + kPF);                                   \
  }
    PCOT_S2_STEP(0)
    PCOT_S2_STEP(1)
    PCOT_S2_STEP(2)
#undef PCOT_S2_STEP
  }
}

template <int BT, bool HOLD>
__global__ void __launch_bounds__(kNT, 2) s2d5_kernel(S2Args a) {
  constexpr int W_LOAD = kNT * kC + 2;
  __shared__ __align__(128) double ring[kPF * W_LOAD];
  __shared__ __align__(16) double edge[2 * (kNT / 32) * 2 * BT];
  __shared__ __align__(8) uint64_t bars[kPF];
  int strip, chunk;
  if (!tile_coords(blockIdx.x, a.nstrips, a.nchunks, a.order, strip, chunk)) return;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kPF; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t c0 = int64_t(strip) * a.w_out;
  const int64_t r0 = a.row_lo + int64_t(chunk) * a.H;
  const int64_t r1 = r0 + a.H < a.row_hi ? r0 + a.H : a.row_hi;
  // Cells whose update can hit the ring (or the outside) need the masked body.
  const bool edge_tile = (c0 - BT <= 0) || (c0 + a.w_out + BT >= a.cols - 1) ||
                         (a.g0 + r0 - BT <= 0) || (a.g0 + r1 + BT >= a.nrows - 1);
  if (edge_tile)
    s2d5_tile<BT, true, HOLD>(a, strip, chunk, ring, bars, edge);
  else
    s2d5_tile<BT, false, HOLD>(a, strip, chunk, ring, bars, edge);
}

template <int BT>
cudaError_t launch_bt(const S2Args& a0, int ring_hold, cudaStream_t stream) {
  S2Args a = a0;
  int grid;
  if (a.order == kOrderMorton) {
    int side = 1;
    while (side < a.nstrips || side < a.nchunks) side <<= 1;
    grid = side * side;
  } else {
    grid = a.nstrips * a.nchunks;
  }
  if (ring_hold)
    s2d5_kernel<BT, true><<<grid, kNT, 0, stream>>>(a);
  else
    s2d5_kernel<BT, false><<<grid, kNT, 0, stream>>>(a);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

int s2d5_max_bt() { return 8; }

cudaError_t s2d5_advance(const Slab2D& in, const Slab2D& out, int64_t g0, int64_t nrows,
                         int bt, int ring_hold, int order, int row_lo, int row_hi,
                         cudaStream_t stream) {
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
  a.w_out = kNT * kC - 2 * bt;
  a.nstrips = int((in.cols + a.w_out - 1) / a.w_out);
  // Enough CTAs for ~8 per SM, chunks no shorter than 16*BT rows.
  const int64_t rows = row_hi - row_lo;
  int64_t want = (148 * 8 + a.nstrips - 1) / a.nstrips;
  int64_t H = (rows + want - 1) / want;
  if (H < 16 * bt) H = 16 * bt;
  if (H > rows) H = rows;
  a.H = int(H);
  a.nchunks = int((rows + H - 1) / H);
  a.order = order;
  // right padding must cover the last strip's W_IN+2 load window
  switch (bt) {
    case 1: return launch_bt<1>(a, ring_hold, stream);
    case 2: return launch_bt<2>(a, ring_hold, stream);
    case 3: return launch_bt<3>(a, ring_hold, stream);
    case 4: return launch_bt<4>(a, ring_hold, stream);
    case 5: return launch_bt<5>(a, ring_hold, stream);
    case 6: return launch_bt<6>(a, ring_hold, stream);
    case 7: return launch_bt<7>(a, ring_hold, stream);
    default: return launch_bt<8>(a, ring_hold, stream);
  }
}

}  // namespace pcotgpu
