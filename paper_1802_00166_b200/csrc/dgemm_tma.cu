// fp64 GEMM, Blackwell load path: tensor TMA + full/empty mbarrier ring,
// DMMA consumers that never meet at a CTA barrier.  sm_100a.
//
// Same computation as dgemm.cu (reference exec_stmt over kernels/gemm.kernel,
// core/src/exec.cpp:347-428: Out = sum_k A'[i,k] * B'[k,j]).  What changes is
// how the operands reach the DMMA pipe:
//   * one elected lane (the duty rotates over the warps, a k-block each) issues
//     `cp.async.bulk.tensor.2d` (SASS UTMALDG) boxes of
//     16 doubles (128 B) x rows with the 128-byte swizzle into a STAGES-deep
//     ring; a stage is published by the TMA engine's complete_tx on its `full`
//     mbarrier and handed back by one arrive per consumer warp on its `empty`
//     mbarrier -- no __syncthreads in the main loop, so the 16 consumer warps
//     drift apart and the DMMA pipe is not drained at every k-block;
//   * the CTA is persistent (tile = blockIdx.x + r * gridDim.x, in the SLT /
//     compact-Morton order of the schedule), so the ring keeps filling with the
//     next tile's first stages while the warps store the finished tile;
//   * fragment loads are bank-conflict free under the swizzle without padding:
//     the DMMA row index g is mapped to tile row (g&3)*2 + (g>>2) (A) and to
//     tile column (g>>2)*2 + ((g>>1)&1)*8 + (g&1) (B), so the 16 lanes of a
//     half-warp touch 16 distinct 8-byte bank pairs (derivation in DESIGN.md).
// Ragged N: the tensor maps carry the true extents, TMA zero-fills the
// out-of-bounds part of a box, the epilogue masks rows/columns >= n.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

namespace {

constexpr int BM = 128, BN = 128;
constexpr int kConsumerWarps = 16;                   // 4 x 4, 32 x 32 warp tiles
constexpr int kThreads = kConsumerWarps * 32;

template <int BK_, int STAGES_>
struct TmaCfg {
  static constexpr int BK = BK_, STAGES = STAGES_;
  static constexpr int A_BOX = BM * 128;              // bytes: 128 rows x 16 doubles
  static constexpr int B_BOX = BK * 128;              // bytes: BK rows x 16 doubles
  static constexpr int A_BYTES = (BK / 16) * A_BOX;   // [kb][m][16]
  static constexpr int B_BYTES = (BN / 16) * B_BOX;   // [nb][k][16]
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE_BYTES + 1024 /* alignment slack */ +
                                 2 * STAGES * sizeof(uint64_t);
};

PCOT_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

PCOT_DEV void tma_load_2d(uint32_t dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

PCOT_DEV double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}

PCOT_DEV void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <class G>
__global__ void __launch_bounds__(kThreads, 1)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap mapA,
                     const __grid_constant__ CUtensorMap mapB, double* __restrict__ C, int n,
                     int64_t ld, int order, int tiles_m, int tiles_n) {
  constexpr int BK = G::BK, STAGES = G::STAGES;
  extern __shared__ unsigned char smraw[];
  const uint32_t ring = (smem_u32(smraw) + 1023u) & ~1023u;  // swizzle atoms are 1024-B aligned
  uint64_t* bars = reinterpret_cast<uint64_t*>(smraw + (ring - smem_u32(smraw)) +
                                               size_t(STAGES) * G::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int ntiles = tiles_m * tiles_n;
  const int nk = (n + BK - 1) / BK;

  auto tile_of = [&](int t, int& tm, int& tn) {
    if (order == kOrderLex) {
      tm = t / tiles_n;
      tn = t - tm * tiles_n;
    } else {
      morton_compact(t, tiles_n, tiles_m, tn, tm);
    }
  };

  // Producer side (no dedicated warp: 16 x 32 x 128 registers fill the file).
  // Global iteration p = (tile round, k-block) is loaded into stage p % STAGES
  // by lane 0 of warp (p % 16) at the top of its iteration p - (STAGES-1), once
  // every consumer warp has handed the stage back (it was read in iteration
  // p - STAGES).  The (tile, k-block) of the next load is tracked in registers.
  int p_it = 0, p_kt = 0, p_tile = blockIdx.x, p_row0 = 0, p_col0 = 0;
  if (p_tile < ntiles) {
    int tm, tn;
    tile_of(p_tile, tm, tn);
    p_row0 = tm * BM, p_col0 = tn * BN;
  }
  auto produce = [&](bool elected) {  // uniform bookkeeping, one lane issues
    if (p_tile >= ntiles) return;
    const int s = p_it % STAGES;
    if (elected) {
      if (p_it >= STAGES) mbar_wait(&empty[s], ((p_it / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], G::STAGE_BYTES);
      const uint32_t a = ring + s * G::STAGE_BYTES, b = a + G::A_BYTES;
      const int k0 = p_kt * BK;
#pragma unroll
      for (int kb = 0; kb < BK / 16; ++kb)
        tma_load_2d(a + kb * G::A_BOX, &mapA, k0 + kb * 16, p_row0, &full[s]);
#pragma unroll
      for (int nb = 0; nb < BN / 16; ++nb)
        tma_load_2d(b + nb * G::B_BOX, &mapB, p_col0 + nb * 16, k0, &full[s]);
    }
    ++p_it;
    if (++p_kt == nk) {
      p_kt = 0;
      p_tile += gridDim.x;
      if (p_tile < ntiles) {
        int tm, tn;
        tile_of(p_tile, tm, tn);
        p_row0 = tm * BM, p_col0 = tn * BN;
      }
    }
  };
#pragma unroll 1
  for (int i = 0; i < STAGES - 1; ++i) produce(tid == 0);

  // ---------------------------------------------------------------- consumers
  const int wm = warp >> 2, wn = warp & 3;
  const int g = lane >> 2, q = lane & 3;
  const int pg = (g & 3) * 2 + (g >> 2);  // tile row (mod 8) of DMMA row g
  // A[m][k]: kb = k / 16, chunk = (k % 16) / 2, physical chunk = chunk ^ (m & 7)
  const uint32_t a_base = (wm * 32 + pg) * 128 + (q & 1) * 8;
  uint32_t offA[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) offA[c] = uint32_t(((c * 2 + (q >> 1)) ^ pg) << 4);
  // B[k][n]: nb = n / 16, chunk = (n % 16) / 2, physical chunk = chunk ^ (k & 7)
  const uint32_t b_base = G::A_BYTES + wn * 2 * G::B_BOX + q * 128 + (g & 1) * 8;
  uint32_t offB[2][2];  // [j & 1][ks & 1]
#pragma unroll
  for (int jj = 0; jj < 2; ++jj)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk)
      offB[jj][kk] = uint32_t(((jj * 2 + (g >> 2) + ((g >> 1) & 1) * 4) ^ (kk * 4 + q)) << 4);

  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    int tm, tn;
    tile_of(t, tm, tn);
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < nk; ++kt, ++it) {
      produce(lane == 0 && warp == (it & (kConsumerWarps - 1)));
      const int s = it % STAGES;
      mbar_wait(&full[s], (it / STAGES) & 1);
      const uint32_t st = ring + s * G::STAGE_BYTES;
      uint32_t pa[4], pb[2][2];
#pragma unroll
      for (int c = 0; c < 4; ++c) pa[c] = st + a_base + offA[c];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj)
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) pb[jj][kk] = st + b_base + offB[jj][kk];
#pragma unroll
      for (int ks = 0; ks < BK / 4; ++ks) {
        double af[4], bf[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          af[i] = lds_f64(pa[ks & 3] + (ks >> 2) * G::A_BOX + i * 1024);
#pragma unroll
        for (int j = 0; j < 4; ++j)
          bf[j] = lds_f64(pb[j & 1][ks & 1] + (j >> 1) * G::B_BOX + ks * 512);
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }

    // epilogue: DMMA row g -> tile row pg, DMMA columns 2q, 2q+1 -> the
    // adjacent tile columns (q>>1)*2 + (q&1)*8 + {0,1}
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t r = int64_t(tm) * BM + wm * 32 + i * 8 + pg;
      if (r >= n) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t c = int64_t(tn) * BN + wn * 32 + (j >> 1) * 16 + (j & 1) * 4 +
                          (q >> 1) * 2 + (q & 1) * 8;
        if (c + 1 < n) {
          *reinterpret_cast<double2*>(C + r * ld + c) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else if (c < n) {
          C[r * ld + c] = acc[i][j][0];
        }
      }
    }
  }
}

// 2-D tensor map over an n x n row-major fp64 matrix with pitch ld: box of 16
// doubles (128 B, one swizzle row) x `rows`, 128-byte swizzle, zero fill.
cudaError_t encode_matrix_map(CUtensorMap* m, const double* base, int64_t n, int64_t ld, int rows) {
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {  // thread-safe one-time lookup
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    return (e == cudaSuccess && q == cudaDriverEntryPointSuccess)
               ? reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn)
               : nullptr;
  }();
  if (!encode) return cudaErrorNotSupported;
  const cuuint64_t dims[2] = {cuuint64_t(n), cuuint64_t(n)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
  const cuuint32_t box[2] = {16, cuuint32_t(rows)};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <class G>
cudaError_t launch_tma(const double* A, const double* B, double* C, int64_t n, int64_t ld,
                       int order, int tiles_m, int tiles_n, cudaStream_t stream) {
  auto fn = dgemm_tma_kernel<G>;
  int slots = 0;
  if (cudaError_t e = kernel_slots(reinterpret_cast<const void*>(fn), kThreads, G::SMEM, &slots))
    return e;
  if (slots <= 0) return cudaErrorInvalidConfiguration;
  CUtensorMap mapA, mapB;
  if (cudaError_t e = encode_matrix_map(&mapA, A, n, ld, BM)) return e;
  if (cudaError_t e = encode_matrix_map(&mapB, B, n, ld, G::BK)) return e;
  const int ntiles = tiles_m * tiles_n;
  const int grid = ntiles < slots ? ntiles : slots;  // persistent: one CTA per SM
  fn<<<grid, kThreads, G::SMEM, stream>>>(mapA, mapB, C, int(n), ld, order, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
}

}  // namespace

// variant 0: BK 32 x 3 stages; 1: BK 16 x 6 stages (same 192 KB ring)
cudaError_t dgemm_nn_tma(const double* A, const double* B, double* C, int64_t n, int64_t ld,
                         int order, int variant, cudaStream_t stream) {
  const int tiles_m = int((n + BM - 1) / BM), tiles_n = int((n + BN - 1) / BN);
  if (variant == 1)
    return launch_tma<TmaCfg<16, 6>>(A, B, C, n, ld, order, tiles_m, tiles_n, stream);
  return launch_tma<TmaCfg<32, 3>>(A, B, C, n, ld, order, tiles_m, tiles_n, stream);
}

}  // namespace pcotgpu
