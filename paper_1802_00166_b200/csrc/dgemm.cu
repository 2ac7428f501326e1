// fp64 GEMM on the B200 DMMA tensor path, sm_100a.
//
// Replaces exec_stmt over kernels/gemm.kernel (reference core/src/exec.cpp:
// 347-428): Out = sum_k A'[i,k] * B'[k,j] with A' = 2A-1, B' = 2B-1.
// tcgen05 has no f64 kind (CUDA 12.9 tcgen05_mma.h), so the fp64 tensor path
// on sm_100a is warp-level mma.sync ... f64 (SASS: DMMA.8x8x4).
//
// CTA tile 128x128xBK, WM x WN warps, warp tile (128/WM) x (128/WN) of 8x8
// DMMA tiles; STAGES-deep cp.async (LDGSTS) pipeline; shared-memory pitches
// chosen so every 64-bit fragment load is bank-conflict free (pitch = 4 mod
// 16 doubles).  Default: 4 x 4 warps (32x32 warp tiles), BK 32, 3 stages;
// PCOTGPU_DGEMM_VARIANT selects another (tools/kbench.py gemm).
// Tile order: lexicographic or Morton (the COT-style recursive order).
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

namespace {

constexpr int BM = 128, BN = 128;

template <int WM_, int WN_, int BK_, int STAGES_>
struct GemmCfg {
  static constexpr int WM = WM_, WN = WN_, BK = BK_, STAGES = STAGES_;
  static constexpr int NTHR = WM * WN * 32;
  static constexpr int TM = BM / WM / 8, TN = BN / WN / 8;  // DMMA tiles per warp
  static constexpr int APITCH = BK + 4;  // A stored [m][k]
  static constexpr int BPITCH = BN + 4;  // B stored [k][n]
  static constexpr int A_STAGE = BM * APITCH;
  static constexpr int B_STAGE = BK * BPITCH;
  static constexpr size_t SMEM = size_t(STAGES) * (A_STAGE + B_STAGE) * sizeof(double);
};

PCOT_DEV void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem));
}
PCOT_DEV void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
PCOT_DEV void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

PCOT_DEV void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

template <class G>
__global__ void __launch_bounds__(G::NTHR, 1)
    dgemm_kernel(const double* __restrict__ A, const double* __restrict__ B,
                 double* __restrict__ C, int n, int64_t ld, int order, int tiles_m,
                 int tiles_n) {
  constexpr int BK = G::BK, STAGES = G::STAGES, NTHR = G::NTHR, TM = G::TM, TN = G::TN;
  constexpr int APITCH = G::APITCH, BPITCH = G::BPITCH, A_STAGE = G::A_STAGE,
                B_STAGE = G::B_STAGE;
  extern __shared__ __align__(128) double sm[];
  double* sA = sm;
  double* sB = sm + STAGES * A_STAGE;
  int tm, tn;
  if (order == kOrderLex) {
    tm = blockIdx.x / tiles_n;
    tn = blockIdx.x - tm * tiles_n;
  } else {
    morton_compact(int(blockIdx.x), tiles_n, tiles_m, tn, tm);
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / G::WN, wn = warp % G::WN;
  const int g = lane >> 2, q = lane & 3;
  const int64_t row0 = int64_t(tm) * BM, col0 = int64_t(tn) * BN;
  const int nk = (n + BK - 1) / BK;

  auto load_stage = [&](int kt, int st) {
    const int64_t k0 = int64_t(kt) * BK;
    double* a = sA + st * A_STAGE;
    double* b = sB + st * B_STAGE;
    constexpr int KC = BK / 2;  // 16-B chunks per A row
#pragma unroll
    for (int r = 0; r < BM * KC / NTHR; ++r) {  // A: 128 rows x KC chunks of 16 B
      const int idx = tid + r * NTHR;
      const int m = idx / KC, kc = (idx % KC) * 2;
      const int64_t gr = row0 + m, gk = k0 + kc;
      double* dst = a + m * APITCH + kc;
      if (gr < n && gk + 1 < n)
        cp_async16(dst, A + gr * ld + gk);
      else {
        dst[0] = (gr < n && gk < n) ? A[gr * ld + gk] : 0.0;
        dst[1] = 0.0;
      }
    }
#pragma unroll
    for (int r = 0; r < BK * 64 / NTHR; ++r) {  // B: BK rows x 64 chunks
      const int idx = tid + r * NTHR;
      const int kk = idx >> 6, nc = (idx & 63) * 2;
      const int64_t gk = k0 + kk, gc = col0 + nc;
      double* dst = b + kk * BPITCH + nc;
      if (gk < n && gc + 1 < n)
        cp_async16(dst, B + gk * ld + gc);
      else {
        dst[0] = (gk < n && gc < n) ? B[gk * ld + gc] : 0.0;
        dst[1] = 0.0;
      }
    }
  };

  double acc[TM][TN][2];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt, nxt % STAGES);
      cp_commit();
    }
    const double* a = sA + (kt % STAGES) * A_STAGE + (wm * TM * 8 + g) * APITCH + q;
    const double* b = sB + (kt % STAGES) * B_STAGE + q * BPITCH + wn * TN * 8 + g;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double af[TM], bf[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) af[i] = a[i * 8 * APITCH + ks * 4];
#pragma unroll
      for (int j = 0; j < TN; ++j) bf[j] = b[ks * 4 * BPITCH + j * 8];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_wait<0>();
  // epilogue: C[g][2q..2q+1] of every 8x8 tile
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t r = row0 + wm * TM * 8 + i * 8 + g;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t c = col0 + wn * TN * 8 + j * 8 + 2 * q;
      if (c + 1 < n) {
        *reinterpret_cast<double2*>(C + r * ld + c) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else if (c < n) {
        C[r * ld + c] = acc[i][j][0];
      }
    }
  }
}

__global__ void affine_kernel(const double* __restrict__ x, double* __restrict__ y, int64_t cnt) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < cnt;
       i += int64_t(gridDim.x) * blockDim.x)
    y[i] = sub(mul(2.0, x[i]), 1.0);  // exact for the [0,1) 53-bit init values
}

}  // namespace

template <class G>
cudaError_t launch_gemm(const double* A, const double* B, double* C, int64_t n, int64_t ld,
                        int order, int tiles_m, int tiles_n, int grid, cudaStream_t stream) {
  int sl = 0;
  if (cudaError_t e = kernel_slots(reinterpret_cast<const void*>(dgemm_kernel<G>), G::NTHR, G::SMEM, &sl))
    return e;
  dgemm_kernel<G><<<grid, G::NTHR, G::SMEM, stream>>>(A, B, C, int(n), ld, order, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
}

cudaError_t dgemm_nn(const double* A, const double* B, double* C, int64_t n, int64_t ld,
                     int order, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if ((ld & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) ||
      (reinterpret_cast<uintptr_t>(C) & 15))
    return cudaErrorInvalidValue;
  const int tiles_m = int((n + BM - 1) / BM), tiles_n = int((n + BN - 1) / BN);
  const int grid = tiles_m * tiles_n;  // both orders (compact Morton rank for COT)
  const int variant = env_int("PCOTGPU_DGEMM_VARIANT", 0);  // 0: default
  // 0 / 10: the TMA kernel (BK 32 x 3 stages / BK 16 x 6 stages); 1-9: the
  // cp.async kernels of round 1 (9 = their best, the previous default)
  if (variant == 0 || variant == 10)
    return dgemm_nn_tma(A, B, C, n, ld, order, variant == 10 ? 1 : 0, stream);
  // measured on the B200 at N=4096 (tools/kbench.py gemm; profiles/dgemm_r01.md)
  switch (variant) {
    case 1: return launch_gemm<GemmCfg<2, 4, 16, 4>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);  // 28.2 TF/s
    case 2: return launch_gemm<GemmCfg<4, 4, 16, 4>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);  // 29.3
    case 3: return launch_gemm<GemmCfg<2, 4, 32, 3>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);  // 29.4
    case 4: return launch_gemm<GemmCfg<4, 2, 16, 4>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);  // 28.2
    case 5: return launch_gemm<GemmCfg<2, 4, 16, 6>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);  // 30.3
    case 6: return launch_gemm<GemmCfg<4, 4, 16, 6>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);  // 30.0
    case 7: return launch_gemm<GemmCfg<4, 4, 24, 4>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);  // 29.1
    case 8: return launch_gemm<GemmCfg<2, 4, 24, 4>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);  // 28.5
    // default: 16 warps (32x32 warp tiles), BK 32, 3 stages: 30.5 TF/s
    default: return launch_gemm<GemmCfg<4, 4, 32, 3>>(A, B, C, n, ld, order, tiles_m, tiles_n, grid, stream);
  }
}

cudaError_t affine_2x_minus_1(const double* x, double* y, int64_t count, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  affine_kernel<<<int(blocks), 256, 0, stream>>>(x, y, count);
  count_launch();
  return cudaGetLastError();
}

}  // namespace pcotgpu
