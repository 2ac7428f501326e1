// fp64 GEMM on the B200 DMMA tensor path, sm_100a.
//
// Replaces exec_stmt over kernels/gemm.kernel (reference core/src/exec.cpp:
// 347-428): Out = sum_k A'[i,k] * B'[k,j] with A' = 2A-1, B' = 2B-1.
// tcgen05 has no f64 kind (CUDA 12.9 tcgen05_mma.h), so the fp64 tensor path
// on sm_100a is warp-level mma.sync ... f64 (SASS: DMMA.8x8x4).
//
// CTA tile 128x128x16, 8 warps (2 x 4), warp tile 64x32 = 8x4 DMMA tiles;
// 4-stage cp.async (LDGSTS) pipeline; shared-memory pitches chosen so every
// 64-bit fragment load is bank-conflict free (pitch = 4 mod 16 doubles).
// Tile order: lexicographic or Morton (the COT-style recursive order).
#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

namespace {

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 4;
constexpr int APITCH = BK + 4;   // A stored [m][k]
constexpr int BPITCH = BN + 4;   // B stored [k][n]
constexpr int A_STAGE = BM * APITCH;
constexpr int B_STAGE = BK * BPITCH;
constexpr int NTHR = 256;

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

__global__ void __launch_bounds__(NTHR, 1)
    dgemm_kernel(const double* __restrict__ A, const double* __restrict__ B,
                 double* __restrict__ C, int n, int64_t ld, int order, int tiles_m,
                 int tiles_n) {
  extern __shared__ __align__(128) double sm[];
  double* sA = sm;
  double* sB = sm + STAGES * A_STAGE;
  int tm, tn;
  if (order == kOrderLex) {
    tm = blockIdx.x / tiles_n;
    tn = blockIdx.x - tm * tiles_n;
  } else {
    int x = 0, y = 0;
    for (int b = 0; b < 12; ++b) {
      x |= ((blockIdx.x >> (2 * b)) & 1) << b;
      y |= ((blockIdx.x >> (2 * b + 1)) & 1) << b;
    }
    tm = y;
    tn = x;
    if (tm >= tiles_m || tn >= tiles_n) return;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps
  const int g = lane >> 2, q = lane & 3;
  const int64_t row0 = int64_t(tm) * BM, col0 = int64_t(tn) * BN;
  const int nk = (n + BK - 1) / BK;

  auto load_stage = [&](int kt, int st) {
    const int64_t k0 = int64_t(kt) * BK;
    double* a = sA + st * A_STAGE;
    double* b = sB + st * B_STAGE;
#pragma unroll
    for (int r = 0; r < 4; ++r) {  // A: 128 rows x 8 chunks of 16 B
      const int idx = tid + r * NTHR;
      const int m = idx >> 3, kc = (idx & 7) * 2;
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
    for (int r = 0; r < 4; ++r) {  // B: 16 rows x 64 chunks
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

  double acc[8][4][2];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

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
    const double* a = sA + (kt % STAGES) * A_STAGE + (wm * 64 + g) * APITCH + q;
    const double* b = sB + (kt % STAGES) * B_STAGE + q * BPITCH + wn * 32 + g;
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double af[8], bf[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) af[i] = a[i * 8 * APITCH + ks * 4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = b[ks * 4 * BPITCH + j * 8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_wait<0>();
  // epilogue: C[g][2q..2q+1] of every 8x8 tile
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t r = row0 + wm * 64 + i * 8 + g;
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = col0 + wn * 32 + j * 8 + 2 * q;
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

cudaError_t dgemm_nn(const double* A, const double* B, double* C, int64_t n, int64_t ld,
                     int order, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  if ((ld & 1) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15) ||
      (reinterpret_cast<uintptr_t>(C) & 15))
    return cudaErrorInvalidValue;
  const int tiles_m = int((n + BM - 1) / BM), tiles_n = int((n + BN - 1) / BN);
  int grid = tiles_m * tiles_n;
  if (order == kOrderMorton) {
    int side = 1;
    while (side < tiles_m || side < tiles_n) side <<= 1;
    grid = side * side;
  }
  const size_t smem = size_t(STAGES) * (A_STAGE + B_STAGE) * sizeof(double);
  cudaError_t e =
      cudaFuncSetAttribute(dgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  dgemm_kernel<<<grid, NTHR, smem, stream>>>(A, B, C, int(n), ld, order, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
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
