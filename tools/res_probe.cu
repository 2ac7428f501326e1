// Timing probe for the resident stencil kernel (compile-time variants):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -I paper_1802_00166_b200/csrc
//        [-DPCOT_RES_...] -o /tmp/res_probe tools/res_probe.cu
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include "../paper_1802_00166_b200/csrc/stencil2d_res.cu"
namespace pcotgpu {
cudaError_t kernel_slots(const void* fn, int nthreads, size_t smem, int* slots) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, nthreads, smem);
  if (slots) *slots = occ * 148;
  return cudaSuccess;
}
int env_int(const char* name, int dflt) { const char* v = getenv(name); return v && *v ? atoi(v) : dflt; }
void count_launch(uint64_t) {}
}
int main(int argc, char** argv) {
  using namespace pcotgpu;
  const int n = argc > 1 ? atoi(argv[1]) : 2048, T = argc > 2 ? atoi(argv[2]) : 256;
  const int64_t ld = 4096;
  double *a, *b;
  cudaMalloc(&a, size_t(n + 32) * ld * 8);
  cudaMalloc(&b, size_t(n + 32) * ld * 8);
  cudaMemset(a, 0, size_t(n + 32) * ld * 8);
  Slab2D in, out;
  in.origin = a + 16 * ld + 16; in.ld = ld; in.rows = n; in.cols = n;
  out = in; out.origin = b + 16 * ld + 16;
  S2ResPlan* p = s2d5_res_create(n, 0);
  if (!p) { printf("no plan\n"); return 1; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int i = 0; i < 5; ++i) {
    cudaEventRecord(e0);
    cudaError_t e = s2d5_res_run(p, in, out, T, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) { printf("err %d\n", int(e)); return 1; }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  printf("%s n=%d T=%d  %.3f ms  %.1f GUpd/s  fault %d\n", argc > 3 ? argv[3] : "", n, T, best,
         double(n) * n * T / best / 1e6, s2d5_res_fault(p));
  return 0;
}
