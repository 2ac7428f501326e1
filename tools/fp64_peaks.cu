// fp64 roofline denominators on the box (MEASURED_PEAKS.json has only HBM and
// bf16): DMMA (mma.sync f64) and DADD/DFMA throughput, DADD latency.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks tools/fp64_peaks.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
  double acc[8][2];
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[i][0]), "+d"(acc[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void dadd_loop(double* out, int iters) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  const double c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = __dadd_rn(x[i], c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1.2345) out[0] = s;
}

__global__ void dadd_chain(double* out, int iters, long long* cycles) {
  double x = threadIdx.x;
  const double c = 1e-9;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) x = __dadd_rn(x, c);
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  if (x == 1.2345) out[0] = x;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  long long* cyc;
  cudaMalloc(&d, 8);
  cudaMalloc(&cyc, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    dmma_loop<<<sms * 2, warps * 32>>>(d, 100);
    cudaEventRecord(e0);
    dmma_loop<<<sms * 2, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 8 * 4 * 8 * double(iters) * sms * 2 * warps;
    printf("{\"probe\":\"dmma_m8n8k4\",\"warps_per_cta\":%d,\"TFLOPs\":%.2f}\n", warps, flops / ms / 1e9);
  }
  for (int warps : {8, 16, 32}) {
    cudaEventRecord(e0);
    dadd_loop<<<sms * 2, warps * 32>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = 8.0 * iters * sms * 2 * warps * 32;
    printf("{\"probe\":\"dadd\",\"warps_per_cta\":%d,\"Gops\":%.1f,\"per_sm_per_clk_at_1965MHz\":%.1f}\n",
           warps, ops / ms / 1e6, ops / ms / 1e6 / sms / 1.965);
  }
  dadd_chain<<<1, 32>>>(d, 10000, cyc);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\":\"dadd_latency_cycles\",\"value\":%.2f}\n", c / 10000.0);
  return 0;
}
