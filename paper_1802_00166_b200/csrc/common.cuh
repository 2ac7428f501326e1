// Shared device helpers for the sm_100a hot-path kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define PCOT_DEV __device__ __forceinline__

namespace pcotgpu {

// ---------------------------------------------------------------- fp64, exact
// Every stencil update is written with explicit round-to-nearest intrinsics so
// no FMA contraction can change a bit (reference exec.cpp:347-428 evaluates
// one rounding per operation; emitted C is built -ffp-contract=off).
PCOT_DEV double add(double a, double b) { return __dadd_rn(a, b); }
PCOT_DEV double sub(double a, double b) { return __dsub_rn(a, b); }
PCOT_DEV double mul(double a, double b) { return __dmul_rn(a, b); }
PCOT_DEV double div(double a, double b) { return __ddiv_rn(a, b); }

// ---------------------------------------------------------------- mbarrier + bulk copy (TMA engine)
PCOT_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

PCOT_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

PCOT_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

PCOT_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

PCOT_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

PCOT_DEV bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

PCOT_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// 1-D bulk copy global -> shared through the TMA engine, completion counted on
// an mbarrier (SASS: UBLKCP).  src/dst 16-B aligned, bytes a multiple of 16.
PCOT_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Tensor TMA: a 3-D box (c0 fastest) of a tensor map -> shared memory, one
// instruction for the whole box (SASS: UTMALDG).
PCOT_DEV void tma_load_3d(void* dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// ---------------------------------------------------------------- programmatic dependent launch
// A grid launched with cudaLaunchAttributeProgrammaticStreamSerialization may
// start while the previous kernel in the stream drains; it must not touch
// global memory before griddep_wait() (which returns once that kernel has
// completed and its writes are visible; a no-op for a plain launch).
PCOT_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Lets the next PDL kernel in the stream begin launching its CTAs (they wait in
// griddep_wait until this grid completes).
PCOT_DEV void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---------------------------------------------------------------- acquire/release flags
PCOT_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

PCOT_DEV void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

PCOT_DEV double ld_cg(const double* p) { return __ldcg(p); }

// ---------------------------------------------------------------- compact Morton (COT) order
// The id-th point, in Morton (Z) order, of the W x H rectangle (x fast bit):
// descends the quadtree of the power-of-two cover, skipping children by the
// number of rectangle points they hold, so a launch of exactly W*H CTAs walks
// the recursive order with no idle CTAs (children in the reference's
// split_orthants bit order, tiler.cpp:98-117).
__host__ __device__ __forceinline__ void morton_compact(int id, int W, int H, int& x, int& y) {
  int side = 1;
  while (side < W || side < H) side <<= 1;
  int x0 = 0, y0 = 0;
  for (int s = side >> 1; s >= 1; s >>= 1) {
    for (int c = 0; c < 4; ++c) {
      const int cx = c & 1, cy = c >> 1;
      const int ox = W - (x0 + cx * s), oy = H - (y0 + cy * s);
      const int cnt = (ox <= 0 || oy <= 0) ? 0 : (ox < s ? ox : s) * (oy < s ? oy : s);
      if (id < cnt) {
        x0 += cx * s;
        y0 += cy * s;
        break;
      }
      id -= cnt;
    }
  }
  x = x0;
  y = y0;
}

// Device-wide nanosecond timer (profiling aids).
PCOT_DEV long long globaltimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace pcotgpu
