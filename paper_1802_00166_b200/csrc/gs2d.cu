// In-place Gauss-Seidel 9-point, skewed tile wavefront, sm_100a.
//
// Replaces exec_stmt over kernels/gs2d.kernel (reference core/src/exec.cpp:
// 347-428) under the in-place storage allocate() derives for it (UOV (1,1,2),
// map (t mod 1, x-t, y-2t): reference memalloc.cpp:542-595).
//
// Tiles are boxes in the kernel's skewed band (t, x = t+i, y = 2t+i+j), where
// every dependence is non-negative (reference tilable_band semantics,
// tiler.cpp:189-243), so a tile only waits for its <= 7 lower neighbours.
// A persistent grid pulls tiles from a global queue in wavefront order and
// spins (acquire) on the predecessors' completion flags — no grid-wide sync.
// Inside a tile, thread (tt, xx) owns the line (t0+tt, x0+xx) and sweeps y;
// clock h = t + x + y (= 4t + 2i + j) is a legal point schedule: every
// dependence distance has positive coordinate sum, so one __syncthreads per
// clock orders the whole tile.  The tile's cells live in shared memory in the
// reference's storage coordinates (i, s = i + j); global memory is written
// through, and the universal occupancy vector makes any dependence-respecting
// concurrent tile schedule safe for in-place storage.
// Per point: 3x3 in row-major order, left-associated sum, IEEE '/ 9.0'.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <tuple>
#include <type_traits>
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace pcotgpu {

struct GsPlan {
  int64_t n = 0, T = 0;
  int bt = 0, bx = 0, by = 0;
  int64_t ntiles = 0;
  int grid = 0;
  int* d_tiles = nullptr;   // [ntiles][3]: tb, xb, yb
  int* d_preds = nullptr;   // [ntiles][8]: predecessor tile ids (-1 = none)
  int* d_state = nullptr;   // [ntiles] flags + [1] queue counter
  int device = 0;
  // systolic pipeline mode (bt == 0): one CTA per 32-row band
  bool pipe = false;
  int nb = 0;       // bands of the longest launch
  int64_t seg = 0;  // levels per launch (the row window drifts one row per level)
  int64_t ebld = 0, ld = 0;
  double* wb[2] = {nullptr, nullptr};
  double* eb = nullptr;
  int* gprog = nullptr;  // split-band progress words
  // fault word: a dependence wait that hit its spin cap (lost co-residency or
  // a scheduling bug) sets it; gs2d_run copies it to h_err after its launches
  int* d_err = nullptr;
  int* h_err = nullptr;  // pinned
  bool setup_failed = false;
};

namespace {

// Correctly rounded x / 9.0 without the general division sequence:
// q0 = RN(x * RN(1/9)) is within 1 ulp of x/9, so r = x - 9*q0 is exact
// (one FMA) and RN(q0 + r * RN(1/9)) is the correctly rounded quotient
// (Markstein's correction theorem for a divisor known in advance).  Verified
// against __ddiv_rn on the device (tests/test_gpu_kernels.py) and through the
// Gauss-Seidel goldens.
PCOT_DEV double div9(double x) {
  const double y = 0.1111111111111111049432054187491303309798240661621094;  // RN(1/9)
  const double q0 = __dmul_rn(x, y);
  const double r = __fma_rn(-q0, 9.0, x);
  return __fma_rn(r, y, q0);
}

__global__ void div9_check_kernel(const double* x, double* q_fast, double* q_ref, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    q_fast[i] = div9(x[i]);
    q_ref[i] = __ddiv_rn(x[i], 9.0);
  }
}

// Acquire-spin on a predecessor's completion flag with exponential backoff:
// thousands of resident warps may be waiting on the wavefront at once, and
// tight polling would flood L2 with acquire loads.
// Bounded (~tens of seconds): on timeout the fault word is set and the run
// reports an error instead of hanging the device or returning silently.
PCOT_DEV void spin_flag(const int* f, int* err) {
  unsigned ns = 64;
  for (long long it = 0; ld_acquire(f) == 0; ++it) {
    if (it > 20000000LL) {
      atomicOr(err, 1);
      return;
    }
    __nanosleep(ns);
    ns = ns < 2048 ? ns * 2 : 2048;
  }
}

struct GsArgs {
  double* a;
  int64_t ld, n, T;
  int bt, bx, by;
  int ni, ns;  // smem region rows / cols
  int64_t ntiles;
  const int* tiles;
  const int* preds;
  int* flags;
  int* counter;
  int* err;
};

__global__ void gs2d_kernel(GsArgs g) {
  extern __shared__ __align__(16) double reg[];
  __shared__ int s_tile;
  const int tid = threadIdx.x;
  const int nthr = g.bt * g.bx;
  for (;;) {
    if (tid == 0) s_tile = atomicAdd(g.counter, 1);
    __syncthreads();
    const int tile = s_tile;
    if (tile >= g.ntiles) return;
    const int tb = g.tiles[tile * 3 + 0], xb = g.tiles[tile * 3 + 1], yb = g.tiles[tile * 3 + 2];
    if (tid < 8) {
      const int p = g.preds[tile * 8 + tid];
      if (p >= 0)
        spin_flag(g.flags + p, g.err);
    }
    __syncthreads();
    const int64_t t0 = 1 + int64_t(tb) * g.bt;
    const int64_t x0 = 2 + int64_t(xb) * g.bx;
    const int64_t y0 = 4 + int64_t(yb) * g.by;
    // region: i in [I0, I0+ni), s = i+j in [S0, S0+ns)
    const int64_t I0 = x0 - t0 - g.bt;
    const int64_t S0 = y0 - 2 * t0 - 2 * g.bt;
    for (int e = tid; e < g.ni * g.ns; e += nthr) {
      const int r = e / g.ns, c = e - r * g.ns;
      const int64_t i = I0 + r;
      const int64_t j = S0 + c - i;
      double v = 0.0;
      if (i >= 0 && i < g.n && j >= 0 && j < g.n) v = ld_cg(g.a + i * g.ld + j);
      reg[e] = v;
    }
    __syncthreads();
    const int tt = tid / g.bx, xx = tid - (tid / g.bx) * g.bx;
    const int64_t t = t0 + tt, x = x0 + xx, i = x - t;
    const bool line_ok = t <= g.T && i >= 1 && i <= g.n - 2;
    const int nclk = g.bt + g.bx + g.by - 2;
    const int ri = int(i - I0);
    for (int clk = 0; clk < nclk; ++clk) {
      const int yy = clk - tt - xx;
      if (line_ok && yy >= 0 && yy < g.by) {
        const int64_t y = y0 + yy;
        const int64_t s = y - 2 * t;
        const int64_t j = s - i;
        if (j >= 1 && j <= g.n - 2) {
          const int cs = int(s - S0);
          const double* up = reg + (ri - 1) * g.ns + cs;
          double* me = reg + ri * g.ns + cs;
          const double* dn = reg + (ri + 1) * g.ns + cs;
          double acc = add(up[-2], up[-1]);
          acc = add(acc, up[0]);
          acc = add(acc, me[-1]);
          acc = add(acc, me[0]);
          acc = add(acc, me[1]);
          acc = add(acc, dn[0]);
          acc = add(acc, dn[1]);
          acc = add(acc, dn[2]);
          const double v = div9(acc);
          me[0] = v;
          g.a[i * g.ld + j] = v;
        }
      }
      __syncthreads();
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_release(g.flags + tile, 1);
  }
}

// One warp per tile (bt * bx == 32): the per-clock ordering is a __syncwarp
// instead of a CTA barrier, the line's own previous value stays in a
// register (off the shared-memory round trip), and only the final version of
// every cell the tile wrote goes back to global memory (a byte mask marks
// written cells).  Intermediate versions are consumed inside the tile only:
// by the universal occupancy vector, any version read outside the tile that
// produced it is that tile's last version of the cell.
__global__ void __launch_bounds__(32) gs2d_warp_kernel(GsArgs g) {
  extern __shared__ __align__(16) double reg[];
  const int cells = g.ni * g.ns;
  unsigned char* wr = reinterpret_cast<unsigned char*>(reg + cells);
  const int lane = threadIdx.x;
  const int tt = lane / g.bx, xx = lane - (lane / g.bx) * g.bx;
  const int nclk = g.bt + g.bx + g.by - 2;
  for (;;) {
    int tile = 0;
    if (lane == 0) tile = atomicAdd(g.counter, 1);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= g.ntiles) return;
    const int tb = g.tiles[tile * 3 + 0], xb = g.tiles[tile * 3 + 1], yb = g.tiles[tile * 3 + 2];
    if (lane < 8) {
      const int p = g.preds[tile * 8 + lane];
      if (p >= 0)
        spin_flag(g.flags + p, g.err);
    }
    __syncwarp();
    const int t0 = 1 + tb * g.bt;
    const int x0 = 2 + xb * g.bx;
    const int y0 = 4 + yb * g.by;
    const int I0 = x0 - t0 - g.bt;
    const int S0 = y0 - 2 * t0 - 2 * g.bt;
#pragma unroll 8
    for (int e = lane; e < cells; e += 32) {
      const int r = e / g.ns, c = e - r * g.ns;
      const int i = I0 + r, j = S0 + c - i;
      double v = 0.0;
      if (i >= 0 && i < g.n && j >= 0 && j < g.n) v = ld_cg(g.a + int64_t(i) * g.ld + j);
      reg[e] = v;
      wr[e] = 0;
    }
    __syncwarp();
    const int t = t0 + tt, i = x0 + xx - t;
    const bool line_ok = t <= g.T && i >= 1 && i <= g.n - 2;
    const int ri = i - I0;
    // s = y - 2t = y0 + clk - tt - xx - 2t ; column in the region = s - S0
    const int cs0 = y0 - tt - xx - 2 * t - S0;  // region column at clk = 0
    const int j0 = y0 - tt - xx - 2 * t - i;     // j at clk = 0
    double* row = reg + ri * g.ns;
    double prev = 0.0;
    bool have_prev = false;
    for (int clk = 0; clk < nclk; ++clk) {
      const int yy = clk - tt - xx;
      const int j = j0 + clk;
      if (line_ok && yy >= 0 && yy < g.by && j >= 1 && j <= g.n - 2) {
        const int cs = cs0 + clk;
        const double* up = row - g.ns + cs;
        double* me = row + cs;
        const double* dn = row + g.ns + cs;
        const double b = have_prev ? prev : me[-1];
        double acc = add(up[-2], up[-1]);
        acc = add(acc, up[0]);
        acc = add(acc, b);
        acc = add(acc, me[0]);
        acc = add(acc, me[1]);
        acc = add(acc, dn[0]);
        acc = add(acc, dn[1]);
        acc = add(acc, dn[2]);
        const double v = div9(acc);
        me[0] = v;
        wr[ri * g.ns + cs] = 1;
        prev = v;
        have_prev = true;
      } else {
        have_prev = false;
      }
      __syncwarp();
    }
    for (int e = lane; e < cells; e += 32) {
      if (wr[e]) {
        const int r = e / g.ns, c = e - r * g.ns;
        const int ii = I0 + r, jj = S0 + c - ii;
        g.a[int64_t(ii) * g.ld + jj] = reg[e];
      }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(g.flags + tile, 1);
  }
}

// ---------------------------------------------------------------------------
// Line-group kernel: one warp per tile of 4 time levels x 32 lines (x), each
// lane owning G = 4 adjacent lines of one time level: lane = tt * 8 + xg,
// lines x0 + 4*xg + q.  Clock h: line (t, x) processes y = y0 + h - tt -
// (x - x0), a legal schedule (all dependence distances have positive
// coordinate sum).  Every value a line needs was produced at clocks h-1..h-4
// by this lane (own lines q-1, q), by lane-8 (t-1, same lines), lane-1
// (t, line x-1) or lane-9 (t-1, line x-1): kept in register histories fed by
// warp shuffles — no block barrier, one __syncwarp per clock for the shared
// tile region (which holds the halo read by boundary lanes and the values
// written back at the end).  A point outside the tile/grid contributes its
// cell's current region value ("virtual output"), which is the right version
// wherever it is consumed (same UOV argument as the tile schedule).
namespace lines {

constexpr int BT = 4, G = 4, NXG = 8, BX = G * NXG;  // 4 x 32 lines per warp

struct Hist {
  double o[G][4];   // own lines, clocks h-1..h-4 (index = clock mod 4)
  double d[G][4];   // lane-8: (t-1, x_q)
  double l[4];      // lane-1: (t, x_0 - 1)
  double dl[4];     // lane-9: (t-1, x_0 - 1)
};

// Region read with the column guarded: lines far outside their valid clock
// range index past the region; such values are never consumed.
PCOT_DEV double rd(const double* reg, int row_base, int col, int ns) {
  return (col >= 0 && col < ns) ? reg[row_base + col] : 0.0;
}

template <int P>  // P = h mod 4 (static ring index)
PCOT_DEV void clock(Hist& H, int h, const GsArgs& g, double* reg, unsigned char* wr,
                    const int (&pr)[G], const int (&pc)[G], const int (&hlo)[G],
                    const int (&hhi)[G], int tt, int xg, int ns) {
  constexpr int M1 = (P + 3) & 3, M2 = (P + 2) & 3, M3 = (P + 1) & 3, M4 = P & 3;
  // neighbours' outputs of clock h-1
#pragma unroll
  for (int q = 0; q < G; ++q) {
    double v = __shfl_up_sync(0xffffffffu, H.o[q][M1], 8);
    if (tt == 0) v = rd(reg, pr[q] + ns, pc[q] + h + 2, ns);  // (t0-1, x_q, y_q): halo
    H.d[q][M1] = v;
  }
  {
    double v = __shfl_up_sync(0xffffffffu, H.o[G - 1][M1], 1);
    if (xg == 0) v = rd(reg, pr[0] - ns, pc[0] + h, ns);  // (t, x0-1, y_0)
    H.l[M1] = v;
    double w = __shfl_up_sync(0xffffffffu, H.o[G - 1][M1], 9);
    if (tt == 0 || xg == 0) w = rd(reg, pr[0], pc[0] + h + 3, ns);  // (t-1, x0-1, y_0 + 1)
    H.dl[M1] = w;
  }
#pragma unroll
  for (int q = 0; q < G; ++q) {
    const int col = pc[q] + h;
    double out;
    if (h >= hlo[q] && h < hhi[q]) {
      const int cell = pr[q] + col;
      const double a1 = q ? H.o[q - 1][M3] : H.l[M3];
      const double a2 = q ? H.o[q - 1][M2] : H.l[M2];
      const double a3 = q ? H.o[q - 1][M1] : H.l[M1];
      const double c1 = q ? H.d[q - 1][M4] : H.dl[M4];
      const double c2 = q ? H.d[q - 1][M3] : H.dl[M3];
      double s = add(a1, a2);
      s = add(s, a3);
      s = add(s, H.o[q][M1]);
      s = add(s, c1);
      s = add(s, c2);
      s = add(s, H.d[q][M3]);
      s = add(s, H.d[q][M2]);
      s = add(s, H.d[q][M1]);
      out = div9(s);
      reg[cell] = out;
      wr[cell] = 1;
    } else {
      out = rd(reg, pr[q], col, ns);
    }
    H.o[q][M4] = out;  // becomes "h-1" at the next clock (slot h mod 4)
  }
  __syncwarp();
}

__global__ void __launch_bounds__(32) gs2d_lines_kernel(GsArgs g) {
  extern __shared__ __align__(16) double reg[];
  const int cells = g.ni * g.ns;
  unsigned char* wr = reinterpret_cast<unsigned char*>(reg + cells);
  const int lane = threadIdx.x;
  const int tt = lane / NXG, xg = lane - (lane / NXG) * NXG;
  const int nclk = BT + BX + g.by - 2;
  for (;;) {
    int tile = 0;
    if (lane == 0) tile = atomicAdd(g.counter, 1);
    tile = __shfl_sync(0xffffffffu, tile, 0);
    if (tile >= g.ntiles) return;
    const int tb = g.tiles[tile * 3 + 0], xb = g.tiles[tile * 3 + 1], yb = g.tiles[tile * 3 + 2];
    if (lane < 8) {
      const int p = g.preds[tile * 8 + lane];
      if (p >= 0)
        spin_flag(g.flags + p, g.err);
    }
    __syncwarp();
    const int t0 = 1 + tb * BT, x0 = 2 + xb * BX, y0 = 4 + yb * g.by;
    const int I0 = x0 - t0 - BT, S0 = y0 - 2 * t0 - 2 * BT;
#pragma unroll 8
    for (int e = lane; e < cells; e += 32) {
      const int r = e / g.ns, c = e - r * g.ns;
      const int i = I0 + r, j = S0 + c - i;
      double v = 0.0;
      if (i >= 0 && i < g.n && j >= 0 && j < g.n) v = ld_cg(g.a + int64_t(i) * g.ld + j);
      reg[e] = v;
      wr[e] = 0;
    }
    __syncwarp();
    const int t = t0 + tt;
    int pr[G], pc[G], hlo[G], hhi[G];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int x = x0 + G * xg + q, i = x - t;
      // y(h) = y0 + h - tt - (x - x0); s = y - 2t; region cell = (i - I0, s - S0)
      const int yoff = y0 - tt - (x - x0);
      pr[q] = (i - I0) * g.ns;
      pc[q] = yoff - 2 * t - S0;  // + h
      // valid: t <= T, 1 <= i <= n-2, y0 <= y < y0 + by, 1 <= j = y - x - t <= n-2
      int lo = tt + (x - x0), hi = lo + g.by;
      const int jlo = 1 + x + t - yoff, jhi = g.n - 2 + x + t - yoff + 1;
      lo = lo > jlo ? lo : jlo;
      hi = hi < jhi ? hi : jhi;
      if (t > g.T || i < 1 || i > g.n - 2) hi = lo;  // empty
      hlo[q] = lo;
      hhi[q] = hi;
    }
    Hist H;
    // warm-up clocks -4..-1: every lane is outside the tile, histories fill
    // with region values (only y >= y0 - 2 entries are ever consumed)
    int h = -4;
    clock<0>(H, h, g, reg, wr, pr, pc, hlo, hhi, tt, xg, g.ns);
    clock<1>(H, h + 1, g, reg, wr, pr, pc, hlo, hhi, tt, xg, g.ns);
    clock<2>(H, h + 2, g, reg, wr, pr, pc, hlo, hhi, tt, xg, g.ns);
    clock<3>(H, h + 3, g, reg, wr, pr, pc, hlo, hhi, tt, xg, g.ns);
    for (h = 0; h < nclk; h += 4) {
      clock<0>(H, h, g, reg, wr, pr, pc, hlo, hhi, tt, xg, g.ns);
      clock<1>(H, h + 1, g, reg, wr, pr, pc, hlo, hhi, tt, xg, g.ns);
      clock<2>(H, h + 2, g, reg, wr, pr, pc, hlo, hhi, tt, xg, g.ns);
      clock<3>(H, h + 3, g, reg, wr, pr, pc, hlo, hhi, tt, xg, g.ns);
    }
    for (int e = lane; e < cells; e += 32) {
      if (wr[e]) {
        const int r = e / g.ns, c = e - r * g.ns;
        const int ii = I0 + r, jj = S0 + c - ii;
        g.a[int64_t(ii) * g.ld + jj] = reg[e];
      }
    }
    __threadfence();
    __syncwarp();
    if (lane == 0) st_release(g.flags + tile, 1);
  }
}

}  // namespace lines

// ---------------------------------------------------------------------------
// Systolic pipeline kernel.  One CTA per band of 32 rows; its NW warps hold NW
// consecutive sweeps (time levels) at once: warp w runs t = w+1, w+1+NW, ...
// Lane l of a warp at clock c updates column j = c - 2l of its row (row i
// needs row i-1 one column ahead, (t, i-1, j+1), so the warp sweeps its rows
// as a skewed wavefront with no barrier at all).
//
// The band's row window moves up one row per level: at level t (1-based
// inside a launch) band b owns rows i0 - (t-1) .. i0 - (t-1) + 31, i0 = 1+32b.
// Then every input of lane l comes from this band or the band above:
//   A (t, i-1, j-1..j+1): lane l-1 (shuffle); lane 0: band b-1's last row;
//   B (t, i, j-1): own previous output;
//   C (t-1, i, j..j+1): producer warp's lane l-1 (lane 0: band b-1's last row
//     at level t-1, or the input row i0 at t = 1);
//   D (t-1, i+1, j-1..j+1): producer warp's lane l;
// so the bands form a one-way chain (band b waits only for band b-1) and the
// pipeline has no cross-band cycle to throttle it.  Warps hand rows over in
// shared-memory rings (consumer waits for its producer; producer waits for
// ring reuse); the last warp's levels go to a global wrap buffer that feeds
// warp 0's next level (no back-pressure around the ring of warps).  Each
// band's last row per level is published in write-once global slots that the
// band below polls as data.  The window drift costs (T-1)/32 extra bands, so
// long runs are split into launches of at most Tseg levels (host side).
// Level T writes the result in place.  All CTAs must be co-resident.
namespace pipe {

// NW warps (= pipelined levels) per CTA, RS-entry producer rings.
constexpr int IRS = 64, SG = 64;  // S (clocks per chunk) is a template parameter
#ifndef PCOT_XLOAD_CLOCK
#define PCOT_XLOAD_CLOCK 3
#endif
constexpr int kXLoadClock = PCOT_XLOAD_CLOCK;  // clock of the chunk that issues the next edge load
constexpr int BIG = 1 << 20;  // progress = level * BIG + completed clocks

struct PipeArgs {
  double* a;        // in-place grid: level 0 at launch, level T at exit
  double* wb[2];    // wrap-level buffers (grid-shaped, pitch ld)
  double* eb;       // last row per (level, band): [((t-1) * nb + b) * ebld + j], kEmpty until written
  int64_t ld;
  int64_t ebld;     // edge-row stride (even, >= n + 2)
  int n, T, nb;
  int nclk;         // clocks per level (c = -1 .. n + 61)
  long long* prof;  // optional per-warp counters [nb * NW][16] (PCOTGPU_GS_PROF dev aid)
  int spin_ns;      // edge-poll backoff cap (ns)
  int* err;         // fault word (spin cap hit)
  int* gprog;       // H > 1: per-CTA progress of its last warp, gpu scope [nb * H]
  int wait_ns;      // sleep per poll of a warp-to-warp progress wait
};

// CTA-scope acquire/release on the shared-memory progress words: the acquire
// load is a plain LDS (no fence), the release a CTA membar + STS.
PCOT_DEV int vld(const volatile int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.s32 %0, [%1];"
               : "=r"(v)
               : "r"(smem_u32(const_cast<const int*>(p)))
               : "memory");
  return v;
}
PCOT_DEV void st_release_cta(volatile int* p, int v) {
  asm volatile("st.release.cta.shared.s32 [%0], %1;" ::"r"(smem_u32(const_cast<const int*>(p))),
               "r"(v)
               : "memory");
}

// Spins are bounded (~seconds): a scheduling bug or lost co-residency then
// sets the fault word (the run fails with an error) instead of hanging the
// device or returning a silently wrong grid.
constexpr long long kSpinCap = 40000000LL;
PCOT_DEV void spin_fault(int* err) {
  if ((threadIdx.x & 31) == 0) atomicOr(err, 1);
}

// Waits are executed by the whole warp (every lane reads the same word, one
// transaction) and exit on a warp vote: a lane-0-only spin leaves the warp
// diverged and every later shuffle takes the compiler's slow collective path.
PCOT_DEV void wait_smem(const volatile int* p, int target, int* err, int ns = 8) {
  long long it = 0;
  for (; !__all_sync(0xffffffffu, vld(p) >= target) && it < kSpinCap; ++it) __nanosleep(ns);
  if (it == kSpinCap) spin_fault(err);
}

// Same wait through a per-warp cache of the last value seen: progress words
// only grow, and an earlier acquire of a value >= target already orders the
// reads that need it, so a producer running ahead costs no shared load.
PCOT_DEV void wait_seen(const volatile int* p, int target, int& seen, int* err, int ns = 8) {
  if (seen >= target) return;
  int v = vld(p);
  long long it = 0;
  for (; !__all_sync(0xffffffffu, v >= target) && it < kSpinCap; ++it) {
    __nanosleep(ns);
    v = vld(p);
  }
  if (it == kSpinCap) spin_fault(err);
  seen = v;
}

// gpu-scope progress (split bands, H > 1): acquire loads by the whole warp.
PCOT_DEV int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
PCOT_DEV void wait_global(const int* p, int target, int& seen, int* err) {
  if (seen >= target) return;
  int v = ld_acquire_gpu(p);
  long long it = 0;
  for (; !__all_sync(0xffffffffu, v >= target) && it < kSpinCap; ++it) {
    __nanosleep(64);
    v = ld_acquire_gpu(p);
  }
  if (it == kSpinCap) spin_fault(err);
  seen = v;
}

// Cross-CTA edge values are polled as data: every slot of the edge arrays
// starts as kEmpty (bytes 0xff, a NaN bit pattern the arithmetic never
// produces — the device returns the canonical NaN 0x7fff...) and is written
// exactly once per run, so a non-empty value is final.  No progress counters,
// no gpu-scope fences: the producer's relaxed store and the consumer's
// relaxed load of the same 8-byte word are the whole protocol.
constexpr long long kEmpty = -1LL;
PCOT_DEV double ld_relaxed(const double* p) {
  double v;
  // no "memory" clobber: a write-once slot needs no ordering with the other
  // accesses, and the load may then be scheduled inside the clock loop
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
PCOT_DEV void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
PCOT_DEV bool is_empty(double v) { return __double_as_longlong(v) == kEmpty; }

// Predicated stores without a branch (SASS @P STG): a per-lane `if` around a
// store inside the clock loop makes the warp diverge, and every later shuffle
// then takes the compiler's collective slow path (WARPSYNC / ENDCOLLECTIVE).
PCOT_DEV void st_relaxed_if(double* p, double v, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.relaxed.gpu.global.f64 [%0], %1;\n}" ::"l"(p),
      "d"(v), "r"(int(pred)));
}
PCOT_DEV void st_global_if(double* p, double v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}" ::"l"(p),
               "d"(v), "r"(int(pred)));
}
// Same with a compile-time element offset folded into the address ([base+imm]):
// one base register per chunk instead of a 64-bit address per store.
template <int OFF>
PCOT_DEV void st_relaxed_if_at(double* base, double v, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.relaxed.gpu.global.f64 [%0+%3], %1;\n}" ::"l"(base),
      "d"(v), "r"(int(pred)), "n"(OFF * 8));
}
template <int OFF>
PCOT_DEV void st_global_if_at(double* base, double v, bool pred) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0+%3], %1;\n}" ::"l"(base),
               "d"(v), "r"(int(pred)), "n"(OFF * 8));
}
// Compile-time unrolled loop: f(std::integral_constant<int, i>) for i in [0, N).
template <int N, class F>
PCOT_DEV void static_for(F&& f) {
  if constexpr (N > 0) {
    static_for<N - 1>(f);
    f(std::integral_constant<int, N - 1>{});
  }
}

// Bits kk in [0, S) with lo <= j0 + kk <= hi.
template <int S>
PCOT_DEV unsigned span_mask(int j0, int lo, int hi) {
  const int klo = max(0, lo - j0), khi = min(S - 1, hi - j0);
  if (klo > khi) return 0u;
  return ((2u << khi) - 1u) & ~((1u << klo) - 1u);
}

// H > 1 splits a band over H CTAs (H x NW warps, level groups of NW levels
// dealt round-robin: CTA h runs groups h, h+H, ...), so the band's work per
// clock spreads over H SMs and the SMs of early and late bands of the
// wavefront overlap; the group-to-group rows go through the wrap buffers (as
// between passes), ordered by a gpu-scope progress word that an extra
// publisher warp mirrors from the last warp's shared-memory progress (the
// release fence stays off the compute warps).
template <int NW, int RS, int S, int H = 1>
__global__ void __launch_bounds__((NW + (H > 1)) * 32, H > 1 ? 2 : 1) gs2d_pipe_kernel(PipeArgs g) {
  static_assert(2 * S <= 32 && 3 * S + 4 <= IRS && S + 2 <= SG / 2, "chunk size");
  constexpr int RSP = RS + 1;  // odd lane pitch: ring accesses are bank-conflict free
  extern __shared__ __align__(16) double sm[];
  double* rb = sm;                              // [NW][32][RSP] producer rings
  double* ir = rb + NW * 32 * RSP;              // [32][IRS] warp 0's staged level t-1 rows
  double* above = ir + 32 * IRS;                // [NW][SG] band b-1's last row, level t
  double* cabove = above + NW * SG;             // [NW][SG] same row, level t-1 (lane 0's C)
  volatile int* prog = reinterpret_cast<volatile int*>(cabove + NW * SG);  // [NW]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int b = H > 1 ? int(blockIdx.x) / H : int(blockIdx.x);
  const int h = H > 1 ? int(blockIdx.x) % H : 0;
  const int i0 = 1 + 32 * b;
  const bool has_above = b > 0;
  if (lane == 0 && w < NW) prog[w] = 0;
  __syncthreads();
  const int nclk_all = ((g.nclk + S - 1) / S) * S - 1;  // every warp's final published clock count
  if constexpr (H > 1) {
    if (w == NW) {  // publisher: mirror the last warp's progress to gpu scope
      int* gp = g.gprog + blockIdx.x;
      int last = 0;
      for (int t = 1 + h * NW + NW - 1; t <= g.T; t += NW * H) {
        const int done = t * BIG + nclk_all;
        for (long long it = 0; last < done && it < kSpinCap; ++it) {
          int v = vld(prog + NW - 1);
          v = __shfl_sync(0xffffffffu, v, 0);
          if (v >= last + 4 * S || v >= done) {  // every 4 chunks and at the level's end
            __threadfence();  // the last warp's wrap-buffer rows before the progress
            if (lane == 0) st_release(gp, v);
            last = v;
          } else {
            __nanosleep(200);
          }
        }
      }
      return;
    }
  }
  double* myring = rb + (w * 32 + lane) * RSP;
  // edge-fetch roles: lanes [0, S) fetch a chunk's A columns (c+1) of band
  // b-1's last row at level t, lanes [S, 2S) the same columns at level t-1
  const bool xa = lane < S, xc = lane >= S && lane < 2 * S;
  double* xring = (xa ? above : cabove) + w * SG;
  const double* ab = above + w * SG;
  const double* cab = cabove + w * SG;
  // producer rows: warp w-1's rings, or (warp 0) the staged wrap rows; the
  // C-term of lane l is producer lane l-1 (lane 0: cab), the D-term lane l
  const double* prowD = w ? rb + ((w - 1) * 32 + lane) * RSP : ir + lane * IRS;
  const double* prowC = lane == 0 ? cab
                                  : (w ? rb + ((w - 1) * 32 + lane - 1) * RSP : ir + (lane - 1) * IRS);
  const int dmask = w ? RS - 1 : IRS - 1;
  const int cmask = lane == 0 ? SG - 1 : dmask;
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int seen_prod = 0, seen_cons = 0, seen_wrap = 0;  // progress words last observed
  long long t_first = 0, c_first = 0;  // globaltimer / clock64 at the first compute (prof)
  const long long t_entry = g.prof ? globaltimer() : 0;
  for (int t = 1 + h * NW + w; t <= g.T; t += NW * H) {
    const int i = i0 - (t - 1) + lane;  // this lane's row at level t
    const bool row_ok = i >= 1 && i <= g.n - 2;
    // (selects, not g.wb[k]: a dynamic index into the parameter struct puts it
    // in local memory)
    const double* src0 = ((((t - 1) / NW) & 1) ? g.wb[1] : g.wb[0]);  // warp 0, t > 1
    double* wb_out = ((t / NW) & 1) ? g.wb[1] : g.wb[0];              // warp NW-1 only
    const double* eb_t = g.eb + (int64_t(t - 1) * g.nb + (b - 1)) * g.ebld;  // band b-1, level t
    const double* xrow = xa ? eb_t : (t == 1 ? g.a + int64_t(i0) * g.ld : eb_t - g.nb * g.ebld);
    const bool xlive = xa ? has_above : (xc && (t == 1 ? i0 <= g.n - 1 : has_above));
    const bool xpoll = xlive && (xa || t > 1);  // level 0 is the input grid
    double* eb_mine = g.eb + (int64_t(t - 1) * g.nb + b) * g.ebld;
    const int lvl = t * BIG, plvl = (t - 1) * BIG, clvl = (t + 1) * BIG;
    const int nchunk = (g.nclk + S - 1) / S;
    // every producer publishes at most `fin` (its last chunk's clock + 1)
    const int fin = ((g.nclk + S - 1) / S) * S - 1;
    auto need = [&](int v) { return v < fin ? v : fin; };
    auto xcol = [&](int k) { return k * S + (xa ? lane : lane - S); };
    auto xload = [&](int k) {
      const int col = xcol(k);
      double v = 0.0;
      if (xlive && col >= 0 && col < g.n) v = xpoll ? ld_relaxed(xrow + col) : xrow[col];
      return v;
    };
    // wait until chunk k's edge values are all non-empty, then stage them
    auto xresolve = [&](int k, double v) {
      const int col = xcol(k);
      const bool mine = xpoll && col >= 0 && col < g.n;
      unsigned ns = 16;
      long long it = 0;
      for (; __any_sync(0xffffffffu, mine && is_empty(v)) && it < kSpinCap; ++it) {
        if (g.spin_ns) __nanosleep(ns);
        ns = ns * 2 < unsigned(g.spin_ns) ? ns * 2 : unsigned(g.spin_ns);
        if (mine && is_empty(v)) v = ld_relaxed(xrow + col);
      }
      if (it == kSpinCap) spin_fault(g.err);
      if ((xa || xc) && col >= 0 && col < g.n) xring[col & (SG - 1)] = v;
    };
    // warp 0: lane q stages level t-1 row i0 - t + 2 + q (the last warp's
    // lane q one level earlier).  Chunk k reads columns [kS-2-2q, kS+S-1-2q]
    // (S+2, even-aligned); the first pair was staged with chunk k-1, so a
    // chunk copies S/2 new 16-byte pairs (chunk 0 one more).
    const int srow = i0 - t + 2 + lane;
    const bool srow_ok = srow >= 0 && srow <= g.n - 1;
    const double* const srcrow = (t == 1 ? g.a : src0) + int64_t(srow) * g.ld;
    double* const irow = ir + lane * IRS;
    // Register-staged copy (loads issued a chunk ahead, stored to the ring at
    // the chunk's start): chunk k needs pairs m = 1..S/2 (m = 0 too at k = 0).
    auto load_pair = [&](int k, int m) {
      const int p = k * S - 2 - 2 * lane + 2 * m;
      double2 v = make_double2(0.0, 0.0);
      if (srow_ok && p >= 0 && p < g.n) v = __ldcg(reinterpret_cast<const double2*>(srcrow + p));
      return v;
    };
    auto store_pair = [&](int k, int m, double2 v) {
      const int p = k * S - 2 - 2 * lane + 2 * m;
      if (p >= 0 && p < g.n) *reinterpret_cast<double2*>(irow + (p & (IRS - 1))) = v;
    };
    double2 pre[S / 2];  // warp 0: chunk k+1's new pairs, in flight during chunk k
    // producer of warp 0's level t-1: this CTA's last warp (H = 1), or the
    // previous group's CTA (gpu scope)
    const int* gprod = H > 1 ? g.gprog + b * H + (h + H - 1) % H : nullptr;
    if (w == 0) {
      if (t > 1) {
        if (H > 1) wait_global(gprod, plvl + need(S - 2 + 2), seen_wrap, g.err);
        else wait_smem(prog + NW - 1, plvl + need(S - 2 + 2), g.err, g.wait_ns);
      }
      store_pair(0, 0, load_pair(0, 0));
#pragma unroll
      for (int m = 1; m <= S / 2; ++m) pre[m - 1] = load_pair(0, m);
    }
    // per-level lane roles of the clock loop
    const bool last = t == g.T;
    const bool wrap_writer = w == NW - 1 && !last && i >= 0 && i <= g.n - 1;
    double* const orow = (last ? g.a : wb_out) + int64_t(i) * g.ld;
    const bool elane = lane == 31;  // publishes the band's last row
    double a1 = 0, a2 = 0, a3 = 0, c1 = 0, c2 = 0, d1 = 0, d2 = 0, d3 = 0, out = 0;
    double xv = xload(0);
    for (int k = 0; k < nchunk; ++k) {
      const int c_lo = k * S - 1;
      const int c_hi = c_lo + S - 1;
      long long tp = g.prof ? clock64() : 0;
#define PCOT_PROF(slot)                                   \
  if (g.prof) {                                           \
    const long long now = clock64();                      \
    pacc[slot] += now - tp;                               \
    tp = now;                                             \
  }
      // Chunk k's edge values (band b-1 only: the wait chain is acyclic).
      xresolve(k, xv);
      PCOT_PROF(0);
      if (w == 0) {
#pragma unroll
        for (int m = 1; m <= S / 2; ++m) store_pair(k, m, pre[m - 1]);
        if (k + 1 < nchunk) {
          if (t > 1) {
            if (H > 1) wait_global(gprod, plvl + need(c_hi + S + 2), seen_wrap, g.err);
            else wait_seen(prog + NW - 1, plvl + need(c_hi + S + 2), seen_wrap, g.err, g.wait_ns);
          }
          PCOT_PROF(1);
#pragma unroll
          for (int m = 1; m <= S / 2; ++m) pre[m - 1] = load_pair(k + 1, m);
        }
      }
      PCOT_PROF(7);
      // producer ahead: D of clock c is producer lane l's column j+1, computed
      // at the producer's clock c+1
      if (w > 0) wait_seen(prog + w - 1, plvl + need(c_hi + 2), seen_prod, g.err, g.wait_ns);
      PCOT_PROF(2);
      if (w < NW - 1) {
        // ring reuse: the consumer (level t+1) must have read what this chunk
        // overwrites; before it starts level t+1 its previous level's reads
        // (of our level t-NW data) must be over — also when there is no level
        // t+1, since every slot is written, out-of-range columns included.
        const int rel = c_hi + 1 - (RS - 4);
        if (rel > 0) {
          if (t + 1 <= g.T) wait_seen(prog + w + 1, clvl + need(rel), seen_cons, g.err, g.wait_ns);
        } else if (t + 1 - NW * H >= 1) {  // the consumer's previous level in this CTA
          wait_seen(prog + w + 1, (t + 1 - NW * H) * BIG + fin, seen_cons, g.err, g.wait_ns);
        }
      }
      PCOT_PROF(3);
      __syncwarp();
      PCOT_PROF(4);
      if (g.prof && t_first == 0) {
        t_first = globaltimer();
        c_first = clock64();
      }
      // Branch-free clock loop (S clocks, fully unrolled): per-lane bit masks
      // over the chunk's clocks replace the per-cell tests, so consecutive
      // clocks' independent work can overlap the serial sum chain.
      const int j0 = c_lo - 2 * lane;  // this lane's column at the chunk's first clock
      const unsigned inb = span_mask<S>(j0, 0, g.n - 1);                // 0 <= j <= n-1
      const unsigned upd = row_ok ? span_mask<S>(j0, 1, g.n - 2) : 0u;  // updated cells
      const unsigned omask = last ? upd : (wrap_writer ? inb : 0u);
      double* const op = orow + j0;
      double* const ep = eb_mine + j0;
      const unsigned emask = elane ? inb : 0u;
      auto clocks = [&](auto OUT) {
      constexpr bool kOut = decltype(OUT)::value;
      static_for<S>([&](auto KK) {
        constexpr int kk = decltype(KK)::value;
        // next chunk's edge values: loaded part-way through this chunk, late
        // enough to be fresh, early enough to land before the next resolve
        if (kk == kXLoadClock && k + 1 < nchunk) xv = xload(k + 1);
        const int q = j0 + kk + 1;
        const double sh = __shfl_up_sync(0xffffffffu, out, 1);
        const double ev = ab[q & (SG - 1)];  // lane 0's band-above value (same address for all)
        a1 = a2;
        a2 = a3;
        a3 = lane ? sh : ev;
        c1 = c2;
        c2 = prowC[q & cmask];
        d1 = d2;
        d2 = d3;
        d3 = prowD[q & dmask];
        double s = add(a1, a2);
        s = add(s, a3);
        s = add(s, out);
        s = add(s, c1);
        s = add(s, c2);
        s = add(s, d1);
        s = add(s, d2);
        s = add(s, d3);
        const double r = div9(s);
        const double v = (upd >> kk) & 1u ? r : 0.0;
        out = v;
        // every column's slot, in range or not: out-of-range slots are only
        // read by consumer cells that are themselves not updated
        myring[(j0 + kk) & (RS - 1)] = v;
        // lane 31: the band's last row (a computed NaN carrying the kEmpty bit
        // pattern would read as "not yet written": stored as the canonical NaN)
        // (computed values never carry the kEmpty pattern: NaNs come only from
        // input NaNs, whose payload the arithmetic propagates, and the copy-in
        // maps the sentinel pattern to its neighbour NaN — copy_rows_nosentinel;
        // test_gs2d_pipeline_nan_input_with_sentinel_bits)
        st_relaxed_if_at<kk>(ep, v, (emask >> kk) & 1u);
        // result / wrap buffer: only the last level's warps and the CTA's last
        // warp store here; the other warps run a body without the predicate
        // arithmetic and the predicated-off store (4 of 31 instructions)
        if constexpr (kOut) st_global_if_at<kk>(op, v, (omask >> kk) & 1u);
      });
      };
      if (last || w == NW - 1)
        clocks(std::true_type{});
      else
        clocks(std::false_type{});
      PCOT_PROF(5);
#ifdef PCOT_EDGE_FENCE
      __threadfence();
#endif
      // publish progress: ring (smem) and wrap-buffer writes are read by other
      // warps of this CTA only -> CTA-scope release of the counter (lane 0's
      // release covers the warp's writes through the __syncwarp)
      __syncwarp();
      if (lane == 0) st_release_cta(prog + w, lvl + c_hi + 1);
      __syncwarp();
      PCOT_PROF(6);
#undef PCOT_PROF
    }
    __syncwarp();
  }
  if (g.prof && lane == 0)
    for (int q = 0; q < 8; ++q) g.prof[(int64_t(blockIdx.x) * NW + w) * 16 + q] = pacc[q];
  if (g.prof && lane == 0) {
    g.prof[(int64_t(blockIdx.x) * NW + w) * 16 + 8] = t_first;
    g.prof[(int64_t(blockIdx.x) * NW + w) * 16 + 9] = globaltimer();
    g.prof[(int64_t(blockIdx.x) * NW + w) * 16 + 10] = c_first;
    g.prof[(int64_t(blockIdx.x) * NW + w) * 16 + 11] = clock64();
    g.prof[(int64_t(blockIdx.x) * NW + w) * 16 + 12] = t_entry;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g.prof[(int64_t(blockIdx.x) * NW + w) * 16 + 13] = smid;
  }
}

}  // namespace pipe

// ---------------------------------------------------------------------------
// Systolic pipeline, K levels per warp (v2).  Same bands, drifting windows,
// edge slots, rings and wrap buffers as gs2d_pipe_kernel, but every warp
// carries K consecutive levels t0 .. t0+K-1 in registers: lane l at clock c
// updates, for every kk, row i0 - (t0+kk-1) + l at column c - 2l - 2kk.  Level
// kk+1 then needs only values its own lane or its upper neighbour produced at
// least one clock earlier:
//   A (t, r-1, j-1..j+1): upper neighbour, level kk, clocks c-3..c-1;
//   B (t, r, j-1):        own output, clock c-1;
//   C (t-1, r, j..j+1):   upper neighbour, level kk-1, clocks c-4, c-3;
//   D (t-1, r+1, j-1..j+1): own level kk-1 outputs, clocks c-3..c-1;
// so the K updates of a clock are independent (K-way ILP), and ONE rotate
// shuffle per level and clock feeds both the A and (four clocks later) the C
// terms.  Lane 31 sends, instead of its own output (which no lane of the warp
// needs), the band-above value lane 0 needs, so lane 0 takes the same path.
// Level kk = 0 reads its C / D terms from the producer warp's ring (or warp
// 0's staged rows) exactly as the one-level kernel does.  Per update: 12 fp64
// operations + one shuffle + a few selects and predicated stores, against ~80
// instructions of the one-level kernel, whose per-chunk overhead (edge resolve,
// staging, progress) is now shared by K levels.
namespace pipe2 {

using pipe::PipeArgs;
using pipe::BIG;
using pipe::IRS;
using pipe::SG;

template <int NW, int K, int RS, int S>
__global__ void __launch_bounds__(NW * 32, 1) gs2d_pipe2_kernel(PipeArgs g) {
  static_assert(S + 2 <= SG / 2 && 3 * S + 4 <= IRS && S % 2 == 0, "chunk size");
  static_assert((K + 1) * S <= 96, "edge slots per chunk: at most three per lane");
  constexpr int RSP = RS + 1;
  constexpr int L = NW * K;  // levels per pass
  constexpr int XS = ((K + 1) * S + 31) / 32;  // edge slots per lane per chunk
  extern __shared__ __align__(16) double sm[];
  double* rb = sm;                          // [NW][32][RSP] last-level rings
  double* ir = rb + NW * 32 * RSP;          // [32][IRS] warp 0's staged rows
  double* above = ir + 32 * IRS;            // [NW][2][K][S] band b-1's last row per level (chunk-relative)
  double* cabove = above + NW * K * SG;     // [NW][SG] same row, level t0 - 1
  volatile int* prog = reinterpret_cast<volatile int*>(cabove + NW * SG);  // [NW]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, b = blockIdx.x;
  const int i0 = 1 + 32 * b;
  const bool has_above = b > 0;
  if (lane == 0) prog[w] = 0;
  __syncthreads();
  double* myring = rb + (w * 32 + lane) * RSP;
  double* const ab = above + w * K * SG;  // (SG >= 2S: the [2][K][S] staging fits the same space)
  double* const cab = cabove + w * SG;
  const double* prowD = w ? rb + ((w - 1) * 32 + lane) * RSP : ir + lane * IRS;
  const double* prowC = lane == 0 ? cab
                                  : (w ? rb + ((w - 1) * 32 + lane - 1) * RSP : ir + (lane - 1) * IRS);
  const int dmask = w ? RS - 1 : IRS - 1;
  const int cmask = lane == 0 ? SG - 1 : dmask;
  const int src_lane = (lane + 31) & 31;  // rotate: lane 0 hears lane 31
  const int nclk = g.n + 63 + 2 * (K - 1);   // clocks -1 .. n + 61 + 2(K-1)
  const int nchunk = (nclk + S - 1) / S;
  const int fin = nchunk * S - 1;            // every warp publishes at most fin
  auto need = [&](int v) { return v < fin ? v : fin; };
  int seen_prod = 0, seen_cons = 0, seen_wrap = 0;
  // optional cycle accounting (PCOTGPU_GS_PROF): same slots as the one-level kernel
  long long pacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t_first = 0, c_first = 0;
  const long long t_entry = g.prof ? globaltimer() : 0;
  long long tp = 0;
#define PCOT_PROF2(slot)            \
  if (g.prof) {                     \
    const long long now = clock64(); \
    pacc[slot] += now - tp;         \
    tp = now;                       \
  }
  for (int p = 0;; ++p) {
    const int t0 = p * L + w * K + 1;  // this warp's first level in pass p
    if (t0 > g.T) break;
    const int plv = (p + 1) * BIG;     // progress base of pass p
    const bool cons_live = w < NW - 1 && t0 + K <= g.T;  // consumer warp has pass p
    const double* src0 = ((p - 1) & 1) ? g.wb[1] : g.wb[0];  // warp 0, p > 0
    double* wb_out = (p & 1) ? g.wb[1] : g.wb[0];             // warp NW-1
    // ---- edge slots of this pass: (K+1) rows x S columns per chunk
    // slot m: row kk = m / S - 1 (-1: level t0 - 1 for lane 0's C at kk = 0),
    // column offset m % S
    const double* xrow[XS];
    int xoff[XS];
    bool xlive[XS], xpoll[XS];
    double* xdst[XS];
#pragma unroll
    for (int x = 0; x < XS; ++x) {
      const int m = lane + 32 * x;
      const int kk = m / S - 1, o = m % S;
      const bool slot = m < (K + 1) * S;
      const int t = t0 + kk;  // level of the row
      const double* row = g.eb + (int64_t(t - 1) * g.nb + (b - 1)) * g.ebld;
      bool live, poll;
      if (kk < 0) {  // lane 0's C at kk = 0: band b-1's last row at t0-1, or the input row i0
        live = slot && (t0 == 1 ? i0 <= g.n - 1 : has_above);
        poll = live && t0 > 1;
        if (t0 == 1) row = g.a + int64_t(i0) * g.ld;
        xoff[x] = o;             // columns kS .. kS + S - 1
        xdst[x] = cab;
      } else {       // lane 31's send for level kk: columns kS + 1 - 2kk ..
        live = slot && has_above && t <= g.T;
        poll = live;
        xoff[x] = o + 1 - 2 * kk;
        xdst[x] = ab + kk * S + o;  // + (k & 1) * K * S: chunk-relative, double buffered
      }
      xrow[x] = row;
      xlive[x] = live;
      xpoll[x] = poll;
    }
    auto xload = [&](int k, double* v) {
#pragma unroll
      for (int x = 0; x < XS; ++x) {
        const int col = k * S + xoff[x];
        v[x] = 0.0;
        if (xlive[x] && col >= 0 && col < g.n) v[x] = xpoll[x] ? pipe::ld_relaxed(xrow[x] + col) : xrow[x][col];
      }
    };
    auto xresolve = [&](int k, double* v) {
      unsigned ns = 16;
#pragma unroll
      for (int x = 0; x < XS; ++x) {
        const int col = k * S + xoff[x];
        const bool mine = xpoll[x] && col >= 0 && col < g.n;
        long long it = 0;
        for (; __any_sync(0xffffffffu, mine && pipe::is_empty(v[x])) && it < pipe::kSpinCap; ++it) {
          if (g.spin_ns) __nanosleep(ns);
          ns = ns * 2 < unsigned(g.spin_ns) ? ns * 2 : unsigned(g.spin_ns);
          if (mine && pipe::is_empty(v[x])) v[x] = pipe::ld_relaxed(xrow[x] + col);
        }
        if (it == pipe::kSpinCap) pipe::spin_fault(g.err);
        if (lane + 32 * x < (K + 1) * S) {
          if (lane + 32 * x < S) xdst[x][col & (SG - 1)] = v[x];  // cab: column-indexed (prowC)
          else xdst[x][(k & 1) * K * S] = v[x];
        }
      }
    };
    // ---- warp 0: level t0-1 rows (input grid or the wrap buffer), as v1
    const int srow = i0 - t0 + 2 + lane;
    const bool srow_ok = srow >= 0 && srow <= g.n - 1;
    const double* const srcrow = (t0 == 1 ? g.a : src0) + int64_t(srow) * g.ld;
    double* const irow = ir + lane * IRS;
    auto load_pair = [&](int k, int m) {
      const int pp = k * S - 2 - 2 * lane + 2 * m;
      double2 v = make_double2(0.0, 0.0);
      if (srow_ok && pp >= 0 && pp < g.n) v = __ldcg(reinterpret_cast<const double2*>(srcrow + pp));
      return v;
    };
    auto store_pair = [&](int k, int m, double2 v) {
      const int pp = k * S - 2 - 2 * lane + 2 * m;
      if (pp >= 0 && pp < g.n) *reinterpret_cast<double2*>(irow + (pp & (IRS - 1))) = v;
    };
    double2 pre[S / 2];
    if (w == 0) {
      if (p > 0) pipe::wait_smem(prog + NW - 1, p * BIG + need(S + 2 * (K - 1)), g.err);
      store_pair(0, 0, load_pair(0, 0));
#pragma unroll
      for (int m = 1; m <= S / 2; ++m) pre[m - 1] = load_pair(0, m);
    }
    // ---- per-level roles
    bool row_ok[K];
    double* orow[K];
    double* erow[K];
    unsigned ofull = 0;  // bit kk: level kk writes every in-range column (wrap buffer)
    unsigned olast = 0;  // bit kk: level kk is t = T (result in place, updated cells)
#pragma unroll
    for (int kk = 0; kk < K; ++kk) {
      const int t = t0 + kk;
      const int i = i0 - (t - 1) + lane;
      row_ok[kk] = t <= g.T && i >= 1 && i <= g.n - 2;
      const bool last = t == g.T;
      const bool wrap = w == NW - 1 && kk == K - 1 && t < g.T && i >= 0 && i <= g.n - 1;
      orow[kk] = (last ? g.a : wb_out) + int64_t(i) * g.ld;
      erow[kk] = g.eb + (int64_t(t - 1) * g.nb + b) * g.ebld;
      if (last) olast |= 1u << kk;
      if (wrap) ofull |= 1u << kk;
    }
    const bool elive = lane == 31;
    const bool has_out = __any_sync(0xffffffffu, (olast | ofull) != 0u);  // warp-uniform
    // ---- register state: h[kk][0..3] = stream (upper neighbour) at c-1..c-4,
    // o[kk][0..2] = own outputs at c-1..c-3; level 0's ring terms
    double h[K][4], o[K][3];
#pragma unroll
    for (int kk = 0; kk < K; ++kk) {
      h[kk][0] = h[kk][1] = h[kk][2] = h[kk][3] = 0.0;
      o[kk][0] = o[kk][1] = o[kk][2] = 0.0;
    }
    double c1 = 0, c2 = 0, d1 = 0, d2 = 0, d3 = 0;
    double xv[XS];
    xload(0, xv);
    for (int k = 0; k < nchunk; ++k) {
      const int c_lo = k * S - 1;
      const int c_hi = c_lo + S - 1;
      if (g.prof) tp = clock64();
      xresolve(k, xv);
      PCOT_PROF2(0);
      if (w == 0) {
#pragma unroll
        for (int m = 1; m <= S / 2; ++m) store_pair(k, m, pre[m - 1]);
        if (k + 1 < nchunk) {
          if (p > 0) pipe::wait_seen(prog + NW - 1, p * BIG + need(c_hi + S + 2 + 2 * (K - 1)), seen_wrap, g.err);
#pragma unroll
          for (int m = 1; m <= S / 2; ++m) pre[m - 1] = load_pair(k + 1, m);
        }
      }
      PCOT_PROF2(1);
      // producer's last level ahead of our level 0 (its column j+1 at our clock c)
      if (w > 0) pipe::wait_seen(prog + w - 1, plv + need(c_hi + 2 + 2 * (K - 1)), seen_prod, g.err);
      PCOT_PROF2(2);
      if (w < NW - 1) {
        // ring reuse (our last level writes column c - 2l - 2(K-1) into slot mod RS)
        const int rel = c_hi + 6 - RS - 2 * (K - 1);
        if (rel > 0 && cons_live) {
          pipe::wait_seen(prog + w + 1, plv + need(rel), seen_cons, g.err);
        } else if (p > 0) {
          pipe::wait_seen(prog + w + 1, p * BIG + fin, seen_cons, g.err);
        }
      }
      PCOT_PROF2(3);
      __syncwarp();
      if (g.prof && t_first == 0) {
        t_first = globaltimer();
        c_first = clock64();
      }
      unsigned upd[K], inb[K];
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const int j0 = c_lo - 2 * lane - 2 * kk;
        inb[kk] = pipe::span_mask<S>(j0, 0, g.n - 1);
        upd[kk] = row_ok[kk] ? pipe::span_mask<S>(j0, 1, g.n - 2) : 0u;
      }
      const int jr = c_lo - 2 * lane - 2 * (K - 1);  // last level's column at the chunk start
      // per-chunk store bases (the clock index then becomes an immediate offset)
      double* ep[K];
      double* op[K];
      unsigned om[K];  // result (level T: updated cells) / wrap buffer (every in-range cell)
#pragma unroll
      for (int kk = 0; kk < K; ++kk) {
        const int j0 = c_lo - 2 * lane - 2 * kk;
        ep[kk] = erow[kk] + j0;
        op[kk] = orow[kk] + j0;
        om[kk] = ((olast >> kk) & 1u) ? upd[kk] : (((ofull >> kk) & 1u) ? inb[kk] : 0u);
        if (!elive) inb[kk] = 0u;  // edge-store mask: lane 31 only
      }
      const double* const abk = ab + (k & 1) * K * S;
#pragma unroll
      for (int cc = 0; cc < S; ++cc) {
        if (cc == pipe::kXLoadClock && k + 1 < nchunk) xload(k + 1, xv);
        const int c = c_lo + cc;
        // level 0's producer terms (columns j..j+1 from lane l-1, j-1..j+1 from lane l)
        const int q = c - 2 * lane + 1;  // level 0: j + 1
        c1 = c2;
        c2 = prowC[q & cmask];
        d1 = d2;
        d2 = d3;
        d3 = prowD[q & dmask];
        // the K sums, operand by operand across the levels: K independent
        // chains interleaved in issue order (the warp issues in order)
        double sum[K];
#pragma unroll
        for (int kk = 0; kk < K; ++kk) sum[kk] = add(h[kk][2], h[kk][1]);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) sum[kk] = add(sum[kk], h[kk][0]);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) sum[kk] = add(sum[kk], o[kk][0]);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) sum[kk] = add(sum[kk], kk ? h[kk - 1][3] : c1);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) sum[kk] = add(sum[kk], kk ? h[kk - 1][2] : c2);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) sum[kk] = add(sum[kk], kk ? o[kk - 1][2] : d1);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) sum[kk] = add(sum[kk], kk ? o[kk - 1][1] : d2);
#pragma unroll
        for (int kk = 0; kk < K; ++kk) sum[kk] = add(sum[kk], kk ? o[kk - 1][0] : d3);
        double nv[K];
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          const double r = div9(sum[kk]);
          nv[kk] = (upd[kk] >> cc) & 1u ? r : 0.0;
        }
        // stores: edge slot (lane 31), result / wrap buffer, ring (last level)
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          const double v = nv[kk];
          pipe::st_relaxed_if(ep[kk] + cc, v, (inb[kk] >> cc) & 1u);
          if (has_out) pipe::st_global_if(op[kk] + cc, v, (om[kk] >> cc) & 1u);
        }
        myring[(jr + cc) & (RS - 1)] = nv[K - 1];
        // shift histories; one rotate shuffle per level (lane 31 sends lane 0's
        // band-above value for the column lane 0 needs next clock)
#pragma unroll
        for (int kk = 0; kk < K; ++kk) {
          o[kk][2] = o[kk][1];
          o[kk][1] = o[kk][0];
          o[kk][0] = nv[kk];
          const double send = elive ? abk[kk * S + cc] : nv[kk];
          const double in = __shfl_sync(0xffffffffu, send, src_lane);
          h[kk][3] = h[kk][2];
          h[kk][2] = h[kk][1];
          h[kk][1] = h[kk][0];
          h[kk][0] = in;
        }
      }
      PCOT_PROF2(5);
      __syncwarp();
      if (lane == 0) pipe::st_release_cta(prog + w, plv + c_hi + 1);
      __syncwarp();
      PCOT_PROF2(6);
    }
    __syncwarp();
  }
#undef PCOT_PROF2
  if (g.prof && lane == 0) {
    long long* pr = g.prof + (int64_t(b) * NW + w) * 16;
    for (int q = 0; q < 8; ++q) pr[q] = pacc[q];
    pr[8] = t_first;
    pr[9] = globaltimer();
    pr[10] = c_first;
    pr[11] = clock64();
    pr[12] = t_entry;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    pr[13] = smid;
  }
}

}  // namespace pipe2

// 2: line-group warp kernel (4 x 32 lines), 1: one-warp tile, 0: CTA tile
int gs_kind(int bt, int bx) {
  if (bt == lines::BT && bx == lines::BX) return 2;
  return bt * bx == 32 ? 1 : 0;
}

}  // namespace

int64_t gs2d_pipe_segment(int64_t n, int64_t T, int device);
int gs2d_pipe_bands(int64_t n, int64_t seg);

GsPlan* gs2d_plan_create(int64_t n, int64_t T, int bt, int bx, int by, int device) {
  GsPlan* p = new GsPlan;
  p->n = n;
  p->T = T;
  p->bt = bt;
  p->bx = bx;
  p->by = by;
  p->device = device;
  if (cudaSetDevice(device) != cudaSuccess || cudaMalloc(&p->d_err, sizeof(int)) != cudaSuccess ||
      cudaMemset(p->d_err, 0, sizeof(int)) != cudaSuccess ||
      cudaHostAlloc(&p->h_err, sizeof(int), cudaHostAllocDefault) != cudaSuccess) {
    p->setup_failed = true;
    return p;
  }
  *p->h_err = 0;
  if (T < 1 || n < 3) return p;  // nothing to do
  if (bt == 0) {  // systolic pipeline: every band's CTA must be resident
    p->pipe = true;
    p->seg = gs2d_pipe_segment(n, T, device);
    p->nb = gs2d_pipe_bands(n, p->seg);
    p->ebld = (n + 3) & ~int64_t(1);
    return p;
  }
  const int64_t NT = (T + bt - 1) / bt;
  const int64_t xmax = T + n - 2, ymax = 2 * T + 2 * (n - 2);
  const int64_t NX = (xmax - 2) / bx + 1, NY = (ymax - 4) / by + 1;
  // Non-empty tiles (exact test per line), then wavefront order.
  std::vector<std::tuple<int64_t, int, int, int>> order;
  std::map<std::tuple<int, int, int>, int> idx;
  auto nonempty = [&](int64_t tb, int64_t xb, int64_t yb) {
    for (int64_t t = 1 + tb * bt; t < 1 + (tb + 1) * bt && t <= T; ++t) {
      const int64_t xlo = 2 + xb * bx, xhi = xlo + bx - 1;
      const int64_t ilo = std::max<int64_t>(1, xlo - t), ihi = std::min<int64_t>(n - 2, xhi - t);
      if (ilo > ihi) continue;
      const int64_t ylo = 4 + yb * by, yhi = ylo + by - 1;
      // y = 2t + i + j, j in [1, n-2], i in [ilo, ihi]
      const int64_t ymin = 2 * t + ilo + 1, ymax2 = 2 * t + ihi + n - 2;
      if (std::max(ylo, ymin) <= std::min(yhi, ymax2)) return true;
    }
    return false;
  };
  for (int64_t tb = 0; tb < NT; ++tb)
    for (int64_t xb = 0; xb < NX; ++xb)
      for (int64_t yb = 0; yb < NY; ++yb)
        if (nonempty(tb, xb, yb)) order.emplace_back(tb + xb + yb, int(tb), int(xb), int(yb));
  std::sort(order.begin(), order.end());
  std::vector<int> tiles, preds;
  for (size_t q = 0; q < order.size(); ++q) {
    auto [w, tb, xb, yb] = order[q];
    idx[{tb, xb, yb}] = int(q);
    tiles.insert(tiles.end(), {tb, xb, yb});
    int np = 0;
    int pr[8] = {-1, -1, -1, -1, -1, -1, -1, -1};
    for (int m = 1; m < 8; ++m) {
      auto it = idx.find({tb - (m >> 2 & 1), xb - (m >> 1 & 1), yb - (m & 1)});
      if (it != idx.end()) pr[np++] = it->second;
    }
    preds.insert(preds.end(), pr, pr + 8);
  }
  p->ntiles = int64_t(order.size());
  const int ni = bx + bt + 1, ns = by + 2 * bt + 2;
  const int kind = gs_kind(bt, bx);
  const size_t smem = size_t(ni) * ns * (kind ? 9 : 8) + 16;
  auto kern = kind == 2 ? lines::gs2d_lines_kernel : kind == 1 ? gs2d_warp_kernel : gs2d_kernel;
  int slots = 0;
  if (cudaMalloc(&p->d_tiles, tiles.size() * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&p->d_preds, preds.size() * sizeof(int)) != cudaSuccess ||
      cudaMalloc(&p->d_state, (p->ntiles + 1) * sizeof(int)) != cudaSuccess ||
      cudaMemcpy(p->d_tiles, tiles.data(), tiles.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(p->d_preds, preds.data(), preds.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess ||
      // legacy-stream copies vs the caller's non-blocking stream
      cudaStreamSynchronize(0) != cudaSuccess ||
      kernel_slots(reinterpret_cast<const void*>(kern), kind ? 32 : bt * bx, smem, &slots) != cudaSuccess ||
      slots <= 0) {
    p->setup_failed = true;
    return p;
  }
  p->grid = int(std::max<int64_t>(1, std::min<int64_t>(p->ntiles, slots)));
  return p;
}

// Fault word of the last runs (call after synchronising the run's stream):
// nonzero if a dependence wait hit its spin cap; reading it re-arms it.
int gs2d_plan_fault(GsPlan* p) {
  if (!p || !p->h_err || !*p->h_err) return 0;
  *p->h_err = 0;
  cudaMemset(p->d_err, 0, sizeof(int));
  cudaDeviceSynchronize();
  return 1;
}

void gs2d_plan_destroy(GsPlan* p) {
  if (!p) return;
  cudaFree(p->d_tiles);
  cudaFree(p->d_preds);
  cudaFree(p->d_state);
  cudaFree(p->wb[0]);
  cudaFree(p->wb[1]);
  cudaFree(p->eb);
  cudaFree(p->gprog);
  cudaFree(p->d_err);
  if (p->h_err) cudaFreeHost(p->h_err);
  delete p;
}

// Pipeline variants: {warps per CTA, ring depth, clocks per chunk, levels per
// warp (1: gs2d_pipe_kernel, K > 1: gs2d_pipe2_kernel)}.
struct PipeVariant {
  int nw, rs, s, k;
  void (*kern)(pipe::PipeArgs);
  int h = 1;  // CTAs per band (split bands)
  int threads() const { return (nw + (h > 1 ? 1 : 0)) * 32; }
};
const PipeVariant kPipeVariants[] = {
    {16, 32, 8, 1, pipe::gs2d_pipe_kernel<16, 32, 8>},
    {12, 64, 8, 1, pipe::gs2d_pipe_kernel<12, 64, 8>},
    {8, 64, 8, 1, pipe::gs2d_pipe_kernel<8, 64, 8>},
    {12, 64, 4, 1, pipe::gs2d_pipe_kernel<12, 64, 4>},
    {12, 64, 16, 1, pipe::gs2d_pipe_kernel<12, 64, 16>},
    {16, 32, 8, 2, pipe2::gs2d_pipe2_kernel<16, 2, 32, 8>},
    {8, 64, 8, 2, pipe2::gs2d_pipe2_kernel<8, 2, 64, 8>},
    {8, 64, 8, 4, pipe2::gs2d_pipe2_kernel<8, 4, 64, 8>},
    {4, 64, 8, 4, pipe2::gs2d_pipe2_kernel<4, 4, 64, 8>},
    {8, 32, 8, 1, pipe::gs2d_pipe_kernel<8, 32, 8, 2>, 2},    // 9: split bands, 2 x 8 warps
    {8, 64, 8, 1, pipe::gs2d_pipe_kernel<8, 64, 8, 2>, 2},    // 10
    {4, 64, 8, 1, pipe::gs2d_pipe_kernel<4, 64, 8, 2>, 2},    // 11: 2 x 4 warps
};
constexpr int kNumPipeVariants = sizeof(kPipeVariants) / sizeof(kPipeVariants[0]);
const PipeVariant& pipe_variant() {
  const char* s = getenv("PCOTGPU_GS_PIPE_V");
  const int v = s ? atoi(s) : 0;  // default: best measured (profiles/gs_pipe_r01.md)
  return kPipeVariants[v < 0 || v >= kNumPipeVariants ? 0 : v];
}

size_t gs2d_pipe_smem(const PipeVariant& v) {
  using namespace pipe;
  if (v.k > 1)  // rings, staged rows, K band-above rows + the level t0-1 row per warp, progress
    return size_t(v.nw) * 32 * (v.rs + 1) * 8 + size_t(32) * IRS * 8 + size_t(v.k + 1) * v.nw * SG * 8 +
           v.nw * 4;
  return size_t(v.nw) * 32 * (v.rs + 1) * 8 + size_t(32) * IRS * 8 + size_t(2) * v.nw * SG * 8 +
         v.nw * 4;
}

// Bands for a launch of `seg` levels: rows 1..n-2 under a window that moves
// up seg-1 rows.
int gs2d_pipe_bands(int64_t n, int64_t seg) { return int((n - 2 + seg - 1 + 31) / 32); }

size_t gs2d_pipe_edge_bytes(int64_t n, int64_t seg) {
  return size_t(seg) * gs2d_pipe_bands(n, seg) * ((n + 3) & ~int64_t(1)) * 8;
}

// Levels per launch for n x n, T sweeps (0: the pipeline does not fit).  All
// bands co-resident (one CTA per SM), progress words level * BIG fit an int,
// the write-once edge rows (8 n bytes per band and level) within a quarter of
// the free memory, and launches of at least min(T, 64) levels.
int64_t gs2d_pipe_segment(int64_t n, int64_t T, int device) {
  if (n < 3 || T < 1) return 0;
  const PipeVariant& v = pipe_variant();
  const size_t smem = gs2d_pipe_smem(v);
  int slots = 0;
  if (cudaSetDevice(device) != cudaSuccess ||
      kernel_slots(reinterpret_cast<const void*>(v.kern), v.threads(), smem, &slots) != cudaSuccess)
    return 0;
  const int64_t cap = slots / v.h;  // bands that can be resident
  int64_t seg = std::min<int64_t>(T, 32 * cap - (n - 2) + 1);
  seg = std::min<int64_t>(seg, (int64_t(1) << 31) / pipe::BIG - 2);
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return 0;
  while (seg > 0 && gs2d_pipe_edge_bytes(n, seg) > free_b / 4) seg /= 2;
  if (seg < std::min<int64_t>(T, 64)) return 0;
  const int64_t launches = (T + seg - 1) / seg;  // balance the launches
  return (T + launches - 1) / launches;
}

bool gs2d_pipe_fits(int64_t n, int64_t T, int device) { return gs2d_pipe_segment(n, T, device) > 0; }

cudaError_t gs2d_pipe_launch(GsPlan* p, const PipeVariant& v, size_t smem, double* a, int64_t ld,
                             int64_t len, cudaStream_t stream);

cudaError_t gs2d_pipe_run(GsPlan* p, double* a, int64_t ld, cudaStream_t stream) {
  using namespace pipe;
  cudaError_t e;
  if (!p->eb || p->ld != ld) {
    cudaFree(p->wb[0]);
    cudaFree(p->wb[1]);
    cudaFree(p->eb);
    p->ld = ld;
    for (int q = 0; q < 2; ++q)
      if ((e = cudaMalloc(&p->wb[q], size_t(p->n) * ld * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&p->eb, gs2d_pipe_edge_bytes(p->n, p->seg))) != cudaSuccess) return e;
  }
  if (!p->gprog) {  // split-band progress words (H <= 4 CTAs per band)
    if ((e = cudaMalloc(&p->gprog, size_t(p->nb + 1) * 4 * sizeof(int))) != cudaSuccess) return e;
  }
  const PipeVariant& v = pipe_variant();
  const size_t smem = gs2d_pipe_smem(v);
  if ((e = kernel_slots(reinterpret_cast<const void*>(v.kern), v.threads(), smem, nullptr)) != cudaSuccess)
    return e;
  for (int64_t t0 = 0; t0 < p->T; t0 += p->seg) {
    const int64_t len = std::min(p->seg, p->T - t0);
    if ((e = gs2d_pipe_launch(p, v, smem, a, ld, len, stream)) != cudaSuccess) return e;
  }
  return cudaMemcpyAsync(p->h_err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, stream);
}

// One launch: `len` levels from the grid in `a` (level 0) back into `a`.
cudaError_t gs2d_pipe_launch(GsPlan* p, const PipeVariant& v, size_t smem, double* a, int64_t ld,
                             int64_t len, cudaStream_t stream) {
  using namespace pipe;
  cudaError_t e;
  const int nb = gs2d_pipe_bands(p->n, len);
  // every edge slot back to kEmpty (written once per launch)
  if ((e = cudaMemsetAsync(p->eb, 0xff, gs2d_pipe_edge_bytes(p->n, len), stream)) != cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(p->gprog, 0, size_t(nb) * v.h * sizeof(int), stream)) != cudaSuccess) return e;
  PipeArgs g;
  g.gprog = p->gprog;
  g.a = a;
  g.wb[0] = p->wb[0];
  g.wb[1] = p->wb[1];
  g.eb = p->eb;
  g.ld = ld;
  g.ebld = p->ebld;
  g.n = int(p->n);
  g.T = int(len);
  g.nb = nb;
  g.nclk = int(p->n) + 63;
  g.prof = nullptr;
  g.err = p->d_err;
  g.spin_ns = env_int("PCOTGPU_GS_SPIN", 256);
  g.wait_ns = env_int("PCOTGPU_GS_WAIT", 8);
  const char* pe = getenv("PCOTGPU_GS_PROF");  // development aid: cycle breakdown
  const size_t np = size_t(nb) * v.h * v.nw * 16;
  if (pe && atoi(pe)) {
    if ((e = cudaMalloc(&g.prof, np * 8)) != cudaSuccess) return e;
    cudaMemsetAsync(g.prof, 0, np * 8, stream);
  }
  // Every band's CTA must be resident (bands wait on the band above):
  // cooperative launch makes that a launch-time guarantee — it fails with
  // cudaErrorCooperativeLaunchTooLarge instead of deadlocking.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb * v.h);
  cfg.blockDim = dim3(v.threads());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if ((e = cudaLaunchKernelEx(&cfg, v.kern, g)) != cudaSuccess) return e;
  count_launch();
  if (g.prof) {
    std::vector<long long> h(np);
    cudaMemcpyAsync(h.data(), g.prof, np * 8, cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    cudaFree(g.prof);
    static const char* names[8] = {"wait_xcta", "wait_wrap", "wait_prod", "wait_ring",
                                   "sync",      "compute",   "publish",  "stage_in"};
    double tot[8] = {0}, all = 0;
    for (size_t q = 0; q < np / 16; ++q)
      for (int m = 0; m < 8; ++m) tot[m] += double(h[q * 16 + m]), all += double(h[q * 16 + m]);
    fprintf(stderr, "gs pipe profile (nw=%d rs=%d, %lld warps):", v.nw, v.rs, (long long)(np / 16));
    for (int m = 0; m < 8; ++m)
      fprintf(stderr, " %s=%.1f%% (%.0f cyc/warp)", names[m], 100 * tot[m] / all, tot[m] / (np / 16));
    fprintf(stderr, "\n");
    for (int q = 0; q < 5; ++q) {  // a few bands: edge wait vs compute per warp
      const int b = int(int64_t(nb - 1) * q / 4);
      double xw = 0, cw = 0, rw = 0;
      for (int w = 0; w < v.nw; ++w) {
        xw += double(h[(size_t(b) * v.h * v.nw + w) * 16 + 0]);
        cw += double(h[(size_t(b) * v.h * v.nw + w) * 16 + 5]);
        rw += double(h[(size_t(b) * v.h * v.nw + w) * 16 + 2] + h[(size_t(b) * v.h * v.nw + w) * 16 + 3]);
      }
      fprintf(stderr, "  band %d: wait_xcta %.0f compute %.0f wait_intra %.0f (cyc/warp)\n", b,
              xw / v.nw, cw / v.nw, rw / v.nw);
    }
    {  // band timeline: warp 0's first compute and warp NW-1's exit (ns from band 0 start)
      const long long t0 = h[8];
      fprintf(stderr, "  timeline (us):");
      for (int q = 0; q <= 8; ++q) {
        const int b = int(int64_t(nb - 1) * q / 8);
        fprintf(stderr, " b%d[%.1f,%.1f]", b, (h[(size_t(b) * v.h * v.nw) * 16 + 8] - t0) * 1e-3,
                (h[(size_t(b) * v.h * v.nw + v.nw - 1) * 16 + 9] - t0) * 1e-3);
      }
      long long emin = h[12], emax = h[12];
      int late = 0;
      for (int bb = 0; bb < nb; ++bb) {
        const long long e = h[(size_t(bb) * v.nw) * 16 + 12];
        emin = std::min(emin, e), emax = std::max(emax, e);
      }
      for (int bb = 0; bb < nb; ++bb)
        if (h[(size_t(bb) * v.nw) * 16 + 12] - emin > 20000) ++late;
      fprintf(stderr, "\n  CTA entry spread %.1f us (%d CTAs > 20 us late)", (emax - emin) * 1e-3, late);
      fprintf(stderr, "\n  band 0 warp 0 clock: %.0f MHz\n",
              double(h[11] - h[10]) / double(h[9] - h[8]) * 1e3);
    }
    if (atoi(pe) > 1) {  // per-warp rows of band PCOTGPU_GS_PROF - 2
      const int b = std::min(atoi(pe) - 2, nb - 1);
      for (int w = 0; w < v.nw; ++w) {
        fprintf(stderr, "  band %d warp %2d:", b, w);
        for (int m = 0; m < 8; ++m)
          fprintf(stderr, " %s=%lld", names[m], h[(size_t(b) * v.h * v.nw + w) * 16 + m]);
        fprintf(stderr, "\n");
      }
    }
  }
  return cudaGetLastError();
}

int64_t gs2d_plan_tiles(const GsPlan* p) { return p ? p->ntiles : 0; }

cudaError_t div9_check(const double* x, double* q_fast, double* q_ref, int64_t n,
                       cudaStream_t stream) {
  div9_check_kernel<<<148 * 8, 256, 0, stream>>>(x, q_fast, q_ref, n);
  count_launch();
  return cudaGetLastError();
}

cudaError_t gs2d_run(GsPlan* p, double* a, int64_t ld, cudaStream_t stream) {
  if (p->setup_failed) return cudaErrorMemoryAllocation;
  if (p->pipe) return gs2d_pipe_run(p, a, ld, stream);
  if (p->ntiles == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(p->d_state, 0, (p->ntiles + 1) * sizeof(int), stream);
  if (e != cudaSuccess) return e;
  GsArgs g;
  g.a = a;
  g.ld = ld;
  g.n = p->n;
  g.T = p->T;
  g.bt = p->bt;
  g.bx = p->bx;
  g.by = p->by;
  g.ni = p->bx + p->bt + 1;
  g.ns = p->by + 2 * p->bt + 2;
  g.ntiles = p->ntiles;
  g.tiles = p->d_tiles;
  g.preds = p->d_preds;
  g.flags = p->d_state;
  g.counter = p->d_state + p->ntiles;
  g.err = p->d_err;
  const int kind = gs_kind(p->bt, p->bx);
  const size_t smem = size_t(g.ni) * g.ns * (kind ? 9 : 8) + 16;
  if (kind == 2)
    lines::gs2d_lines_kernel<<<p->grid, 32, smem, stream>>>(g);
  else if (kind == 1)
    gs2d_warp_kernel<<<p->grid, 32, smem, stream>>>(g);
  else
    gs2d_kernel<<<p->grid, p->bt * p->bx, smem, stream>>>(g);
  count_launch();
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return cudaMemcpyAsync(p->h_err, p->d_err, sizeof(int), cudaMemcpyDeviceToHost, stream);
}

}  // namespace pcotgpu
