// Internal launch interface of the sm_100a kernels (host side, no torch types).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pcotgpu {

// Row-sharded 2-D grid slab.  `origin` points at local cell (0,0); rows
// [-ghost, R+ghost) and columns [-padl, ld-padl) are addressable.
struct Slab2D {
  double* origin = nullptr;
  int64_t ld = 0;       // row pitch in doubles (multiple of 16)
  int64_t rows = 0;     // R, local rows owned
  int64_t cols = 0;     // N, grid columns
  int64_t ghost = 0;    // ghost rows above and below
  int64_t padl = 0;     // addressable columns left of column 0
};

enum TileOrderMode { kOrderLex = 0, kOrderMorton = 1 };

// Advance a 2-D 5-point slab by `bt` steps (1 <= bt <= 8): out = S^bt(in) on
// local rows [0, R).  Rows [-bt, 0) and [R, R+bt) of `in` must hold step-t0
// values of the neighbouring rows (ghost rows; ignored outside the grid).
// g0 = global row of local row 0; nrows = global row count (ring detection).
// ring_hold: 0 -> ring cells are 0.0 (jacobi2d.kernel), 1 -> ring cells keep
// their value (reference heat2d.kernel S2-S5).
cudaError_t s2d5_advance(const Slab2D& in, const Slab2D& out, int64_t g0, int64_t nrows,
                         int bt, int ring_hold, int order, int row_lo, int row_hi,
                         cudaStream_t stream);
// Same, and the owned rows [0, mirror_rows) / [rows - mirror_rows, rows) of the
// output are also stored at mirror_up / mirror_dn + row * out.ld + col (peer
// ghost rows, P2P over NVLink); a null mirror is skipped.
cudaError_t s2d5_advance_p2p(const Slab2D& in, const Slab2D& out, int64_t g0, int64_t nrows,
                             int bt, int ring_hold, int order, int row_lo, int row_hi,
                             double* mirror_up, double* mirror_dn, int mirror_rows,
                             cudaStream_t stream);
int s2d5_max_bt();
// Grid resident on chip for the whole run (stencil2d_res.cu): one persistent
// CTA per SM owns a band of rows in shared memory and steps it T times;
// neighbours exchange boundary rows through flags (no grid barrier).  create()
// returns null when the grid does not fit (n outside [64, 2048], band larger
// than shared memory, no cooperative launch).  `in` must hold the step-0 grid
// with its ring already zeroed / held; `out` receives step T.
struct S2ResPlan;
S2ResPlan* s2d5_res_create(int64_t n, int device);
void s2d5_res_destroy(S2ResPlan* p);
cudaError_t s2d5_res_run(S2ResPlan* p, const Slab2D& in, const Slab2D& out, int64_t T,
                         cudaStream_t stream);
// Nonzero if a neighbour wait of the runs since the last call hit its spin cap
// (the grid is then invalid); call after synchronising the run's stream.
int s2d5_res_fault(S2ResPlan* p);
// Programmatic dependent launch for the stencil depth blocks (PCOTGPU_PDL=0: off).
bool pdl_enabled();

// 3-D 7-point, dense N^3 cube with halo padding (see Grid3D).
struct Grid3D {
  double* origin = nullptr;  // cell (0,0,0)
  int64_t n = 0;             // N
  int64_t pitch_j = 0;       // doubles between j rows (multiple of 16)
  int64_t pitch_i = 0;       // doubles between i planes
  int64_t halo = 0;          // addressable halo planes/rows/cols on each side
};
// rule 0: c + 0.125*(sum6 - 6c) (heat3d_b); rule 1: 0.1*(c + sum6) (heat3d).
cudaError_t s3d7_advance(const Grid3D& in, const Grid3D& out, int bt, int rule, int ring_hold,
                         int order, cudaStream_t stream);
int s3d7_max_bt();

// In-place Gauss-Seidel 9-point, T sweeps, tile wavefront.  `a` is an N x N
// row-major array with pitch `ld` (ring cells fixed at their value).
struct GsPlan;  // host-side tile plan (device buffers owned by the plan)
// bt == 0 selects the systolic pipeline kernel (requires gs2d_pipe_fits).
GsPlan* gs2d_plan_create(int64_t n, int64_t T, int bt, int bx, int by, int device);
bool gs2d_pipe_fits(int64_t n, int64_t T, int device);
void gs2d_plan_destroy(GsPlan* p);
cudaError_t gs2d_run(GsPlan* p, double* a, int64_t ld, cudaStream_t stream);
int64_t gs2d_plan_tiles(const GsPlan* p);
// Nonzero if a dependence wait of the runs since the last call hit its spin
// cap (the grid is then invalid); call after synchronising the run's stream.
int gs2d_plan_fault(GsPlan* p);
// Test hook: the Gauss-Seidel kernel's x/9 vs the IEEE division, elementwise.
cudaError_t div9_check(const double* x, double* q_fast, double* q_ref, int64_t n,
                       cudaStream_t stream);

// C = A*B, fp64 DMMA tensor cores, row-major N x N with pitch ld.
cudaError_t dgemm_nn(const double* A, const double* B, double* C, int64_t n, int64_t ld,
                     int order, cudaStream_t stream);
// The tensor-TMA + mbarrier-ring kernel behind dgemm_nn's default (dgemm_tma.cu);
// variant 0: BK 32 x 3 stages, 1: BK 16 x 6 stages.
cudaError_t dgemm_nn_tma(const double* A, const double* B, double* C, int64_t n, int64_t ld,
                         int order, int variant, cudaStream_t stream);
// y = 2x - 1 elementwise (exact for x in [0,1) of the reference init_value).
cudaError_t affine_2x_minus_1(const double* x, double* y, int64_t count, cudaStream_t stream);

// Reference init_value (exec.cpp:21-28) on device: dst[r*ld + c] =
// init_value(name, flat0 + r*ncols + c) for r < nrows, c < ncols.
cudaError_t fill_init_value(double* dst, int64_t ld, int64_t nrows, int64_t ncols,
                            uint64_t name_hash, uint64_t flat0, cudaStream_t stream);
// 3-D variant over an N^3 cube with pitches.
cudaError_t fill_init_value_3d(const Grid3D& g, uint64_t name_hash, cudaStream_t stream);
// Copy a dense row-major [nrows x ncols] block between pitched layouts.
// With plane pitches (pd, rows_per_plane) the destination row r lands at
// plane r / rows_per_plane, row r % rows_per_plane (dense source).
cudaError_t copy_rows(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t nrows,
                      int64_t ncols, cudaStream_t stream, int64_t pd = 0, int64_t rows_per_plane = 0);
// copy_rows (2-D, dense source) that maps the Gauss-Seidel edge-slot sentinel
// bit pattern 0xffff...ffff to 0xffff...fffe (both NaN).
cudaError_t copy_rows_nosentinel(double* dst, int64_t ldd, const double* src, int64_t lds, int64_t nrows,
                                 int64_t ncols, cudaStream_t stream);
// Zero (or keep) the ring of a 2-D grid: cells on rows 0/N-1, cols 0/N-1.
cudaError_t zero_ring_2d(double* origin, int64_t ld, int64_t n, cudaStream_t stream);
cudaError_t zero_ring_3d(const Grid3D& g, cudaStream_t stream);

// Per-(kernel, device) launch preparation, thread-safe and cached: sets the
// dynamic shared-memory opt-in for `smem` on the current device and returns the
// number of CTAs of `nthreads` that can be resident at once (occupancy x SMs;
// 0 if none fits).
cudaError_t kernel_slots(const void* fn, int nthreads, size_t smem, int* slots);
// Integer environment override (read on every call: cheap, no shared state).
int env_int(const char* name, int dflt);

// Launch counter (every kernel launched by this library increments it).
uint64_t launches();
void count_launch(uint64_t n = 1);

}  // namespace pcotgpu
