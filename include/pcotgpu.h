/* pcotgpu — C ABI of the B200 (sm_100a) executor for the PCOT hot path.
 *
 * The reference toolkit has no FFI; its run API is the C++ class
 * pcot::Executor (reference proj/core/include/pcot/exec.hpp:62-82) fed by the
 * kernel registration API (kernel_io.hpp:11-22).  Each entry point below
 * replaces one of those calls; the reference-side binding a maintainer adds is
 * in INTEGRATION.md.  Plain pointers and sizes only; every function returns a
 * status (0 = ok, else 1 + pcot::ErrorKind ordinal, reference error.hpp:8-16,
 * or PCOTGPU_E_CUDA) and pcotgpu_last_error() holds the message (per thread).
 */
#ifndef PCOTGPU_H
#define PCOTGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCOTGPU_ABI_VERSION 1

enum pcotgpu_status {
  PCOTGPU_OK = 0,
  PCOTGPU_E_OVERFLOW = 1,      /* pcot::ErrorKind::Overflow    */
  PCOTGPU_E_DIM_MISMATCH = 2,  /* pcot::ErrorKind::DimMismatch */
  PCOTGPU_E_UNBOUNDED = 3,     /* pcot::ErrorKind::Unbounded   */
  PCOTGPU_E_PARSE = 4,         /* pcot::ErrorKind::Parse       */
  PCOTGPU_E_VALIDATION = 5,    /* pcot::ErrorKind::Validation  */
  PCOTGPU_E_IO = 6,            /* pcot::ErrorKind::Io          */
  PCOTGPU_E_UNSUPPORTED = 7,   /* pcot::ErrorKind::Unsupported */
  PCOTGPU_E_CUDA = 8           /* device error (no reference counterpart) */
};

enum pcotgpu_family {
  PCOTGPU_STENCIL2D5 = 1, /* heat2d (ring copied) / jacobi2d (ring 0.0) */
  PCOTGPU_STENCIL3D7 = 2, /* heat3d (0.1 rule) / heat3d_b (BASELINE rule) */
  PCOTGPU_GS2D9 = 3,      /* in-place Gauss-Seidel 9-point */
  PCOTGPU_GEMM = 4        /* Out = (2A-1)(2B-1), fp64 */
};

/* reference tiler.hpp:21 enum class Scheme { Untiled, Slt, Cot } */
enum pcotgpu_scheme { PCOTGPU_UNTILED = 0, PCOTGPU_SLT = 1, PCOTGPU_COT = 2 };

enum pcotgpu_run_flags {
  PCOTGPU_SKIP_CHECKSUM = 1, /* leave result.checksum = 0 (no device->host copy) */
  PCOTGPU_SPACE_TIME = 2     /* COT on 2-D stencils: recursive order over (depth block,
                                row band) across launches, bands of leaf[1] rows */
};

/* What the recognizer proved about a kernel at a parameter binding. */
typedef struct {
  int32_t family;    /* pcotgpu_family */
  int32_t rule;      /* 3-D: 0 = c + 0.125*(sum6 - 6c), 1 = 0.1*(c + sum6) */
  int32_t ring_hold; /* 0: ring is literal 0.0; 1: ring copied forward */
  int32_t ndim;      /* spatial dimensions */
  int64_t T, N;      /* time steps, grid extent (GEMM: T = 0, N = order) */
  uint64_t points, reads, writes; /* ExecResult counters in closed form */
  char name[64];
} pcotgpu_kernel_info;

/* TileOrder + TileSpec (reference tiler.hpp:12-31): leaf[0] is the time-leaf
 * size (= temporal block depth on the GPU), leaf[1..] the spatial tile. */
typedef struct {
  int32_t scheme; /* pcotgpu_scheme */
  int32_t ndim;   /* entries used in leaf[] (0 = defaults) */
  int64_t leaf[8];
  int32_t flags;  /* pcotgpu_run_flags */
  int32_t reserved;
} pcotgpu_schedule;

/* ExecResult (reference exec.hpp:45-52) + device time. */
typedef struct {
  uint64_t points, reads, writes;
  int32_t violation; /* always 0: legality holds by construction */
  int32_t bt;        /* temporal block depth actually used; device interpreter
                        (family 5): 0 sequential, 1 dataflow grid over ready
                        flags, 2 dataflow grid over storage shadows (maps) */
  uint64_t checksum; /* FNV-1a over output bytes (formats.md CHECKSUM) */
  double device_ms;  /* CUDA-event time of the device work */
  uint64_t launches; /* kernels launched by this run */
} pcotgpu_result;

/* MemoryMap (reference memalloc.hpp:14-33) of one array:
 *   storage_k = (sum_c linear[k * rank + c] * cell_c + constant[k]) mod moduli[k]
 * (moduli[k] == 0: no modulo), storage_k in [0, extents[k]), row-major. */
typedef struct {
  const char* array;
  int32_t rank;            /* the array's (cell) rank */
  int32_t storage_rank;    /* entries of constant / moduli / extents */
  const int64_t* linear;   /* storage_rank x rank, row-major */
  const int64_t* constant;
  const int64_t* moduli;
  const int64_t* extents;
  int32_t single_assignment;
  int32_t reserved;
} pcotgpu_map;

typedef struct pcotgpu_handle pcotgpu_handle;

/* ---- registration (host only; no GPU needed) ---------------------------- */
/* parse_kernel + recognizer: reference kernel_io.cpp:118-197. */
int pcotgpu_recognize(const char* kernel_json, const int64_t* params, size_t nparams,
                      pcotgpu_kernel_info* out);
/* find_kernel_file: reference kernel_io.cpp:250-276 (path, PCOT_KERNEL_PATH,
 * ./kernels); writes "" when not found. */
int pcotgpu_find_kernel_file(const char* name_or_path, char* out, size_t cap);

/* Host only: the map checks pcotgpu_create_mapped makes (one map per array,
 * arities; Validation for out-of-extent storage) and whether the hand-written
 * kernel keeps the run (*hot_path = 1) or the interpreter takes it (0); `why`
 * (may be NULL) receives the reason the hot path declined. */
int pcotgpu_check_maps(const char* kernel_json, const int64_t* params, size_t nparams,
                       const pcotgpu_map* maps, size_t nmaps, int* hot_path, char* why, size_t cap);

/* Host only: the PRDG -> CUDA emitter's source for a kernel (the device
 * interpreter's compiled form), written to `buf` (needs
 * `*need` bytes incl. the NUL); with compile != 0 it is also compiled by NVRTC
 * for sm_100a and `buf` receives the compiler log instead on failure. */
int pcotgpu_generic_source(const char* kernel_json, const int64_t* params, size_t nparams, int compile,
                           char* buf, size_t cap, size_t* need);
/* After a run on the device interpreter: its schedule (0 sequential, 1 dataflow
 * over ready flags, 2 dataflow over storage shadows) and whether the emitter's
 * compiled kernels ran (else the interpreter); `why` gets the build status. */
int pcotgpu_generic_info(const pcotgpu_handle* h, int* mode, int* compiled, char* why, size_t cap);

/* ---- Executor ------------------------------------------------------------ */
/* Executor(p, params, maps) — exec.hpp:64.  Allocates device storage and
 * initialises inputs with init_value (exec.cpp:21-28, 281-294). */
int pcotgpu_create(const char* kernel_json, const int64_t* params, size_t nparams, int device,
                   pcotgpu_handle** out);
/* Executor(p, params, maps) with the caller's memory maps (one per array, as
 * the reference requires: exec.cpp:134-141).  The hand-written kernels run
 * when their device layout reproduces the reference's storage semantics
 * (inputs/outputs: identity at the declared extents; the temp: single
 * assignment, or folded along a multiple of the kernel's occupancy vector —
 * what allocate() derives); any other map set runs on the device interpreter
 * with storage laid out exactly by the maps.  Out-of-extent maps: Validation. */
int pcotgpu_create_mapped(const char* kernel_json, const int64_t* params, size_t nparams,
                          const pcotgpu_map* maps, size_t nmaps, int device, pcotgpu_handle** out);
/* Executor::run(order, opts) — exec.hpp:71; sched == NULL means untiled. */
int pcotgpu_run(pcotgpu_handle* h, const pcotgpu_schedule* sched, pcotgpu_result* res);
/* Executor::run_untiled — exec.hpp:73. */
int pcotgpu_run_untiled(pcotgpu_handle* h, pcotgpu_result* res);
/* Beyond the reference: `count` independent runs straight from host memory
 * (what a caller of Executor::run does around it: set the inputs, run, read
 * the output — exec.hpp:71-80), with instance k+1's input copies and instance
 * k-1's output copy overlapped with instance k's compute.
 * host_inputs[k * ninputs + q] = instance k's input q (dense, array_words
 * doubles, inputs in kernel-declaration order); host_outputs[k] = instance k's
 * output.  res->device_ms covers the whole batch (copies included);
 * res->checksum is the last instance's output checksum.  Use pinned host
 * memory for asynchronous copies. */
int pcotgpu_run_batch(pcotgpu_handle* h, const pcotgpu_schedule* sched, size_t count,
                      const double* const* host_inputs, double* const* host_outputs,
                      pcotgpu_result* res);
/* Executor::reset — exec.hpp:75. */
int pcotgpu_reset(pcotgpu_handle* h);
/* Executor::array_data — exec.hpp:76 (inputs and outputs; temps live in the
 * device layout and report PCOTGPU_E_UNSUPPORTED). n must equal the word count. */
int pcotgpu_read_array(pcotgpu_handle* h, const char* array, double* host_dst, size_t n);
/* Load an input array from host memory (replaces init_value for that array). */
int pcotgpu_write_array(pcotgpu_handle* h, const char* array, const double* host_src, size_t n);
/* Executor::array_base — exec.hpp:77 (64-byte aligned, reference layout). */
int pcotgpu_array_base(const pcotgpu_handle* h, const char* array, uint64_t* base);
int pcotgpu_array_words(const pcotgpu_handle* h, const char* array, uint64_t* words);
int pcotgpu_info(const pcotgpu_handle* h, pcotgpu_kernel_info* out);
/* Device pointer + pitch of the array's current storage (advanced use). */
int pcotgpu_device_view(pcotgpu_handle* h, const char* array, double** ptr, int64_t* ld);
/* Run on this CUDA stream (cudaStream_t as void*); default is a private stream. */
int pcotgpu_set_stream(pcotgpu_handle* h, void* stream);
void pcotgpu_destroy(pcotgpu_handle* h);

/* ---- slab kernels on caller-owned device memory (row-sharded grids) ------ */
/* Geometry a 2-D slab of `rows` x `cols` must be allocated with. */
int pcotgpu_s2d5_layout(int64_t rows, int64_t cols, int64_t* ld, int64_t* ghost, int64_t* padl,
                        int64_t* total_doubles);
/* Advance a slab `bt` steps on local rows [row_lo, row_hi); origin pointers
 * address local cell (0,0) of buffers laid out by pcotgpu_s2d5_layout. */
int pcotgpu_s2d5_advance(const double* in_origin, double* out_origin, int64_t rows, int64_t cols,
                         int64_t g0, int64_t nrows_global, int bt, int ring_hold, int order,
                         int64_t row_lo, int64_t row_hi, void* stream);
/* Same, with the halo exchange fused into the kernel (P2P stores over NVLink):
 * owned output rows [0, mirror_rows) are also written to
 * mirror_up + row*ld + col and rows [rows - mirror_rows, rows) to
 * mirror_dn + row*ld + col, where mirror_up = upper neighbour's out origin +
 * rows*ld (its ghost rows below) and mirror_dn = lower neighbour's out origin -
 * rows*ld (its ghost rows above); NULL mirrors are skipped.  Replaces the
 * NCCL send/recv of sharded.py's exchange; mirror_rows <= ghost rows. */
int pcotgpu_s2d5_advance_p2p(const double* in_origin, double* out_origin, int64_t rows,
                             int64_t cols, int64_t g0, int64_t nrows_global, int bt, int ring_hold,
                             int order, int64_t row_lo, int64_t row_hi, double* mirror_up,
                             double* mirror_dn, int64_t mirror_rows, void* stream);
/* init_value(name, flat0 + r*cols + c) into a pitched block. */
int pcotgpu_fill_init_value(double* dst, int64_t ld, int64_t nrows, int64_t ncols,
                            const char* name, uint64_t flat0, void* stream);
/* zero the global ring rows/cols of a slab (rows with global index 0 / N-1). */
int pcotgpu_s2d5_prepare(double* origin, int64_t rows, int64_t cols, int64_t g0,
                         int64_t nrows_global, int ring_hold, void* stream);

/* Test hook: q_fast[i] = the Gauss-Seidel kernel's x[i] / 9.0, q_ref[i] =
 * IEEE __ddiv_rn(x[i], 9.0); device pointers. */
int pcotgpu_test_div9(const double* x, double* q_fast, double* q_ref, int64_t n, void* stream);

/* ---- misc ---------------------------------------------------------------- */
const char* pcotgpu_last_error(void);
uint64_t pcotgpu_launch_count(void);
int pcotgpu_abi_version(void);
int pcotgpu_device_count(int* n);
uint64_t pcotgpu_fnv1a(const void* data, size_t n, uint64_t h);

#ifdef __cplusplus
}
#endif
#endif /* PCOTGPU_H */
