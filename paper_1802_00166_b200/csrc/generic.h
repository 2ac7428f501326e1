// Generic device execution of any embedded-or-embeddable PRDG kernel (the
// reference's Executor semantics, core/src/exec.cpp:347-498) for kernels the
// hot-path recognizer does not map onto a hand-written kernel (SURVEY §8f.2:
// the remaining corpus kernels — triangle, lud, osp, heat1d-fig7 — run on the
// device instead of being rejected).
//
// Storage: laid out by the caller's memory maps (reference exec.cpp:142-185,
// 234-245: words = product of the map extents, storage_k = map_k(cell) mod
// moduli_k, out-of-extent checks on the unfolded dims), or dense at the
// declared extents when no maps are given (single-assignment layout).
// Schedule:
//   * single-assignment kernels (every logical cell written at most once, and
//     every write before its reads in the reference's order — both checked on
//     the device by a counting pass over the logical cells): a persistent grid
//     takes points in the reference's lexicographic order from an atomic
//     counter; every read waits for its cell (dense storage: a ready flag;
//     folded storage: the storage cell's shadow = logical id of the value it
//     holds, the reference's shadow array), every write publishes it.  A read
//     only ever waits on a point earlier in that order, which is already
//     running or done, so the grid cannot deadlock; folded storage is safe
//     because allocate()'s maps fold along universal occupancy vectors (any
//     dependence-respecting order), and a reused cell is detected, not read;
//   * otherwise (cells overwritten, e.g. osp's C): one device thread walks the
//     points in the reference's order.
// Per point, the statements whose domains contain it run in declaration
// order; bodies are evaluated as the reference's postfix program (one IEEE
// rounding per operation, no contraction), so outputs are bit-identical.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "spec.h"

namespace pcotgpu {

struct GenericPlan;

// Parse-time plan at a parameter binding: embeds shallow statements
// (reference prdg.cpp:72-119: missing inner indices pinned to 0), evaluates
// extents, projects every statement domain onto each index (Fourier-Motzkin)
// for the point box, compiles bodies to postfix programs.  Throws Unbounded /
// Validation like the reference.
// `maps` (may be empty): the reference's MemoryMaps — storage of each mapped
// array is laid out exactly by its map (words, modulo folding, extents), as the
// reference's ArrayStore is; unmapped arrays are dense at declared extents.
// host_only: the plan tables without device storage (the emitter's source).
GenericPlan* generic_plan_create(const KernelSpec& k, const IntVec& params,
                                 const std::vector<MemoryMap>& maps, int device,
                                 bool host_only = false);
void generic_plan_destroy(GenericPlan* p);

// Array access (dense, declaration extents).
size_t generic_array_count(const GenericPlan* p);
const std::string& generic_array_name(const GenericPlan* p, size_t i);
ArrayKind generic_array_kind(const GenericPlan* p, size_t i);
uint64_t generic_array_words(const GenericPlan* p, size_t i);
double* generic_array_ptr(GenericPlan* p, size_t i);

// Inputs <- init_value, temps/outputs <- 0.0 (reference init_storage,
// exec.cpp:281-294); the inputs are kept, everything else is reset per run.
cudaError_t generic_init_inputs(GenericPlan* p, cudaStream_t s);
struct GenericCounts {
  uint64_t points = 0, reads = 0, writes = 0;
  bool parallel = false;  // dataflow grid (true) or sequential walk
  int mode = 0;           // 0 sequential, 1 dataflow over dense flags, 2 dataflow over shadows
  bool compiled = false;  // the emitter's NVRTC-compiled kernels ran (else the interpreter)
};
// One run.  Errors: cudaErrorInvalidValue with `err_msg` set for an
// out-of-extent access (reference exec.cpp:318-323).
cudaError_t generic_run(GenericPlan* p, cudaStream_t s, GenericCounts* counts, std::string* err_msg);

// PRDG -> CUDA emitter (the GPU analogue of the reference's emit_c): the
// plan's statements as device source (host only), and its NVRTC build; the
// runs use the compiled kernels when the build succeeds (PCOTGPU_GENERIC_JIT=0:
// interpreter).  generic_jit_status: "compiled" or why not.
std::string generic_emit_source(const GenericPlan* p);
bool generic_jit_build(GenericPlan* p);
const std::string& generic_jit_status(const GenericPlan* p);
bool generic_jit_compile_check(const GenericPlan* p, std::string* log);

}  // namespace pcotgpu
