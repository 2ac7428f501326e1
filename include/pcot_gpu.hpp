// pcotgpu C++ API — the GPU executor as a drop-in for pcot::Executor.
//
// Same member names, argument meaning and error behaviour as the reference
// Executor (reference proj/core/include/pcot/exec.hpp:40-82) and kernel
// registration API (kernel_io.hpp:11-22).  Types are this library's own
// mirrors (the reference headers are not a dependency); INTEGRATION.md shows
// the adapter from pcot::Prdg (print_kernel) to this class.
#pragma once
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../paper_1802_00166_b200/csrc/spec.h"

namespace pcotgpu {

// reference tiler.hpp:12-31
struct TileSpec {
  IntVec leaf;
};
enum class Scheme { Untiled, Slt, Cot };
struct TileOrder {
  Scheme scheme = Scheme::Untiled;
  TileSpec tile;  // leaf sizes of the order (leaf[0]: time -> temporal block depth)
  // COT only: the recursive order spans time too (reference cot_order recurses
  // over the whole band box, t included, tiler.cpp:150-203): 2-D stencils run
  // one launch per (depth block, row band of tile.leaf[1] rows), visited in
  // Morton order over the skewed (block, band + 2 block) box, so a band goes
  // through several depth blocks while it is L2-resident.
  bool space_time = false;
};

// reference exec.hpp:40-52
struct ExecOptions {
  bool check_oracle = true;  // legality holds by construction on the device
  void* sink = nullptr;      // per-access traces are not produced: non-null -> Unsupported
  bool skip_checksum = false;
};
struct ExecResult {
  uint64_t points = 0, reads = 0, writes = 0;
  bool violation = false;
  std::string violation_msg;
  uint64_t checksum = 0;
  double device_ms = 0.0;
  int bt = 0;
  uint64_t launches = 0;
};

// MemoryMap: reference memalloc.hpp:14-33 (declared in spec.h).  Maps the
// hand-written kernels' device layouts reproduce (identity inputs/outputs,
// the temp single-assignment or folded along a multiple of the kernel's
// occupancy vector: allocate()'s maps) keep the hot path; any other map set
// runs on the device interpreter with storage laid out by the maps.

class GpuExecutor {
 public:
  GpuExecutor(const KernelSpec& embedded, const IntVec& params,
              const std::vector<MemoryMap>& maps = {}, int device = 0);
  ~GpuExecutor();
  GpuExecutor(const GpuExecutor&) = delete;
  GpuExecutor& operator=(const GpuExecutor&) = delete;

  ExecResult run(const TileOrder& order, const ExecOptions& opts = {});
  ExecResult run_untiled(const ExecOptions& opts = {});
  // beyond the reference API: `count` independent runs from host memory with
  // the host<->device copies overlapped with the compute (two copy streams).
  // host_inputs[k * ninputs + q]: instance k's input q (dense, array_words);
  // host_outputs[k]: instance k's output.  Pinned host memory keeps the copies
  // asynchronous.  Inputs of the last instance remain the executor's inputs.
  ExecResult run_batch(const TileOrder& order, size_t count, const double* const* host_inputs,
                       double* const* host_outputs, const ExecOptions& opts = {});
  void reset();
  const std::vector<double>& array_data(const std::string& array) const;
  uint64_t array_base(const std::string& array) const;
  uint64_t array_words(const std::string& array) const;

  // beyond the reference API
  const Recognized& recognized() const;
  // device interpreter only: last run's schedule, compiled (emitter) or not, build status
  void generic_info(int* mode, int* compiled, std::string* why) const;
  void write_array(const std::string& array, const double* host, size_t n);
  void read_array(const std::string& array, double* host, size_t n) const;
  double* device_view(const std::string& array, int64_t* ld);
  void set_stream(void* stream);

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};

}  // namespace pcotgpu
