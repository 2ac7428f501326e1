// pcot::GpuExecutor — the reference-side binding of the B200 executor.
//
// This is the file a maintainer adds to the reference tree
// (proj/core/include/pcot/gpu_executor.hpp).  It is a drop-in for
// pcot::Executor (reference core/include/pcot/exec.hpp:62-82): same
// constructor (embedded Prdg, params, MemoryMaps), same run / run_untiled /
// reset / array_data / array_base, same error kinds (pcot::Error with the
// reference ErrorKind, error.hpp:8-16).  Everything crosses the C ABI of
// include/pcotgpu.h: the Prdg is re-serialised with the reference's own
// print_kernel (kernel_io.hpp:17), the maps are passed field by field.
//
// Compiled against the unmodified reference headers by
// tests/c/ref_adapter_demo.cpp (oracle/Makefile), which runs the reference's
// own parse_kernel_file -> allocate -> slt_order / cot_order -> run ->
// array_data sequence through it (tests/test_ref_adapter.py).
#pragma once

#include <pcotgpu.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "pcot/exec.hpp"
#include "pcot/kernel_io.hpp"
#include "pcot/memalloc.hpp"
#include "pcot/tiler.hpp"

namespace pcot {

class GpuExecutor {
 public:
  GpuExecutor(const Prdg& embedded, const IntVec& params, const std::vector<MemoryMap>& maps,
              int device = 0) {
    const std::string json = print_kernel(embedded);
    // flatten the maps into the ABI's plain arrays (kept alive for the call)
    std::vector<std::vector<std::int64_t>> lin(maps.size());
    std::vector<pcotgpu_map> cm(maps.size());
    for (std::size_t i = 0; i < maps.size(); ++i) {
      const MemoryMap& m = maps[i];
      const std::size_t rank = m.map.linear.empty() ? 0 : m.map.linear[0].size();
      for (const auto& row : m.map.linear) lin[i].insert(lin[i].end(), row.begin(), row.end());
      pcotgpu_map& c = cm[i];
      c.array = m.array.c_str();
      c.rank = std::int32_t(rank);
      c.storage_rank = std::int32_t(m.extents.size());
      c.linear = lin[i].data();
      c.constant = m.map.constant.data();
      c.moduli = m.moduli.data();
      c.extents = m.extents.data();
      c.single_assignment = m.single_assignment ? 1 : 0;
      c.reserved = 0;
    }
    check(pcotgpu_create_mapped(json.c_str(), params.data(), params.size(), cm.data(), cm.size(),
                                device, &h_));
  }
  ~GpuExecutor() { pcotgpu_destroy(h_); }
  GpuExecutor(const GpuExecutor&) = delete;
  GpuExecutor& operator=(const GpuExecutor&) = delete;

  // The order's scheme and its leaf size (the TileSpec it was built from)
  // select the GPU schedule; leaf[0] (time) is the temporal block depth.
  ExecResult run(const TileOrder& order, const ExecOptions& opts = {}) {
    if (opts.sink) fail(ErrorKind::Unsupported, "GpuExecutor: per-access traces are not produced");
    pcotgpu_schedule s{};
    s.scheme = order.scheme == Scheme::Slt ? PCOTGPU_SLT
             : order.scheme == Scheme::Cot ? PCOTGPU_COT : PCOTGPU_UNTILED;
    if (order.scheme != Scheme::Untiled && !order.leaves.empty()) {
      const OrthantBox& b = order.leaves.front();
      s.ndim = std::int32_t(b.size.size() < 8 ? b.size.size() : 8);
      for (std::int32_t i = 0; i < s.ndim; ++i) s.leaf[i] = b.size[std::size_t(i)];
    }
    return convert(&s);
  }
  ExecResult run_untiled(const ExecOptions& opts = {}) {
    if (opts.sink) fail(ErrorKind::Unsupported, "GpuExecutor: per-access traces are not produced");
    return convert(nullptr);
  }
  void reset() {
    check(pcotgpu_reset(h_));
    cache_.clear();
  }
  const std::vector<double>& array_data(const std::string& a) const {
    std::uint64_t w = 0;
    check(pcotgpu_array_words(h_, a.c_str(), &w));
    std::vector<double>& v = cache_[a];
    v.resize(w);
    check(pcotgpu_read_array(h_, a.c_str(), v.data(), w));
    return v;
  }
  std::uint64_t array_base(const std::string& a) const {
    std::uint64_t b = 0;
    check(pcotgpu_array_base(h_, a.c_str(), &b));
    return b;
  }
  // pcotgpu_result.bt of the last run (temporal depth; interpreter schedule)
  int last_bt() const { return last_bt_; }
  int family() const {
    pcotgpu_kernel_info i{};
    check(pcotgpu_info(h_, &i));
    return i.family;
  }

 private:
  static void check(int st) {
    if (st == PCOTGPU_OK) return;
    // device failures have no reference kind: reported as Validation (the run
    // produced no valid result), with the CUDA message
    if (st == PCOTGPU_E_CUDA) fail(ErrorKind::Validation, pcotgpu_last_error());
    fail(ErrorKind(st - 1), pcotgpu_last_error());
  }
  ExecResult convert(const pcotgpu_schedule* s) {
    pcotgpu_result r{};
    check(pcotgpu_run(h_, s, &r));
    cache_.clear();
    last_bt_ = r.bt;
    ExecResult e;
    e.points = r.points;
    e.reads = r.reads;
    e.writes = r.writes;
    e.violation = r.violation != 0;
    e.checksum = r.checksum;
    return e;
  }
  pcotgpu_handle* h_ = nullptr;
  int last_bt_ = 0;
  mutable std::map<std::string, std::vector<double>> cache_;
};

}  // namespace pcot
