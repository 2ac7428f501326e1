// TEST INFRASTRUCTURE — the reference-side boundary, exercised for real.
//
// Compiled against the UNMODIFIED reference headers and library
// (oracle/Makefile -> oracle/_ref/ref_adapter_demo; the library is the
// checker) together with integration/pcot/gpu_executor.hpp, the adapter a
// maintainer adds to the reference tree.  It runs the reference's own call
// sequence — parse_kernel_file -> allocate (or single_assignment_maps) ->
// slt_order / cot_order -> run -> array_data (reference tools/pcot.cpp:
// 238-336, tests/acceptance.cpp:154-165 run_order) — once through
// pcot::GpuExecutor (the B200) and, unless --gpu-only, once through the
// reference pcot::Executor on the CPU, and prints both results.
//
//   ref_adapter_demo <kernel> T=..,N=.. [--single] [--scheme untiled|slt|cot]
//                    [--tile a,b,c] [--gpu-only] [--maps-only] [--fold-modulus k]
//
// --maps-only prints the maps and exits (no device needed); --fold-modulus k
// rewrites the temp's folded modulus to k (a map the hot path must not accept).
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "pcot/exec.hpp"
#include "pcot/gpu_executor.hpp"
#include "pcot/kernel_io.hpp"
#include "pcot/memalloc.hpp"
#include "pcot/tiler.hpp"

namespace {

pcot::IntVec split_ints(const std::string& s) {
  pcot::IntVec v;
  std::size_t i = 0;
  while (i < s.size()) {
    std::size_t j = s.find(',', i);
    if (j == std::string::npos) j = s.size();
    v.push_back(std::stoll(s.substr(i, j - i)));
    i = j + 1;
  }
  return v;
}

pcot::IntVec bind(const pcot::Prdg& p, const std::string& spec) {
  pcot::IntVec out(p.params.size(), 0);
  std::size_t i = 0;
  while (i < spec.size()) {
    std::size_t j = spec.find(',', i);
    if (j == std::string::npos) j = spec.size();
    const std::string kv = spec.substr(i, j - i);
    const std::size_t eq = kv.find('=');
    for (std::size_t q = 0; q < p.params.size(); ++q)
      if (p.params[q] == kv.substr(0, eq)) out[q] = std::stoll(kv.substr(eq + 1));
    i = j + 1;
  }
  return out;
}

void print_maps(const std::vector<pcot::MemoryMap>& maps) {
  for (const auto& m : maps) {
    std::printf("MAP %s moduli", m.array.c_str());
    for (auto v : m.moduli) std::printf(" %" PRId64, v);
    std::printf(" extents");
    for (auto v : m.extents) std::printf(" %" PRId64, v);
    std::printf(" linear");
    for (const auto& row : m.map.linear) {
      std::printf(" [");
      for (auto v : row) std::printf(" %" PRId64, v);
      std::printf(" ]");
    }
    std::printf(" constant");
    for (auto v : m.map.constant) std::printf(" %" PRId64, v);
    std::printf("\n");
  }
}

pcot::TileOrder make_order(const pcot::Prdg& e, const pcot::IntVec& params, const std::string& scheme,
                           const pcot::IntVec& tile) {
  if (scheme == "slt") return pcot::slt_order(e, params, pcot::TileSpec{tile});
  if (scheme == "cot") return pcot::cot_order(e, params, pcot::TileSpec{tile});
  return pcot::TileOrder{};
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s <kernel> T=..,N=.. [options]\n", argv[0]);
    return 2;
  }
  bool single = false, gpu_only = false, maps_only = false;
  std::string scheme = "untiled";
  pcot::IntVec tile;
  std::int64_t fold = 0;
  for (int i = 3; i < argc; ++i) {
    const std::string a = argv[i];
    if (a == "--single") single = true;
    else if (a == "--gpu-only") gpu_only = true;
    else if (a == "--maps-only") maps_only = true;
    else if (a == "--scheme" && i + 1 < argc) scheme = argv[++i];
    else if (a == "--tile" && i + 1 < argc) tile = split_ints(argv[++i]);
    else if (a == "--fold-modulus" && i + 1 < argc) fold = std::stoll(argv[++i]);
  }
  try {
    const std::string path = pcot::find_kernel_file(argv[1]);
    if (path.empty()) throw std::runtime_error(std::string("kernel not found: ") + argv[1]);
    const pcot::Prdg p = pcot::parse_kernel_file(path);
    const pcot::IntVec params = bind(p, argv[2]);
    pcot::Prdg e;
    std::vector<pcot::MemoryMap> maps;
    if (single) {
      e = p.is_perfect() ? p : pcot::embed(p);
      maps = pcot::single_assignment_maps(e, params);
    } else {
      pcot::AllocResult ar = pcot::allocate(p, params);
      e = std::move(ar.transformed);
      maps = std::move(ar.maps);
    }
    if (fold > 0)
      for (auto& m : maps)
        for (auto& mod : m.moduli)
          if (mod > 0) mod = fold, m.extents[std::size_t(&mod - m.moduli.data())] = fold;
    print_maps(maps);
    if (maps_only) return 0;
    if (scheme != "untiled" && tile.empty()) tile.assign(e.tilable_band.size(), 8);
    const pcot::TileOrder order = make_order(e, params, scheme, tile);

    pcot::GpuExecutor gx(e, params, maps);
    const pcot::ExecResult g = scheme == "untiled" ? gx.run_untiled() : gx.run(order);
    std::printf("GPU_FAMILY %d\n", gx.family());
    std::printf("GPU_MODE %d\n", gx.last_bt());
    std::printf("GPU_CHECKSUM %016" PRIx64 "\n", g.checksum);
    std::printf("GPU_COUNTS %" PRIu64 " %" PRIu64 " %" PRIu64 "\n", g.points, g.reads, g.writes);
    for (const auto& a : e.arrays)
      if (a.kind != pcot::ArrayKind::Temp)
        std::printf("GPU_ARRAY %s base %" PRIu64 " words %zu\n", a.name.c_str(), gx.array_base(a.name),
                    gx.array_data(a.name).size());
    gx.reset();
    const pcot::ExecResult g2 = scheme == "untiled" ? gx.run_untiled() : gx.run(order);
    std::printf("GPU_RERUN_CHECKSUM %016" PRIx64 "\n", g2.checksum);
    if (!gpu_only) {
      pcot::Executor rx(e, params, maps);
      pcot::ExecOptions opts;
      opts.check_oracle = false;
      const pcot::ExecResult r = scheme == "untiled" ? rx.run_untiled(opts) : rx.run(order, opts);
      std::printf("REF_CHECKSUM %016" PRIx64 "\n", r.checksum);
      std::printf("REF_COUNTS %" PRIu64 " %" PRIu64 " %" PRIu64 "\n", r.points, r.reads, r.writes);
      for (const auto& a : e.arrays)
        if (a.kind != pcot::ArrayKind::Temp)
          std::printf("REF_ARRAY %s base %" PRIu64 " words %zu\n", a.name.c_str(), rx.array_base(a.name),
                      rx.array_data(a.name).size());
    }
  } catch (const pcot::Error& err) {
    std::printf("ERROR %d %s\n", int(err.kind()), err.what());
    return 3;
  } catch (const std::exception& err) {
    std::printf("ERROR -1 %s\n", err.what());
    return 3;
  }
  return 0;
}
