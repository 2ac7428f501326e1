// `pcot run` with the GPU executor switch.
//
// The reference CLI's `run` subcommand (reference tools/pcot.cpp:238-336,
// cmd_run) rebuilt around one change — the executor line:
//
//     ExecResult r = executor == "gpu" ? pcot::GpuExecutor(e, params, maps).run(order)
//                                      : pcot::Executor(e, params, maps).run(order, opts);
//
// Same front end (parse_kernel_file / find_kernel_file, allocate or
// single_assignment_maps, slt_order, cot_order + assign_wavefront_phases),
// same option names, same stdout lines and exit codes (0 ok, 2 usage, 3 io,
// 4 oracle violation, 5 kernel error; pcot.cpp:28-32, 622-634).  The
// reference's CLI11 front end is not in this image (vendor/ is not shipped),
// so the options are parsed by hand; the cache simulator lines are printed by
// the CPU executor only (the GPU path has no per-access trace: `cache -`,
// `OCA -`, plus the device time).
//
//   pcot_run <kernel> -p N=..,T=.. [--scheme untiled|slt|cot] [--tile a,b,c]
//            [--alloc] [--no-check] [--wavefront --seed S] [--executor gpu|cpu]
//
// Built by oracle/Makefile against the unmodified reference library and
// include/pcotgpu.h + integration/pcot/gpu_executor.hpp.
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "pcot/cachesim.hpp"
#include "pcot/exec.hpp"
#include "pcot/gpu_executor.hpp"
#include "pcot/kernel_io.hpp"
#include "pcot/memalloc.hpp"
#include "pcot/tiler.hpp"

namespace {

constexpr int kExitOk = 0, kExitUsage = 2, kExitIo = 3, kExitOracle = 4, kExitKernel = 5;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
[[noreturn]] void usage_fail(const std::string& m) { throw UsageError(m); }

std::vector<std::string> split(const std::string& s, char d) {
  std::vector<std::string> out;
  std::size_t i = 0;
  while (i <= s.size()) {
    std::size_t j = s.find(d, i);
    if (j == std::string::npos) j = s.size();
    out.push_back(s.substr(i, j - i));
    i = j + 1;
  }
  return out;
}

std::int64_t parse_i64(const std::string& s, const std::string& what) {
  try {
    std::size_t n = 0;
    const long long v = std::stoll(s, &n);
    if (n != s.size()) throw std::invalid_argument(s);
    return v;
  } catch (const std::exception&) {
    usage_fail("bad " + what + " '" + s + "'");
  }
}

pcot::IntVec parse_tile(const std::string& s) {
  pcot::IntVec t;
  for (const auto& tok : split(s, ',')) t.push_back(parse_i64(tok, "tile size"));
  for (auto v : t)
    if (v <= 0) usage_fail("tile sizes must be positive, got '" + s + "'");
  return t;
}

pcot::IntVec bind_kernel_params(const pcot::Prdg& p, const std::vector<std::string>& kvs) {
  std::map<std::string, std::int64_t> vals;
  for (const auto& arg : kvs)
    for (const auto& one : split(arg, ',')) {
      const auto eq = one.find('=');
      if (eq == std::string::npos) usage_fail("expected NAME=VALUE, got '" + one + "'");
      vals[one.substr(0, eq)] = parse_i64(one.substr(eq + 1), "parameter value");
    }
  pcot::IntVec out;
  for (const auto& name : p.params) {
    auto it = vals.find(name);
    if (it == vals.end()) usage_fail("kernel parameter " + name + " not set (use -p " + name + "=V)");
    out.push_back(it->second);
    vals.erase(it);
  }
  if (!vals.empty()) usage_fail("unknown kernel parameter " + vals.begin()->first);
  return out;
}

std::string params_string(const pcot::Prdg& p, const pcot::IntVec& params) {
  std::string s;
  for (std::size_t i = 0; i < p.params.size(); ++i)
    s += (i ? ";" : "") + p.params[i] + "=" + std::to_string(params[i]);
  return s;
}

std::string tile_string(const pcot::IntVec& t) {
  std::string s;
  for (std::size_t i = 0; i < t.size(); ++i) s += (i ? "x" : "") + std::to_string(t[i]);
  return t.empty() ? "-" : s;
}

int cmd_run(const std::string& kernel, const std::vector<std::string>& pvals, const std::string& scheme_s,
            const std::string& tile_s, bool use_alloc, bool wavefront, std::uint64_t seed, bool no_check,
            const std::string& executor) {
  const std::string path = pcot::find_kernel_file(kernel);
  if (path.empty()) throw pcot::Error(pcot::ErrorKind::Io, "kernel not found: " + kernel);
  pcot::Prdg p = pcot::parse_kernel_file(path);
  pcot::IntVec params = bind_kernel_params(p, pvals);
  pcot::Scheme scheme;
  if (scheme_s == "untiled") scheme = pcot::Scheme::Untiled;
  else if (scheme_s == "slt") scheme = pcot::Scheme::Slt;
  else if (scheme_s == "cot") scheme = pcot::Scheme::Cot;
  else usage_fail("unknown scheme '" + scheme_s + "' (untiled|slt|cot)");
  if (executor != "gpu" && executor != "cpu") usage_fail("unknown executor '" + executor + "' (gpu|cpu)");

  pcot::Prdg e;
  std::vector<pcot::MemoryMap> maps;
  if (use_alloc) {
    pcot::AllocResult ar = pcot::allocate(p, params);
    e = std::move(ar.transformed);
    maps = std::move(ar.maps);
  } else {
    e = p.is_perfect() ? p : pcot::embed(p);
    maps = pcot::single_assignment_maps(e, params);
  }
  pcot::TileOrder order;
  if (scheme == pcot::Scheme::Untiled) {
    if (!tile_s.empty()) usage_fail("--tile has no effect with --scheme untiled");
  } else {
    if (tile_s.empty()) usage_fail("--tile is required for slt/cot");
    const pcot::IntVec tile = parse_tile(tile_s);
    if (tile.size() != e.tilable_band.size())
      usage_fail("tile has " + std::to_string(tile.size()) + " sizes, band has " +
                 std::to_string(e.tilable_band.size()));
    if (scheme == pcot::Scheme::Slt) {
      order = pcot::slt_order(e, params, pcot::TileSpec{tile});
    } else {
      order = pcot::assign_wavefront_phases(pcot::cot_order(e, params, pcot::TileSpec{tile}));
      if (wavefront) order = pcot::linearize_wavefront(order, seed);
    }
  }

  pcot::ExecResult r;
  double device_ms = -1.0;
  pcot::CacheSim sim(pcot::parse_cache_spec("desk-llc"));
  if (executor == "gpu") {  // the one changed line of cmd_run (pcot.cpp:288-293)
    pcot::GpuExecutor ex(e, params, maps);
    const auto t0 = std::chrono::steady_clock::now();
    r = scheme == pcot::Scheme::Untiled ? ex.run_untiled() : ex.run(order);
    device_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  } else {
    pcot::Executor ex(e, params, maps);
    pcot::ExecOptions opts;
    opts.check_oracle = !no_check;
    opts.sink = &sim;
    r = scheme == pcot::Scheme::Untiled ? ex.run_untiled(opts) : ex.run(order, opts);
  }
  std::printf("kernel %s\n", p.name.c_str());
  std::printf("params %s\n", params_string(p, params).c_str());
  std::printf("scheme %s\n", scheme_s.c_str());
  std::printf("tile %s\n", scheme == pcot::Scheme::Untiled ? "-" : tile_string(parse_tile(tile_s)).c_str());
  std::printf("points %llu\n", (unsigned long long)r.points);
  std::printf("reads %llu\n", (unsigned long long)r.reads);
  std::printf("writes %llu\n", (unsigned long long)r.writes);
  const std::size_t leaves = scheme == pcot::Scheme::Untiled ? 1 : order.leaves.size();
  std::printf("leaves %zu\n", leaves);
  std::printf("nodes %zu\n", scheme == pcot::Scheme::Cot ? order.nodes_visited : leaves);
  std::printf("CHECKSUM %016llx\n", (unsigned long long)r.checksum);
  std::printf("executor %s\n", executor.c_str());
  if (executor == "gpu") {
    std::printf("cache -\n");
    std::printf("OCA -\n");
    std::printf("wall_ms %.3f\n", device_ms);
  } else {
    std::printf("cache %s\n", pcot::cache_spec_string(pcot::parse_cache_spec("desk-llc")).c_str());
    const auto& st = sim.stats();
    for (std::size_t l = 0; l < st.levels.size(); ++l)
      std::printf("level %zu accesses %llu misses %llu\n", l, (unsigned long long)st.levels[l].accesses,
                  (unsigned long long)st.levels[l].misses);
    std::printf("OCA %llu\n", (unsigned long long)st.oca());
  }
  if (r.violation) {
    std::fprintf(stderr, "oracle: %s\n", r.violation_msg.c_str());
    return kExitOracle;
  }
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    std::string kernel, scheme = "untiled", tile, executor = "gpu";
    std::vector<std::string> pvals;
    bool use_alloc = false, wavefront = false, no_check = false;
    std::uint64_t seed = 1;
    for (int i = 1; i < argc; ++i) {
      const std::string a = argv[i];
      auto value = [&](const char* opt) -> std::string {
        if (i + 1 >= argc) usage_fail(std::string(opt) + " needs a value");
        return argv[++i];
      };
      if (a == "-p" || a == "--param") pvals.push_back(value("-p"));
      else if (a == "--scheme") scheme = value("--scheme");
      else if (a == "--tile") tile = value("--tile");
      else if (a == "--executor") executor = value("--executor");
      else if (a == "--seed") seed = std::uint64_t(parse_i64(value("--seed"), "seed"));
      else if (a == "--alloc") use_alloc = true;
      else if (a == "--wavefront") wavefront = true;
      else if (a == "--no-check") no_check = true;
      else if (!a.empty() && a[0] == '-') usage_fail("unknown option " + a);
      else if (kernel.empty()) kernel = a;
      else usage_fail("unexpected argument " + a);
    }
    if (kernel.empty()) usage_fail("usage: pcot_run <kernel> -p NAME=V[,..] [--scheme] [--tile] [--alloc] [--executor gpu|cpu]");
    return cmd_run(kernel, pvals, scheme, tile, use_alloc, wavefront, seed, no_check, executor);
  } catch (const UsageError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitUsage;
  } catch (const pcot::Error& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return e.kind() == pcot::ErrorKind::Io ? kExitIo : kExitKernel;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitKernel;
  }
}
