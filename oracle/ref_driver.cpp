// TEST INFRASTRUCTURE — part of the parity oracle, never part of the product.
//
// pcot_ref: a thin driver around the UNMODIFIED reference library compiled
// from /root/reference/proj/core/src (see oracle/Makefile).  It exercises the
// reference's own public API exactly as its CLI does (tools/pcot.cpp:238-336):
//   parse_kernel_file -> allocate / single_assignment_maps -> slt/cot order
//   -> Executor::run / run_untiled -> ExecResult.checksum
// and the reference's compiled path (emit_c, emit_c.cpp:342-380) used as the
// large-size oracle and as the timed CPU baseline.
//
// Usage:
//   pcot_ref run  <kernel> T=..,N=.. [--alloc] [--scheme untiled|slt|cot]
//                 [--tile a,b,c] [--no-oracle] [--dump <file>]
//   pcot_ref emit <kernel> T=..,N=.. [--openmp] [--leaf a,b,c] -o <file.c>
//   pcot_ref parse <kernel>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "pcot/emit_c.hpp"
#include "pcot/exec.hpp"
#include "pcot/kernel_io.hpp"
#include "pcot/memalloc.hpp"
#include "pcot/tiler.hpp"

namespace {

std::vector<std::int64_t> split_ints(const std::string& s) {
  std::vector<std::int64_t> v;
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
  std::vector<bool> seen(p.params.size(), false);
  std::size_t i = 0;
  while (i < spec.size()) {
    std::size_t j = spec.find(',', i);
    if (j == std::string::npos) j = spec.size();
    std::string kv = spec.substr(i, j - i);
    std::size_t eq = kv.find('=');
    if (eq == std::string::npos) throw std::runtime_error("bad param " + kv);
    std::string k = kv.substr(0, eq);
    bool found = false;
    for (std::size_t q = 0; q < p.params.size(); ++q)
      if (p.params[q] == k) {
        out[q] = std::stoll(kv.substr(eq + 1));
        seen[q] = found = true;
      }
    if (!found) throw std::runtime_error("unknown param " + k);
    i = j + 1;
  }
  for (std::size_t q = 0; q < seen.size(); ++q)
    if (!seen[q]) throw std::runtime_error("missing param " + p.params[q]);
  return out;
}

pcot::Prdg load(const std::string& name) {
  std::string path = pcot::find_kernel_file(name);
  if (path.empty()) throw std::runtime_error("kernel not found: " + name);
  return pcot::parse_kernel_file(path);
}

int cmd_run(int argc, char** argv) {
  pcot::Prdg p = load(argv[2]);
  pcot::IntVec params = bind(p, argv[3]);
  bool use_alloc = false, oracle = true;
  std::string scheme = "untiled", tile, dump;
  for (int i = 4; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--alloc") use_alloc = true;
    else if (a == "--no-oracle") oracle = false;
    else if (a == "--scheme") scheme = argv[++i];
    else if (a == "--tile") tile = argv[++i];
    else if (a == "--dump") dump = argv[++i];
    else throw std::runtime_error("unknown flag " + a);
  }
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
  pcot::Executor ex(e, params, maps);
  pcot::ExecOptions opts;
  opts.check_oracle = oracle;
  auto t0 = std::chrono::steady_clock::now();
  pcot::ExecResult r;
  if (scheme == "untiled") {
    r = ex.run_untiled(opts);
  } else {
    pcot::TileSpec ts{split_ints(tile)};
    pcot::TileOrder order = scheme == "slt" ? pcot::slt_order(e, params, ts)
                                            : pcot::cot_order(e, params, ts);
    r = ex.run(order, opts);
  }
  double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("kernel %s\n", p.name.c_str());
  std::printf("points %" PRIu64 "\nreads %" PRIu64 "\nwrites %" PRIu64 "\n", r.points,
              r.reads, r.writes);
  std::printf("violation %d\n", r.violation ? 1 : 0);
  if (r.violation) std::printf("violation_msg %s\n", r.violation_msg.c_str());
  std::printf("seconds %.6f\n", secs);
  std::printf("CHECKSUM %016" PRIx64 "\n", r.checksum);
  if (!dump.empty()) {
    std::ofstream f(dump, std::ios::binary);
    for (const auto& a : e.arrays)
      if (a.kind == pcot::ArrayKind::Output) {
        const auto& d = ex.array_data(a.name);
        f.write(reinterpret_cast<const char*>(d.data()), std::streamsize(d.size() * 8));
      }
  }
  return r.violation ? 4 : 0;
}

int cmd_emit(int argc, char** argv) {
  pcot::Prdg p = load(argv[2]);
  pcot::IntVec params = bind(p, argv[3]);
  pcot::EmitOptions opts;
  opts.use_alloc = true;
  std::string outp;
  for (int i = 4; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--openmp") opts.openmp = true;
    else if (a == "--no-alloc") opts.use_alloc = false;
    else if (a == "--leaf") opts.leaf_defaults = split_ints(argv[++i]);
    else if (a == "-o") outp = argv[++i];
    else throw std::runtime_error("unknown flag " + a);
  }
  std::string src = pcot::emit_c(p, params, opts);
  std::ofstream f(outp);
  f << src;
  return f ? 0 : 3;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: pcot_ref run|emit|parse <kernel> ...\n");
    return 2;
  }
  try {
    std::string cmd = argv[1];
    if (cmd == "parse") {
      pcot::Prdg p = load(argv[2]);
      std::printf("ok %s statements %zu\n", p.name.c_str(), p.statements.size());
      return 0;
    }
    if (argc < 4) return 2;
    if (cmd == "run") return cmd_run(argc, argv);
    if (cmd == "emit") return cmd_emit(argc, argv);
  } catch (const pcot::Error& e) {
    std::fprintf(stderr, "pcot error (kind %d): %s\n", int(e.kind()), e.what());
    return 5;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 5;
  }
  return 2;
}
