// GpuExecutor (drop-in for pcot::Executor, reference exec.hpp:62-82) and the
// C ABI in include/pcotgpu.h.
//
// Device layout (HBM):
//   2-D stencils: two ping-pong slabs of (N + 2*ghost) rows x ld doubles, ld a
//     multiple of 16 (128 B) with >= 16 pad columns left and a right pad that
//     covers the last strip's TMA window; the input F kept dense N x N.
//   3-D stencils: two padded cubes (halo planes/rows/cols), F dense N^3.
//   Gauss-Seidel: one in-place N x ld grid (the reference allocate() map
//     (t mod 1, x-t, y-2t) is a bijection with (i, j), so cell (i,j) holds
//     every version in place), F dense.
//   GEMM: A, B (init values), A' = 2A-1, B' = 2B-1, Out, all N x ld.
// Every run starts from the inputs, as the reference's run does (its init
// statement re-reads F every time), so storage persists across runs exactly
// as the reference describes (exec.hpp:69-75).
#include "../../include/pcot_gpu.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/pcotgpu.h"
#include "generic.h"
#include "kernels.h"

namespace pcotgpu {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    fail(ErrorKind::Cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

constexpr int64_t kGhost = 16;  // ghost rows / halo planes (>= max bt + 3)
constexpr int64_t kPadL = 16;   // left pad columns (128 B)
constexpr int64_t kPadR2 = 1040; // right pad for the 2-D strip window (>= W_IN + 2, widest variant)
constexpr int64_t kPadR3 = 80;  // right pad for the 3-D window (>= 66 + halo)

struct DevBuf {
  double* p = nullptr;
  size_t n = 0;
  void alloc(size_t count) {
    n = count;
    ck(cudaMalloc(&p, count * sizeof(double)), "cudaMalloc");
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

}  // namespace

struct GpuExecutor::Impl {
  KernelSpec spec;
  IntVec params;
  std::vector<MemoryMap> maps;  // the caller's (empty: device layouts / dense)
  Recognized rec;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  int64_t n = 0, T = 0;
  // inputs (dense)
  DevBuf in[2];
  int64_t in_ld = 0;
  // 2-D slabs
  DevBuf slab[2];
  Slab2D sg[2];
  // 3-D cubes
  DevBuf cube[2];
  Grid3D cg[2];
  // GS grid
  DevBuf gsa;
  int64_t gs_ld = 0;
  GsPlan* gs_plan = nullptr;
  S2ResPlan* res_plan = nullptr;  // on-chip resident 2-D stencil (small grids)
  bool res_tried = false;
  int gs_cfg[3] = {0, 0, 0};
  int gs_pipe_ok = -1;
  // GEMM
  DevBuf gA, gB, gC;
  int64_t g_ld = 0;
  int result_slot = -1;  // which buffer holds the output after a run (-1: none)
  mutable std::map<std::string, std::vector<double>> mirror;
  // generic device interpreter (kernels outside the hot-path registry)
  bool generic = false;
  GenericPlan* gplan = nullptr;
  GenericCounts gcounts;
  int garray(const std::string& a) const {
    for (size_t i = 0; i < generic_array_count(gplan); ++i)
      if (generic_array_name(gplan, i) == a) return int(i);
    return -1;
  }
  // batched host runs (run_batch): copy streams and device staging
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t e_start = nullptr, e_in = nullptr, e_prev = nullptr, e_out = nullptr, e_free = nullptr;
  DevBuf stage_in[2], stage_out;

  ~Impl() {
    for (cudaEvent_t e : {e_start, e_in, e_prev, e_out, e_free})
      if (e) cudaEventDestroy(e);
    if (h2d) cudaStreamDestroy(h2d);
    if (d2h) cudaStreamDestroy(d2h);
    if (gs_plan) gs2d_plan_destroy(gs_plan);
    if (res_plan) s2d5_res_destroy(res_plan);
    if (gplan) generic_plan_destroy(gplan);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }

  uint64_t words_of(const std::string& a) const {
    const ArrayDecl* d = spec.find_array(a);
    if (!d) fail(ErrorKind::Validation, "array_data: unknown array " + a);
    if (generic) return generic_array_words(gplan, size_t(garray(a)));
    if (rec.family == Family::Gemm) return uint64_t(n) * uint64_t(n);
    uint64_t w = 1;
    for (int i = 0; i < rec.ndim; ++i) w *= uint64_t(n);
    if (d->kind == ArrayKind::Temp && rec.family != Family::GaussSeidel2D9) w *= 2;  // ping-pong
    return w;
  }

  void init_inputs() {
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (generic) {
      ck(generic_init_inputs(gplan, stream), "generic init");
      for (size_t i = 0; i < generic_array_count(gplan); ++i)  // temps/outputs: 0.0
        if (generic_array_kind(gplan, i) != ArrayKind::Input && generic_array_words(gplan, i))
          ck(cudaMemsetAsync(generic_array_ptr(gplan, i), 0, generic_array_words(gplan, i) * 8, stream),
             "cudaMemset");
      ck(cudaStreamSynchronize(stream), "init inputs");
      mirror.clear();
      return;
    }
    for (size_t q = 0; q < rec.inputs.size(); ++q) {
      const std::string& nm = rec.inputs[q];
      uint64_t h = fnv1a(nm.data(), nm.size());
      if (rec.ndim == 3) {
        Grid3D g;
        g.origin = in[q].p;
        g.n = n;
        g.pitch_j = n;
        g.pitch_i = n * n;
        ck(fill_init_value_3d(g, h, stream), "fill_init_value_3d");
      } else {
        ck(fill_init_value(in[q].p, in_ld, n, n, h, 0, stream), "fill_init_value");
      }
    }
    ck(cudaStreamSynchronize(stream), "init inputs");
    mirror.clear();
  }

  void setup() {
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "cudaStreamCreate");
    own_stream = true;
    ck(cudaEventCreate(&ev0), "cudaEventCreate");
    ck(cudaEventCreate(&ev1), "cudaEventCreate");
    n = rec.N;
    T = rec.T;
    if (generic) {
      gplan = generic_plan_create(spec, params, maps, device);
      rec = Recognized();
      rec.family = Family::Generic;
      rec.ndim = 0;
      for (const auto& a : spec.arrays) {
        if (a.kind == ArrayKind::Input) rec.inputs.push_back(a.name);
        if (a.kind == ArrayKind::Output && rec.output.empty()) rec.output = a.name;
        if (a.kind == ArrayKind::Temp && rec.temp.empty()) rec.temp = a.name;
      }
      init_inputs();
      return;
    }
    switch (rec.family) {
      case Family::Stencil2D5: {
        in_ld = n;
        in[0].alloc(size_t(n * n));
        const int64_t ld = round_up(kPadL + n + kPadR2, 16);
        for (int b = 0; b < 2; ++b) {
          slab[b].alloc(size_t((n + 2 * kGhost) * ld));
          ck(cudaMemsetAsync(slab[b].p, 0, slab[b].n * sizeof(double), stream), "cudaMemset");
          sg[b].origin = slab[b].p + kGhost * ld + kPadL;
          sg[b].ld = ld;
          sg[b].rows = n;
          sg[b].cols = n;
          sg[b].ghost = kGhost;
          sg[b].padl = kPadL;
        }
        break;
      }
      case Family::Stencil3D7: {
        in[0].alloc(size_t(n * n * n));
        const int64_t pj = round_up(kGhost + n + kPadR3, 16);
        const int64_t pi = pj * (n + 2 * kGhost);
        for (int b = 0; b < 2; ++b) {
          cube[b].alloc(size_t(pi * (n + 2 * kGhost)));
          ck(cudaMemsetAsync(cube[b].p, 0, cube[b].n * sizeof(double), stream), "cudaMemset");
          cg[b].origin = cube[b].p + kGhost * pi + kGhost * pj + kGhost;
          cg[b].n = n;
          cg[b].pitch_j = pj;
          cg[b].pitch_i = pi;
          cg[b].halo = kGhost;
        }
        break;
      }
      case Family::GaussSeidel2D9: {
        in_ld = n;
        in[0].alloc(size_t(n * n));
        gs_ld = round_up(n, 2);
        gsa.alloc(size_t(n * gs_ld));
        break;
      }
      case Family::Gemm: {
        g_ld = round_up(n, 2);
        in_ld = g_ld;
        for (int q = 0; q < 2; ++q) {
          in[q].alloc(size_t(n * g_ld));
          // on the executor's stream: a legacy-stream cudaMemset is not ordered
          // with the non-blocking stream's init kernels and raced them
          ck(cudaMemsetAsync(in[q].p, 0, in[q].n * sizeof(double), stream), "cudaMemset");
        }
        gA.alloc(size_t(n * g_ld));
        gB.alloc(size_t(n * g_ld));
        gC.alloc(size_t(n * g_ld));
        break;
      }
    }
    init_inputs();
  }

  // ---------------------------------------------------------------- runs
  int pick_bt(const TileOrder& o, int dflt, int maxbt) const {
    int bt = dflt;
    if (o.scheme != Scheme::Untiled && !o.tile.leaf.empty()) bt = int(o.tile.leaf[0]);
    return std::max(1, std::min(bt, maxbt));
  }

  int run_stencil2d(const TileOrder& o) {
    // default depth: 6 for HBM-streaming grids (power-capped optimum, bench.py),
    // 8 for L2-resident ones (<= 2^24 cells: the fewest launches of short
    // chunks; 2048^2 T=256: bt=8 907, bt=6 790, bt=4 648-800 GUpd/s)
    const int bt = pick_bt(o, env_int("PCOTGPU_BT2D", n * n <= (int64_t(1) << 24) ? 8 : 6),
                           s2d5_max_bt());
    const int order = o.scheme == Scheme::Cot ? kOrderMorton : kOrderLex;
    ck(copy_rows(sg[0].origin, sg[0].ld, in[0].p, in_ld, n, n, stream), "copy_rows");
    if (!rec.ring_hold) ck(zero_ring_2d(sg[0].origin, sg[0].ld, n, stream), "zero_ring");
    // Opt-in experiment (PCOTGPU_RESIDENT=1, untiled schedule, grids up to 2048^2):
    // one persistent launch keeps every row band in shared memory for all T
    // steps (stencil2d_res.cu).  Bit-exact, but measured slower than the
    // streaming kernel on the B200 (2048^2 T=256: 2.2 ms vs 1.19 ms): the
    // band-to-band row exchange moves 19 MB through L2 per step
    // (profiles/cfg0_resident_r02.md), so the default stays the streaming path.
    if (o.scheme == Scheme::Untiled && T >= 4 && env_int("PCOTGPU_RESIDENT", 0) != 0) {
      if (!res_tried) {
        res_tried = true;
        res_plan = s2d5_res_create(n, device);
      }
      if (res_plan) {
        ck(s2d5_res_run(res_plan, sg[0], sg[1], T, stream), "s2d5_res_run");
        result_slot = 1;
        return 0;  // no depth blocks: the whole run is one launch
      }
    }
    if (o.scheme == Scheme::Cot && o.space_time && T > 0) {
      // Space-time recursive order (reference cot_order over the band box with
      // time, tiler.cpp:150-203, 98-117): cells (d, r) = (depth block, row band).
      // Cell (d, r) reads rows of bands r-1..r+1 at time d*bt from slab d&1 and
      // writes band r at time (d+1)*bt into slab (d+1)&1; in the skewed
      // coordinates (d, s = r + 2d) every flow and ping-pong anti-dependence
      // is a componentwise non-negative vector ((1,1), (1,2), (1,3), (2,4)), so
      // the Morton order of the skewed box (time bit most significant, empty
      // cells skipped) is a legal schedule with two slabs.
      const int64_t hb = std::max<int64_t>(2 * bt, std::min<int64_t>(
          n, o.tile.leaf.size() > 1 && o.tile.leaf[1] > 0 ? o.tile.leaf[1] : 256));
      const int64_t nband = (n + hb - 1) / hb, nblk = (T + bt - 1) / bt;
      const int64_t ns = nband + 2 * (nblk - 1);
      int bits = 0;
      while ((int64_t(1) << bits) < std::max(nblk, ns)) ++bits;
      std::vector<std::pair<uint64_t, std::pair<int64_t, int64_t>>> cells;
      for (int64_t d = 0; d < nblk; ++d)
        for (int64_t r = 0; r < nband; ++r) {
          const uint64_t sv = uint64_t(r + 2 * d), dv = uint64_t(d);
          uint64_t key = 0;
          for (int q = bits - 1; q >= 0; --q) key = (key << 2) | (((dv >> q) & 1) << 1) | ((sv >> q) & 1);
          cells.push_back({key, {d, r}});
        }
      std::sort(cells.begin(), cells.end());
      for (const auto& c : cells) {
        const int64_t d = c.second.first, r = c.second.second;
        const int step = int(std::min<int64_t>(bt, T - d * bt));
        const int lo = int(r * hb), hi = int(std::min<int64_t>(n, (r + 1) * hb));
        ck(s2d5_advance(sg[d & 1], sg[(d + 1) & 1], 0, n, step, rec.ring_hold, kOrderLex, lo, hi, stream),
           "s2d5_advance");
      }
      result_slot = int(nblk & 1);
      return bt;
    }
    int cur = 0;
    for (int64_t t = 0; t < T; t += bt) {
      const int step = int(std::min<int64_t>(bt, T - t));
      ck(s2d5_advance(sg[cur], sg[cur ^ 1], 0, n, step, rec.ring_hold, order, 0, int(n), stream),
         "s2d5_advance");
      cur ^= 1;
    }
    result_slot = cur;
    return bt;
  }

  int run_stencil3d(const TileOrder& o) {
    const int bt = pick_bt(o, env_int("PCOTGPU_BT3D", 2), s3d7_max_bt());
    const int order = o.scheme == Scheme::Cot ? kOrderMorton : kOrderLex;
    // dense F -> padded cube: one pitched copy (n*n rows of n doubles)
    ck(copy_rows(cg[0].origin, cg[0].pitch_j, in[0].p, n, n * n, n, stream, cg[0].pitch_i, n),
       "copy_rows");
    if (!rec.ring_hold) ck(zero_ring_3d(cg[0], stream), "zero_ring_3d");
    int cur = 0;
    for (int64_t t = 0; t < T; t += bt) {
      const int step = int(std::min<int64_t>(bt, T - t));
      ck(s3d7_advance(cg[cur], cg[cur ^ 1], step, rec.rule, rec.ring_hold, order, stream),
         "s3d7_advance");
      cur ^= 1;
    }
    result_slot = cur;
    return bt;
  }

  // A Gauss-Seidel dependence wait that timed out leaves an invalid grid:
  // report it as a CUDA-level failure (PCOTGPU_E_CUDA), never a silent result.
  void check_gs_fault() {
    if (rec.family == Family::GaussSeidel2D9 && gs_plan && gs2d_plan_fault(gs_plan))
      ck(cudaErrorLaunchTimeout, "Gauss-Seidel: a dependence wait hit its spin cap "
                                 "(CTAs not co-resident?); the grid is invalid");
    if (rec.family == Family::Stencil2D5 && res_plan && s2d5_res_fault(res_plan))
      ck(cudaErrorLaunchTimeout, "resident stencil: a neighbour-band wait hit its spin cap "
                                 "(CTAs not co-resident?); the grid is invalid");
  }

  int run_gs(const TileOrder& o) {
    // default tile = best measured (profiles/kbench_r01.md)
    int bt = env_int("PCOTGPU_GS_BT", 2), bx = env_int("PCOTGPU_GS_BX", 64),
        by = env_int("PCOTGPU_GS_BY", 64);
    const bool tiled = o.scheme != Scheme::Untiled && o.tile.leaf.size() >= 3;
    if (tiled) {
      bt = int(o.tile.leaf[0]);
      bx = int(o.tile.leaf[1]);
      by = int(o.tile.leaf[2]);
    }
    // the fit check queries the device (occupancy, free memory): once per
    // executor, outside the timed region of later runs
    if (gs_pipe_ok < 0) gs_pipe_ok = gs2d_pipe_fits(n, T, device) ? 1 : 0;
    if (!tiled && env_int("PCOTGPU_GS_PIPE", 1) && gs_pipe_ok) {
      bt = bx = by = 0;  // systolic pipeline (one CTA per 32-row band)
    } else {
      bt = std::max(1, std::min(bt, 32));
      bx = std::max(1, std::min(bx, 1024 / bt));
      by = std::max(2, std::min(by, 2048));
      while (size_t(bx + bt + 1) * size_t(by + 2 * bt + 2) * 8 > 200 * 1024 && by > 16) by /= 2;
    }
    if (!gs_plan || gs_cfg[0] != bt || gs_cfg[1] != bx || gs_cfg[2] != by) {
      if (gs_plan) gs2d_plan_destroy(gs_plan);
      gs_plan = gs2d_plan_create(n, T, bt, bx, by, device);
      gs_cfg[0] = bt, gs_cfg[1] = bx, gs_cfg[2] = by;
    }
    ck(copy_rows_nosentinel(gsa.p, gs_ld, in[0].p, in_ld, n, n, stream), "copy_rows");
    ck(zero_ring_2d(gsa.p, gs_ld, n, stream), "zero_ring");
    ck(gs2d_run(gs_plan, gsa.p, gs_ld, stream), "gs2d_run");
    result_slot = 0;
    return bt;
  }

  int run_gemm(const TileOrder& o) {
    // untiled default: the recursive (Morton) CTA order — same time, up to 44%
    // less DRAM traffic once A and B exceed the L2 (profiles/sweep_slt_cot_r01.md)
    const int order = o.scheme == Scheme::Slt ? kOrderLex : kOrderMorton;
    ck(affine_2x_minus_1(in[0].p, gA.p, n * g_ld, stream), "affine A");
    ck(affine_2x_minus_1(in[1].p, gB.p, n * g_ld, stream), "affine B");
    ck(dgemm_nn(gA.p, gB.p, gC.p, n, g_ld, order, stream), "dgemm");
    result_slot = 0;
    return 0;
  }

  ExecResult run(const TileOrder& o, const ExecOptions& opts) {
    if (opts.sink) fail(ErrorKind::Unsupported, "GpuExecutor: trace sinks are not supported on the device");
    ck(cudaSetDevice(device), "cudaSetDevice");
    ExecResult r;
    const uint64_t l0 = launches();
    ck(cudaEventRecord(ev0, stream), "cudaEventRecord");
    switch (rec.family) {
      case Family::Stencil2D5: r.bt = run_stencil2d(o); break;
      case Family::Stencil3D7: r.bt = run_stencil3d(o); break;
      case Family::GaussSeidel2D9: r.bt = run_gs(o); break;
      case Family::Gemm: r.bt = run_gemm(o); break;
      case Family::Generic: run_generic(); r.bt = gcounts.mode; break;  // interpreter schedule
    }
    ck(cudaEventRecord(ev1, stream), "cudaEventRecord");
    ck(cudaEventSynchronize(ev1), "run");
    check_gs_fault();
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, ev0, ev1), "cudaEventElapsedTime");
    r.device_ms = ms;
    r.launches = launches() - l0;
    r.points = generic ? gcounts.points : rec.points;
    r.reads = generic ? gcounts.reads : rec.reads;
    r.writes = generic ? gcounts.writes : rec.writes;
    mirror.clear();
    if (!opts.skip_checksum) {
      if (generic) {  // every Output array in declaration order (exec.cpp:492-495)
        uint64_t h = 0xcbf29ce484222325ULL;
        for (const auto& a : spec.arrays)
          if (a.kind == ArrayKind::Output) {
            const std::vector<double>& out = array_data(a.name);
            h = fnv1a(out.data(), out.size() * sizeof(double), h);
          }
        r.checksum = h;
      } else {
        const std::vector<double>& out = array_data(rec.output);
        r.checksum = fnv1a(out.data(), out.size() * sizeof(double));
      }
    }
    return r;
  }

  void run_generic() {
    std::string msg;
    cudaError_t e = generic_run(gplan, stream, &gcounts, &msg);
    if (e == cudaErrorInvalidValue && !msg.empty()) fail(ErrorKind::Validation, msg);
    ck(e, "generic run");
    result_slot = 0;
  }

  // ---------------------------------------------------------------- host <-> device
  // output device view: pointer + pitch (2-D), or copy-out for 3-D
  void read_generic(int i, double* host) const {
    const uint64_t w = generic_array_words(gplan, size_t(i));
    if (w)
      ck(cudaMemcpyAsync(host, generic_array_ptr(gplan, size_t(i)), w * 8, cudaMemcpyDeviceToHost, stream),
         "D2H");
    ck(cudaStreamSynchronize(stream), "D2H");
  }

  void read_output(double* host) const {
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (generic) return read_generic(garray(rec.output), host);
    if (result_slot < 0) {  // never run: reference outputs start at 0.0
      std::memset(host, 0, words_of(rec.output) * sizeof(double));
      return;
    }
    switch (rec.family) {
      case Family::Stencil2D5: {
        const Slab2D& s = sg[result_slot];
        ck(cudaMemcpy2DAsync(host, n * 8, s.origin, s.ld * 8, n * 8, n, cudaMemcpyDeviceToHost, stream),
           "D2H");
        break;
      }
      case Family::Stencil3D7: {
        const Grid3D& g = cg[result_slot];
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr(g.origin, size_t(g.pitch_j) * 8, size_t(n) * 8,
                                       size_t(g.pitch_i / g.pitch_j));
        p.dstPtr = make_cudaPitchedPtr(host, size_t(n) * 8, size_t(n) * 8, size_t(n));
        p.extent = make_cudaExtent(size_t(n) * 8, size_t(n), size_t(n));
        p.kind = cudaMemcpyDeviceToHost;
        ck(cudaMemcpy3DAsync(&p, stream), "D2H");
        break;
      }
      case Family::GaussSeidel2D9:
        ck(cudaMemcpy2DAsync(host, n * 8, gsa.p, gs_ld * 8, n * 8, n, cudaMemcpyDeviceToHost, stream),
           "D2H");
        break;
      case Family::Gemm:
        ck(cudaMemcpy2DAsync(host, n * 8, gC.p, g_ld * 8, n * 8, n, cudaMemcpyDeviceToHost, stream),
           "D2H");
        break;
    }
    ck(cudaStreamSynchronize(stream), "D2H");
  }

  // ---------------------------------------------------------------- batched host runs
  // Dense host input q -> device input buffer `dst` (same layout as in[q]).
  void h2d_input(int q, double* dst, const double* host, cudaStream_t s) const {
    const uint64_t w = words_of(rec.inputs[q]);
    if (rec.ndim == 3 || in_ld == n)
      ck(cudaMemcpyAsync(dst, host, w * 8, cudaMemcpyHostToDevice, s), "H2D");
    else
      ck(cudaMemcpy2DAsync(dst, in_ld * 8, host, n * 8, n * 8, n, cudaMemcpyHostToDevice, s), "H2D");
  }

  // The output of the last run -> dense device buffer (D2D, on `stream`).
  void output_to_dense(double* dst) const {
    switch (rec.family) {
      case Family::Stencil2D5: {
        const Slab2D& sl = sg[result_slot];
        ck(cudaMemcpy2DAsync(dst, n * 8, sl.origin, sl.ld * 8, n * 8, n, cudaMemcpyDeviceToDevice, stream),
           "D2D");
        break;
      }
      case Family::Stencil3D7: {
        const Grid3D& g = cg[result_slot];
        cudaMemcpy3DParms p = {};
        p.srcPtr = make_cudaPitchedPtr(g.origin, size_t(g.pitch_j) * 8, size_t(n) * 8,
                                       size_t(g.pitch_i / g.pitch_j));
        p.dstPtr = make_cudaPitchedPtr(dst, size_t(n) * 8, size_t(n) * 8, size_t(n));
        p.extent = make_cudaExtent(size_t(n) * 8, size_t(n), size_t(n));
        p.kind = cudaMemcpyDeviceToDevice;
        ck(cudaMemcpy3DAsync(&p, stream), "D2D");
        break;
      }
      case Family::GaussSeidel2D9:
        ck(cudaMemcpy2DAsync(dst, n * 8, gsa.p, gs_ld * 8, n * 8, n, cudaMemcpyDeviceToDevice, stream),
           "D2D");
        break;
      case Family::Gemm:
        ck(cudaMemcpy2DAsync(dst, n * 8, gC.p, g_ld * 8, n * 8, n, cudaMemcpyDeviceToDevice, stream),
           "D2D");
        break;
    }
  }

  int run_family(const TileOrder& o) {
    switch (rec.family) {
      case Family::Stencil2D5: return run_stencil2d(o);
      case Family::Stencil3D7: return run_stencil3d(o);
      case Family::GaussSeidel2D9: return run_gs(o);
      case Family::Gemm: return run_gemm(o);
    }
    return 0;
  }

  // `count` independent runs from host memory.  Instance k's inputs are copied
  // in on the h2d stream while instance k-1 computes, and its output leaves on
  // the d2h stream (through a dense device staging buffer) while instance k+1
  // computes, so the copies overlap the compute in both directions.
  ExecResult run_batch(const TileOrder& o, size_t count, const double* const* hin,
                       double* const* hout, const ExecOptions& opts) {
    if (opts.sink) fail(ErrorKind::Unsupported, "GpuExecutor: trace sinks are not supported on the device");
    if (count == 0) fail(ErrorKind::Validation, "run_batch: count must be positive");
    const size_t ni = rec.inputs.size();
    for (size_t k = 0; k < count; ++k) {
      if (!hout || !hout[k]) fail(ErrorKind::Validation, "run_batch: null output pointer");
      for (size_t q = 0; q < ni; ++q)
        if (!hin || !hin[k * ni + q]) fail(ErrorKind::Validation, "run_batch: null input pointer");
    }
    if (generic) {  // interpreter path: instances one after the other
      ExecResult r;
      double ms = 0;
      uint64_t l0 = launches();
      for (size_t k = 0; k < count; ++k) {
        for (size_t q = 0; q < ni; ++q) write_input(int(q), hin[k * ni + q]);
        ExecOptions o2 = opts;
        o2.skip_checksum = true;
        r = run(o, o2);
        ms += r.device_ms;
        read_output(hout[k]);
      }
      r.device_ms = ms;
      r.launches = launches() - l0;
      if (!opts.skip_checksum) r.checksum = fnv1a(hout[count - 1], words_of(rec.output) * sizeof(double));
      return r;
    }
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (!h2d) {
      ck(cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking), "cudaStreamCreate");
      ck(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking), "cudaStreamCreate");
      for (cudaEvent_t* e : {&e_start, &e_in, &e_prev, &e_out, &e_free})
        ck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
    }
    if (count > 1)
      for (size_t q = 0; q < ni; ++q)
        if (!stage_in[q].p) stage_in[q].alloc(in[q].n);
    if (!stage_out.p) stage_out.alloc(words_of(rec.output));
    ExecResult r;
    const uint64_t l0 = launches();
    const uint64_t ow = words_of(rec.output);
    ck(cudaEventRecord(ev0, stream), "cudaEventRecord");
    ck(cudaEventRecord(e_start, stream), "cudaEventRecord");
    ck(cudaStreamWaitEvent(h2d, e_start, 0), "wait");
    ck(cudaStreamWaitEvent(d2h, e_start, 0), "wait");
    for (size_t q = 0; q < ni; ++q) h2d_input(int(q), in[q].p, hin[q], h2d);
    ck(cudaEventRecord(e_in, h2d), "cudaEventRecord");
    for (size_t k = 0; k < count; ++k) {
      ck(cudaStreamWaitEvent(stream, e_in, 0), "wait");  // instance k's inputs landed
      if (k > 0)
        for (size_t q = 0; q < ni; ++q) std::swap(in[q].p, stage_in[q].p);
      ck(cudaEventRecord(e_prev, stream), "cudaEventRecord");  // instance k-1 done with its inputs
      if (k + 1 < count) {
        ck(cudaStreamWaitEvent(h2d, e_prev, 0), "wait");
        for (size_t q = 0; q < ni; ++q)
          h2d_input(int(q), stage_in[q].p, hin[(k + 1) * ni + q], h2d);
        ck(cudaEventRecord(e_in, h2d), "cudaEventRecord");
      }
      r.bt = run_family(o);
      ck(cudaStreamWaitEvent(stream, e_free, 0), "wait");  // staging free (previous D2H done)
      output_to_dense(stage_out.p);
      ck(cudaEventRecord(e_out, stream), "cudaEventRecord");
      ck(cudaStreamWaitEvent(d2h, e_out, 0), "wait");
      ck(cudaMemcpyAsync(hout[k], stage_out.p, ow * 8, cudaMemcpyDeviceToHost, d2h), "D2H");
      ck(cudaEventRecord(e_free, d2h), "cudaEventRecord");
    }
    ck(cudaStreamWaitEvent(stream, e_free, 0), "wait");
    ck(cudaEventRecord(ev1, stream), "cudaEventRecord");
    ck(cudaEventSynchronize(ev1), "run_batch");
    check_gs_fault();
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, ev0, ev1), "cudaEventElapsedTime");
    r.device_ms = ms;
    r.launches = launches() - l0;
    r.points = rec.points;
    r.reads = rec.reads;
    r.writes = rec.writes;
    mirror.clear();
    if (!opts.skip_checksum) r.checksum = fnv1a(hout[count - 1], ow * sizeof(double));
    return r;
  }

  int input_slot(const std::string& a) const {
    for (size_t q = 0; q < rec.inputs.size(); ++q)
      if (rec.inputs[q] == a) return int(q);
    return -1;
  }

  void read_input(int q, double* host) const {
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (generic) return read_generic(garray(rec.inputs[size_t(q)]), host);
    const uint64_t w = words_of(rec.inputs[q]);
    if (rec.ndim == 3)
      ck(cudaMemcpyAsync(host, in[q].p, w * 8, cudaMemcpyDeviceToHost, stream), "D2H");
    else
      ck(cudaMemcpy2DAsync(host, n * 8, in[q].p, in_ld * 8, n * 8, n, cudaMemcpyDeviceToHost, stream),
         "D2H");
    ck(cudaStreamSynchronize(stream), "D2H");
  }

  void write_input(int q, const double* host) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    if (generic) {
      const int i = garray(rec.inputs[size_t(q)]);
      const uint64_t w = generic_array_words(gplan, size_t(i));
      if (w)
        ck(cudaMemcpyAsync(generic_array_ptr(gplan, size_t(i)), host, w * 8, cudaMemcpyHostToDevice, stream),
           "H2D");
      ck(cudaStreamSynchronize(stream), "H2D");
      mirror.clear();
      return;
    }
    const uint64_t w = words_of(rec.inputs[q]);
    if (rec.ndim == 3)
      ck(cudaMemcpyAsync(in[q].p, host, w * 8, cudaMemcpyHostToDevice, stream), "H2D");
    else
      ck(cudaMemcpy2DAsync(in[q].p, in_ld * 8, host, n * 8, n * 8, n, cudaMemcpyHostToDevice, stream),
         "H2D");
    ck(cudaStreamSynchronize(stream), "H2D");
    mirror.clear();
  }

  const std::vector<double>& array_data(const std::string& a) const {
    const ArrayDecl* d = spec.find_array(a);
    if (!d) fail(ErrorKind::Validation, "array_data: unknown array " + a);
    auto it = mirror.find(a);
    if (it != mirror.end()) return it->second;
    std::vector<double> v(words_of(a));
    if (generic) read_generic(garray(a), v.data());  // dense storage: temps too
    else if (d->kind == ArrayKind::Output) read_output(v.data());
    else if (d->kind == ArrayKind::Input) read_input(input_slot(a), v.data());
    else fail(ErrorKind::Unsupported, "array_data: temp array " + a + " lives in the device layout");
    return mirror.emplace(a, std::move(v)).first->second;
  }
};

GpuExecutor::GpuExecutor(const KernelSpec& embedded, const IntVec& params,
                         const std::vector<MemoryMap>& maps, int device)
    : impl_(new Impl) {
  impl_->spec = embedded;
  impl_->params = params;
  impl_->device = device;
  if (!maps.empty()) check_maps(embedded, maps);  // reference map_of / build_ref checks
  impl_->maps = maps;
  // Hot-path kernels go to their hand-written kernels; anything else the
  // reference can run goes to the device interpreter (generic.h).
  try {
    impl_->rec = recognize(embedded, params);
  } catch (const Error& e) {
    const bool shallow = e.kind() == ErrorKind::Validation &&
                         std::string(e.what()).find("embedded") != std::string::npos;
    if (e.kind() != ErrorKind::Unsupported && !shallow) throw;
    impl_->generic = true;
  }
  if (env_int("PCOTGPU_FORCE_GENERIC", 0)) impl_->generic = true;
  // Caller maps: the hand-written kernels only where their layout reproduces
  // the reference's storage semantics; otherwise the interpreter, which lays
  // storage out by the maps themselves.
  if (!impl_->generic && !maps.empty()) {
    std::string why;
    if (!hot_path_honours(impl_->rec, embedded, params, maps, &why)) impl_->generic = true;
  }
  impl_->setup();
}

GpuExecutor::~GpuExecutor() = default;

ExecResult GpuExecutor::run(const TileOrder& order, const ExecOptions& opts) {
  return impl_->run(order, opts);
}
ExecResult GpuExecutor::run_untiled(const ExecOptions& opts) { return impl_->run(TileOrder{}, opts); }
ExecResult GpuExecutor::run_batch(const TileOrder& order, size_t count, const double* const* host_inputs,
                                  double* const* host_outputs, const ExecOptions& opts) {
  return impl_->run_batch(order, count, host_inputs, host_outputs, opts);
}
void GpuExecutor::reset() {
  impl_->init_inputs();
  impl_->result_slot = -1;
}
const std::vector<double>& GpuExecutor::array_data(const std::string& a) const {
  return impl_->array_data(a);
}
uint64_t GpuExecutor::array_words(const std::string& a) const { return impl_->words_of(a); }
uint64_t GpuExecutor::array_base(const std::string& a) const {
  // reference exec.cpp:234-245: arrays laid out from byte 64, 64-B aligned
  uint64_t base = 64;
  for (const auto& d : impl_->spec.arrays) {
    if (d.name == a) return base;
    uint64_t w = impl_->words_of(d.name);
    for (const auto& m : impl_->maps)  // storage words of the caller's maps
      if (m.array == d.name) w = uint64_t(m.words());
    base += (w * 8 + 63) / 64 * 64;
  }
  fail(ErrorKind::Validation, "array_base: unknown array " + a);
}
const Recognized& GpuExecutor::recognized() const { return impl_->rec; }
void GpuExecutor::generic_info(int* mode, int* compiled, std::string* why) const {
  if (!impl_->generic) fail(ErrorKind::Unsupported, "generic_info: this kernel runs on a hand-written kernel");
  if (mode) *mode = impl_->gcounts.mode;
  if (compiled) *compiled = impl_->gcounts.compiled ? 1 : 0;
  if (why) *why = generic_jit_status(impl_->gplan);
}
void GpuExecutor::write_array(const std::string& a, const double* host, size_t n) {
  int q = impl_->input_slot(a);
  if (q < 0) fail(ErrorKind::Validation, "write_array: " + a + " is not an input");
  if (n != impl_->words_of(a)) fail(ErrorKind::DimMismatch, "write_array: word count");
  impl_->write_input(q, host);
}
void GpuExecutor::read_array(const std::string& a, double* host, size_t n) const {
  if (n != impl_->words_of(a)) fail(ErrorKind::DimMismatch, "read_array: word count");
  const ArrayDecl* d = impl_->spec.find_array(a);
  if (d && d->kind == ArrayKind::Output) return impl_->read_output(host);
  int q = impl_->input_slot(a);
  if (q < 0) fail(ErrorKind::Unsupported, "read_array: temp array " + a + " lives in the device layout");
  impl_->read_input(q, host);
}
double* GpuExecutor::device_view(const std::string& a, int64_t* ld) {
  Impl& m = *impl_;
  int q = m.input_slot(a);
  if (q >= 0) {
    if (ld) *ld = m.rec.ndim == 3 ? m.n : m.in_ld;
    return m.in[q].p;
  }
  if (m.generic) {
    const int i = m.garray(a);
    if (i < 0) fail(ErrorKind::Validation, "device_view: unknown array " + a);
    if (ld) *ld = int64_t(generic_array_words(m.gplan, size_t(i)));
    return generic_array_ptr(m.gplan, size_t(i));
  }
  if (a != m.rec.output || m.result_slot < 0) fail(ErrorKind::Validation, "device_view: no device data for " + a);
  switch (m.rec.family) {
    case Family::Stencil2D5: if (ld) *ld = m.sg[m.result_slot].ld; return m.sg[m.result_slot].origin;
    case Family::Stencil3D7: if (ld) *ld = m.cg[m.result_slot].pitch_j; return m.cg[m.result_slot].origin;
    case Family::GaussSeidel2D9: if (ld) *ld = m.gs_ld; return m.gsa.p;
    case Family::Gemm: if (ld) *ld = m.g_ld; return m.gC.p;
    case Family::Generic: break;
  }
  return nullptr;
}
void GpuExecutor::set_stream(void* s) {
  if (impl_->own_stream && impl_->stream) cudaStreamDestroy(impl_->stream);
  impl_->stream = static_cast<cudaStream_t>(s);
  impl_->own_stream = false;
}

}  // namespace pcotgpu

// ======================================================================== C ABI
using namespace pcotgpu;

struct pcotgpu_handle {
  std::unique_ptr<GpuExecutor> ex;
};

namespace {
thread_local std::string t_err;

int status_of(ErrorKind k) { return int(k) + 1; }

template <class F>
int guarded(F&& f) {
  try {
    f();
    t_err.clear();
    return PCOTGPU_OK;
  } catch (const Error& e) {
    t_err = e.what();
    return status_of(e.kind());
  } catch (const std::exception& e) {
    t_err = e.what();
    return PCOTGPU_E_VALIDATION;
  }
}

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return PCOTGPU_OK;
  t_err = cudaGetErrorString(e);
  return e == cudaErrorInvalidValue ? PCOTGPU_E_VALIDATION : PCOTGPU_E_CUDA;
}

void fill_info(const Recognized& r, const std::string& name, pcotgpu_kernel_info* out) {
  std::memset(out, 0, sizeof(*out));
  out->family = int32_t(r.family);
  out->rule = r.rule;
  out->ring_hold = r.ring_hold;
  out->ndim = r.ndim;
  out->T = r.T;
  out->N = r.N;
  out->points = r.points;
  out->reads = r.reads;
  out->writes = r.writes;
  std::strncpy(out->name, name.c_str(), sizeof(out->name) - 1);
}

TileOrder order_of(const pcotgpu_schedule* s) {
  TileOrder o;
  if (!s) return o;
  o.scheme = s->scheme == PCOTGPU_SLT ? Scheme::Slt : s->scheme == PCOTGPU_COT ? Scheme::Cot : Scheme::Untiled;
  for (int i = 0; i < s->ndim && i < 8; ++i) o.tile.leaf.push_back(s->leaf[i]);
  o.space_time = (s->flags & PCOTGPU_SPACE_TIME) != 0;
  return o;
}

void fill_result(const ExecResult& r, pcotgpu_result* out) {
  std::memset(out, 0, sizeof(*out));
  out->points = r.points;
  out->reads = r.reads;
  out->writes = r.writes;
  out->violation = r.violation ? 1 : 0;
  out->bt = r.bt;
  out->checksum = r.checksum;
  out->device_ms = r.device_ms;
  out->launches = r.launches;
}
}  // namespace

extern "C" {

int pcotgpu_abi_version(void) { return PCOTGPU_ABI_VERSION; }
const char* pcotgpu_last_error(void) { return t_err.c_str(); }
uint64_t pcotgpu_launch_count(void) { return launches(); }
uint64_t pcotgpu_fnv1a(const void* data, size_t n, uint64_t h) { return fnv1a(data, n, h); }

int pcotgpu_device_count(int* n) {
  int c = 0;
  cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) c = 0;
  if (n) *n = c;
  return cuda_status(e == cudaErrorNoDevice ? cudaSuccess : e);
}

int pcotgpu_recognize(const char* kernel_json, const int64_t* params, size_t nparams,
                      pcotgpu_kernel_info* out) {
  return guarded([&] {
    if (!kernel_json || !out) fail(ErrorKind::Validation, "null argument");
    KernelSpec k = parse_kernel(kernel_json);
    Recognized r = recognize(k, IntVec(params, params + nparams));
    fill_info(r, k.name, out);
  });
}

int pcotgpu_find_kernel_file(const char* name, char* out, size_t cap) {
  return guarded([&] {
    std::string p = find_kernel_file(name ? name : "");
    if (cap) {
      std::strncpy(out, p.c_str(), cap - 1);
      out[cap - 1] = 0;
    }
    if (p.size() >= cap) fail(ErrorKind::Io, "path buffer too small");
  });
}

int pcotgpu_create(const char* kernel_json, const int64_t* params, size_t nparams, int device,
                   pcotgpu_handle** out) {
  return guarded([&] {
    if (!kernel_json || !out) fail(ErrorKind::Validation, "null argument");
    *out = nullptr;
    KernelSpec k = parse_kernel(kernel_json);
    auto h = std::make_unique<pcotgpu_handle>();
    h->ex = std::make_unique<GpuExecutor>(k, IntVec(params, params + nparams),
                                          std::vector<MemoryMap>{}, device);
    *out = h.release();
  });
}

namespace {
std::vector<MemoryMap> maps_of(const pcotgpu_map* maps, size_t nmaps) {
    std::vector<MemoryMap> mm;
    for (size_t i = 0; i < nmaps; ++i) {
      const pcotgpu_map& c = maps[i];
      if (!c.array || c.rank < 0 || c.storage_rank < 0 ||
          (c.storage_rank && (!c.constant || !c.moduli || !c.extents || (c.rank && !c.linear))))
        fail(ErrorKind::Validation, "pcotgpu_create_mapped: malformed map " + std::to_string(i));
      MemoryMap m;
      m.array = c.array;
      for (int32_t q = 0; q < c.storage_rank; ++q) {
        m.linear.emplace_back(c.linear + size_t(q) * c.rank, c.linear + size_t(q + 1) * c.rank);
        m.constant.push_back(c.constant[q]);
        m.moduli.push_back(c.moduli[q]);
        m.extents.push_back(c.extents[q]);
      }
      m.single_assignment = c.single_assignment != 0;
      mm.push_back(std::move(m));
    }
    return mm;
}
}  // namespace

int pcotgpu_check_maps(const char* kernel_json, const int64_t* params, size_t nparams,
                       const pcotgpu_map* maps, size_t nmaps, int* hot_path, char* why, size_t cap) {
  return guarded([&] {
    if (!kernel_json || !hot_path || (nmaps && !maps)) fail(ErrorKind::Validation, "null argument");
    KernelSpec k = parse_kernel(kernel_json);
    const IntVec prm(params, params + nparams);
    const std::vector<MemoryMap> mm = maps_of(maps, nmaps);
    check_maps(k, mm);
    std::string w;
    bool hot = false;
    try {
      const Recognized R = recognize(k, prm);
      hot = hot_path_honours(R, k, prm, mm, &w);
    } catch (const Error& e) {
      if (e.kind() != ErrorKind::Unsupported) throw;
      w = e.what();
    }
    *hot_path = hot ? 1 : 0;
    if (why && cap) {
      std::strncpy(why, w.c_str(), cap - 1);
      why[cap - 1] = 0;
    }
  });
}

int pcotgpu_create_mapped(const char* kernel_json, const int64_t* params, size_t nparams,
                          const pcotgpu_map* maps, size_t nmaps, int device, pcotgpu_handle** out) {
  return guarded([&] {
    if (!kernel_json || !out || (nmaps && !maps)) fail(ErrorKind::Validation, "null argument");
    *out = nullptr;
    KernelSpec k = parse_kernel(kernel_json);
    std::vector<MemoryMap> mm = maps_of(maps, nmaps);
    auto h = std::make_unique<pcotgpu_handle>();
    h->ex = std::make_unique<GpuExecutor>(k, IntVec(params, params + nparams), mm, device);
    *out = h.release();
  });
}

int pcotgpu_run(pcotgpu_handle* h, const pcotgpu_schedule* sched, pcotgpu_result* res) {
  return guarded([&] {
    if (!h || !res) fail(ErrorKind::Validation, "null argument");
    ExecOptions o;
    o.skip_checksum = sched && (sched->flags & PCOTGPU_SKIP_CHECKSUM);
    fill_result(h->ex->run(order_of(sched), o), res);
  });
}

int pcotgpu_run_untiled(pcotgpu_handle* h, pcotgpu_result* res) { return pcotgpu_run(h, nullptr, res); }

int pcotgpu_run_batch(pcotgpu_handle* h, const pcotgpu_schedule* sched, size_t count,
                      const double* const* host_inputs, double* const* host_outputs,
                      pcotgpu_result* res) {
  return guarded([&] {
    if (!h || !res) fail(ErrorKind::Validation, "null argument");
    ExecOptions o;
    o.skip_checksum = sched && (sched->flags & PCOTGPU_SKIP_CHECKSUM);
    fill_result(h->ex->run_batch(order_of(sched), count, host_inputs, host_outputs, o), res);
  });
}

int pcotgpu_reset(pcotgpu_handle* h) {
  return guarded([&] { h->ex->reset(); });
}

int pcotgpu_read_array(pcotgpu_handle* h, const char* array, double* dst, size_t n) {
  return guarded([&] { h->ex->read_array(array, dst, n); });
}

int pcotgpu_write_array(pcotgpu_handle* h, const char* array, const double* src, size_t n) {
  return guarded([&] { h->ex->write_array(array, src, n); });
}

int pcotgpu_array_base(const pcotgpu_handle* h, const char* array, uint64_t* base) {
  return guarded([&] { *base = h->ex->array_base(array); });
}

int pcotgpu_array_words(const pcotgpu_handle* h, const char* array, uint64_t* words) {
  return guarded([&] { *words = h->ex->array_words(array); });
}

int pcotgpu_generic_source(const char* kernel_json, const int64_t* params, size_t nparams, int compile,
                           char* buf, size_t cap, size_t* need) {
  return guarded([&] {
    if (!kernel_json) fail(ErrorKind::Validation, "null argument");
    KernelSpec k = parse_kernel(kernel_json);
    std::unique_ptr<GenericPlan, void (*)(GenericPlan*)> plan(
        generic_plan_create(k, IntVec(params, params + nparams), {}, 0, true), generic_plan_destroy);
    std::string text = generic_emit_source(plan.get());
    if (compile) {
      std::string log;
      if (!generic_jit_compile_check(plan.get(), &log)) {
        text = log;
        if (buf && cap) {
          std::strncpy(buf, text.c_str(), cap - 1);
          buf[cap - 1] = 0;
        }
        if (need) *need = text.size() + 1;
        fail(ErrorKind::Unsupported, "NVRTC could not compile the emitted kernel");
      }
    }
    if (need) *need = text.size() + 1;
    if (buf && cap) {
      std::strncpy(buf, text.c_str(), cap - 1);
      buf[cap - 1] = 0;
    }
  });
}

int pcotgpu_generic_info(const pcotgpu_handle* h, int* mode, int* compiled, char* why, size_t cap) {
  return guarded([&] {
    if (!h) fail(ErrorKind::Validation, "null argument");
    std::string w;
    h->ex->generic_info(mode, compiled, &w);
    if (why && cap) {
      std::strncpy(why, w.c_str(), cap - 1);
      why[cap - 1] = 0;
    }
  });
}

int pcotgpu_info(const pcotgpu_handle* h, pcotgpu_kernel_info* out) {
  return guarded([&] { fill_info(h->ex->recognized(), "", out); });
}

int pcotgpu_device_view(pcotgpu_handle* h, const char* array, double** ptr, int64_t* ld) {
  return guarded([&] { *ptr = h->ex->device_view(array, ld); });
}

int pcotgpu_set_stream(pcotgpu_handle* h, void* stream) {
  return guarded([&] { h->ex->set_stream(stream); });
}

void pcotgpu_destroy(pcotgpu_handle* h) { delete h; }

int pcotgpu_s2d5_layout(int64_t rows, int64_t cols, int64_t* ld, int64_t* ghost, int64_t* padl,
                        int64_t* total) {
  const int64_t l = round_up(kPadL + cols + kPadR2, 16);
  if (ld) *ld = l;
  if (ghost) *ghost = kGhost;
  if (padl) *padl = kPadL;
  if (total) *total = (rows + 2 * kGhost) * l;
  return PCOTGPU_OK;
}

int pcotgpu_s2d5_advance(const double* in_origin, double* out_origin, int64_t rows, int64_t cols,
                         int64_t g0, int64_t nrows_global, int bt, int ring_hold, int order,
                         int64_t row_lo, int64_t row_hi, void* stream) {
  return pcotgpu_s2d5_advance_p2p(in_origin, out_origin, rows, cols, g0, nrows_global, bt,
                                  ring_hold, order, row_lo, row_hi, nullptr, nullptr, 0, stream);
}

int pcotgpu_s2d5_advance_p2p(const double* in_origin, double* out_origin, int64_t rows,
                             int64_t cols, int64_t g0, int64_t nrows_global, int bt, int ring_hold,
                             int order, int64_t row_lo, int64_t row_hi, double* mirror_up,
                             double* mirror_dn, int64_t mirror_rows, void* stream) {
  Slab2D a, b;
  int64_t ld = 0;
  pcotgpu_s2d5_layout(rows, cols, &ld, nullptr, nullptr, nullptr);
  a.origin = const_cast<double*>(in_origin);
  b.origin = out_origin;
  a.ld = b.ld = ld;
  a.rows = b.rows = rows;
  a.cols = b.cols = cols;
  a.ghost = b.ghost = kGhost;
  a.padl = b.padl = kPadL;
  if (mirror_rows < 0 || mirror_rows > std::min<int64_t>(rows, kGhost))
    return cuda_status(cudaErrorInvalidValue);
  return cuda_status(s2d5_advance_p2p(a, b, g0, nrows_global, bt, ring_hold, order, int(row_lo),
                                      int(row_hi), mirror_up, mirror_dn, int(mirror_rows),
                                      static_cast<cudaStream_t>(stream)));
}

int pcotgpu_test_div9(const double* x, double* q_fast, double* q_ref, int64_t n, void* stream) {
  return cuda_status(div9_check(x, q_fast, q_ref, n, static_cast<cudaStream_t>(stream)));
}

int pcotgpu_fill_init_value(double* dst, int64_t ld, int64_t nrows, int64_t ncols, const char* name,
                            uint64_t flat0, void* stream) {
  const uint64_t h = fnv1a(name, std::strlen(name));
  return cuda_status(fill_init_value(dst, ld, nrows, ncols, h, flat0, static_cast<cudaStream_t>(stream)));
}

int pcotgpu_s2d5_prepare(double* origin, int64_t rows, int64_t cols, int64_t g0,
                         int64_t nrows_global, int ring_hold, void* stream) {
  if (ring_hold) return PCOTGPU_OK;
  int64_t ld = 0;
  pcotgpu_s2d5_layout(rows, cols, &ld, nullptr, nullptr, nullptr);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  // columns 0 and N-1 of every local row, rows with global index 0 / N-1
  for (int64_t r = 0; r < rows && e == cudaSuccess; ++r) {
    const int64_t g = g0 + r;
    if (g == 0 || g == nrows_global - 1) {
      e = cudaMemsetAsync(origin + r * ld, 0, cols * 8, s);
    }
  }
  if (e == cudaSuccess) e = cudaMemset2DAsync(origin, ld * 8, 0, 8, rows, s);
  if (e == cudaSuccess) e = cudaMemset2DAsync(origin + cols - 1, ld * 8, 0, 8, rows, s);
  return cuda_status(e);
}

}  // extern "C"
