// Host-side kernel registration for the GPU executor: the reference's
// kernel-spec JSON (reference docs/formats.md:7-85), its body grammar
// (formats.md:55-68, expr.cpp:163-195) and a recognizer that maps a parsed
// kernel onto one of the sm_100a hot-path kernels.
#pragma once
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace pcotgpu {

// Same ordinals as pcot::ErrorKind (reference core/include/pcot/error.hpp:8-16);
// Cuda is this library's addition.
enum class ErrorKind { Overflow, DimMismatch, Unbounded, Parse, Validation, Io, Unsupported, Cuda };

class Error : public std::runtime_error {
 public:
  Error(ErrorKind k, const std::string& m) : std::runtime_error(m), kind_(k) {}
  ErrorKind kind() const { return kind_; }

 private:
  ErrorKind kind_;
};

[[noreturn]] inline void fail(ErrorKind k, const std::string& m) { throw Error(k, m); }

using IntVec = std::vector<int64_t>;

// Affine form over indices ++ params, plus constant (reference expr.hpp:13-28).
struct Affine {
  IntVec c;
  int64_t k = 0;
  bool operator==(const Affine& o) const { return c == o.c && k == o.k; }
};

struct Expr {
  enum class Kind { Lit, Aff, Read, Add, Sub, Mul, Div, Min, Max, Neg, Sqrt };
  Kind kind = Kind::Lit;
  double lit = 0.0;
  Affine aff;
  std::string array;
  std::vector<Affine> subs;
  std::shared_ptr<const Expr> l, r;
};
using ExprPtr = std::shared_ptr<const Expr>;

enum class ArrayKind { Input, Output, Temp };

struct ArrayDecl {
  std::string name;
  size_t rank = 0;
  std::vector<Affine> extents;  // over params only (index coefficients zero)
  ArrayKind kind = ArrayKind::Temp;
};

struct Statement {
  std::string id;
  size_t depth = 0;
  std::vector<IntVec> domain;  // rows over depth indices ++ params ++ [1], >= 0
  std::string write_array;
  std::vector<Affine> write_subs;
  ExprPtr body;
  std::string body_text;
};

// Mirror of the reference's Prdg as far as the executor needs it
// (reference core/include/pcot/prdg.hpp:60-106).
struct KernelSpec {
  std::string name;
  std::vector<std::string> params, indices;
  IntVec check_params;
  std::vector<ArrayDecl> arrays;
  std::vector<Statement> statements;
  std::vector<size_t> tilable_band;
  const ArrayDecl* find_array(const std::string& n) const {
    for (const auto& a : arrays)
      if (a.name == n) return &a;
    return nullptr;
  }
};

// reference kernel_io.hpp:11-22
KernelSpec parse_kernel(const std::string& text);
KernelSpec parse_kernel_file(const std::string& path);
std::string find_kernel_file(const std::string& name_or_path);
ExprPtr parse_expr(const std::string& text, const std::vector<std::string>& indices,
                   const std::vector<std::string>& params);

// Generic: any other embeddable kernel, run by the device interpreter
// (generic.h) instead of a hand-written hot-path kernel.
enum class Family { Stencil2D5 = 1, Stencil3D7 = 2, GaussSeidel2D9 = 3, Gemm = 4, Generic = 5 };

struct StmtBox {
  std::string id;
  std::string role;       // init | ring | update | final
  IntVec lo, hi;          // unskewed box (time first); empty if any lo > hi
  uint64_t points = 0;
  uint64_t reads_per_point = 0;
};

// Storage map of one array (reference memalloc.hpp:14-33):
//   storage_k = (linear[k] . cell + constant[k]) mod moduli[k]  (moduli 0: none),
// in [0, extents[k]); storage is row-major over `extents`.
struct MemoryMap {
  std::string array;
  std::vector<IntVec> linear;  // storage rank x array rank
  IntVec constant, moduli, extents;
  bool single_assignment = false;
  int64_t words() const {
    int64_t w = 1;
    for (int64_t e : extents) w *= e;
    return w;
  }
};

// What the recognizer established about a kernel at a parameter binding.
struct Recognized {
  Family family = Family::Stencil2D5;
  int rule = 0;       // 3-D: 0 = c + 0.125*(sum6 - 6c), 1 = 0.1*(c + sum6)
  int ring_hold = 0;  // 0: ring literal 0.0 (every t); 1: ring copied forward
  int ndim = 2;
  int64_t T = 0, N = 0;
  std::vector<std::string> inputs;
  std::string temp, output;
  std::vector<StmtBox> stmts;
  uint64_t points = 0, reads = 0, writes = 0;  // closed-form ExecResult counters
  // kernel index z of un-skewed point u (box coordinates): z = Ainv (u - b)
  std::vector<IntVec> Ainv;
  IntVec b;
};

Recognized recognize(const KernelSpec& k, const IntVec& params);

// The structural checks the reference makes when it builds storage from maps
// (exec.cpp:134-141 map_of, 142-185 build_ref): one map per array, arities.
void check_maps(const KernelSpec& k, const std::vector<MemoryMap>& maps);
// True if a recognized kernel's device layout reproduces the reference's
// results under `maps`: inputs/outputs stored as the identity at their
// declared extents, the temp either single-assignment or folded along a
// positive multiple of the kernel's occupancy vector (the allocate() maps,
// memalloc.cpp:542-595).  Storage extents that cannot hold the cells the run
// touches raise Validation, as the reference's out-of-extent check does
// (exec.cpp:318-323).  `why` says what did not match.
bool hot_path_honours(const Recognized& R, const KernelSpec& k, const IntVec& prm,
                      const std::vector<MemoryMap>& maps, std::string* why);
const char* family_name(Family f);

uint64_t fnv1a(const void* data, size_t n, uint64_t h = 0xcbf29ce484222325ULL);
double init_value(const std::string& array, uint64_t flat);  // reference exec.cpp:21-28

}  // namespace pcotgpu
