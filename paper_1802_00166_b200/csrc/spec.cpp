// Kernel-spec loading and recognition (host C++, no CUDA).
//
// parse_kernel follows the reference's normative format (docs/formats.md:7-85)
// and validation intent (kernel_io.cpp:54-114); parse_expr follows the body
// grammar (formats.md:55-68) with left-associative + - * / (expr.cpp:163-195)
// and literals read with strtod (expr.cpp:116-123).
//
// recognize() proves, at a parameter binding, that a kernel is one of the
// hot-path shapes the sm_100a kernels implement:
//   * the output statement fixes the time parameter and the un-skewing map
//     u = U(z) from loop indices to (t, grid cell);
//   * every temp-writing statement is classified by its body (init from the
//     input, ring literal 0.0, ring copy-forward, or the update), the update
//     body is canonicalised with reads expressed as un-skewed offsets and
//     compared with the registry;
//   * every domain is mapped to u-space and must be a box; the boxes must
//     tile exactly: init at t=0, update over [1,T] x interior, ring pieces
//     pairwise disjoint and covering the ring, final at t=T over the grid.
// Anything else is ErrorKind::Unsupported (the executor never guesses).
#include "spec.h"

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <map>
#include <sstream>
#include <sys/stat.h>

namespace pcotgpu {

// ====================================================================== util
uint64_t fnv1a(const void* data, size_t n, uint64_t h) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

double init_value(const std::string& array, uint64_t flat) {
  uint64_t x = fnv1a(array.data(), array.size()) ^ (flat * 0x9E3779B97F4A7C15ULL);
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  x ^= x >> 31;
  return double(x >> 11) * 0x1.0p-53;
}

const char* family_name(Family f) {
  switch (f) {
    case Family::Stencil2D5: return "stencil2d5";
    case Family::Stencil3D7: return "stencil3d7";
    case Family::GaussSeidel2D9: return "gs2d9";
    case Family::Gemm: return "gemm";
    case Family::Generic: return "generic";
  }
  return "?";
}

// ====================================================================== JSON
namespace {

struct JVal {
  enum class T { Null, Bool, Num, Str, Arr, Obj } t = T::Null;
  double num = 0;
  bool isint = false;
  int64_t inum = 0;
  bool b = false;
  std::string s;
  std::vector<JVal> arr;
  std::vector<std::pair<std::string, JVal>> obj;
  const JVal* get(const std::string& k) const {
    for (const auto& kv : obj)
      if (kv.first == k) return &kv.second;
    return nullptr;
  }
};

struct JParser {
  const std::string& s;
  size_t p = 0;
  explicit JParser(const std::string& t) : s(t) {}
  [[noreturn]] void err(const std::string& m) {
    fail(ErrorKind::Parse, "kernel JSON: " + m + " at offset " + std::to_string(p));
  }
  void ws() {
    while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
  }
  JVal value() {
    ws();
    if (p >= s.size()) err("unexpected end");
    char c = s[p];
    JVal v;
    if (c == '{') {
      v.t = JVal::T::Obj;
      ++p;
      ws();
      if (p < s.size() && s[p] == '}') return ++p, v;
      for (;;) {
        ws();
        if (p >= s.size() || s[p] != '"') err("expected key");
        std::string k = str();
        ws();
        if (p >= s.size() || s[p] != ':') err("expected ':'");
        ++p;
        v.obj.emplace_back(k, value());
        ws();
        if (p < s.size() && s[p] == ',') { ++p; continue; }
        if (p < s.size() && s[p] == '}') { ++p; break; }
        err("expected ',' or '}'");
      }
    } else if (c == '[') {
      v.t = JVal::T::Arr;
      ++p;
      ws();
      if (p < s.size() && s[p] == ']') return ++p, v;
      for (;;) {
        v.arr.push_back(value());
        ws();
        if (p < s.size() && s[p] == ',') { ++p; continue; }
        if (p < s.size() && s[p] == ']') { ++p; break; }
        err("expected ',' or ']'");
      }
    } else if (c == '"') {
      v.t = JVal::T::Str;
      v.s = str();
    } else if (s.compare(p, 4, "true") == 0) {
      v.t = JVal::T::Bool, v.b = true, p += 4;
    } else if (s.compare(p, 5, "false") == 0) {
      v.t = JVal::T::Bool, p += 5;
    } else if (s.compare(p, 4, "null") == 0) {
      p += 4;
    } else {
      size_t q = p;
      if (s[q] == '-') ++q;
      bool frac = false;
      while (q < s.size() && (std::isdigit(static_cast<unsigned char>(s[q])) || s[q] == '.' ||
                              s[q] == 'e' || s[q] == 'E' || s[q] == '+' || s[q] == '-')) {
        if (s[q] == '.' || s[q] == 'e' || s[q] == 'E') frac = true;
        ++q;
      }
      if (q == p) err("bad value");
      std::string t = s.substr(p, q - p);
      v.t = JVal::T::Num;
      v.num = std::strtod(t.c_str(), nullptr);
      v.isint = !frac;
      if (!frac) v.inum = std::strtoll(t.c_str(), nullptr, 10);
      p = q;
    }
    return v;
  }
  std::string str() {
    ++p;  // opening quote
    std::string out;
    while (p < s.size() && s[p] != '"') {
      if (s[p] == '\\') {
        ++p;
        if (p >= s.size()) err("bad escape");
        char e = s[p];
        out += e == 'n' ? '\n' : e == 't' ? '\t' : e;
      } else {
        out += s[p];
      }
      ++p;
    }
    if (p >= s.size()) err("unterminated string");
    ++p;
    return out;
  }
};

// ====================================================================== expressions
struct EParser {
  const std::string& s;
  const std::vector<std::string>& idx;
  const std::vector<std::string>& prm;
  size_t p = 0;
  EParser(const std::string& t, const std::vector<std::string>& i,
          const std::vector<std::string>& q)
      : s(t), idx(i), prm(q) {}
  [[noreturn]] void err(const std::string& m) {
    fail(ErrorKind::Parse, "body '" + s + "': " + m + " at position " + std::to_string(p));
  }
  void ws() {
    while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
  }
  bool eat(char c) {
    ws();
    if (p < s.size() && s[p] == c) return ++p, true;
    return false;
  }
  size_t width() const { return idx.size() + prm.size(); }
  static ExprPtr bin(Expr::Kind k, ExprPtr a, ExprPtr b) {
    auto e = std::make_shared<Expr>();
    e->kind = k;
    e->l = std::move(a);
    e->r = std::move(b);
    return e;
  }
  ExprPtr expr() {
    ExprPtr a = term();
    for (;;) {
      if (eat('+')) a = bin(Expr::Kind::Add, a, term());
      else if (eat('-')) a = bin(Expr::Kind::Sub, a, term());
      else return a;
    }
  }
  ExprPtr term() {
    ExprPtr a = factor();
    for (;;) {
      if (eat('*')) a = bin(Expr::Kind::Mul, a, factor());
      else if (eat('/')) a = bin(Expr::Kind::Div, a, factor());
      else return a;
    }
  }
  ExprPtr factor() {
    ws();
    if (p >= s.size()) err("unexpected end");
    char c = s[p];
    if (c == '(') {
      ++p;
      ExprPtr e = expr();
      if (!eat(')')) err("expected ')'");
      return e;
    }
    if (c == '-') {
      ++p;
      auto e = std::make_shared<Expr>();
      e->kind = Expr::Kind::Neg;
      e->l = factor();
      return e;
    }
    if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') {
      const char* b = s.c_str() + p;
      char* end = nullptr;
      double v = std::strtod(b, &end);
      if (end == b) err("bad number");
      p += size_t(end - b);
      auto e = std::make_shared<Expr>();
      e->kind = Expr::Kind::Lit;
      e->lit = v;
      return e;
    }
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      size_t q = p;
      while (q < s.size() && (std::isalnum(static_cast<unsigned char>(s[q])) || s[q] == '_')) ++q;
      std::string id = s.substr(p, q - p);
      p = q;
      if (id == "min" || id == "max") {
        if (!eat('(')) err("expected '('");
        ExprPtr a = expr();
        if (!eat(',')) err("expected ','");
        ExprPtr b = expr();
        if (!eat(')')) err("expected ')'");
        return bin(id == "min" ? Expr::Kind::Min : Expr::Kind::Max, a, b);
      }
      if (id == "sqrt") {
        if (!eat('(')) err("expected '('");
        auto e = std::make_shared<Expr>();
        e->kind = Expr::Kind::Sqrt;
        e->l = expr();
        if (!eat(')')) err("expected ')'");
        return e;
      }
      if (eat('[')) {
        auto e = std::make_shared<Expr>();
        e->kind = Expr::Kind::Read;
        e->array = id;
        do {
          e->subs.push_back(to_affine(expr()));
        } while (eat(','));
        if (!eat(']')) err("expected ']'");
        return e;
      }
      auto e = std::make_shared<Expr>();
      e->kind = Expr::Kind::Aff;
      e->aff.c.assign(width(), 0);
      for (size_t i = 0; i < idx.size(); ++i)
        if (idx[i] == id) return e->aff.c[i] = 1, e;
      for (size_t i = 0; i < prm.size(); ++i)
        if (prm[i] == id) return e->aff.c[idx.size() + i] = 1, e;
      err("unknown name '" + id + "'");
    }
    err(std::string("unexpected '") + c + "'");
  }
  // subscripts / extents must reduce to an affine form with integer coefficients
  Affine to_affine(const ExprPtr& e) {
    Affine a;
    a.c.assign(width(), 0);
    switch (e->kind) {
      case Expr::Kind::Aff: return e->aff;
      case Expr::Kind::Lit:
        if (e->lit != std::floor(e->lit)) err("non-integer literal in affine position");
        a.k = int64_t(e->lit);
        return a;
      case Expr::Kind::Neg: {
        Affine x = to_affine(e->l);
        for (auto& v : x.c) v = -v;
        x.k = -x.k;
        return x;
      }
      case Expr::Kind::Add:
      case Expr::Kind::Sub: {
        Affine x = to_affine(e->l), y = to_affine(e->r);
        int64_t sg = e->kind == Expr::Kind::Add ? 1 : -1;
        for (size_t i = 0; i < x.c.size(); ++i) x.c[i] += sg * y.c[i];
        x.k += sg * y.k;
        return x;
      }
      case Expr::Kind::Mul: {
        Affine x = to_affine(e->l), y = to_affine(e->r);
        bool xc = std::all_of(x.c.begin(), x.c.end(), [](int64_t v) { return v == 0; });
        bool yc = std::all_of(y.c.begin(), y.c.end(), [](int64_t v) { return v == 0; });
        if (!xc && !yc) err("non-affine product");
        if (xc) std::swap(x, y);
        for (auto& v : x.c) v *= y.k;
        x.k *= y.k;
        return x;
      }
      default: err("non-affine subscript");
    }
  }
};

IntVec int_array(const JVal* v, const std::string& what) {
  if (!v || v->t != JVal::T::Arr) fail(ErrorKind::Validation, "kernel: " + what + " must be an array");
  IntVec out;
  for (const auto& x : v->arr) {
    if (x.t != JVal::T::Num || !x.isint) fail(ErrorKind::Validation, "kernel: " + what + " must hold integers");
    out.push_back(x.inum);
  }
  return out;
}

std::vector<std::string> str_array(const JVal* v, const std::string& what) {
  if (!v || v->t != JVal::T::Arr) fail(ErrorKind::Validation, "kernel: " + what + " must be an array");
  std::vector<std::string> out;
  for (const auto& x : v->arr) {
    if (x.t != JVal::T::Str) fail(ErrorKind::Validation, "kernel: " + what + " must hold strings");
    out.push_back(x.s);
  }
  return out;
}

const JVal& need(const JVal& o, const char* key) {
  const JVal* v = o.get(key);
  if (!v) fail(ErrorKind::Validation, std::string("kernel: missing key '") + key + "'");
  return *v;
}

}  // namespace

ExprPtr parse_expr(const std::string& text, const std::vector<std::string>& indices,
                   const std::vector<std::string>& params) {
  EParser ep(text, indices, params);
  ExprPtr e = ep.expr();
  ep.ws();
  if (ep.p != text.size()) ep.err("trailing input");
  return e;
}

KernelSpec parse_kernel(const std::string& text) {
  JParser jp(text);
  JVal root = jp.value();
  jp.ws();
  if (jp.p != text.size()) jp.err("trailing input");
  if (root.t != JVal::T::Obj) fail(ErrorKind::Parse, "kernel JSON: top level must be an object");
  static const char* keys[] = {"name", "params", "indices", "check_params", "arrays",
                               "statements", "edges", "tilable_band"};
  for (const auto& kv : root.obj)
    if (std::find_if(std::begin(keys), std::end(keys),
                     [&](const char* k) { return kv.first == k; }) == std::end(keys))
      fail(ErrorKind::Validation, "kernel: unknown key '" + kv.first + "'");
  KernelSpec k;
  const JVal& name = need(root, "name");
  if (name.t != JVal::T::Str) fail(ErrorKind::Validation, "kernel: name must be a string");
  k.name = name.s;
  k.params = str_array(&need(root, "params"), "params");
  k.indices = str_array(&need(root, "indices"), "indices");
  const JVal& cp = need(root, "check_params");
  for (const auto& p : k.params) {
    const JVal* v = cp.get(p);
    if (!v || v->t != JVal::T::Num || !v->isint)
      fail(ErrorKind::Validation, "kernel: check_params lacks " + p);
    k.check_params.push_back(v->inum);
  }
  const JVal& arrays = need(root, "arrays");
  if (arrays.t != JVal::T::Arr) fail(ErrorKind::Validation, "kernel: arrays must be an array");
  static const std::vector<std::string> none;
  for (const auto& a : arrays.arr) {
    ArrayDecl d;
    d.name = need(a, "name").s;
    const JVal& rk = need(a, "rank");
    d.rank = size_t(rk.inum);
    for (const auto& ex : str_array(&need(a, "extents"), "extents")) {
      EParser ep(ex, none, k.params);
      Affine af = ep.to_affine(ep.expr());
      d.extents.push_back(af);
    }
    if (d.extents.size() != d.rank) fail(ErrorKind::Validation, "kernel: rank != extents for " + d.name);
    const std::string kind = need(a, "kind").s;
    if (kind == "input") d.kind = ArrayKind::Input;
    else if (kind == "output") d.kind = ArrayKind::Output;
    else if (kind == "temp") d.kind = ArrayKind::Temp;
    else fail(ErrorKind::Validation, "kernel: bad array kind " + kind);
    if (k.find_array(d.name)) fail(ErrorKind::Validation, "kernel: duplicate array " + d.name);
    k.arrays.push_back(std::move(d));
  }
  const JVal& stmts = need(root, "statements");
  if (stmts.t != JVal::T::Arr) fail(ErrorKind::Validation, "kernel: statements must be an array");
  for (const auto& sj : stmts.arr) {
    Statement st;
    st.id = need(sj, "id").s;
    st.depth = size_t(need(sj, "depth").inum);
    if (st.depth > k.indices.size()) fail(ErrorKind::Validation, "kernel: depth too large in " + st.id);
    std::vector<std::string> sidx(k.indices.begin(), k.indices.begin() + st.depth);
    const JVal& dom = need(sj, "domain");
    if (dom.t != JVal::T::Arr) fail(ErrorKind::Validation, "kernel: domain must be an array");
    for (const auto& row : dom.arr) {
      IntVec r = int_array(&row, "domain row");
      if (r.size() != st.depth + k.params.size() + 1)
        fail(ErrorKind::DimMismatch, "kernel: domain row width in " + st.id);
      st.domain.push_back(r);
    }
    const JVal& w = need(sj, "writes");
    st.write_array = need(w, "array").s;
    const ArrayDecl* wa = k.find_array(st.write_array);
    if (!wa) fail(ErrorKind::Validation, "kernel: " + st.id + " writes unknown array");
    if (wa->kind == ArrayKind::Input) fail(ErrorKind::Validation, "kernel: " + st.id + " writes an input");
    for (const auto& sub : str_array(&need(w, "subscripts"), "subscripts")) {
      EParser ep(sub, sidx, k.params);
      st.write_subs.push_back(ep.to_affine(ep.expr()));
    }
    if (st.write_subs.size() != wa->rank) fail(ErrorKind::DimMismatch, "kernel: write arity in " + st.id);
    st.body_text = need(sj, "body").s;
    st.body = parse_expr(st.body_text, sidx, k.params);
    k.statements.push_back(std::move(st));
  }
  // structural validation, reference kernel_io.cpp:54-76
  if (k.indices.empty()) fail(ErrorKind::Validation, "kernel has no indices");
  std::function<void(const ExprPtr&, const std::string&)> walk = [&](const ExprPtr& e,
                                                                     const std::string& where) {
    if (!e) return;
    if (e->kind == Expr::Kind::Read) {
      const ArrayDecl* a = k.find_array(e->array);
      if (!a) fail(ErrorKind::Validation, where + ": read of undeclared array " + e->array);
      if (e->subs.size() != a->rank) fail(ErrorKind::Validation, where + ": read arity mismatch");
    }
    walk(e->l, where);
    walk(e->r, where);
  };
  for (const auto& st : k.statements) {
    if (st.depth == 0) fail(ErrorKind::Validation, "statement " + st.id + ": bad depth");
    walk(st.body, "statement " + st.id);
  }
  for (auto v : int_array(&need(root, "tilable_band"), "tilable_band")) {
    if (v < 0 || size_t(v) >= k.indices.size()) fail(ErrorKind::Validation, "kernel: band index");
    k.tilable_band.push_back(size_t(v));
  }
  for (size_t i = 0; i < k.tilable_band.size(); ++i)
    if (k.tilable_band[i] != i) fail(ErrorKind::Validation, "kernel: band must be the leading indices");
  return k;
}

KernelSpec parse_kernel_file(const std::string& path) {
  std::ifstream f(path);
  if (!f) fail(ErrorKind::Io, "cannot open kernel file " + path);
  std::stringstream ss;
  ss << f.rdbuf();
  return parse_kernel(ss.str());
}

// reference kernel_io.cpp:250-276: path, then PCOT_KERNEL_PATH dirs, then ./kernels
std::string find_kernel_file(const std::string& name) {
  auto exists = [](const std::string& p) {
    struct stat sb;
    return stat(p.c_str(), &sb) == 0 && S_ISREG(sb.st_mode);
  };
  if (exists(name)) return name;
  std::vector<std::string> dirs;
  if (const char* env = std::getenv("PCOT_KERNEL_PATH")) {
    std::string s = env;
    size_t i = 0;
    while (i <= s.size()) {
      size_t j = s.find(':', i);
      if (j == std::string::npos) j = s.size();
      if (j > i) dirs.push_back(s.substr(i, j - i));
      i = j + 1;
    }
  }
  dirs.push_back("kernels");
  for (const auto& d : dirs) {
    if (exists(d + "/" + name)) return d + "/" + name;
    if (exists(d + "/" + name + ".kernel")) return d + "/" + name + ".kernel";
  }
  return "";
}

// ====================================================================== recognizer
namespace {

[[noreturn]] void unsupported(const std::string& m) { fail(ErrorKind::Unsupported, "GpuExecutor: " + m); }

int64_t eval_aff(const Affine& a, const IntVec& z, const IntVec& prm) {
  int64_t v = a.k;
  for (size_t i = 0; i < z.size(); ++i) v += a.c[i] * z[i];
  for (size_t j = 0; j < prm.size(); ++j) v += a.c[z.size() + j] * prm[j];
  return v;
}

// exact inverse of a small unimodular integer matrix (Gauss-Jordan on rationals
// that stay integral because det = +-1)
std::vector<IntVec> inverse_unimodular(std::vector<IntVec> m) {
  const size_t n = m.size();
  std::vector<std::vector<double>> a(n, std::vector<double>(2 * n, 0.0));
  for (size_t i = 0; i < n; ++i) {
    for (size_t j = 0; j < n; ++j) a[i][j] = double(m[i][j]);
    a[i][n + i] = 1.0;
  }
  for (size_t c = 0; c < n; ++c) {
    size_t piv = c;
    while (piv < n && a[piv][c] == 0.0) ++piv;
    if (piv == n) unsupported("singular un-skewing map");
    std::swap(a[piv], a[c]);
    double d = a[c][c];
    for (auto& v : a[c]) v /= d;
    for (size_t r = 0; r < n; ++r)
      if (r != c && a[r][c] != 0.0) {
        double f = a[r][c];
        for (size_t j = 0; j < 2 * n; ++j) a[r][j] -= f * a[c][j];
      }
  }
  std::vector<IntVec> inv(n, IntVec(n));
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < n; ++j) {
      double v = a[i][n + j];
      if (v != std::round(v)) unsupported("un-skewing map is not unimodular");
      inv[i][j] = int64_t(std::llround(v));
    }
  return inv;
}

std::string fmt_lit(double v) {
  char buf[40];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

struct Skew {
  size_t nidx = 0, nprm = 0;
  std::vector<IntVec> A;  // u = A z + b (rows: t, cell dims)
  IntVec b;
  std::vector<IntVec> Ainv;
};

// Canonical text of a body; reads of `temp` at z+delta become un-skewed offsets.
std::string canon(const ExprPtr& e, const Skew& sk, const std::string& temp, int& nreads) {
  using K = Expr::Kind;
  switch (e->kind) {
    case K::Lit: return fmt_lit(e->lit);
    case K::Aff: unsupported("affine scalar in an update body");
    case K::Read: {
      ++nreads;
      if (e->array != temp) unsupported("update reads array " + e->array);
      IntVec d(sk.nidx);
      for (size_t q = 0; q < sk.nidx; ++q) {
        const Affine& s = e->subs[q];
        for (size_t i = 0; i < sk.nidx + sk.nprm; ++i)
          if (s.c[i] != (i == q ? 1 : 0)) unsupported("non-uniform read in update body");
        d[q] = s.k;
      }
      std::string out = temp + "[";
      for (size_t r = 0; r < sk.nidx; ++r) {
        int64_t v = 0;
        for (size_t q = 0; q < sk.nidx; ++q) v += sk.A[r][q] * d[q];
        out += (r ? "," : "") + std::to_string(v);
      }
      return out + "]";
    }
    case K::Add: return "(" + canon(e->l, sk, temp, nreads) + "+" + canon(e->r, sk, temp, nreads) + ")";
    case K::Sub: return "(" + canon(e->l, sk, temp, nreads) + "-" + canon(e->r, sk, temp, nreads) + ")";
    case K::Mul: return "(" + canon(e->l, sk, temp, nreads) + "*" + canon(e->r, sk, temp, nreads) + ")";
    case K::Div: return "(" + canon(e->l, sk, temp, nreads) + "/" + canon(e->r, sk, temp, nreads) + ")";
    case K::Min: return "min(" + canon(e->l, sk, temp, nreads) + "," + canon(e->r, sk, temp, nreads) + ")";
    case K::Max: return "max(" + canon(e->l, sk, temp, nreads) + "," + canon(e->r, sk, temp, nreads) + ")";
    case K::Neg: return "-(" + canon(e->l, sk, temp, nreads) + ")";
    case K::Sqrt: return "sqrt(" + canon(e->l, sk, temp, nreads) + ")";
  }
  return "";
}

// Canonical text with affine subscripts written over positional index names.
std::string canon_plain(const ExprPtr& e, size_t nidx, int& nreads) {
  using K = Expr::Kind;
  auto aff = [&](const Affine& a) {
    std::string s;
    for (size_t i = 0; i < a.c.size(); ++i)
      if (a.c[i]) s += (a.c[i] > 0 ? "+" : "-") + std::to_string(std::llabs(a.c[i])) + "*" +
                       (i < nidx ? "$" + std::to_string(i) : "p" + std::to_string(i - nidx));
    if (a.k || s.empty()) s += (a.k >= 0 ? "+" : "-") + std::to_string(std::llabs(a.k));
    return s;
  };
  switch (e->kind) {
    case K::Lit: return fmt_lit(e->lit);
    case K::Aff: return "aff(" + aff(e->aff) + ")";
    case K::Read: {
      ++nreads;
      std::string s = e->array + "[";
      for (size_t i = 0; i < e->subs.size(); ++i) s += (i ? "," : "") + aff(e->subs[i]);
      return s + "]";
    }
    case K::Add: return "(" + canon_plain(e->l, nidx, nreads) + "+" + canon_plain(e->r, nidx, nreads) + ")";
    case K::Sub: return "(" + canon_plain(e->l, nidx, nreads) + "-" + canon_plain(e->r, nidx, nreads) + ")";
    case K::Mul: return "(" + canon_plain(e->l, nidx, nreads) + "*" + canon_plain(e->r, nidx, nreads) + ")";
    case K::Div: return "(" + canon_plain(e->l, nidx, nreads) + "/" + canon_plain(e->r, nidx, nreads) + ")";
    default: return "?";
  }
}

int count_reads(const ExprPtr& e) {
  if (!e) return 0;
  return (e->kind == Expr::Kind::Read ? 1 : 0) + count_reads(e->l) + count_reads(e->r);
}

// Box of a domain in u-space at bound params (throws Unsupported if not a box).
// Rows that couple several coordinates are accepted when all but one of those
// coordinates are pinned (lo == hi) by other rows, e.g. "x >= 0" at t = 0.
void domain_box(const Statement& st, const Skew& sk, const IntVec& prm, IntVec& lo, IntVec& hi) {
  const size_t n = sk.nidx;
  lo.assign(n, INT64_MIN / 4);
  hi.assign(n, INT64_MAX / 4);
  struct URow {
    IntVec cu;
    int64_t cst;
    bool done;
  };
  std::vector<URow> rows;
  for (const auto& row : st.domain) {
    // row . z + rp . p + rc >= 0 with z = Ainv (u - b)
    int64_t cst = row.back();
    for (size_t j = 0; j < sk.nprm; ++j) cst += row[n + j] * prm[j];
    IntVec cu(n, 0);
    for (size_t q = 0; q < n; ++q)
      for (size_t r = 0; r < n; ++r) cu[r] += row[q] * sk.Ainv[q][r];
    for (size_t r = 0; r < n; ++r) cst -= cu[r] * sk.b[r];
    rows.push_back({cu, cst, false});
  }
  auto apply = [&](size_t which, int64_t a, int64_t cst) {
    if (a > 0) {  // a*u + cst >= 0  ->  u >= ceil(-cst/a)
      int64_t v = -cst >= 0 ? (-cst + a - 1) / a : -((cst) / a);
      lo[which] = std::max(lo[which], v);
    } else {      // -|a| u + cst >= 0 -> u <= floor(cst/|a|)
      int64_t m = -a;
      int64_t v = cst >= 0 ? cst / m : -((-cst + m - 1) / m);
      hi[which] = std::min(hi[which], v);
    }
  };
  bool infeasible = false;
  for (bool changed = true; changed;) {
    changed = false;
    for (auto& r : rows) {
      if (r.done) continue;
      int64_t cst = r.cst;
      int free = 0;
      size_t which = 0;
      for (size_t q = 0; q < n; ++q) {
        if (!r.cu[q]) continue;
        if (lo[q] == hi[q]) cst += r.cu[q] * lo[q];
        else ++free, which = q;
      }
      if (free > 1) continue;
      r.done = changed = true;
      if (free == 0) {
        if (cst < 0) infeasible = true;
        continue;
      }
      apply(which, r.cu[which], cst);
    }
  }
  for (const auto& r : rows)
    if (!r.done) unsupported("domain of " + st.id + " is not a box in un-skewed coordinates");
  if (infeasible) lo[0] = 1, hi[0] = 0;
  for (size_t r = 0; r < n; ++r)
    if (!infeasible && (lo[r] <= INT64_MIN / 8 || hi[r] >= INT64_MAX / 8))
      fail(ErrorKind::Unbounded, "domain of " + st.id + " is unbounded");
}

bool box_empty(const IntVec& lo, const IntVec& hi) {
  for (size_t i = 0; i < lo.size(); ++i)
    if (lo[i] > hi[i]) return true;
  return false;
}

uint64_t box_volume(const IntVec& lo, const IntVec& hi) {
  if (box_empty(lo, hi)) return 0;
  uint64_t v = 1;
  for (size_t i = 0; i < lo.size(); ++i) v *= uint64_t(hi[i] - lo[i] + 1);
  return v;
}

const std::string kS2D5 =
    "(0.20000000000000001*((((X[-1,0,0]+X[-1,-1,0])+X[-1,1,0])+X[-1,0,-1])+X[-1,0,1]))";
const std::string kGS9 =
    "(((((((((X[0,-1,-1]+X[0,-1,0])+X[0,-1,1])+X[0,0,-1])+X[-1,0,0])+X[-1,0,1])+X[-1,1,-1])+X[-1,1,0])+"
    "X[-1,1,1])/9)";
const std::string kS3D7R0 =
    "(X[-1,0,0,0]+(0.125*((((((X[-1,-1,0,0]+X[-1,1,0,0])+X[-1,0,-1,0])+X[-1,0,1,0])+X[-1,0,0,-1])+"
    "X[-1,0,0,1])-(6*X[-1,0,0,0]))))";
const std::string kS3D7R1 =
    "(0.10000000000000001*((((((X[-1,0,0,0]+X[-1,-1,0,0])+X[-1,1,0,0])+X[-1,0,-1,0])+X[-1,0,1,0])+"
    "X[-1,0,0,-1])+X[-1,0,0,1]))";
const std::string kGEMM = "(C[+1*$0,+1*$1,+1*$2-1]+(((2*A[+1*$0,+1*$2-1])-1)*((2*B[+1*$2-1,+1*$1])-1)))";

std::string replace_all(std::string s, const std::string& from, const std::string& to) {
  size_t p = 0;
  while ((p = s.find(from, p)) != std::string::npos) s.replace(p, from.size(), to), p += to.size();
  return s;
}

Recognized recognize_stencil(const KernelSpec& k, const IntVec& prm) {
  Recognized R;
  const size_t nidx = k.indices.size(), d = nidx - 1, nprm = k.params.size();
  const ArrayDecl *in = nullptr, *tmp = nullptr, *out = nullptr;
  for (const auto& a : k.arrays)
    (a.kind == ArrayKind::Input ? in : a.kind == ArrayKind::Temp ? tmp : out) = &a;
  if (in->rank != d || out->rank != d || tmp->rank != nidx) unsupported("array ranks do not fit a stencil");
  R.inputs = {in->name};
  R.temp = tmp->name;
  R.output = out->name;
  R.ndim = int(d);
  // ---- final statement: Out[U(z)] = X[z], domain pins t to a parameter
  const Statement* fin = nullptr;
  for (const auto& s : k.statements)
    if (s.write_array == out->name) {
      if (fin) unsupported("more than one statement writes the output");
      fin = &s;
    }
  if (!fin) unsupported("no statement writes the output");
  if (fin->body->kind != Expr::Kind::Read || fin->body->array != tmp->name) unsupported("output is not a copy of the temp");
  for (size_t q = 0; q < nidx; ++q) {
    const Affine& s = fin->body->subs[q];
    for (size_t i = 0; i < nidx + nprm; ++i)
      if (s.c[i] != (i == q ? 1 : 0) || s.k != 0) unsupported("output copy is not X[indices]");
  }
  int tparam = -1;
  for (size_t j = 0; j < nprm && tparam < 0; ++j) {
    bool ge = false, le = false;
    for (const auto& row : fin->domain) {
      bool only = row.back() == 0;
      for (size_t i = 1; i < nidx; ++i) only = only && row[i] == 0;
      for (size_t jj = 0; jj < nprm; ++jj) only = only && (jj == j || row[nidx + jj] == 0);
      if (!only) continue;
      if (row[0] == 1 && row[nidx + j] == -1) ge = true;
      if (row[0] == -1 && row[nidx + j] == 1) le = true;
    }
    if (ge && le) tparam = int(j);
  }
  if (tparam < 0) unsupported("output statement does not fix time to a parameter");
  Skew sk;
  sk.nidx = nidx;
  sk.nprm = nprm;
  sk.A.assign(nidx, IntVec(nidx, 0));
  sk.b.assign(nidx, 0);
  sk.A[0][0] = 1;
  for (size_t r = 0; r < d; ++r) {
    Affine u = fin->write_subs[r];
    u.c[0] += u.c[nidx + tparam];
    u.c[nidx + tparam] = 0;
    for (size_t j = 0; j < nprm; ++j)
      if (u.c[nidx + j]) unsupported("un-skewing map depends on a parameter");
    for (size_t q = 0; q < nidx; ++q) sk.A[r + 1][q] = u.c[q];
    sk.b[r + 1] = u.k;
  }
  sk.Ainv = inverse_unimodular(sk.A);
  R.Ainv = sk.Ainv;
  R.b = sk.b;
  R.T = prm[tparam];
  // ---- classify temp-writing statements
  std::string update_canon;
  int n_update = 0;
  struct Piece { IntVec lo, hi; };
  std::vector<Piece> ring_zero, ring_copy, init;
  for (const auto& s : k.statements) {
    StmtBox b;
    b.id = s.id;
    domain_box(s, sk, prm, b.lo, b.hi);
    b.points = box_volume(b.lo, b.hi);
    b.reads_per_point = uint64_t(count_reads(s.body));
    if (&s == fin) {
      b.role = "final";
      R.stmts.push_back(b);
      continue;
    }
    if (s.write_array != tmp->name) unsupported("statement " + s.id + " writes an unexpected array");
    for (size_t q = 0; q < nidx; ++q) {
      const Affine& w = s.write_subs[q];
      for (size_t i = 0; i < nidx + nprm; ++i)
        if (w.c[i] != (i == q ? 1 : 0) || w.k != 0) unsupported("statement " + s.id + " does not write X[indices]");
    }
    const Expr& e = *s.body;
    if (e.kind == Expr::Kind::Lit && e.lit == 0.0 && !std::signbit(e.lit)) {
      b.role = "ring";
      ring_zero.push_back({b.lo, b.hi});
    } else if (e.kind == Expr::Kind::Read && e.array == tmp->name) {
      int nr = 0;
      std::string c = canon(s.body, sk, tmp->name, nr);
      std::string want = tmp->name + "[-1";
      for (size_t r = 0; r < d; ++r) want += ",0";
      if (c != want + "]") unsupported("statement " + s.id + " copies an unexpected cell");
      b.role = "ring";
      ring_copy.push_back({b.lo, b.hi});
    } else if (e.kind == Expr::Kind::Read && e.array == in->name) {
      // F[cell] at t = 0: subscripts must equal U(z) restricted to t = 0
      for (size_t r = 0; r < d; ++r) {
        const Affine& f = e.subs[r];
        for (size_t q = 1; q < nidx; ++q)
          if (f.c[q] != sk.A[r + 1][q]) unsupported("init statement " + s.id + " reads a skewed cell");
        for (size_t j = 0; j < nprm; ++j)
          if (f.c[nidx + j]) unsupported("init statement " + s.id + " depends on a parameter");
        if (f.k != sk.b[r + 1]) unsupported("init statement " + s.id + " reads a shifted cell");
      }
      if (!box_empty(b.lo, b.hi) && (b.lo[0] != 0 || b.hi[0] != 0)) unsupported("init statement " + s.id + " is not at t = 0");
      b.role = "init";
      init.push_back({b.lo, b.hi});
    } else {
      int nr = 0;
      update_canon = canon(s.body, sk, tmp->name, nr);
      update_canon = replace_all(update_canon, tmp->name + "[", "X[");
      b.role = "update";
      ++n_update;
      // the update box must be [1,T] x interior (checked below)
      R.stmts.push_back(b);
      continue;
    }
    R.stmts.push_back(b);
  }
  if (n_update != 1) unsupported("expected exactly one update statement");
  if (d == 2 && update_canon == kS2D5) R.family = Family::Stencil2D5;
  else if (d == 2 && update_canon == kGS9) R.family = Family::GaussSeidel2D9;
  else if (d == 3 && update_canon == kS3D7R0) R.family = Family::Stencil3D7, R.rule = 0;
  else if (d == 3 && update_canon == kS3D7R1) R.family = Family::Stencil3D7, R.rule = 1;
  else unsupported("update body not in the registry: " + update_canon);
  // ---- grid extent from the output statement: [T,T] x [0, n-1]^d
  const StmtBox* fb = nullptr;
  for (const auto& b : R.stmts)
    if (b.role == "final") fb = &b;
  if (fb->lo[0] != R.T || fb->hi[0] != R.T) unsupported("output statement is not at t = T");
  const int64_t n = fb->hi[1] - fb->lo[1] + 1;
  for (size_t r = 1; r <= d; ++r)
    if (fb->lo[r] != 0 || fb->hi[r] != n - 1) unsupported("output does not cover the square grid");
  R.N = n;
  for (const auto& a : {in, out}) {
    for (const auto& ex : a->extents)
      if (eval_aff(ex, {}, prm) != n) unsupported("array " + a->name + " extent differs from the grid");
  }
  if (R.T < 0 || n < 3) unsupported("grid smaller than 3 or negative T");
  // ---- update box
  for (const auto& b : R.stmts)
    if (b.role == "update") {
      if (R.T >= 1 && box_empty(b.lo, b.hi)) unsupported("update statement has an empty domain");
      if (R.T >= 1 && (b.lo[0] != 1 || b.hi[0] != R.T)) unsupported("update does not span t = 1..T");
      for (size_t r = 1; r <= d; ++r)
        if (b.lo[r] != 1 || b.hi[r] != n - 2) unsupported("update does not cover the interior");
    }
  // ---- ring + init partition
  auto ring_volume = [&](int64_t t0) {
    (void)t0;
    uint64_t full = 1, inner = 1;
    for (size_t r = 0; r < d; ++r) full *= uint64_t(n), inner *= uint64_t(n - 2);
    return full - inner;
  };
  auto check_ring = [&](const std::vector<Piece>& ps, int64_t t0) {
    uint64_t vol = 0;
    for (size_t a = 0; a < ps.size(); ++a) {
      const Piece& p = ps[a];
      if (box_empty(p.lo, p.hi)) continue;
      if (p.lo[0] != t0 || p.hi[0] != R.T) unsupported("ring piece does not span the time range");
      bool on_ring = false;
      for (size_t r = 1; r <= d; ++r) {
        if (p.lo[r] < 0 || p.hi[r] > n - 1) unsupported("ring piece leaves the grid");
        if ((p.lo[r] == 0 && p.hi[r] == 0) || (p.lo[r] == n - 1 && p.hi[r] == n - 1)) on_ring = true;
      }
      if (!on_ring) unsupported("ring piece is not on the ring");
      for (size_t b2 = a + 1; b2 < ps.size(); ++b2) {
        bool overlap = !box_empty(ps[b2].lo, ps[b2].hi);
        for (size_t r = 1; r <= d && overlap; ++r)
          overlap = std::max(p.lo[r], ps[b2].lo[r]) <= std::min(p.hi[r], ps[b2].hi[r]);
        if (overlap) unsupported("ring pieces overlap");
      }
      uint64_t v = 1;
      for (size_t r = 1; r <= d; ++r) v *= uint64_t(p.hi[r] - p.lo[r] + 1);
      vol += v;
    }
    if (vol != ring_volume(t0)) unsupported("ring pieces do not cover the ring");
  };
  if (init.size() != 1) unsupported("expected one init statement");
  const Piece& ip = init[0];
  bool init_full = true, init_inner = true;
  for (size_t r = 1; r <= d; ++r) {
    init_full = init_full && ip.lo[r] == 0 && ip.hi[r] == n - 1;
    init_inner = init_inner && ip.lo[r] == 1 && ip.hi[r] == n - 2;
  }
  if (!ring_zero.empty() && ring_copy.empty() && init_inner) {
    check_ring(ring_zero, 0);
    R.ring_hold = 0;
  } else if (ring_zero.empty() && !ring_copy.empty() && init_full) {
    if (R.T >= 1) check_ring(ring_copy, 1);
    R.ring_hold = 1;
  } else {
    unsupported("ring/init statements do not match a zero or copied ring");
  }
  if (R.family == Family::GaussSeidel2D9 && R.ring_hold) unsupported("Gauss-Seidel with a copied ring");
  return R;
}

Recognized recognize_gemm(const KernelSpec& k, const IntVec& prm) {
  Recognized R;
  R.family = Family::Gemm;
  R.ndim = 2;
  const ArrayDecl *tmp = nullptr, *out = nullptr;
  std::vector<const ArrayDecl*> ins;
  for (const auto& a : k.arrays) {
    if (a.kind == ArrayKind::Input) ins.push_back(&a);
    else if (a.kind == ArrayKind::Temp) tmp = &a;
    else out = &a;
  }
  R.temp = tmp->name;
  R.output = out->name;
  if (!tmp || !out) unsupported("gemm needs one temp and one output array");
  std::string upd;
  const size_t nidx = k.indices.size();
  int nfinal = 0, ninit = 0, nupdate = 0;
  // canonical form of a statement's write reference (same notation as reads)
  auto write_ref = [&](const Statement& s) {
    auto e = std::make_shared<Expr>();
    e->kind = Expr::Kind::Read;
    e->array = s.write_array;
    e->subs = s.write_subs;
    int nr = 0;
    std::string c = canon_plain(e, nidx, nr);
    c = replace_all(c, tmp->name + "[", "C[");
    return replace_all(c, out->name + "[", "Out[");
  };
  const std::string kTmpIJK = "C[+1*$0,+1*$1,+1*$2]";
  for (const auto& s : k.statements) {
    StmtBox b;
    b.id = s.id;
    Skew sk;
    sk.nidx = nidx;
    sk.nprm = k.params.size();
    sk.A.assign(nidx, IntVec(nidx, 0));
    for (size_t i = 0; i < nidx; ++i) sk.A[i][i] = 1;
    sk.b.assign(nidx, 0);
    sk.Ainv = sk.A;
    domain_box(s, sk, prm, b.lo, b.hi);
    b.points = box_volume(b.lo, b.hi);
    b.reads_per_point = uint64_t(count_reads(s.body));
    int nr = 0;
    std::string c = canon_plain(s.body, nidx, nr);
    if (s.write_array == out->name) {
      b.role = "final";
      ++nfinal;
      // Out[i, j] = C[i, j, k] (at k = N): a plain copy, identity subscripts
      if (write_ref(s) != "Out[+1*$0,+1*$1]" || replace_all(c, tmp->name + "[", "C[") != kTmpIJK)
        unsupported("gemm output statement is not Out[i,j] = C[i,j,k]");
    } else if (s.body->kind == Expr::Kind::Lit && s.body->lit == 0.0) {
      b.role = "init";
      ++ninit;
      if (write_ref(s) != kTmpIJK) unsupported("gemm init statement does not write C[i,j,k]");
    } else {
      b.role = "update";
      ++nupdate;
      if (write_ref(s) != kTmpIJK) unsupported("gemm update statement does not write C[i,j,k]");
      upd = c;
      // A/B are the two inputs in declaration order: substitute their names
      if (ins.size() != 2) unsupported("gemm needs two inputs");
      upd = replace_all(upd, ins[0]->name + "[", "A[");
      upd = replace_all(upd, ins[1]->name + "[", "B[");
      upd = replace_all(upd, tmp->name + "[", "C[");
    }
    R.stmts.push_back(b);
  }
  if (nfinal != 1 || ninit != 1 || nupdate != 1)
    unsupported("gemm needs exactly one init, one update and one output statement");
  if (upd != kGEMM) unsupported("update body not in the registry: " + upd);
  const StmtBox* fb = nullptr;
  for (const auto& b : R.stmts)
    if (b.role == "final") fb = &b;
  if (!fb) unsupported("no output statement");
  const int64_t n = fb->hi[0] - fb->lo[0] + 1;
  if (n < 1 || fb->lo[0] != 0 || fb->lo[1] != 0 || fb->hi[1] != n - 1 || fb->lo[2] != n || fb->hi[2] != n)
    unsupported("gemm output box");
  for (const auto& b : R.stmts) {
    if (b.role == "update" && (b.lo[0] != 0 || b.hi[0] != n - 1 || b.lo[1] != 0 || b.hi[1] != n - 1 ||
                               b.lo[2] != 1 || b.hi[2] != n))
      unsupported("gemm update box");
    if (b.role == "init" && (b.lo[0] != 0 || b.hi[0] != n - 1 || b.lo[1] != 0 || b.hi[1] != n - 1 ||
                             b.lo[2] != 0 || b.hi[2] != 0))
      unsupported("gemm init box");
  }
  R.N = n;
  R.inputs = {ins[0]->name, ins[1]->name};
  R.Ainv.assign(nidx, IntVec(nidx, 0));
  for (size_t i = 0; i < nidx; ++i) R.Ainv[i][i] = 1;
  R.b.assign(nidx, 0);
  return R;
}


int64_t eval_param_affine(const Affine& a, size_t nidx, const IntVec& prm) {
  int64_t v = a.k;
  const size_t off = a.c.size() >= nidx + prm.size() ? nidx : 0;
  for (size_t j = 0; j < prm.size(); ++j)
    if (off + j < a.c.size()) v += a.c[off + j] * prm[j];
  return v;
}

}  // namespace

void check_maps(const KernelSpec& k, const std::vector<MemoryMap>& maps) {
  for (const auto& m : maps) {
    const ArrayDecl* a = k.find_array(m.array);
    if (!a) fail(ErrorKind::Validation, "Executor: memory map for unknown array " + m.array);
    const size_t pd = m.extents.size();
    if (m.linear.size() != pd || m.constant.size() != pd || m.moduli.size() != pd)
      fail(ErrorKind::DimMismatch, "Executor: malformed memory map for " + m.array);
    for (const auto& row : m.linear)
      if (row.size() != a->rank) fail(ErrorKind::DimMismatch, "Executor: memory map arity for " + m.array);
    for (size_t q = 0; q < pd; ++q)
      if (m.extents[q] < 0 || m.moduli[q] < 0)
        fail(ErrorKind::Validation, "Executor: negative extent or modulus in the map of " + m.array);
  }
  for (const auto& a : k.arrays) {
    int n = 0;
    for (const auto& m : maps) n += m.array == a.name;
    if (n == 0) fail(ErrorKind::Validation, "Executor: no memory map for array " + a.name);
  }
}

bool hot_path_honours(const Recognized& R, const KernelSpec& k, const IntVec& prm,
                      const std::vector<MemoryMap>& maps, std::string* why) {
  const size_t nidx = k.indices.size();
  auto no = [&](const std::string& m) {
    if (why) *why = m;
    return false;
  };
  // occupancy vector of the temp, in its cell coordinates (= kernel indices)
  IntVec u0(nidx, 0);
  switch (R.family) {
    case Family::Stencil2D5:
    case Family::Stencil3D7: u0.assign(nidx, 2); break;        // (t mod 2, x - t, ...)
    case Family::GaussSeidel2D9: u0 = {1, 1, 2}; break;        // (t mod 1, x - t, y - 2t)
    case Family::Gemm: u0 = {0, 0, 1}; break;                  // (i, j, k mod 1)
    default: return no("not a hot-path kernel");
  }
  for (const auto& a : k.arrays) {
    const MemoryMap* m = nullptr;
    for (const auto& mm : maps)
      if (mm.array == a.name) m = &mm;
    if (!m) return no("no map for " + a.name);
    const size_t r = a.rank, pd = m->extents.size();
    bool identity = pd == r;
    for (size_t q = 0; identity && q < pd; ++q) {
      identity = m->constant[q] == 0 && m->moduli[q] == 0;
      for (size_t c = 0; c < r; ++c) identity = identity && m->linear[q][c] == (q == c ? 1 : 0);
    }
    IntVec decl(r);
    for (size_t q = 0; q < r; ++q) decl[q] = eval_param_affine(a.extents[q], nidx, prm);
    if (a.kind != ArrayKind::Temp) {
      if (!identity || m->extents != decl)
        return no("the " + a.name + " map is not the identity at the declared extents");
      continue;
    }
    if (identity) {  // single assignment: every cell the run touches lies in the declared box
      for (size_t q = 0; q < r; ++q)
        if (m->extents[q] < decl[q]) return no("the " + a.name + " map is smaller than its declared extents");
      continue;
    }
    // folded along u = c * (e_j0 - sum_i alpha_i e_i): linear = I except column j0
    if (pd != r) return no("the " + a.name + " map changes the rank");
    int j0 = -1;
    for (size_t q = 0; q < pd; ++q)
      if (m->moduli[q] > 0) {
        if (j0 >= 0) return no("the " + a.name + " map folds more than one dimension");
        j0 = int(q);
      }
    if (j0 < 0) return no("the " + a.name + " map is neither single-assignment nor folded");
    const int64_t c = m->moduli[size_t(j0)];
    IntVec u(r, 0);
    u[size_t(j0)] = c;
    for (size_t q = 0; q < pd; ++q)
      for (size_t cc = 0; cc < r; ++cc) {
        const int64_t v = m->linear[q][cc];
        if (cc == size_t(j0) && q != size_t(j0)) {
          u[q] = -v * c;
        } else if (v != (q == cc ? 1 : 0)) {
          return no("the " + a.name + " map is not an occupancy-vector fold");
        }
      }
    // u must be a positive multiple of the kernel's occupancy vector
    int64_t mult = 0;
    for (size_t q = 0; q < r; ++q)
      if (u0[q]) {
        if (u[q] % u0[q]) return no("the " + a.name + " map folds along a vector the kernel does not allow");
        mult = u[q] / u0[q];
        break;
      }
    if (mult < 1) return no("the " + a.name + " map folds along a vector the kernel does not allow");
    for (size_t q = 0; q < r; ++q)
      if (u[q] != mult * u0[q]) return no("the " + a.name + " map folds along a vector the kernel does not allow");
    // extents: every cell the temp-writing statements touch must map inside
    // (the modulo dimension needs extent >= modulus)
    if (m->extents[size_t(j0)] < c)
      fail(ErrorKind::Validation, "out-of-extent storage for " + a.name + ": folded extent below its modulus");
    IntVec lo(pd, INT64_MAX), hi(pd, INT64_MIN);
    for (const auto& b : R.stmts) {
      if (b.role == "final" || b.lo.empty()) continue;
      bool empty = false;
      for (size_t q = 0; q < b.lo.size(); ++q) empty = empty || b.lo[q] > b.hi[q];
      if (empty) continue;
      const size_t nb = b.lo.size();
      for (uint64_t corner = 0; corner < (uint64_t(1) << nb); ++corner) {
        IntVec uu(nb), z(nidx, 0);
        for (size_t q = 0; q < nb; ++q) uu[q] = (corner >> q & 1) ? b.hi[q] : b.lo[q];
        for (size_t i = 0; i < nidx; ++i)
          for (size_t j = 0; j < nidx && j < nb; ++j) z[i] += R.Ainv[i][j] * (uu[j] - R.b[j]);
        for (size_t q = 0; q < pd; ++q) {
          int64_t v = m->constant[q];
          for (size_t cc = 0; cc < r; ++cc) v += m->linear[q][cc] * z[cc];
          lo[q] = std::min(lo[q], v);
          hi[q] = std::max(hi[q], v);
        }
      }
    }
    for (size_t q = 0; q < pd; ++q)
      if (q != size_t(j0) && lo[q] <= hi[q] && (lo[q] < 0 || hi[q] >= m->extents[q]))
        fail(ErrorKind::Validation, "out-of-extent access to " + a.name + " dim " + std::to_string(q) +
                                        " under its memory map (storage range [" + std::to_string(lo[q]) +
                                        ", " + std::to_string(hi[q]) + "])");
  }
  return true;
}

Recognized recognize(const KernelSpec& k, const IntVec& params) {
  if (params.size() != k.params.size()) fail(ErrorKind::DimMismatch, "GpuExecutor: parameter count");
  for (const auto& s : k.statements)
    if (s.depth != k.indices.size()) fail(ErrorKind::Validation, "GpuExecutor: kernel must be embedded");
  int nin = 0, ntmp = 0, nout = 0;
  for (const auto& a : k.arrays)
    (a.kind == ArrayKind::Input ? nin : a.kind == ArrayKind::Temp ? ntmp : nout)++;
  Recognized R;
  if (nin == 1 && ntmp == 1 && nout == 1 && (k.indices.size() == 3 || k.indices.size() == 4))
    R = recognize_stencil(k, params);
  else if (nin == 2 && ntmp == 1 && nout == 1 && k.indices.size() == 3)
    R = recognize_gemm(k, params);
  else
    unsupported("kernel '" + k.name + "' does not match a supported array signature");
  for (const auto& b : R.stmts) {
    R.points += b.points;
    R.writes += b.points;
    R.reads += b.points * b.reads_per_point;
  }
  return R;
}

}  // namespace pcotgpu
