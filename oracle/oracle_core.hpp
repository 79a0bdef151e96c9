// oracle_core.hpp — TEST INFRASTRUCTURE ONLY (parity checker, never the product path).
//
// CPU restatement of the reference `rannddm` primitives (/root/reference/proj/include/rannddm/)
// with the same floating-point operation order, so that assembly reproduces the reference's
// golden exports (proj/h_export.txt) bit for bit. Each item cites the reference file:line it
// restates. Bit-level parity requires the reference's expressions and their grouping, so the
// jet arithmetic here (random.hpp:9-37, geometry.hpp:26-75, jet.hpp:13-156) is a close
// transliteration of those headers, with Eigen (absent here) replaced by plain column-major
// storage. The reference itself is compiled separately (oracle/_ref, oracle/eigen_shim) and
// this restatement is pinned against it (tests/test_reference_build.py).
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

constexpr int kMaxDim = 4;                       // geometry.hpp:13
constexpr double kPi = 3.14159265358979323846;   // problems.hpp:18
using Point = std::array<double, kMaxDim>;       // geometry.hpp:16

// ---- random.hpp:9-37 ------------------------------------------------------------------
struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next_u64() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
  }
  double next_unit() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
  double next_symmetric() { return 2.0 * next_unit() - 1.0; }
  double next_in(double lo, double hi) { return lo + (hi - lo) * next_unit(); }
};
inline uint64_t subdomain_seed(uint64_t base, int j) {
  SplitMix64 mix(base ^ (0xD1B54A32D192ED03ULL * static_cast<uint64_t>(j + 1)));
  return mix.next_u64();
}

// ---- geometry.hpp:26-75 ---------------------------------------------------------------
struct Box {
  int dim = 0;
  Point lo{}, hi{};
  double width(int a) const { return hi[a] - lo[a]; }
  double center(int a) const { return 0.5 * (lo[a] + hi[a]); }
};
inline bool contains(const Box& b, const Point& x) {  // geometry.hpp:51-57 (closed)
  for (int a = 0; a < b.dim; ++a)
    if (x[a] < b.lo[a] || x[a] > b.hi[a]) return false;
  return true;
}
inline Point normalize_to_box(const Box& b, const Point& x) {  // geometry.hpp:61-68
  Point o{};
  for (int a = 0; a < b.dim; ++a) o[a] = 2.0 * (x[a] - b.center(a)) / b.width(a);
  return o;
}
inline Point normalize_scales(const Box& b) {  // geometry.hpp:71-75
  Point s{};
  for (int a = 0; a < b.dim; ++a) s[a] = 2.0 / b.width(a);
  return s;
}

// ---- jet.hpp:13-156 -------------------------------------------------------------------
constexpr int jet_len(int d) { return 1 + d + d * (d + 1) / 2; }
constexpr int hess_index(int i, int j, int d) { return i * d - i * (i - 1) / 2 + (j - i); }
struct Triple { double f = 0, df = 0, d2f = 0; };
inline Triple triple_tanh(double s) {
  const double t = std::tanh(s);
  const double sech2 = 1.0 - t * t;
  return {t, sech2, -2.0 * t * sech2};
}
inline Triple triple_sin(double s) { return {std::sin(s), std::cos(s), -std::sin(s)}; }
inline Triple triple_cos(double s) { return {std::cos(s), -std::sin(s), -std::cos(s)}; }
inline Triple triple_recip(double s) {
  const double r = 1.0 / s;
  return {r, -r * r, 2.0 * r * r * r};
}
inline Triple triple_exp(double s) {
  const double e = std::exp(s);
  return {e, e, e};
}

struct Jet2 {
  int dim = 0;
  double v = 0.0;
  std::array<double, kMaxDim> g{};
  std::array<double, kMaxDim*(kMaxDim + 1) / 2> h{};
  double hess(int i, int j) const {
    if (i > j) std::swap(i, j);
    return h[hess_index(i, j, dim)];
  }
  static Jet2 constant(int d, double val) {
    Jet2 o;
    o.dim = d;
    o.v = val;
    return o;
  }
  static Jet2 variable(int d, int axis, double val, double scale = 1.0) {
    Jet2 o;
    o.dim = d;
    o.v = val;
    o.g[axis] = scale;
    return o;
  }
};
inline Jet2 operator+(const Jet2& a, const Jet2& b) {
  Jet2 o = a;
  o.v += b.v;
  const int nh = a.dim * (a.dim + 1) / 2;
  for (int i = 0; i < a.dim; ++i) o.g[i] += b.g[i];
  for (int i = 0; i < nh; ++i) o.h[i] += b.h[i];
  return o;
}
inline Jet2 operator*(double c, const Jet2& a) {
  Jet2 o = a;
  o.v *= c;
  const int nh = a.dim * (a.dim + 1) / 2;
  for (int i = 0; i < a.dim; ++i) o.g[i] *= c;
  for (int i = 0; i < nh; ++i) o.h[i] *= c;
  return o;
}
inline Jet2 operator-(const Jet2& a, const Jet2& b) { return a + (-1.0 * b); }
inline Jet2 operator*(const Jet2& a, const Jet2& b) {  // jet.hpp:107-124 (Leibniz, grouped)
  Jet2 o;
  o.dim = a.dim;
  o.v = a.v * b.v;
  for (int i = 0; i < a.dim; ++i) o.g[i] = a.v * b.g[i] + b.v * a.g[i];
  for (int i = 0; i < a.dim; ++i)
    for (int j = i; j < a.dim; ++j) {
      const int k = hess_index(i, j, a.dim);
      o.h[k] = (a.v * b.h[k] + b.v * a.h[k]) + (a.g[i] * b.g[j] + a.g[j] * b.g[i]);
    }
  return o;
}
inline Jet2 compose(const Triple& t, const Jet2& a) {  // jet.hpp:127-138
  Jet2 o;
  o.dim = a.dim;
  o.v = t.f;
  for (int i = 0; i < a.dim; ++i) o.g[i] = t.df * a.g[i];
  for (int i = 0; i < a.dim; ++i)
    for (int j = i; j < a.dim; ++j) {
      const int k = hess_index(i, j, a.dim);
      o.h[k] = t.df * a.h[k] + t.d2f * a.g[i] * a.g[j];
    }
  return o;
}
inline Jet2 tanh_of_linear(int d, int axis, double x, double alpha, double beta = 0.0) {
  const Jet2 arg = Jet2::variable(d, axis, alpha * x + beta, alpha);
  return compose(triple_tanh(arg.v), arg);
}
inline Jet2 sin_of_linear(int d, int axis, double x, double alpha, double beta = 0.0) {
  const Jet2 arg = Jet2::variable(d, axis, alpha * x + beta, alpha);
  return compose(triple_sin(arg.v), arg);
}
inline Jet2 cos_of_linear(int d, int axis, double x, double alpha, double beta = 0.0) {
  const Jet2 arg = Jet2::variable(d, axis, alpha * x + beta, alpha);
  return compose(triple_cos(arg.v), arg);
}

}  // namespace orc
