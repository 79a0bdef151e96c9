// rdd_eigen_shim.hpp — TEST INFRASTRUCTURE ONLY.
//
// A small stand-in for the part of Eigen 3's API that the reference headers
// (/root/reference/proj/include/rannddm/*.hpp) use, so that the UNMODIFIED reference can be
// compiled here (Eigen is not installed and there is no network). It is used to build
// oracle/_ref (the reference itself, the strongest oracle) and the level-2 drop-in test that
// runs the reference's own Krylov drivers over the device operators (tests/cpp/).
//
// Semantics: dynamic-size double matrices in column-major storage, evaluated eagerly (no
// expression templates); vectors are n x 1 matrices; blocks/rows/columns/segments are
// writable strided views. Sums run in index order (Eigen's vectorised kernels sum in a
// different order, so results agree with a real Eigen build to rounding, not bitwise).
// Decompositions call LAPACK from scipy's bundled OpenBLAS, loaded with dlopen from
// $RDD_LAPACK_PATH (the oracle's loader sets it; oracle/oracle.py lapack_path()):
//   JacobiSVD               -> column-pivoted QR preconditioner (dgeqp3) + one-sided Jacobi
//                              on R (dgesvj), Eigen's default QR-preconditioned form
//   SelfAdjointEigenSolver  -> dsyevd (ascending eigenvalues, lower triangle read)
//   ColPivHouseholderQR     -> dgeqp3 + dormqr + triangular solve with Eigen's rank rule
//   EigenSolver / BDCSVD    -> dgeev / dgesvd
// This is an API-compatible re-implementation written for this repository, not Eigen code.
#pragma once

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdlib>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;
enum UpLoType { Lower = 1, Upper = 2 };
enum DecompositionOptions { ComputeFullU = 0x04, ComputeThinU = 0x08, ComputeFullV = 0x10, ComputeThinV = 0x20,
                            EigenvaluesOnly = 0x40, ComputeEigenvectors = 0x80 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

class MatrixXd;
class Block;
class ArrayRef;

namespace shim {
[[noreturn]] inline void fail(const char* what) { throw std::logic_error(std::string("eigen shim: ") + what); }

// ---- LAPACK (scipy-openblas, `scipy_` symbol prefix)
struct Lapack {
  void* h = nullptr;
  void* sym(const char* n) {
    if (!h) {
      const char* p = std::getenv("RDD_LAPACK_PATH");
      if (!p || !*p) fail("RDD_LAPACK_PATH not set (scipy's bundled OpenBLAS)");
      h = dlopen(p, RTLD_NOW | RTLD_LOCAL);
      if (!h) fail("dlopen of RDD_LAPACK_PATH failed");
      if (auto st = reinterpret_cast<void (*)(int)>(dlsym(h, "scipy_openblas_set_num_threads"))) st(1);
    }
    void* f = dlsym(h, n);
    if (!f) fail(n);
    return f;
  }
};
inline Lapack& lapack() {
  static Lapack L;
  return L;
}
}  // namespace shim

// ---------------------------------------------------------------- dense storage
class MatrixXd {
 public:
  MatrixXd() = default;
  explicit MatrixXd(Index n) : r_(n), c_(1), a_(static_cast<size_t>(n), 0.0) {}
  MatrixXd(Index r, Index c) : r_(r), c_(c), a_(static_cast<size_t>(r * c), 0.0) {}
  MatrixXd(const Block& b);  // NOLINT (implicit, like Eigen's expression conversion)
  MatrixXd& operator=(const Block& b);

  static MatrixXd Zero(Index n) { return MatrixXd(n); }
  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
  static MatrixXd Ones(Index n) { return Constant(n, 1, 1.0); }
  static MatrixXd Ones(Index r, Index c) { return Constant(r, c, 1.0); }
  static MatrixXd Constant(Index n, double v) { return Constant(n, 1, v); }
  static MatrixXd Constant(Index r, Index c, double v) {
    MatrixXd m(r, c);
    std::fill(m.a_.begin(), m.a_.end(), v);
    return m;
  }
  static MatrixXd Identity(Index r, Index c) {
    MatrixXd m(r, c);
    for (Index i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }

  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  void resize(Index n) { resize(n, 1); }
  void resize(Index r, Index c) {
    if (r * c != size()) a_.assign(static_cast<size_t>(r * c), 0.0);
    r_ = r;
    c_ = c;
  }
  void setZero() { std::fill(a_.begin(), a_.end(), 0.0); }
  void setZero(Index n) { resize(n); setZero(); }
  void setZero(Index r, Index c) { resize(r, c); setZero(); }
  void setConstant(double v) { std::fill(a_.begin(), a_.end(), v); }

  double& operator()(Index i) { return a_[static_cast<size_t>(i)]; }
  double operator()(Index i) const { return a_[static_cast<size_t>(i)]; }
  double& operator()(Index i, Index j) { return a_[static_cast<size_t>(j * r_ + i)]; }
  double operator()(Index i, Index j) const { return a_[static_cast<size_t>(j * r_ + i)]; }
  double& operator[](Index i) { return a_[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return a_[static_cast<size_t>(i)]; }

  // views
  Block block(Index i, Index j, Index r, Index c) const;
  Block col(Index j) const;
  Block row(Index i) const;
  Block segment(Index i, Index n) const;
  Block head(Index n) const;
  Block tail(Index n) const;
  Block topRows(Index n) const;
  Block bottomRows(Index n) const;
  Block leftCols(Index n) const;
  Block rightCols(Index n) const;
  Block topLeftCorner(Index r, Index c) const;
  MatrixXd& noalias() { return *this; }
  ArrayRef array() const;
  MatrixXd eval() const { return *this; }

  double trace() const {
    double t = 0.0;
    for (Index i = 0; i < std::min(r_, c_); ++i) t += (*this)(i, i);
    return t;
  }
  Block diagonal() const;
  class CommaInit operator<<(double v);
  class LdltSolve ldlt() const;
  bool operator==(const MatrixXd& o) const { return r_ == o.r_ && c_ == o.c_ && a_ == o.a_; }
  bool operator!=(const MatrixXd& o) const { return !(*this == o); }

  MatrixXd transpose() const {
    MatrixXd t(c_, r_);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  MatrixXd adjoint() const { return transpose(); }

  // reductions (linear index order)
  double dot(const MatrixXd& o) const {
    if (o.size() != size()) shim::fail("dot: size mismatch");
    double s = 0.0;
    for (Index i = 0; i < size(); ++i) s += a_[i] * o.a_[i];
    return s;
  }
  double squaredNorm() const { return dot(*this); }
  double norm() const { return std::sqrt(squaredNorm()); }
  double sum() const {
    double s = 0.0;
    for (double v : a_) s += v;
    return s;
  }
  double mean() const { return sum() / static_cast<double>(size()); }
  double maxCoeff() const { return *std::max_element(a_.begin(), a_.end()); }
  double minCoeff() const { return *std::min_element(a_.begin(), a_.end()); }
  double lpNorm_inf() const {
    double m = 0.0;
    for (double v : a_) m = std::max(m, std::abs(v));
    return m;
  }
  bool allFinite() const {
    for (double v : a_)
      if (!std::isfinite(v)) return false;
    return true;
  }
  bool hasNaN() const {
    for (double v : a_)
      if (std::isnan(v)) return true;
    return false;
  }

  // coefficient-wise
  template <class F>
  MatrixXd unaryExpr(F f) const {
    MatrixXd m = *this;
    for (double& v : m.a_) v = f(v);
    return m;
  }
  MatrixXd cwiseAbs() const { return unaryExpr([](double v) { return std::abs(v); }); }
  MatrixXd cwiseInverse() const { return unaryExpr([](double v) { return 1.0 / v; }); }
  MatrixXd cwiseSqrt() const { return unaryExpr([](double v) { return std::sqrt(v); }); }
  MatrixXd cwiseProduct(const MatrixXd& o) const {
    MatrixXd m = *this;
    for (Index i = 0; i < size(); ++i) m.a_[i] *= o.a_[i];
    return m;
  }
  MatrixXd cwiseQuotient(const MatrixXd& o) const {
    MatrixXd m = *this;
    for (Index i = 0; i < size(); ++i) m.a_[i] /= o.a_[i];
    return m;
  }

  MatrixXd& operator+=(const MatrixXd& o) {
    for (Index i = 0; i < size(); ++i) a_[i] += o.a_[i];
    return *this;
  }
  MatrixXd& operator-=(const MatrixXd& o) {
    for (Index i = 0; i < size(); ++i) a_[i] -= o.a_[i];
    return *this;
  }
  MatrixXd& operator*=(double s) {
    for (double& v : a_) v *= s;
    return *this;
  }
  MatrixXd& operator/=(double s) {
    for (double& v : a_) v /= s;
    return *this;
  }

  // decompositions and triangular views
  class ColPivQR colPivHouseholderQr() const;
  template <int Mode>
  class TriView triangularView() const;

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> a_;
};

using VectorXd = MatrixXd;
using RowVectorXd = MatrixXd;

// ---------------------------------------------------------------- strided writable view
class Block {
 public:
  Block(double* base, Index r, Index c, Index ld, Index rs = 1) : p_(base), r_(r), c_(c), ld_(ld), rs_(rs) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double& operator()(Index i, Index j) const { return p_[j * ld_ + i * rs_]; }
  double& operator()(Index i) const {
    return c_ == 1 ? p_[i * rs_] : (r_ == 1 ? p_[i * ld_] : p_[(i / r_) * ld_ + (i % r_) * rs_]);
  }
  class CommaInit operator<<(double v);

  Block& operator=(const MatrixXd& m) {
    if (m.size() != size()) shim::fail("block assignment: size mismatch");
    const bool vec = (r_ == 1 || c_ == 1) && (m.rows() == 1 || m.cols() == 1);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) = vec ? m(j * r_ + i) : m(i, j);
    return *this;
  }
  Block& operator=(const Block& b) { return *this = MatrixXd(b); }
  Block& noalias() { return *this; }
  Block& operator+=(const MatrixXd& m);
  Block& operator-=(const MatrixXd& m);
  Block& operator*=(double s) {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) *= s;
    return *this;
  }
  Block& operator/=(double s) {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) (*this)(i, j) /= s;
    return *this;
  }
  void setZero() { *this *= 0.0; }

  Block block(Index i, Index j, Index r, Index c) const { return Block(&(*this)(i, j), r, c, ld_, rs_); }
  Block segment(Index i, Index n) const { return c_ == 1 ? block(i, 0, n, 1) : block(0, i, 1, n); }
  Block head(Index n) const { return segment(0, n); }
  Block tail(Index n) const { return segment(size() - n, n); }
  Block col(Index j) const { return block(0, j, r_, 1); }
  Block row(Index i) const { return block(i, 0, 1, c_); }
  Block leftCols(Index n) const { return block(0, 0, r_, n); }
  Block rightCols(Index n) const { return block(0, c_ - n, r_, n); }
  Block topLeftCorner(Index r, Index c) const { return block(0, 0, r, c); }

  MatrixXd eval() const { return MatrixXd(*this); }
  MatrixXd transpose() const { return MatrixXd(*this).transpose(); }
  double dot(const MatrixXd& o) const { return MatrixXd(*this).dot(o); }
  double norm() const { return MatrixXd(*this).norm(); }
  double squaredNorm() const { return MatrixXd(*this).squaredNorm(); }
  double sum() const { return MatrixXd(*this).sum(); }
  double maxCoeff() const { return MatrixXd(*this).maxCoeff(); }
  double minCoeff() const { return MatrixXd(*this).minCoeff(); }
  bool allFinite() const { return MatrixXd(*this).allFinite(); }
  MatrixXd cwiseAbs() const { return MatrixXd(*this).cwiseAbs(); }
  MatrixXd cwiseInverse() const { return MatrixXd(*this).cwiseInverse(); }
  MatrixXd cwiseProduct(const MatrixXd& o) const { return MatrixXd(*this).cwiseProduct(o); }
  template <int Mode>
  class TriView triangularView() const;
  ArrayRef array() const;

 private:
  double* p_;
  Index r_, c_, ld_, rs_;
};

inline MatrixXd::MatrixXd(const Block& b) : r_(b.rows()), c_(b.cols()), a_(static_cast<size_t>(b.size())) {
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) (*this)(i, j) = b(i, j);
}
inline MatrixXd& MatrixXd::operator=(const Block& b) { return *this = MatrixXd(b); }

inline Block MatrixXd::block(Index i, Index j, Index r, Index c) const {
  if (i < 0 || j < 0 || i + r > r_ || j + c > c_) shim::fail("block out of range");
  return Block(const_cast<double*>(a_.data()) + j * r_ + i, r, c, r_);
}
inline Block MatrixXd::col(Index j) const { return block(0, j, r_, 1); }
inline Block MatrixXd::row(Index i) const { return block(i, 0, 1, c_); }
inline Block MatrixXd::segment(Index i, Index n) const { return c_ == 1 ? block(i, 0, n, 1) : block(0, i, 1, n); }
inline Block MatrixXd::head(Index n) const { return segment(0, n); }
inline Block MatrixXd::tail(Index n) const { return segment(size() - n, n); }
inline Block MatrixXd::topRows(Index n) const { return block(0, 0, n, c_); }
inline Block MatrixXd::bottomRows(Index n) const { return block(r_ - n, 0, n, c_); }
inline Block MatrixXd::leftCols(Index n) const { return block(0, 0, r_, n); }
inline Block MatrixXd::rightCols(Index n) const { return block(0, c_ - n, r_, n); }
inline Block MatrixXd::topLeftCorner(Index r, Index c) const { return block(0, 0, r, c); }
inline Block MatrixXd::diagonal() const {
  return Block(const_cast<double*>(a_.data()), std::min(r_, c_), 1, r_, r_ + 1);
}

// comma initializer (M << a, b, ...): row after row, as Eigen fills
class CommaInit {
 public:
  CommaInit(MatrixXd* m, Block* b, double v) : m_(m), b_(b) { put(v); }
  CommaInit& operator,(double v) {
    put(v);
    return *this;
  }

 private:
  void put(double v) {
    const Index r = m_ ? m_->rows() : b_->rows(), c = m_ ? m_->cols() : b_->cols();
    if (k_ >= r * c) shim::fail("comma initializer: too many coefficients");
    const Index i = k_ / c, j = k_ % c;
    if (m_) (*m_)(i, j) = v;
    else (*b_)(i, j) = v;
    ++k_;
  }
  MatrixXd* m_;
  Block* b_;
  Index k_ = 0;
};
inline CommaInit MatrixXd::operator<<(double v) { return CommaInit(this, nullptr, v); }
inline CommaInit Block::operator<<(double v) { return CommaInit(nullptr, this, v); }

// ---------------------------------------------------------------- arithmetic (eager)
inline MatrixXd operator+(const MatrixXd& a, const MatrixXd& b) {
  if (a.size() != b.size()) shim::fail("+: size mismatch");
  MatrixXd m = a;
  m += b;
  return m;
}
inline MatrixXd operator-(const MatrixXd& a, const MatrixXd& b) {
  if (a.size() != b.size()) shim::fail("-: size mismatch");
  MatrixXd m = a;
  m -= b;
  return m;
}
inline MatrixXd operator-(const MatrixXd& a) { return a.unaryExpr([](double v) { return -v; }); }
inline MatrixXd operator*(const MatrixXd& a, double s) { return a.unaryExpr([s](double v) { return v * s; }); }
inline MatrixXd operator*(double s, const MatrixXd& a) { return a.unaryExpr([s](double v) { return s * v; }); }
inline MatrixXd operator/(const MatrixXd& a, double s) { return a.unaryExpr([s](double v) { return v / s; }); }
// matrix product: c(i,j) = Σ_k a(i,k) b(k,j), k ascending
inline MatrixXd operator*(const MatrixXd& a, const MatrixXd& b) {
  if (a.cols() != b.rows()) shim::fail("*: inner dimensions differ");
  MatrixXd c(a.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index k = 0; k < a.cols(); ++k) {
      const double bk = b(k, j);
      for (Index i = 0; i < a.rows(); ++i) c(i, j) += a(i, k) * bk;
    }
  return c;
}
// Block operands convert to MatrixXd
inline MatrixXd operator+(const Block& a, const MatrixXd& b) { return MatrixXd(a) + b; }
inline MatrixXd operator-(const Block& a, const MatrixXd& b) { return MatrixXd(a) - b; }
inline MatrixXd operator-(const Block& a) { return -MatrixXd(a); }
inline MatrixXd operator*(const Block& a, double s) { return MatrixXd(a) * s; }
inline MatrixXd operator*(double s, const Block& a) { return s * MatrixXd(a); }
inline MatrixXd operator/(const Block& a, double s) { return MatrixXd(a) / s; }
inline MatrixXd operator*(const Block& a, const MatrixXd& b) { return MatrixXd(a) * b; }
inline MatrixXd operator*(const MatrixXd& a, const Block& b) { return a * MatrixXd(b); }
inline MatrixXd operator*(const Block& a, const Block& b) { return MatrixXd(a) * MatrixXd(b); }

inline Block& Block::operator+=(const MatrixXd& m) { return *this = MatrixXd(*this) + m; }
inline Block& Block::operator-=(const MatrixXd& m) { return *this = MatrixXd(*this) - m; }

// ---------------------------------------------------------------- array view (coefficient-wise)
class ArrayRef {
 public:
  explicit ArrayRef(MatrixXd m) : m_(std::move(m)) {}
  ArrayRef(MatrixXd* target, MatrixXd m) : m_(std::move(m)), tgt_(target) {}
  ArrayRef operator-(double s) const { return ArrayRef(m_.unaryExpr([s](double v) { return v - s; })); }
  ArrayRef operator+(double s) const { return ArrayRef(m_.unaryExpr([s](double v) { return v + s; })); }
  ArrayRef operator*(const ArrayRef& o) const { return ArrayRef(m_.cwiseProduct(o.m_)); }
  ArrayRef operator/(const ArrayRef& o) const { return ArrayRef(m_.cwiseQuotient(o.m_)); }
  ArrayRef operator-(const ArrayRef& o) const { return ArrayRef(m_ - o.m_); }
  ArrayRef square() const { return ArrayRef(m_.unaryExpr([](double v) { return v * v; })); }
  ArrayRef abs() const { return ArrayRef(m_.cwiseAbs()); }
  ArrayRef sqrt() const { return ArrayRef(m_.cwiseSqrt()); }
  double sum() const { return m_.sum(); }
  double mean() const { return m_.mean(); }
  double maxCoeff() const { return m_.maxCoeff(); }
  MatrixXd matrix() const { return m_; }
  // W.array().colwise() /= s.array(): every column divided coefficient-wise by s
  struct Colwise {
    MatrixXd* tgt;
    void operator/=(const ArrayRef& s) const {
      for (Index j = 0; j < tgt->cols(); ++j)
        for (Index i = 0; i < tgt->rows(); ++i) (*tgt)(i, j) /= s.m_(i);
    }
    void operator*=(const ArrayRef& s) const {
      for (Index j = 0; j < tgt->cols(); ++j)
        for (Index i = 0; i < tgt->rows(); ++i) (*tgt)(i, j) *= s.m_(i);
    }
  };
  Colwise colwise() const {
    if (!tgt_) shim::fail("colwise on a temporary");
    return Colwise{tgt_};
  }

 private:
  MatrixXd m_;
  MatrixXd* tgt_ = nullptr;
};
inline ArrayRef MatrixXd::array() const { return ArrayRef(const_cast<MatrixXd*>(this), *this); }
inline ArrayRef Block::array() const { return ArrayRef(MatrixXd(*this)); }

// ---------------------------------------------------------------- triangular solve
class TriView {
 public:
  TriView(MatrixXd m, int mode) : m_(std::move(m)), mode_(mode) {}
  MatrixXd solve(const MatrixXd& b) const {
    const Index n = m_.rows();
    MatrixXd x = b;
    if (mode_ == Upper) {
      for (Index i = n - 1; i >= 0; --i) {
        double s = x(i);
        for (Index k = i + 1; k < n; ++k) s -= m_(i, k) * x(k);
        x(i) = s / m_(i, i);
      }
    } else {
      for (Index i = 0; i < n; ++i) {
        double s = x(i);
        for (Index k = 0; k < i; ++k) s -= m_(i, k) * x(k);
        x(i) = s / m_(i, i);
      }
    }
    return x;
  }

 private:
  MatrixXd m_;
  int mode_;
};
template <int Mode>
TriView MatrixXd::triangularView() const { return TriView(*this, Mode); }
template <int Mode>
TriView Block::triangularView() const { return TriView(MatrixXd(*this), Mode); }

// ---------------------------------------------------------------- decompositions (LAPACK)
namespace shim {
using gesvj_t = void (*)(const char*, const char*, const char*, const int*, const int*, double*, const int*, double*,
                         const int*, double*, const int*, double*, const int*, int*, size_t, size_t, size_t);
using geqp3_t = void (*)(const int*, const int*, double*, const int*, int*, double*, double*, const int*, int*);
using ormqr_t = void (*)(const char*, const char*, const int*, const int*, const int*, const double*, const int*,
                         const double*, double*, const int*, double*, const int*, int*, size_t, size_t);
using syevd_t = void (*)(const char*, const char*, const int*, double*, const int*, double*, double*, const int*,
                         int*, const int*, int*, size_t, size_t);
using gesvd_t = void (*)(const char*, const char*, const int*, const int*, double*, const int*, double*, double*,
                         const int*, double*, const int*, double*, const int*, int*, size_t, size_t);
using geev_t = void (*)(const char*, const char*, const int*, double*, const int*, double*, double*, double*,
                        const int*, double*, const int*, double*, const int*, int*, size_t, size_t);

struct PivotedQR {
  MatrixXd qr;
  std::vector<int> jpvt;  // 1-based, LAPACK
  std::vector<double> tau;
};
inline PivotedQR geqp3(const MatrixXd& A) {
  PivotedQR f{A, std::vector<int>(static_cast<size_t>(A.cols()), 0), std::vector<double>(static_cast<size_t>(std::min(A.rows(), A.cols())) + 1)};
  auto fn = reinterpret_cast<geqp3_t>(lapack().sym("scipy_dgeqp3_"));
  const int m = static_cast<int>(A.rows()), n = static_cast<int>(A.cols()), lda = std::max(1, m);
  int info = 0, lw = -1;
  double wq = 0.0;
  fn(&m, &n, f.qr.data(), &lda, f.jpvt.data(), f.tau.data(), &wq, &lw, &info);
  lw = std::max(1, static_cast<int>(wq));
  std::vector<double> w(static_cast<size_t>(lw));
  fn(&m, &n, f.qr.data(), &lda, f.jpvt.data(), f.tau.data(), w.data(), &lw, &info);
  if (info < 0) fail("dgeqp3");
  return f;
}
}  // namespace shim

template <class MatrixType>
class JacobiSVD {
 public:
  JacobiSVD(const MatrixXd& A, unsigned opts = 0) { compute(A, opts); }
  const MatrixXd& singularValues() const { return sv_; }
  const MatrixXd& matrixV() const { return V_; }
  ComputationInfo info() const { return Success; }

 private:
  void compute(const MatrixXd& A, unsigned) {
    // square or tall: QR-preconditioned (Eigen's default ColPivHouseholderQRPreconditioner);
    // wide: work on the transpose, whose left vectors are A's right vectors
    const Index M = A.rows(), N = A.cols();
    auto gesvj = reinterpret_cast<shim::gesvj_t>(shim::lapack().sym("scipy_dgesvj_"));
    if (M >= N) {
      shim::PivotedQR f = shim::geqp3(A);
      const int n = static_cast<int>(N);
      MatrixXd R(N, N), VR(N, N);
      for (Index c = 0; c < N; ++c)
        for (Index r = 0; r <= c; ++r) R(r, c) = f.qr(r, c);
      MatrixXd s(N);
      int lw = std::max(6, 2 * n), info = 0, mv = 0, ld = std::max(1, n);
      std::vector<double> w(static_cast<size_t>(lw));
      gesvj("U", "N", "V", &n, &n, R.data(), &ld, s.data(), &mv, VR.data(), &ld, w.data(), &lw, &info, 1, 1, 1);
      if (info < 0) shim::fail("dgesvj");
      for (Index i = 0; i < N; ++i) s(i) *= w[0];
      MatrixXd V(N, N);
      for (Index c = 0; c < N; ++c)
        for (Index r = 0; r < N; ++r) V(f.jpvt[r] - 1, c) = VR(r, c);
      sort_(s, V);
    } else {
      MatrixXd T = A.transpose();  // N x M, tall
      const int m2 = static_cast<int>(N), n2 = static_cast<int>(M);
      MatrixXd s(M), dummy(1, 1);
      int lw = std::max(6, m2 + n2), info = 0, mv = 0, ldv = 1, lda = std::max(1, m2);
      std::vector<double> w(static_cast<size_t>(lw));
      gesvj("G", "U", "N", &m2, &n2, T.data(), &lda, s.data(), &mv, dummy.data(), &ldv, w.data(), &lw, &info, 1, 1,
            1);
      if (info < 0) shim::fail("dgesvj");
      for (Index i = 0; i < M; ++i) s(i) *= w[0];
      sort_(s, T);
    }
  }
  void sort_(const MatrixXd& s, const MatrixXd& V) {
    const Index k = s.size();
    std::vector<Index> ord(static_cast<size_t>(k));
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](Index a, Index b) { return s(a) > s(b); });
    sv_ = MatrixXd(k);
    V_ = MatrixXd(V.rows(), k);
    for (Index i = 0; i < k; ++i) {
      sv_(i) = s(ord[i]);
      for (Index r = 0; r < V.rows(); ++r) V_(r, i) = V(r, ord[i]);
    }
  }
  MatrixXd sv_, V_;
};

template <class MatrixType>
class SelfAdjointEigenSolver {
 public:
  SelfAdjointEigenSolver() = default;
  explicit SelfAdjointEigenSolver(const MatrixXd& A, int opts = ComputeEigenvectors) { compute(A, opts); }
  SelfAdjointEigenSolver& compute(const MatrixXd& A, int opts = ComputeEigenvectors) {
    auto syevd = reinterpret_cast<shim::syevd_t>(shim::lapack().sym("scipy_dsyevd_"));
    const int n = static_cast<int>(A.rows()), lda = std::max(1, n);
    V_ = A;
    ev_ = MatrixXd(n);
    const char* jobz = (opts & EigenvaluesOnly) ? "N" : "V";
    int info = 0, lw = -1, liw = -1, iwq = 0;
    double wq = 0.0;
    syevd(jobz, "L", &n, V_.data(), &lda, ev_.data(), &wq, &lw, &iwq, &liw, &info, 1, 1);
    lw = std::max(1, static_cast<int>(wq));
    liw = std::max(1, iwq);
    std::vector<double> w(static_cast<size_t>(lw));
    std::vector<int> iw(static_cast<size_t>(liw));
    syevd(jobz, "L", &n, V_.data(), &lda, ev_.data(), w.data(), &lw, iw.data(), &liw, &info, 1, 1);
    info_ = info == 0 ? Success : NoConvergence;
    return *this;
  }
  const MatrixXd& eigenvalues() const { return ev_; }
  const MatrixXd& eigenvectors() const { return V_; }
  ComputationInfo info() const { return info_; }

 private:
  MatrixXd V_, ev_;
  ComputationInfo info_ = Success;
};

class ColPivQR {
 public:
  explicit ColPivQR(const MatrixXd& A) : f_(shim::geqp3(A)), m_(A.rows()), n_(A.cols()) {
    // Eigen's default threshold: |R_ii| > ε·diagSize·max|R_ii| counts toward the rank
    const Index d = std::min(m_, n_);
    double maxp = 0.0;
    for (Index i = 0; i < d; ++i) maxp = std::max(maxp, std::abs(f_.qr(i, i)));
    const double thr = std::numeric_limits<double>::epsilon() * static_cast<double>(d) * maxp;
    rank_ = 0;
    for (Index i = 0; i < d; ++i)
      if (std::abs(f_.qr(i, i)) > thr) ++rank_;
  }
  Index rank() const { return rank_; }
  MatrixXd solve(const MatrixXd& b) const {
    auto ormqr = reinterpret_cast<shim::ormqr_t>(shim::lapack().sym("scipy_dormqr_"));
    const int m = static_cast<int>(m_), k = static_cast<int>(std::min(m_, n_)), lda = std::max(1, m);
    const int nrhs = static_cast<int>(b.cols());
    MatrixXd c = b;
    int info = 0, lw = -1;
    double wq = 0.0;
    ormqr("L", "T", &m, &nrhs, &k, f_.qr.data(), &lda, f_.tau.data(), c.data(), &lda, &wq, &lw, &info, 1, 1);
    lw = std::max(1, static_cast<int>(wq));
    std::vector<double> w(static_cast<size_t>(lw));
    ormqr("L", "T", &m, &nrhs, &k, f_.qr.data(), &lda, f_.tau.data(), c.data(), &lda, w.data(), &lw, &info, 1, 1);
    MatrixXd x(n_, b.cols());
    for (Index col = 0; col < b.cols(); ++col) {
      std::vector<double> z(static_cast<size_t>(n_), 0.0);
      for (Index i = rank_ - 1; i >= 0; --i) {
        double s = c(i, col);
        for (Index q = i + 1; q < rank_; ++q) s -= f_.qr(i, q) * z[q];
        z[i] = s / f_.qr(i, i);
      }
      for (Index i = 0; i < n_; ++i) x(f_.jpvt[i] - 1, col) = z[i];
    }
    return x;
  }

 private:
  shim::PivotedQR f_;
  Index m_, n_, rank_ = 0;
};
template <class MatrixType>
using ColPivHouseholderQR = ColPivQR;
inline ColPivQR MatrixXd::colPivHouseholderQr() const { return ColPivQR(*this); }
// ldlt().solve (used by the reference's tests on small SPD systems): a column-pivoted QR solve
class LdltSolve {
 public:
  explicit LdltSolve(const MatrixXd& A) : qr_(A) {}
  MatrixXd solve(const MatrixXd& b) const { return qr_.solve(b); }

 private:
  ColPivQR qr_;
};
inline LdltSolve MatrixXd::ldlt() const { return LdltSolve(*this); }

template <int Size>
class PermutationMatrix {
 public:
  explicit PermutationMatrix(Index n) : idx_(std::vector<int>(static_cast<size_t>(n), 0)) {}
  void setIdentity() {
    for (size_t i = 0; i < idx_.v.size(); ++i) idx_.v[i] = static_cast<int>(i);
  }
  struct Indices {
    std::vector<int> v;
    int& operator()(Index i) { return v[static_cast<size_t>(i)]; }
    int operator()(Index i) const { return v[static_cast<size_t>(i)]; }
  };
  Indices& indices() { return idx_; }
  const Indices& indices() const { return idx_; }
  // (P A).row(indices(i)) = A.row(i)
  friend MatrixXd operator*(const PermutationMatrix& P, const MatrixXd& A) {
    MatrixXd out(A.rows(), A.cols());
    for (Index i = 0; i < A.rows(); ++i)
      for (Index j = 0; j < A.cols(); ++j) out(P.idx_(i), j) = A(i, j);
    return out;
  }

 private:
  Indices idx_;
};

class VectorXcd {
 public:
  explicit VectorXcd(Index n = 0) : a_(static_cast<size_t>(n)) {}
  Index size() const { return static_cast<Index>(a_.size()); }
  std::complex<double>& operator()(Index i) { return a_[i]; }
  const std::complex<double>& operator()(Index i) const { return a_[i]; }

 private:
  std::vector<std::complex<double>> a_;
};

template <class MatrixType>
class EigenSolver {
 public:
  EigenSolver(const MatrixXd& A, bool /*computeEigenvectors*/ = true) : ev_(A.rows()) {
    auto geev = reinterpret_cast<shim::geev_t>(shim::lapack().sym("scipy_dgeev_"));
    const int n = static_cast<int>(A.rows()), lda = std::max(1, n), one = 1;
    MatrixXd a = A;
    std::vector<double> wr(static_cast<size_t>(n)), wi(static_cast<size_t>(n));
    double dummy = 0.0, wq = 0.0;
    int info = 0, lw = -1;
    geev("N", "N", &n, a.data(), &lda, wr.data(), wi.data(), &dummy, &one, &dummy, &one, &wq, &lw, &info, 1, 1);
    lw = std::max(1, static_cast<int>(wq));
    std::vector<double> w(static_cast<size_t>(lw));
    geev("N", "N", &n, a.data(), &lda, wr.data(), wi.data(), &dummy, &one, &dummy, &one, w.data(), &lw, &info, 1, 1);
    for (Index i = 0; i < n; ++i) ev_(i) = {wr[i], wi[i]};
  }
  const VectorXcd& eigenvalues() const { return ev_; }

 private:
  VectorXcd ev_;
};

template <class MatrixType>
class BDCSVD {
 public:
  explicit BDCSVD(const MatrixXd& A, unsigned = 0) {
    auto gesvd = reinterpret_cast<shim::gesvd_t>(shim::lapack().sym("scipy_dgesvd_"));
    const int m = static_cast<int>(A.rows()), n = static_cast<int>(A.cols()), lda = std::max(1, m), one = 1;
    MatrixXd a = A;
    sv_ = MatrixXd(std::min(m, n));
    double dummy = 0.0, wq = 0.0;
    int info = 0, lw = -1;
    gesvd("N", "N", &m, &n, a.data(), &lda, sv_.data(), &dummy, &one, &dummy, &one, &wq, &lw, &info, 1, 1);
    lw = std::max(1, static_cast<int>(wq));
    std::vector<double> w(static_cast<size_t>(lw));
    gesvd("N", "N", &m, &n, a.data(), &lda, sv_.data(), &dummy, &one, &dummy, &one, w.data(), &lw, &info, 1, 1);
  }
  const MatrixXd& singularValues() const { return sv_; }

 private:
  MatrixXd sv_;
};

}  // namespace Eigen
