// Minimal Eigen-API shim: just enough of Eigen 3's dense interface for the
// reference library's own sources (/root/reference/proj/src/*.cpp) to compile
// UNCHANGED, with the arithmetic delegated to LAPACK/BLAS.
//
// TEST INFRASTRUCTURE ONLY (oracle/_ref).  It exists because Eigen3 is not
// installed in this image and the reference cannot be built
// against the real thing.  It is our own code, written against Eigen's public
// API as the reference uses it; it is not Eigen.
//
// What the reference needs (grep of proj/src + proj/include):
//   * MatrixXd / VectorXd (column-major, dynamic), Map<const MatrixXd>,
//     Map<MatrixXd>, Ref<const MatrixXd>                 dense_tensor.hpp:14-16
//   * blocks: col/row/leftCols/rightCols/middleCols/topRows/topLeftCorner/head,
//     writable when the owner is                          tt_ice.cpp:113-118
//   * products, +, -, unary -, transpose, asDiagonal      tt_ice.cpp:40,100
//   * norm/squaredNorm/cwiseAbs/maxCoeff(&i)/allFinite   truncated_svd.cpp:16-30
//   * Identity/Zero, triangularView<Upper>                truncated_svd.cpp:53-55
//   * HouseholderQR (matrixQR, householderQ, applyOnTheLeft)
//                                                         truncated_svd.cpp:53, update_common.hpp:30
//   * BDCSVD (ComputeThinU|ComputeThinV, info, singularValues, matrixU/V)
//                                                         truncated_svd.cpp:61
//
// Arithmetic mapping (all through numpy's bundled ILP64 OpenBLAS, the same
// library the numpy oracle uses):
//   GEMM            -> cblas_dgemm
//   HouseholderQR   -> dgeqrf (reflectors with Eigen's convention:
//                      beta = -sign(x0)|x|, tau = 0 for a zero tail)
//   householderQ()  -> dormqr applied on the left
//   BDCSVD          -> dgesdd (divide and conquer, JOBZ='S').  Singular
//                      values/vectors agree with Eigen's BDCSVD to rounding;
//                      the reference's own sign rule (truncated_svd.cpp:16-25)
//                      then fixes the column signs.
//   norms/reductions-> plain loops (Eigen's vectorised reduction order differs
//                      at rounding level only).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <limits>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

using Index = std::ptrdiff_t;
constexpr int Dynamic = -1;

enum UpLoType { Lower = 0x1, Upper = 0x2 };
enum DecompositionOptions {
  ComputeFullU = 0x04,
  ComputeThinU = 0x08,
  ComputeFullV = 0x10,
  ComputeThinV = 0x20
};
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

namespace shim {
extern "C" {
// ILP64 OpenBLAS as bundled with numpy (symbol suffix 64_).
void scipy_cblas_dgemm64_(int order, int ta, int tb, long long m, long long n, long long k, double alpha,
                          const double* a, long long lda, const double* b, long long ldb, double beta, double* c,
                          long long ldc);
void scipy_dgeqrf_64_(const long long* m, const long long* n, double* a, const long long* lda, double* tau,
                      double* work, const long long* lwork, long long* info);
void scipy_dormqr_64_(const char* side, const char* trans, const long long* m, const long long* n,
                      const long long* k, const double* a, const long long* lda, const double* tau, double* c,
                      const long long* ldc, double* work, const long long* lwork, long long* info, std::size_t,
                      std::size_t);
void scipy_dgesdd_64_(const char* jobz, const long long* m, const long long* n, double* a, const long long* lda,
                      double* s, double* u, const long long* ldu, double* vt, const long long* ldvt, double* work,
                      const long long* lwork, long long* iwork, long long* info, std::size_t);
}
constexpr int kColMajor = 102, kNoTrans = 111, kTrans = 112;
}  // namespace shim

class MatrixXd;
class VectorXd;
template <class T>
class Block;
class DiagonalWrapper;
class Transposed;

// Read-only column-major view: element (i, j) at p_[i + j * ld_].  Every
// matrix-like type of the shim (owning matrices, maps, blocks, refs) is one.
class ConstBase {
 protected:
  const double* p_ = nullptr;
  Index r_ = 0, c_ = 0, ld_ = 1;
  ConstBase() = default;
  ConstBase(const double* p, Index r, Index c, Index ld) : p_(p), r_(r), c_(c), ld_(ld < 1 ? 1 : ld) {}
  void set_view(const double* p, Index r, Index c, Index ld) {
    p_ = p;
    r_ = r;
    c_ = c;
    ld_ = ld < 1 ? 1 : ld;
  }

 public:
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  Index outerStride() const { return ld_; }
  const double* data() const { return p_; }
  double operator()(Index i, Index j) const { return p_[i + j * ld_]; }
  // Linear access for vectors (one row or one column).
  double operator()(Index i) const { return c_ == 1 ? p_[i] : p_[i * ld_]; }
  double coeff(Index i, Index j) const { return (*this)(i, j); }

  Block<const double> block(Index i, Index j, Index r, Index c) const;
  Block<const double> col(Index j) const;
  Block<const double> row(Index i) const;
  Block<const double> leftCols(Index n) const;
  Block<const double> rightCols(Index n) const;
  Block<const double> middleCols(Index j, Index n) const;
  Block<const double> topRows(Index n) const;
  Block<const double> bottomRows(Index n) const;
  Block<const double> topLeftCorner(Index r, Index c) const;
  Block<const double> head(Index n) const;

  Transposed transpose() const;
  MatrixXd cwiseAbs() const;
  MatrixXd eval() const;
  DiagonalWrapper asDiagonal() const;
  template <int Mode>
  MatrixXd triangularView() const;

  double squaredNorm() const {
    double s = 0.0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) {
        const double v = p_[i + j * ld_];
        s += v * v;
      }
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double sum() const {
    double s = 0.0;
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) s += p_[i + j * ld_];
    return s;
  }
  bool allFinite() const {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i)
        if (!std::isfinite(p_[i + j * ld_])) return false;
    return true;
  }
  double maxCoeff() const {
    double m = -std::numeric_limits<double>::infinity();
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) m = std::max(m, p_[i + j * ld_]);
    return m;
  }
  double minCoeff() const {
    double m = std::numeric_limits<double>::infinity();
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) m = std::min(m, p_[i + j * ld_]);
    return m;
  }
  // Vector form: index of the FIRST maximum (Eigen's visitor keeps the first).
  template <class I>
  double maxCoeff(I* index) const {
    const Index n = size();
    Index best = 0;
    double m = n > 0 ? (*this)(0) : 0.0;
    for (Index k = 1; k < n; ++k) {
      const double v = (*this)(k);
      if (v > m) {
        m = v;
        best = k;
      }
    }
    *index = static_cast<I>(best);
    return m;
  }
};

// Writable view.
class MutBase : public ConstBase {
 protected:
  MutBase() = default;
  MutBase(double* p, Index r, Index c, Index ld) : ConstBase(p, r, c, ld) {}
  double* mp() const { return const_cast<double*>(p_); }
  void assign_from(const ConstBase& o) {
    if (o.rows() != r_ || o.cols() != c_) throw std::logic_error("Eigen shim: block assignment size mismatch");
    // Copy through a temporary when source and destination could overlap.
    std::vector<double> tmp(static_cast<std::size_t>(size()));
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) tmp[static_cast<std::size_t>(i + j * r_)] = o(i, j);
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) mp()[i + j * ld_] = tmp[static_cast<std::size_t>(i + j * r_)];
  }

 public:
  using ConstBase::operator();
  double* data() const { return mp(); }
  double& operator()(Index i, Index j) { return mp()[i + j * ld_]; }
  double& operator()(Index i) { return c_ == 1 ? mp()[i] : mp()[i * ld_]; }
  using ConstBase::block;
  using ConstBase::col;
  using ConstBase::head;
  using ConstBase::leftCols;
  using ConstBase::middleCols;
  using ConstBase::rightCols;
  using ConstBase::row;
  using ConstBase::topLeftCorner;
  using ConstBase::topRows;
  using ConstBase::bottomRows;
  Block<double> block(Index i, Index j, Index r, Index c);
  Block<double> col(Index j);
  Block<double> row(Index i);
  Block<double> leftCols(Index n);
  Block<double> rightCols(Index n);
  Block<double> middleCols(Index j, Index n);
  Block<double> topRows(Index n);
  Block<double> bottomRows(Index n);
  Block<double> topLeftCorner(Index r, Index c);
  Block<double> head(Index n);
  void setZero() {
    for (Index j = 0; j < c_; ++j)
      for (Index i = 0; i < r_; ++i) mp()[i + j * ld_] = 0.0;
  }
};

template <>
class Block<const double> : public ConstBase {
 public:
  Block(const double* p, Index r, Index c, Index ld) : ConstBase(p, r, c, ld) {}
};

template <>
class Block<double> : public MutBase {
 public:
  Block(double* p, Index r, Index c, Index ld) : MutBase(p, r, c, ld) {}
  Block& operator=(const Block& o) {
    assign_from(o);
    return *this;
  }
  Block& operator=(const ConstBase& o) {
    assign_from(o);
    return *this;
  }
  Block& operator=(const MatrixXd& o);
  Block& operator=(const Transposed& o);
};

class HouseholderSequence;

class MatrixXd : public MutBase {
 protected:
  std::vector<double> v_;
  void bind() { set_view(v_.data(), r_, c_, r_); }
  void resize_keep_nothing(Index r, Index c) {
    v_.assign(static_cast<std::size_t>(r * c), 0.0);
    r_ = r;
    c_ = c;
    bind();
  }

 public:
  MatrixXd() { bind(); }
  MatrixXd(Index r, Index c) { resize_keep_nothing(r, c); }
  MatrixXd(const MatrixXd& o) : MutBase(), v_(o.v_) {
    r_ = o.r_;
    c_ = o.c_;
    bind();
  }
  MatrixXd(MatrixXd&& o) noexcept : MutBase(), v_(std::move(o.v_)) {
    r_ = o.r_;
    c_ = o.c_;
    bind();
    o.r_ = o.c_ = 0;
    o.bind();
  }
  MatrixXd(const ConstBase& o) { copy_from(o); }  // NOLINT: implicit like Eigen
  MatrixXd(const Transposed& t);                   // NOLINT
  MatrixXd& operator=(const MatrixXd& o) {
    if (this != &o) {
      v_ = o.v_;
      r_ = o.r_;
      c_ = o.c_;
      bind();
    }
    return *this;
  }
  MatrixXd& operator=(MatrixXd&& o) noexcept {
    if (this != &o) {
      v_ = std::move(o.v_);
      r_ = o.r_;
      c_ = o.c_;
      bind();
      o.r_ = o.c_ = 0;
      o.bind();
    }
    return *this;
  }
  MatrixXd& operator=(const ConstBase& o) {
    copy_from(o);
    return *this;
  }
  MatrixXd& operator=(const Transposed& t);

  void copy_from(const ConstBase& o) {
    std::vector<double> nv(static_cast<std::size_t>(o.rows() * o.cols()));
    for (Index j = 0; j < o.cols(); ++j)
      for (Index i = 0; i < o.rows(); ++i) nv[static_cast<std::size_t>(i + j * o.rows())] = o(i, j);
    const Index r = o.rows(), c = o.cols();
    v_ = std::move(nv);
    r_ = r;
    c_ = c;
    bind();
  }
  void resize(Index r, Index c) {
    if (r * c != r_ * c_) v_.resize(static_cast<std::size_t>(r * c));
    r_ = r;
    c_ = c;
    bind();
  }

  static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
  static MatrixXd Identity(Index r, Index c) {
    MatrixXd m(r, c);
    for (Index k = 0; k < std::min(r, c); ++k) m(k, k) = 1.0;
    return m;
  }

  void applyOnTheLeft(const HouseholderSequence& h);
};

class VectorXd : public MatrixXd {
 public:
  VectorXd() = default;
  explicit VectorXd(Index n) : MatrixXd(n, 1) {}
  VectorXd(const ConstBase& o) : MatrixXd(o) { flatten(); }  // NOLINT
  VectorXd& operator=(const ConstBase& o) {
    copy_from(o);
    flatten();
    return *this;
  }
  Index size() const { return r_ * c_; }

 private:
  void flatten() {
    r_ = r_ * c_;
    c_ = 1;
    bind();
  }
};

template <class T>
class Map;

template <>
class Map<const MatrixXd> : public ConstBase {
 public:
  Map(const double* p, Index r, Index c) : ConstBase(p, r, c, r) {}
};

template <>
class Map<MatrixXd> : public MutBase {
 public:
  Map(double* p, Index r, Index c) : MutBase(p, r, c, r) {}
  Map& operator=(const ConstBase& o) {
    assign_from(o);
    return *this;
  }
  Map& operator=(const Map& o) {
    assign_from(o);
    return *this;
  }
  Map& operator=(const MatrixXd& o) {
    assign_from(o);
    return *this;
  }
};

template <class T>
class Ref;

// Ref<const MatrixXd>: binds to any column-major view (never copies here:
// every shim type has unit inner stride).
template <>
class Ref<const MatrixXd> : public ConstBase {
 public:
  Ref(const ConstBase& o) : ConstBase(o.data(), o.rows(), o.cols(), o.outerStride()) {}  // NOLINT
};

// transpose(): a lazy transposed view, consumed by the products (BLAS trans
// flags) or materialised on assignment.
class Transposed {
 public:
  explicit Transposed(const ConstBase& m) : m_(m.data(), m.rows(), m.cols(), m.outerStride()) {}
  const Block<const double>& nested() const { return m_; }
  Index rows() const { return m_.cols(); }
  Index cols() const { return m_.rows(); }
  double operator()(Index i, Index j) const { return m_(j, i); }

 private:
  Block<const double> m_;
};

class DiagonalWrapper {
 public:
  explicit DiagonalWrapper(const ConstBase& v) : v_(v.data(), v.rows(), v.cols(), v.outerStride()) {}
  const Block<const double>& diag() const { return v_; }

 private:
  Block<const double> v_;
};

// ---- block accessors ----------------------------------------------------
inline Block<const double> ConstBase::block(Index i, Index j, Index r, Index c) const {
  return Block<const double>(p_ + i + j * ld_, r, c, ld_);
}
inline Block<const double> ConstBase::col(Index j) const { return block(0, j, r_, 1); }
inline Block<const double> ConstBase::row(Index i) const { return block(i, 0, 1, c_); }
inline Block<const double> ConstBase::leftCols(Index n) const { return block(0, 0, r_, n); }
inline Block<const double> ConstBase::rightCols(Index n) const { return block(0, c_ - n, r_, n); }
inline Block<const double> ConstBase::middleCols(Index j, Index n) const { return block(0, j, r_, n); }
inline Block<const double> ConstBase::topRows(Index n) const { return block(0, 0, n, c_); }
inline Block<const double> ConstBase::bottomRows(Index n) const { return block(r_ - n, 0, n, c_); }
inline Block<const double> ConstBase::topLeftCorner(Index r, Index c) const { return block(0, 0, r, c); }
inline Block<const double> ConstBase::head(Index n) const {
  return c_ == 1 ? block(0, 0, n, 1) : block(0, 0, 1, n);
}
inline Block<double> MutBase::block(Index i, Index j, Index r, Index c) {
  return Block<double>(mp() + i + j * ld_, r, c, ld_);
}
inline Block<double> MutBase::col(Index j) { return block(0, j, r_, 1); }
inline Block<double> MutBase::row(Index i) { return block(i, 0, 1, c_); }
inline Block<double> MutBase::leftCols(Index n) { return block(0, 0, r_, n); }
inline Block<double> MutBase::rightCols(Index n) { return block(0, c_ - n, r_, n); }
inline Block<double> MutBase::middleCols(Index j, Index n) { return block(0, j, r_, n); }
inline Block<double> MutBase::topRows(Index n) { return block(0, 0, n, c_); }
inline Block<double> MutBase::bottomRows(Index n) { return block(r_ - n, 0, n, c_); }
inline Block<double> MutBase::topLeftCorner(Index r, Index c) { return block(0, 0, r, c); }
inline Block<double> MutBase::head(Index n) { return c_ == 1 ? block(0, 0, n, 1) : block(0, 0, 1, n); }

inline Block<double>& Block<double>::operator=(const MatrixXd& o) {
  assign_from(o);
  return *this;
}
inline Block<double>& Block<double>::operator=(const Transposed& t) {
  assign_from(MatrixXd(t));
  return *this;
}

inline MatrixXd::MatrixXd(const Transposed& t) {
  const Index r = t.rows(), c = t.cols();
  resize_keep_nothing(r, c);
  for (Index j = 0; j < c; ++j)
    for (Index i = 0; i < r; ++i) v_[static_cast<std::size_t>(i + j * r)] = t(i, j);
}
inline MatrixXd& MatrixXd::operator=(const Transposed& t) {
  MatrixXd m(t);
  *this = std::move(m);
  return *this;
}

inline Transposed ConstBase::transpose() const { return Transposed(*this); }
inline MatrixXd ConstBase::eval() const { return MatrixXd(*this); }
inline MatrixXd ConstBase::cwiseAbs() const {
  MatrixXd m(r_, c_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i) m(i, j) = std::fabs((*this)(i, j));
  return m;
}
inline DiagonalWrapper ConstBase::asDiagonal() const { return DiagonalWrapper(*this); }
template <int Mode>
inline MatrixXd ConstBase::triangularView() const {
  static_assert(Mode == Upper || Mode == Lower, "Eigen shim: Upper/Lower only");
  MatrixXd m(r_, c_);
  for (Index j = 0; j < c_; ++j)
    for (Index i = 0; i < r_; ++i)
      if ((Mode == Upper && i <= j) || (Mode == Lower && i >= j)) m(i, j) = (*this)(i, j);
  return m;
}

// ---- products and elementwise arithmetic ----------------------------------
namespace shim {
inline MatrixXd gemm(const ConstBase& a, bool ta, const ConstBase& b, bool tb) {
  const Index m = ta ? a.cols() : a.rows();
  const Index k = ta ? a.rows() : a.cols();
  const Index kb = tb ? b.cols() : b.rows();
  const Index n = tb ? b.rows() : b.cols();
  if (k != kb) throw std::logic_error("Eigen shim: product size mismatch");
  MatrixXd c(m, n);
  if (m == 0 || n == 0 || k == 0) return c;
  scipy_cblas_dgemm64_(kColMajor, ta ? kTrans : kNoTrans, tb ? kTrans : kNoTrans, m, n, k, 1.0, a.data(),
                       a.outerStride(), b.data(), b.outerStride(), 0.0, c.data(), std::max<Index>(1, m));
  return c;
}
}  // namespace shim

inline MatrixXd operator*(const ConstBase& a, const ConstBase& b) { return shim::gemm(a, false, b, false); }
inline MatrixXd operator*(const Transposed& a, const ConstBase& b) {
  return shim::gemm(a.nested(), true, b, false);
}
inline MatrixXd operator*(const ConstBase& a, const Transposed& b) {
  return shim::gemm(a, false, b.nested(), true);
}
inline MatrixXd operator*(const Transposed& a, const Transposed& b) {
  return shim::gemm(a.nested(), true, b.nested(), true);
}
inline MatrixXd operator*(const DiagonalWrapper& d, const ConstBase& b) {
  const auto& v = d.diag();
  if (v.size() != b.rows()) throw std::logic_error("Eigen shim: diagonal product size mismatch");
  MatrixXd m(b.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < b.rows(); ++i) m(i, j) = v(i) * b(i, j);
  return m;
}
inline MatrixXd operator*(double s, const ConstBase& b) {
  MatrixXd m(b.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < b.rows(); ++i) m(i, j) = s * b(i, j);
  return m;
}
inline MatrixXd operator*(const ConstBase& b, double s) { return s * b; }
inline MatrixXd operator/(const ConstBase& b, double s) {
  MatrixXd m(b.rows(), b.cols());
  for (Index j = 0; j < b.cols(); ++j)
    for (Index i = 0; i < b.rows(); ++i) m(i, j) = b(i, j) / s;
  return m;
}
inline MatrixXd operator-(const ConstBase& a) { return -1.0 * a; }
inline MatrixXd operator-(const ConstBase& a, const ConstBase& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::logic_error("Eigen shim: difference size mismatch");
  MatrixXd m(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) m(i, j) = a(i, j) - b(i, j);
  return m;
}
inline MatrixXd operator+(const ConstBase& a, const ConstBase& b) {
  if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::logic_error("Eigen shim: sum size mismatch");
  MatrixXd m(a.rows(), a.cols());
  for (Index j = 0; j < a.cols(); ++j)
    for (Index i = 0; i < a.rows(); ++i) m(i, j) = a(i, j) + b(i, j);
  return m;
}

// ---- HouseholderQR ---------------------------------------------------------
class HouseholderSequence {
 public:
  HouseholderSequence(const MatrixXd* qr, const std::vector<double>* tau) : qr_(qr), tau_(tau) {}
  const MatrixXd& qr() const { return *qr_; }
  const std::vector<double>& tau() const { return *tau_; }

 private:
  const MatrixXd* qr_;
  const std::vector<double>* tau_;
};

template <class M>
class HouseholderQR {
 public:
  explicit HouseholderQR(const ConstBase& a) : qr_(a) {
    const long long m = qr_.rows(), n = qr_.cols(), lda = std::max<long long>(1, m);
    const long long k = std::min(m, n);
    tau_.assign(static_cast<std::size_t>(std::max<long long>(k, 1)), 0.0);
    if (k == 0) return;
    long long info = 0, lwork = -1;
    double wq = 0.0;
    shim::scipy_dgeqrf_64_(&m, &n, qr_.data(), &lda, tau_.data(), &wq, &lwork, &info);
    lwork = std::max<long long>(1, static_cast<long long>(wq));
    std::vector<double> work(static_cast<std::size_t>(lwork));
    shim::scipy_dgeqrf_64_(&m, &n, qr_.data(), &lda, tau_.data(), work.data(), &lwork, &info);
    if (info != 0) throw std::runtime_error("Eigen shim: dgeqrf failed");
  }
  const MatrixXd& matrixQR() const { return qr_; }
  HouseholderSequence householderQ() const { return HouseholderSequence(&qr_, &tau_); }

 private:
  MatrixXd qr_;
  std::vector<double> tau_;
};

// this <- H_0 H_1 ... H_{k-1} * this (Eigen: m.applyOnTheLeft(qr.householderQ())).
inline void MatrixXd::applyOnTheLeft(const HouseholderSequence& h) {
  const long long m = r_, n = c_;
  const long long k = std::min<long long>(h.qr().rows(), h.qr().cols());
  if (m != h.qr().rows()) throw std::logic_error("Eigen shim: householder size mismatch");
  if (k == 0 || n == 0 || m == 0) return;
  const long long lda = std::max<long long>(1, h.qr().rows()), ldc = std::max<long long>(1, m);
  long long info = 0, lwork = -1;
  double wq = 0.0;
  shim::scipy_dormqr_64_("L", "N", &m, &n, &k, h.qr().data(), &lda, h.tau().data(), data(), &ldc, &wq, &lwork,
                         &info, 1, 1);
  lwork = std::max<long long>(1, static_cast<long long>(wq));
  std::vector<double> work(static_cast<std::size_t>(lwork));
  shim::scipy_dormqr_64_("L", "N", &m, &n, &k, h.qr().data(), &lda, h.tau().data(), data(), &ldc, work.data(),
                         &lwork, &info, 1, 1);
  if (info != 0) throw std::runtime_error("Eigen shim: dormqr failed");
}

// ---- BDCSVD (thin) -------------------------------------------------------------
template <class M>
class BDCSVD {
 public:
  BDCSVD(const ConstBase& a, unsigned int options) {
    if (!(options & ComputeThinU) || !(options & ComputeThinV))
      throw std::logic_error("Eigen shim: BDCSVD supports ComputeThinU|ComputeThinV only");
    const long long m = a.rows(), n = a.cols(), k = std::min(m, n);
    s_ = VectorXd(k);
    u_ = MatrixXd(m, k);
    v_ = MatrixXd(n, k);
    if (k == 0) return;
    MatrixXd work_a(a);
    MatrixXd vt(k, n);
    const long long lda = std::max<long long>(1, m), ldu = std::max<long long>(1, m),
                    ldvt = std::max<long long>(1, k);
    std::vector<long long> iwork(static_cast<std::size_t>(8 * k));
    long long info = 0, lwork = -1;
    double wq = 0.0;
    shim::scipy_dgesdd_64_("S", &m, &n, work_a.data(), &lda, s_.data(), u_.data(), &ldu, vt.data(), &ldvt, &wq,
                           &lwork, iwork.data(), &info, 1);
    lwork = std::max<long long>(1, static_cast<long long>(wq));
    std::vector<double> work(static_cast<std::size_t>(lwork));
    shim::scipy_dgesdd_64_("S", &m, &n, work_a.data(), &lda, s_.data(), u_.data(), &ldu, vt.data(), &ldvt,
                           work.data(), &lwork, iwork.data(), &info, 1);
    if (info != 0) {
      info_ = info > 0 ? NoConvergence : InvalidInput;
      return;
    }
    v_ = MatrixXd(vt.transpose());
  }
  ComputationInfo info() const { return info_; }
  const VectorXd& singularValues() const { return s_; }
  const MatrixXd& matrixU() const { return u_; }
  const MatrixXd& matrixV() const { return v_; }

 private:
  VectorXd s_;
  MatrixXd u_, v_;
  ComputationInfo info_ = Success;
};

}  // namespace Eigen
