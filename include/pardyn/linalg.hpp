// Small dense value types for the pardyn drop-in API (include/pardyn/pardyn.hpp).
//
// The reference spells its public types with Eigen (types.hpp:12-17:
// Vec3 = Vector3d, Mat3 = Matrix3d, Vec6, Mat6, JointVector = VectorXd;
// forward_dynamics.hpp:27 Vec5). Eigen is not a dependency of the drop-in,
// so these are fixed-size stand-ins with the subset of Eigen's interface that
// the reference API and its callers use: Zero() / Identity() / UnitX..Z(),
// component constructors, (i) / (i, j) / [i] access, data() in Eigen's
// column-major order, + - * / with scalars and matrices, transpose(), dot(),
// norm(), squaredNorm(), head<K>() / tail<K>() / segment<K>(), col(j),
// allFinite(), setZero(). Every element starts at zero (Eigen leaves
// fixed-size storage uninitialised; zero is a valid refinement of that).
#pragma once

#include <array>
#include <cmath>
#include <cstddef>
#include <initializer_list>
#include <vector>

namespace pardyn {

template <int R, int C>
class Matrix {
 public:
  static constexpr int RowsAtCompileTime = R;
  static constexpr int ColsAtCompileTime = C;

  Matrix() { v_.fill(0.0); }
  // Vector constructors (Eigen's Vector3d(x, y, z), Vector2d(x, y), ...).
  Matrix(double x, double y) requires(R * C == 2 && (R == 1 || C == 1)) : v_{x, y} {}
  Matrix(double x, double y, double z) requires(R * C == 3 && (R == 1 || C == 1)) : v_{x, y, z} {}
  Matrix(double a, double b, double c, double d) requires(R * C == 4 && (R == 1 || C == 1)) : v_{a, b, c, d} {}

  static Matrix Zero() { return Matrix(); }
  static Matrix Constant(double c) {
    Matrix m;
    m.v_.fill(c);
    return m;
  }
  static Matrix Identity() {
    Matrix m;
    for (int k = 0; k < (R < C ? R : C); ++k) m(k, k) = 1.0;
    return m;
  }
  static Matrix Unit(int i) requires(C == 1) {
    Matrix m;
    m.v_[static_cast<std::size_t>(i)] = 1.0;
    return m;
  }
  static Matrix UnitX() requires(C == 1) { return Unit(0); }
  static Matrix UnitY() requires(C == 1 && R >= 2) { return Unit(1); }
  static Matrix UnitZ() requires(C == 1 && R >= 3) { return Unit(2); }

  // Row-major initialiser-list fill, the order Eigen's comma initialiser reads.
  static Matrix FromRowMajor(const double* rm) {
    Matrix m;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C; ++j) m(i, j) = rm[i * C + j];
    return m;
  }
  static Matrix FromRowMajor(std::initializer_list<double> rm) { return FromRowMajor(rm.begin()); }
  void toRowMajor(double* out) const {
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C; ++j) out[i * C + j] = (*this)(i, j);
  }

  static constexpr int rows() { return R; }
  static constexpr int cols() { return C; }
  static constexpr int size() { return R * C; }

  double& operator()(int i, int j) { return v_[static_cast<std::size_t>(j * R + i)]; }
  double operator()(int i, int j) const { return v_[static_cast<std::size_t>(j * R + i)]; }
  double& operator()(int i) { return v_[static_cast<std::size_t>(i)]; }
  double operator()(int i) const { return v_[static_cast<std::size_t>(i)]; }
  double& operator[](int i) { return v_[static_cast<std::size_t>(i)]; }
  double operator[](int i) const { return v_[static_cast<std::size_t>(i)]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double* begin() { return v_.data(); }
  double* end() { return v_.data() + R * C; }
  const double* begin() const { return v_.data(); }
  const double* end() const { return v_.data() + R * C; }

  Matrix<C, R> transpose() const {
    Matrix<C, R> t;
    for (int i = 0; i < R; ++i)
      for (int j = 0; j < C; ++j) t(j, i) = (*this)(i, j);
    return t;
  }
  Matrix<R, 1> col(int j) const {
    Matrix<R, 1> c;
    for (int i = 0; i < R; ++i) c(i) = (*this)(i, j);
    return c;
  }
  template <int K>
  Matrix<K, 1> segment(int start) const requires(C == 1) {
    Matrix<K, 1> s;
    for (int i = 0; i < K; ++i) s(i) = v_[static_cast<std::size_t>(start + i)];
    return s;
  }
  template <int K>
  Matrix<K, 1> head() const requires(C == 1) { return segment<K>(0); }
  template <int K>
  Matrix<K, 1> tail() const requires(C == 1) { return segment<K>(R - K); }

  double squaredNorm() const {
    double s = 0.0;
    for (double x : v_) s += x * x;
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double dot(const Matrix& o) const requires(C == 1) {
    double s = 0.0;
    for (int i = 0; i < R; ++i) s += v_[static_cast<std::size_t>(i)] * o.v_[static_cast<std::size_t>(i)];
    return s;
  }
  Matrix<3, 1> cross(const Matrix<3, 1>& o) const requires(R == 3 && C == 1) {
    const Matrix& a = *this;
    return {a(1) * o(2) - a(2) * o(1), a(2) * o(0) - a(0) * o(2), a(0) * o(1) - a(1) * o(0)};
  }
  bool allFinite() const {
    for (double x : v_)
      if (!std::isfinite(x)) return false;
    return true;
  }
  void setZero() { v_.fill(0.0); }

  Matrix& operator+=(const Matrix& o) {
    for (int k = 0; k < R * C; ++k) v_[static_cast<std::size_t>(k)] += o.v_[static_cast<std::size_t>(k)];
    return *this;
  }
  Matrix& operator-=(const Matrix& o) {
    for (int k = 0; k < R * C; ++k) v_[static_cast<std::size_t>(k)] -= o.v_[static_cast<std::size_t>(k)];
    return *this;
  }
  Matrix& operator*=(double s) {
    for (double& x : v_) x *= s;
    return *this;
  }
  friend Matrix operator+(Matrix a, const Matrix& b) { return a += b; }
  friend Matrix operator-(Matrix a, const Matrix& b) { return a -= b; }
  friend Matrix operator-(Matrix a) { return a *= -1.0; }
  friend Matrix operator*(Matrix a, double s) { return a *= s; }
  friend Matrix operator*(double s, Matrix a) { return a *= s; }
  friend Matrix operator/(Matrix a, double s) {
    for (double& x : a.v_) x /= s;
    return a;
  }
  friend bool operator==(const Matrix& a, const Matrix& b) { return a.v_ == b.v_; }
  friend bool operator!=(const Matrix& a, const Matrix& b) { return !(a == b); }

 private:
  std::array<double, static_cast<std::size_t>(R * C)> v_;
};

template <int R, int K, int C>
Matrix<R, C> operator*(const Matrix<R, K>& a, const Matrix<K, C>& b) {
  Matrix<R, C> m;
  for (int j = 0; j < C; ++j)
    for (int k = 0; k < K; ++k) {
      const double bkj = b(k, j);
      for (int i = 0; i < R; ++i) m(i, j) += a(i, k) * bkj;
    }
  return m;
}

using Vec3 = Matrix<3, 1>;
using Vec5 = Matrix<5, 1>;
using Vec6 = Matrix<6, 1>;
using Mat3 = Matrix<3, 3>;
using Mat5 = Matrix<5, 5>;
using Mat6 = Matrix<6, 6>;
using Mat65 = Matrix<6, 5>;

// Eigen::VectorXd stand-in (types.hpp:17 JointVector).
class JointVector {
 public:
  JointVector() = default;
  explicit JointVector(std::size_t n) : v_(n, 0.0) {}
  explicit JointVector(int n) : v_(static_cast<std::size_t>(n < 0 ? 0 : n), 0.0) {}
  JointVector(std::initializer_list<double> l) : v_(l) {}
  template <class It>
  JointVector(It first, It last) : v_(first, last) {}
  static JointVector Zero(std::size_t n) { return JointVector(n); }
  static JointVector Constant(std::size_t n, double c) {
    JointVector v(n);
    for (double& x : v.v_) x = c;
    return v;
  }
  std::size_t size() const { return v_.size(); }
  void resize(std::size_t n) { v_.assign(n, 0.0); }
  double& operator[](std::size_t i) { return v_[i]; }
  double operator[](std::size_t i) const { return v_[i]; }
  double& operator()(std::size_t i) { return v_[i]; }
  double operator()(std::size_t i) const { return v_[i]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double* begin() { return v_.data(); }
  double* end() { return v_.data() + v_.size(); }
  const double* begin() const { return v_.data(); }
  const double* end() const { return v_.data() + v_.size(); }
  double squaredNorm() const {
    double s = 0.0;
    for (double x : v_) s += x * x;
    return s;
  }
  double norm() const { return std::sqrt(squaredNorm()); }
  double dot(const JointVector& o) const {
    double s = 0.0;
    for (std::size_t i = 0; i < v_.size(); ++i) s += v_[i] * o.v_[i];
    return s;
  }
  bool allFinite() const {
    for (double x : v_)
      if (!std::isfinite(x)) return false;
    return true;
  }
  JointVector& operator+=(const JointVector& o) {
    for (std::size_t i = 0; i < v_.size(); ++i) v_[i] += o.v_[i];
    return *this;
  }
  JointVector& operator-=(const JointVector& o) {
    for (std::size_t i = 0; i < v_.size(); ++i) v_[i] -= o.v_[i];
    return *this;
  }
  JointVector& operator*=(double s) {
    for (double& x : v_) x *= s;
    return *this;
  }
  friend JointVector operator+(JointVector a, const JointVector& b) { return a += b; }
  friend JointVector operator-(JointVector a, const JointVector& b) { return a -= b; }
  friend JointVector operator*(double s, JointVector a) { return a *= s; }
  friend JointVector operator*(JointVector a, double s) { return a *= s; }
  friend bool operator==(const JointVector& a, const JointVector& b) { return a.v_ == b.v_; }
  friend bool operator!=(const JointVector& a, const JointVector& b) { return !(a == b); }

 private:
  std::vector<double> v_;
};

// Eigen::MatrixXd stand-in (joint_space_inertia, forward_dynamics.hpp:34-35),
// row-major storage.
class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(std::size_t r, std::size_t c) : r_(r), c_(c), v_(r * c, 0.0) {}
  static MatrixXd Identity(std::size_t r, std::size_t c) {
    MatrixXd m(r, c);
    for (std::size_t k = 0; k < (r < c ? r : c); ++k) m(k, k) = 1.0;
    return m;
  }
  std::size_t rows() const { return r_; }
  std::size_t cols() const { return c_; }
  double& operator()(std::size_t i, std::size_t j) { return v_[i * c_ + j]; }
  double operator()(std::size_t i, std::size_t j) const { return v_[i * c_ + j]; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  MatrixXd transpose() const {
    MatrixXd t(c_, r_);
    for (std::size_t i = 0; i < r_; ++i)
      for (std::size_t j = 0; j < c_; ++j) t(j, i) = (*this)(i, j);
    return t;
  }
  double norm() const {
    double s = 0.0;
    for (double x : v_) s += x * x;
    return std::sqrt(s);
  }
  friend MatrixXd operator-(const MatrixXd& a, const MatrixXd& b) {
    MatrixXd m(a.r_, a.c_);
    for (std::size_t k = 0; k < a.v_.size(); ++k) m.v_[k] = a.v_[k] - b.v_[k];
    return m;
  }
  friend MatrixXd operator*(const MatrixXd& a, const MatrixXd& b) {
    MatrixXd m(a.r_, b.c_);
    for (std::size_t i = 0; i < a.r_; ++i)
      for (std::size_t k = 0; k < a.c_; ++k)
        for (std::size_t j = 0; j < b.c_; ++j) m(i, j) += a(i, k) * b(k, j);
    return m;
  }
  friend JointVector operator*(const MatrixXd& a, const JointVector& x) {
    JointVector y(a.r_);
    for (std::size_t i = 0; i < a.r_; ++i)
      for (std::size_t j = 0; j < a.c_; ++j) y[i] += a(i, j) * x[j];
    return y;
  }

 private:
  std::size_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};

}  // namespace pardyn
