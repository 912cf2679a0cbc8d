// eigen_subset.hpp -- ORACLE TEST INFRASTRUCTURE, not product code.
//
// A from-scratch stand-in for the small part of the Eigen 3 API the reference
// C++ sources use (Vector2d/3d/3i/4d, Matrix3d, Quaterniond, AngleAxisd), so
// the reference's own hot-path translation units -- renderer.cpp,
// likelihood.cpp, inference.cpp, tracking.cpp, ... -- compile here unmodified
// into oracle/_ref/ (Eigen itself is absent from this container and is not
// vendored by the reference: proj/CMakeLists.txt:13-18).
//
// Arithmetic order follows Eigen's scalar (non-SIMD) evaluation, the same
// convention the C restatement (oracle/b3d_oracle.c) and the CUDA path use:
//   * every reduction (dot, squaredNorm, sum, trace, the inner sum of a
//     matrix product) splits its terms in halves recursively:
//     3 terms -> a0 + (a1 + a2), 4 terms -> (a0 + a1) + (a2 + a3);
//   * normalized() divides each coefficient by sqrt(squaredNorm) (no
//     reciprocal), and leaves a zero vector unchanged;
//   * quaternion coefficients are stored (x, y, z, w); the Hamilton product,
//     q * v = v + w*uv + vec x uv with uv = 2 (vec x v), the rotation matrix
//     from 2x/2y/2z products and the trace-branch matrix->quaternion are the
//     textbook formulas Eigen documents.
// A SIMD Eigen build may associate a few of these sums differently; that is
// an ulp-level, unpinned difference.
#pragma once

// Eigen/Dense pulls these in transitively and the reference relies on it
// (geometry.hpp uses std::array without including <array>).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstddef>
#include <cstdlib>
#include <functional>
#include <limits>
#include <type_traits>
#include <vector>

namespace Eigen {

namespace shim {

// Sum of n terms f(lo) ... f(lo + n - 1), split in halves recursively.
template <typename T, typename F>
inline T halving_sum(int lo, int n, const F& f) {
  if (n == 1) return f(lo);
  const int h = n / 2;
  return halving_sum<T>(lo, h, f) + halving_sum<T>(lo + h, n - h, f);
}

}  // namespace shim

template <typename Scalar, int Rows, int Cols>
class Matrix;

// Writable view of one column of a matrix (rot.col(0) = v).
template <typename Scalar, int Rows, int Cols>
class ColumnRef {
 public:
  ColumnRef(Matrix<Scalar, Rows, Cols>& m, int c) : m_(m), c_(c) {}
  ColumnRef& operator=(const Matrix<Scalar, Rows, 1>& v) {
    for (int r = 0; r < Rows; ++r) m_(r, c_) = v[r];
    return *this;
  }
  operator Matrix<Scalar, Rows, 1>() const {
    Matrix<Scalar, Rows, 1> v;
    for (int r = 0; r < Rows; ++r) v[r] = m_(r, c_);
    return v;
  }

 private:
  Matrix<Scalar, Rows, Cols>& m_;
  int c_;
};

template <typename Scalar, int Rows, int Cols>
class Matrix {
 public:
  static constexpr int kSize = Rows * Cols;
  static constexpr bool kVector = (Cols == 1);

  Matrix() {
    for (int i = 0; i < kSize; ++i) a_[i] = Scalar(0);
  }
  Matrix(Scalar x, Scalar y) {
    static_assert(kSize == 2, "two-coefficient constructor");
    a_[0] = x;
    a_[1] = y;
  }
  Matrix(Scalar x, Scalar y, Scalar z) {
    static_assert(kSize == 3, "three-coefficient constructor");
    a_[0] = x;
    a_[1] = y;
    a_[2] = z;
  }
  Matrix(Scalar x, Scalar y, Scalar z, Scalar w) {
    static_assert(kSize == 4, "four-coefficient constructor");
    a_[0] = x;
    a_[1] = y;
    a_[2] = z;
    a_[3] = w;
  }

  static Matrix Zero() { return Matrix(); }
  static Matrix Constant(Scalar s) {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = s;
    return m;
  }
  static Matrix Ones() { return Constant(Scalar(1)); }
  static Matrix Identity() {
    Matrix m;
    for (int i = 0; i < Rows && i < Cols; ++i) m(i, i) = Scalar(1);
    return m;
  }
  static Matrix Unit(int i) {
    Matrix m;
    m.a_[i] = Scalar(1);
    return m;
  }
  static Matrix UnitX() { return Unit(0); }
  static Matrix UnitY() { return Unit(1); }
  static Matrix UnitZ() { return Unit(2); }

  // column-major storage, like Eigen's default
  Scalar& operator()(int r, int c) { return a_[c * Rows + r]; }
  Scalar operator()(int r, int c) const { return a_[c * Rows + r]; }
  Scalar& operator()(int i) { return a_[i]; }
  Scalar operator()(int i) const { return a_[i]; }
  Scalar& operator[](int i) { return a_[i]; }
  Scalar operator[](int i) const { return a_[i]; }
  Scalar coeff(int r, int c) const { return (*this)(r, c); }
  Scalar coeff(int i) const { return a_[i]; }
  Scalar& coeffRef(int r, int c) { return (*this)(r, c); }
  Scalar& coeffRef(int i) { return a_[i]; }
  Scalar& x() { return a_[0]; }
  Scalar& y() { return a_[1]; }
  Scalar& z() { return a_[2]; }
  Scalar& w() { return a_[3]; }
  Scalar x() const { return a_[0]; }
  Scalar y() const { return a_[1]; }
  Scalar z() const { return a_[2]; }
  Scalar w() const { return a_[3]; }
  Scalar* data() { return a_; }
  const Scalar* data() const { return a_; }
  static constexpr int rows() { return Rows; }
  static constexpr int cols() { return Cols; }
  static constexpr int size() { return kSize; }

  ColumnRef<Scalar, Rows, Cols> col(int c) { return ColumnRef<Scalar, Rows, Cols>(*this, c); }
  Matrix<Scalar, Rows, 1> col(int c) const {
    Matrix<Scalar, Rows, 1> v;
    for (int r = 0; r < Rows; ++r) v[r] = (*this)(r, c);
    return v;
  }
  Matrix<Scalar, Cols, Rows> transpose() const {
    Matrix<Scalar, Cols, Rows> t;
    for (int r = 0; r < Rows; ++r)
      for (int c = 0; c < Cols; ++c) t(c, r) = (*this)(r, c);
    return t;
  }

  template <typename T>
  Matrix<T, Rows, Cols> cast() const {
    Matrix<T, Rows, Cols> m;
    for (int i = 0; i < kSize; ++i) m[i] = static_cast<T>(a_[i]);
    return m;
  }

  // ---- coefficient-wise arithmetic
  Matrix operator+(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = a_[i] + o.a_[i];
    return m;
  }
  Matrix operator-(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = a_[i] - o.a_[i];
    return m;
  }
  Matrix operator-() const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = -a_[i];
    return m;
  }
  Matrix operator*(Scalar s) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = a_[i] * s;
    return m;
  }
  Matrix operator/(Scalar s) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = a_[i] / s;
    return m;
  }
  Matrix& operator+=(const Matrix& o) { return *this = *this + o; }
  Matrix& operator-=(const Matrix& o) { return *this = *this - o; }
  Matrix& operator*=(Scalar s) { return *this = *this * s; }
  Matrix& operator/=(Scalar s) { return *this = *this / s; }
  bool operator==(const Matrix& o) const {
    for (int i = 0; i < kSize; ++i)
      if (!(a_[i] == o.a_[i])) return false;
    return true;
  }
  bool operator!=(const Matrix& o) const { return !(*this == o); }

  Matrix cwiseMin(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = o.a_[i] < a_[i] ? o.a_[i] : a_[i];
    return m;
  }
  Matrix cwiseMax(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = a_[i] < o.a_[i] ? o.a_[i] : a_[i];
    return m;
  }
  Matrix cwiseProduct(const Matrix& o) const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = a_[i] * o.a_[i];
    return m;
  }
  Matrix cwiseAbs() const {
    Matrix m;
    for (int i = 0; i < kSize; ++i) m.a_[i] = a_[i] < Scalar(0) ? -a_[i] : a_[i];
    return m;
  }
  Scalar minCoeff() const {
    Scalar v = a_[0];
    for (int i = 1; i < kSize; ++i) v = a_[i] < v ? a_[i] : v;
    return v;
  }
  Scalar maxCoeff() const {
    Scalar v = a_[0];
    for (int i = 1; i < kSize; ++i) v = v < a_[i] ? a_[i] : v;
    return v;
  }

  // ---- reductions (halving order)
  Scalar sum() const {
    return shim::halving_sum<Scalar>(0, kSize, [&](int i) { return a_[i]; });
  }
  Scalar prod() const {
    Scalar p = a_[0];
    for (int i = 1; i < kSize; ++i) p *= a_[i];
    return p;
  }
  Scalar trace() const {
    return shim::halving_sum<Scalar>(0, Rows < Cols ? Rows : Cols,
                                     [&](int i) { return (*this)(i, i); });
  }
  Scalar dot(const Matrix& o) const {
    return shim::halving_sum<Scalar>(0, kSize, [&](int i) { return a_[i] * o.a_[i]; });
  }
  Scalar squaredNorm() const { return dot(*this); }
  Scalar norm() const { return std::sqrt(squaredNorm()); }
  Matrix normalized() const {
    const Scalar z = squaredNorm();
    if (z > Scalar(0)) return *this / std::sqrt(z);
    return *this;
  }
  void normalize() {
    const Scalar z = squaredNorm();
    if (z > Scalar(0)) *this /= std::sqrt(z);
  }
  Matrix cross(const Matrix& o) const {
    static_assert(kSize == 3, "cross product of 3-vectors");
    return Matrix(a_[1] * o.a_[2] - a_[2] * o.a_[1], a_[2] * o.a_[0] - a_[0] * o.a_[2],
                  a_[0] * o.a_[1] - a_[1] * o.a_[0]);
  }

  void setZero() { *this = Zero(); }

 private:
  Scalar a_[kSize];
};

template <typename Scalar, int Rows, int Cols>
inline Matrix<Scalar, Rows, Cols> operator*(Scalar s, const Matrix<Scalar, Rows, Cols>& m) {
  return m * s;
}
// int * Vector3d etc. (Eigen requires the same scalar; the reference only
// multiplies by doubles, but literal ints would otherwise be ambiguous)
template <typename Scalar, int Rows, int Cols, typename S,
          typename = std::enable_if_t<std::is_arithmetic_v<S> && !std::is_same_v<S, Scalar>>>
inline Matrix<Scalar, Rows, Cols> operator*(S s, const Matrix<Scalar, Rows, Cols>& m) {
  return m * static_cast<Scalar>(s);
}

// Matrix product: each coefficient is the halving sum over the inner index.
template <typename Scalar, int R, int K, int C>
inline Matrix<Scalar, R, C> operator*(const Matrix<Scalar, R, K>& a, const Matrix<Scalar, K, C>& b) {
  Matrix<Scalar, R, C> m;
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c)
      m(r, c) = shim::halving_sum<Scalar>(0, K, [&](int k) { return a(r, k) * b(k, c); });
  return m;
}

using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Vector2i = Matrix<int, 2, 1>;
using Vector3i = Matrix<int, 3, 1>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;

template <typename Scalar>
class AngleAxis {
 public:
  AngleAxis() = default;
  AngleAxis(Scalar angle, const Matrix<Scalar, 3, 1>& axis) : angle_(angle), axis_(axis) {}
  Scalar angle() const { return angle_; }
  const Matrix<Scalar, 3, 1>& axis() const { return axis_; }

 private:
  Scalar angle_ = 0;
  Matrix<Scalar, 3, 1> axis_;
};

template <typename Scalar>
class Quaternion {
 public:
  using Vec3 = Matrix<Scalar, 3, 1>;
  using Mat3 = Matrix<Scalar, 3, 3>;

  Quaternion() = default;
  Quaternion(Scalar w, Scalar x, Scalar y, Scalar z) : c_(x, y, z, w) {}
  // half-angle form: w = cos(a/2), vec = sin(a/2) * axis
  explicit Quaternion(const AngleAxis<Scalar>& aa) {
    const Scalar ha = Scalar(0.5) * aa.angle();
    const Scalar s = std::sin(ha);
    c_ = Matrix<Scalar, 4, 1>(s * aa.axis()[0], s * aa.axis()[1], s * aa.axis()[2],
                              std::cos(ha));
  }
  // rotation matrix -> quaternion (trace branch, else largest diagonal)
  explicit Quaternion(const Mat3& m) {
    Scalar t = m.trace();
    if (t > Scalar(0)) {
      t = std::sqrt(t + Scalar(1));
      w() = Scalar(0.5) * t;
      t = Scalar(0.5) / t;
      x() = (m(2, 1) - m(1, 2)) * t;
      y() = (m(0, 2) - m(2, 0)) * t;
      z() = (m(1, 0) - m(0, 1)) * t;
    } else {
      int i = 0;
      if (m(1, 1) > m(0, 0)) i = 1;
      if (m(2, 2) > m(i, i)) i = 2;
      const int j = (i + 1) % 3;
      const int k = (j + 1) % 3;
      t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + Scalar(1));
      c_[i] = Scalar(0.5) * t;
      t = Scalar(0.5) / t;
      w() = (m(k, j) - m(j, k)) * t;
      c_[j] = (m(j, i) + m(i, j)) * t;
      c_[k] = (m(k, i) + m(i, k)) * t;
    }
  }

  static Quaternion Identity() { return Quaternion(Scalar(1), Scalar(0), Scalar(0), Scalar(0)); }

  Scalar& x() { return c_[0]; }
  Scalar& y() { return c_[1]; }
  Scalar& z() { return c_[2]; }
  Scalar& w() { return c_[3]; }
  Scalar x() const { return c_[0]; }
  Scalar y() const { return c_[1]; }
  Scalar z() const { return c_[2]; }
  Scalar w() const { return c_[3]; }
  Vec3 vec() const { return Vec3(c_[0], c_[1], c_[2]); }
  Matrix<Scalar, 4, 1>& coeffs() { return c_; }
  const Matrix<Scalar, 4, 1>& coeffs() const { return c_; }

  Scalar squaredNorm() const { return c_.squaredNorm(); }
  Scalar norm() const { return c_.norm(); }
  Scalar dot(const Quaternion& o) const { return c_.dot(o.c_); }
  Quaternion normalized() const {
    Quaternion q;
    q.c_ = c_.normalized();
    return q;
  }
  void normalize() { c_.normalize(); }
  Quaternion conjugate() const { return Quaternion(w(), -x(), -y(), -z()); }
  Quaternion inverse() const {
    const Scalar n2 = squaredNorm();
    if (n2 > Scalar(0)) {
      const Quaternion c = conjugate();
      Quaternion q;
      q.c_ = c.c_ / n2;
      return q;
    }
    Quaternion q;
    q.c_ = Matrix<Scalar, 4, 1>::Zero();
    return q;
  }
  Scalar angularDistance(const Quaternion& o) const {
    const Quaternion d = *this * o.conjugate();
    const Scalar vn = d.vec().norm();
    const Scalar aw = d.w() < Scalar(0) ? -d.w() : d.w();
    return Scalar(2) * std::atan2(vn, aw);
  }

  Quaternion operator*(const Quaternion& b) const {
    const Quaternion& a = *this;
    return Quaternion(a.w() * b.w() - a.x() * b.x() - a.y() * b.y() - a.z() * b.z(),
                      a.w() * b.x() + a.x() * b.w() + a.y() * b.z() - a.z() * b.y(),
                      a.w() * b.y() + a.y() * b.w() + a.z() * b.x() - a.x() * b.z(),
                      a.w() * b.z() + a.z() * b.w() + a.x() * b.y() - a.y() * b.x());
  }
  Quaternion& operator*=(const Quaternion& b) { return *this = *this * b; }

  // rotate a vector: v + w*uv + vec x uv, uv = 2 (vec x v)
  Vec3 operator*(const Vec3& v) const {
    Vec3 uv = vec().cross(v);
    uv += uv;
    return v + w() * uv + vec().cross(uv);
  }

  Mat3 toRotationMatrix() const {
    Mat3 r;
    const Scalar tx = Scalar(2) * x(), ty = Scalar(2) * y(), tz = Scalar(2) * z();
    const Scalar twx = tx * w(), twy = ty * w(), twz = tz * w();
    const Scalar txx = tx * x(), txy = ty * x(), txz = tz * x();
    const Scalar tyy = ty * y(), tyz = tz * y(), tzz = tz * z();
    r(0, 0) = Scalar(1) - (tyy + tzz);
    r(0, 1) = txy - twz;
    r(0, 2) = txz + twy;
    r(1, 0) = txy + twz;
    r(1, 1) = Scalar(1) - (txx + tzz);
    r(1, 2) = tyz - twx;
    r(2, 0) = txz - twy;
    r(2, 1) = tyz + twx;
    r(2, 2) = Scalar(1) - (txx + tyy);
    return r;
  }

 private:
  Matrix<Scalar, 4, 1> c_{Scalar(0), Scalar(0), Scalar(0), Scalar(1)};
};

using Quaterniond = Quaternion<double>;
using AngleAxisd = AngleAxis<double>;

}  // namespace Eigen
