// cbp::core value types for the B200 build (reference proj/core/include/cbp/types.hpp).
// The reference aliases Eigen's dynamic column-major matrices; Eigen is not available
// here, so these are minimal owning column-major containers with the members the
// reference API and tests use: rows(), cols(), size(), operator()(r, c), data().
#pragma once

#include <complex>
#include <cstddef>
#include <vector>

namespace cbp {

using cplx = std::complex<double>;

template <class T>
class Matrix {
 public:
  Matrix() = default;
  Matrix(long rows, long cols, T fill = T()) : r_(rows), c_(cols), v_(size_t(rows * cols), fill) {}
  static Matrix Zero(long rows, long cols) { return Matrix(rows, cols, T(0)); }
  static Matrix Ones(long rows, long cols) { return Matrix(rows, cols, T(1)); }
  long rows() const { return r_; }
  long cols() const { return c_; }
  long size() const { return r_ * c_; }
  T& operator()(long r, long c) { return v_[size_t(c * r_ + r)]; }  // column-major
  const T& operator()(long r, long c) const { return v_[size_t(c * r_ + r)]; }
  T* data() { return v_.data(); }
  const T* data() const { return v_.data(); }
  T sum() const {
    T s(0);
    for (const T& x : v_) s += x;
    return s;
  }

 private:
  long r_ = 0, c_ = 0;
  std::vector<T> v_;
};

template <class T>
class Vector {
 public:
  Vector() = default;
  explicit Vector(long n, T fill = T()) : v_(size_t(n), fill) {}
  Vector(std::initializer_list<T> init) : v_(init) {}
  long size() const { return long(v_.size()); }
  T& operator[](long i) { return v_[size_t(i)]; }
  const T& operator[](long i) const { return v_[size_t(i)]; }
  T& operator()(long i) { return v_[size_t(i)]; }
  const T& operator()(long i) const { return v_[size_t(i)]; }
  T* data() { return v_.data(); }
  const T* data() const { return v_.data(); }

 private:
  std::vector<T> v_;
};

using Mat = Matrix<double>;
using CMat = Matrix<cplx>;
using Vec = Vector<double>;
using CVec = Vector<cplx>;

/* Image planes are coefficient arrays of bivariate polynomials: row index m is the
   z1 power, column index n the z2 power (types.hpp:15-17). */
using ImagePlane = Mat;

enum class Axis { Z1, Z2 };

inline const char* axis_name(Axis a) { return a == Axis::Z1 ? "z1" : "z2"; }

}  // namespace cbp
