// Minimal owning dense containers with Eigen's storage contract: column-major,
// contiguous data(), (rows, cols) shape, Index = std::ptrdiff_t.  Only what the
// host layer and its tests need -- no expression templates.
#pragma once

#include <algorithm>
#include <cstddef>
#include <initializer_list>
#include <stdexcept>
#include <vector>

namespace noma::dense {

using Index = std::ptrdiff_t;

template <class T>
class Matrix {
  public:
    Matrix() = default;
    Matrix(Index rows, Index cols) : rows_(rows), cols_(cols), v_(rows * cols, T{}) {}
    static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
    static Matrix Constant(Index rows, Index cols, T value) {
        Matrix m(rows, cols);
        std::fill(m.v_.begin(), m.v_.end(), value);
        return m;
    }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    T *data() { return v_.data(); }
    const T *data() const { return v_.data(); }
    T &operator()(Index r, Index c) { return v_[c * rows_ + r]; }
    const T &operator()(Index r, Index c) const { return v_[c * rows_ + r]; }
    void resize(Index rows, Index cols) {
        rows_ = rows;
        cols_ = cols;
        v_.assign(rows * cols, T{});
    }
    void setZero() { std::fill(v_.begin(), v_.end(), T{}); }
    bool operator==(const Matrix &o) const {
        return rows_ == o.rows_ && cols_ == o.cols_ && v_ == o.v_;
    }

  private:
    Index rows_ = 0, cols_ = 0;
    std::vector<T> v_;
};

template <class T>
class Vector {
  public:
    Vector() = default;
    explicit Vector(Index n) : v_(n, T{}) {}
    Vector(std::initializer_list<T> init) : v_(init) {}
    static Vector Zero(Index n) { return Vector(n); }
    Index size() const { return static_cast<Index>(v_.size()); }
    T *data() { return v_.data(); }
    const T *data() const { return v_.data(); }
    T &operator[](Index i) { return v_[i]; }
    const T &operator[](Index i) const { return v_[i]; }
    T &operator()(Index i) { return v_[i]; }
    const T &operator()(Index i) const { return v_[i]; }
    void resize(Index n) { v_.assign(n, T{}); }
    bool operator==(const Vector &o) const { return v_ == o.v_; }

  private:
    std::vector<T> v_;
};

}  // namespace noma::dense
