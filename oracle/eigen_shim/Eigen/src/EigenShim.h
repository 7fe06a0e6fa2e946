// Eigen-subset shim for building the UNMODIFIED FaSS-MVS reference sources
// (/root/reference/proj) as the parity oracle. TEST INFRASTRUCTURE ONLY.
//
// Eigen3 is a hard dependency of the reference (proj/CMakeLists.txt:12) and is
// absent from this image, so this header provides exactly the API subset the
// reference uses. Evaluation is eager, coefficient by
// coefficient, with NO fused multiply-add and with every reduction evaluated
// strictly left to right starting from the first term:
//     dot / squaredNorm / (A*B)(i,j) / (A*v)(i)  =  ((e0 + e1) + e2) [+ e3 ...]
// This order is the parity pin shared by the oracle and the B200 host code
// (paper_2112_00821_b200/csrc/host/geom.hpp implements the same order).
#pragma once

// Real Eigen pulls these standard headers in transitively; the reference
// relies on that (e.g. colorize.cpp uses std::array without <array>).
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <vector>
#include <initializer_list>
#include <ostream>
#include <type_traits>

namespace Eigen {

using Index = std::ptrdiff_t;

template <typename S, int R, int C>
class Matrix;

namespace shim_detail {

template <typename S, int R, int C>
class ColRef {
public:
    ColRef(Matrix<S, R, C>& m, int j) : m_(m), j_(j) {}
    ColRef& operator=(const Matrix<S, R, 1>& v) {
        for (int i = 0; i < R; ++i)
            m_(i, j_) = v(i);
        return *this;
    }
    operator Matrix<S, R, 1>() const {
        Matrix<S, R, 1> v;
        for (int i = 0; i < R; ++i)
            v(i) = m_(i, j_);
        return v;
    }

private:
    Matrix<S, R, C>& m_;
    int j_;
};

template <typename S, int R, int C, int N>
class LeftColsRef {
public:
    explicit LeftColsRef(Matrix<S, R, C>& m) : m_(m) {}
    LeftColsRef& operator=(const Matrix<S, R, N>& v) {
        for (int j = 0; j < N; ++j)
            for (int i = 0; i < R; ++i)
                m_(i, j) = v(i, j);
        return *this;
    }

private:
    Matrix<S, R, C>& m_;
};

template <typename S, int R, int C>
class CommaInit {
public:
    CommaInit(Matrix<S, R, C>& m, S first) : m_(m), k_(0) { put(first); }
    template <typename T>
    CommaInit& operator,(T v) {
        put(static_cast<S>(v));
        return *this;
    }

private:
    // Comma initialisation fills row by row (Eigen semantics).
    void put(S v) {
        m_(k_ / C, k_ % C) = v;
        ++k_;
    }
    Matrix<S, R, C>& m_;
    int k_;
};

}  // namespace shim_detail

template <typename S, int R, int C>
class Matrix {
public:
    using Scalar = S;
    static constexpr int RowsAtCompileTime = R;
    static constexpr int ColsAtCompileTime = C;

    Matrix() {
        for (int i = 0; i < R * C; ++i)
            d_[i] = S(0);
    }
    template <typename A, typename B,
              typename = std::enable_if_t<std::is_arithmetic_v<A> && std::is_arithmetic_v<B> &&
                                          R * C == 2>>
    Matrix(A a, B b) {
        d_[0] = static_cast<S>(a);
        d_[1] = static_cast<S>(b);
    }
    template <typename A, typename B, typename D,
              typename = std::enable_if_t<std::is_arithmetic_v<A> && std::is_arithmetic_v<B> &&
                                          std::is_arithmetic_v<D> && R * C == 3>>
    Matrix(A a, B b, D c) {
        d_[0] = static_cast<S>(a);
        d_[1] = static_cast<S>(b);
        d_[2] = static_cast<S>(c);
    }
    template <typename A, typename B, typename D, typename E,
              typename = std::enable_if_t<std::is_arithmetic_v<A> && R * C == 4>>
    Matrix(A a, B b, D c, E e) {
        d_[0] = static_cast<S>(a);
        d_[1] = static_cast<S>(b);
        d_[2] = static_cast<S>(c);
        d_[3] = static_cast<S>(e);
    }

    static Matrix Zero() { return Matrix(); }
    static Matrix Constant(S v) {
        Matrix m;
        for (int i = 0; i < R * C; ++i)
            m.d_[i] = v;
        return m;
    }
    static Matrix Ones() { return Constant(S(1)); }
    static Matrix Identity() {
        Matrix m;
        for (int i = 0; i < R && i < C; ++i)
            m(i, i) = S(1);
        return m;
    }
    static Matrix Unit(int k) {
        Matrix m;
        m.d_[k] = S(1);
        return m;
    }
    static Matrix UnitX() { return Unit(0); }
    static Matrix UnitY() { return Unit(1); }
    static Matrix UnitZ() { return Unit(2); }

    static constexpr Index rows() { return R; }
    static constexpr Index cols() { return C; }
    static constexpr Index size() { return R * C; }

    S& operator()(Index i, Index j) { return d_[j * R + i]; }
    const S& operator()(Index i, Index j) const { return d_[j * R + i]; }
    S& operator()(Index k) { return d_[k]; }
    const S& operator()(Index k) const { return d_[k]; }
    S& operator[](Index k) { return d_[k]; }
    const S& operator[](Index k) const { return d_[k]; }
    S& coeffRef(Index i, Index j) { return (*this)(i, j); }
    S coeff(Index i, Index j) const { return (*this)(i, j); }
    S* data() { return d_; }
    const S* data() const { return d_; }

    S& x() { return d_[0]; }
    S& y() { return d_[1]; }
    S& z() { return d_[2]; }
    S x() const { return d_[0]; }
    S y() const { return d_[1]; }
    S z() const { return d_[2]; }

    shim_detail::CommaInit<S, R, C> operator<<(S v) { return {*this, v}; }

    Matrix& setZero() {
        for (int i = 0; i < R * C; ++i)
            d_[i] = S(0);
        return *this;
    }

    Matrix<S, C, R> transpose() const {
        Matrix<S, C, R> t;
        for (int i = 0; i < R; ++i)
            for (int j = 0; j < C; ++j)
                t(j, i) = (*this)(i, j);
        return t;
    }

    Matrix<S, R, 1> col(Index j) const {
        Matrix<S, R, 1> v;
        for (int i = 0; i < R; ++i)
            v(i) = (*this)(i, j);
        return v;
    }
    shim_detail::ColRef<S, R, C> col(Index j) { return {*this, static_cast<int>(j)}; }
    Matrix<S, 1, C> row(Index i) const {
        Matrix<S, 1, C> v;
        for (int j = 0; j < C; ++j)
            v(0, j) = (*this)(i, j);
        return v;
    }
    template <int N>
    shim_detail::LeftColsRef<S, R, C, N> leftCols() {
        return shim_detail::LeftColsRef<S, R, C, N>(*this);
    }

    template <typename T>
    Matrix<T, R, C> cast() const {
        Matrix<T, R, C> m;
        for (int i = 0; i < R * C; ++i)
            m(i) = static_cast<T>(d_[i]);
        return m;
    }

    // Reductions: strictly left to right from the first term.
    S sum() const {
        S acc = d_[0];
        for (int i = 1; i < R * C; ++i)
            acc = acc + d_[i];
        return acc;
    }
    S dot(const Matrix& o) const {
        S acc = d_[0] * o.d_[0];
        for (int i = 1; i < R * C; ++i)
            acc = acc + d_[i] * o.d_[i];
        return acc;
    }
    S squaredNorm() const { return dot(*this); }
    S norm() const { return std::sqrt(squaredNorm()); }
    Matrix normalized() const {
        const S z = squaredNorm();
        if (z > S(0))
            return *this / std::sqrt(z);
        return *this;
    }
    void normalize() {
        const S z = squaredNorm();
        if (z > S(0))
            *this /= std::sqrt(z);
    }
    S maxCoeff() const {
        S m = d_[0];
        for (int i = 1; i < R * C; ++i)
            if (d_[i] > m)
                m = d_[i];
        return m;
    }
    S minCoeff() const {
        S m = d_[0];
        for (int i = 1; i < R * C; ++i)
            if (d_[i] < m)
                m = d_[i];
        return m;
    }
    Matrix cwiseAbs() const {
        Matrix m;
        for (int i = 0; i < R * C; ++i)
            m.d_[i] = std::abs(d_[i]);
        return m;
    }
    Matrix cwiseProduct(const Matrix& o) const {
        Matrix m;
        for (int i = 0; i < R * C; ++i)
            m.d_[i] = d_[i] * o.d_[i];
        return m;
    }

    // 3-vector cross product (Eigen's coefficient formulas).
    Matrix cross(const Matrix& b) const {
        static_assert(R * C == 3, "cross needs 3-vectors");
        return Matrix(d_[1] * b.d_[2] - d_[2] * b.d_[1], d_[2] * b.d_[0] - d_[0] * b.d_[2],
                      d_[0] * b.d_[1] - d_[1] * b.d_[0]);
    }

    Matrix<S, R + 1, 1> homogeneous() const {
        static_assert(C == 1, "homogeneous needs a column vector");
        Matrix<S, R + 1, 1> h;
        for (int i = 0; i < R; ++i)
            h(i) = d_[i];
        h(R) = S(1);
        return h;
    }
    Matrix<S, R - 1, 1> hnormalized() const {
        static_assert(C == 1, "hnormalized needs a column vector");
        Matrix<S, R - 1, 1> h;
        for (int i = 0; i < R - 1; ++i)
            h(i) = d_[i] / d_[R - 1];
        return h;
    }

    S determinant() const {
        static_assert(R == 3 && C == 3, "determinant implemented for 3x3");
        const Matrix& m = *this;
        const auto h = [&](int a, int b, int c) {
            return m(0, a) * (m(1, b) * m(2, c) - m(1, c) * m(2, b));
        };
        return h(0, 1, 2) - h(1, 0, 2) + h(2, 0, 1);
    }

    // Elementwise arithmetic.
    Matrix operator+(const Matrix& o) const {
        Matrix m;
        for (int i = 0; i < R * C; ++i)
            m.d_[i] = d_[i] + o.d_[i];
        return m;
    }
    Matrix operator-(const Matrix& o) const {
        Matrix m;
        for (int i = 0; i < R * C; ++i)
            m.d_[i] = d_[i] - o.d_[i];
        return m;
    }
    Matrix operator-() const {
        Matrix m;
        for (int i = 0; i < R * C; ++i)
            m.d_[i] = -d_[i];
        return m;
    }
    template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
    Matrix operator*(T s) const {
        const S ss = static_cast<S>(s);
        Matrix m;
        for (int i = 0; i < R * C; ++i)
            m.d_[i] = d_[i] * ss;
        return m;
    }
    template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
    Matrix operator/(T s) const {
        const S ss = static_cast<S>(s);
        Matrix m;
        for (int i = 0; i < R * C; ++i)
            m.d_[i] = d_[i] / ss;
        return m;
    }
    Matrix& operator+=(const Matrix& o) { return *this = *this + o; }
    Matrix& operator-=(const Matrix& o) { return *this = *this - o; }
    template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
    Matrix& operator*=(T s) {
        return *this = *this * s;
    }
    template <typename T, typename = std::enable_if_t<std::is_arithmetic_v<T>>>
    Matrix& operator/=(T s) {
        return *this = *this / s;
    }

    // Matrix product; each coefficient reduced left to right.
    template <int K>
    Matrix<S, R, K> operator*(const Matrix<S, C, K>& o) const {
        Matrix<S, R, K> m;
        for (int i = 0; i < R; ++i)
            for (int j = 0; j < K; ++j) {
                S acc = (*this)(i, 0) * o(0, j);
                for (int k = 1; k < C; ++k)
                    acc = acc + (*this)(i, k) * o(k, j);
                m(i, j) = acc;
            }
        return m;
    }

    bool operator==(const Matrix& o) const {
        for (int i = 0; i < R * C; ++i)
            if (!(d_[i] == o.d_[i]))
                return false;
        return true;
    }
    bool operator!=(const Matrix& o) const { return !(*this == o); }

    bool isApprox(const Matrix& o, S prec = S(1e-12)) const {
        return (*this - o).norm() <= prec * std::min(norm(), o.norm());
    }

private:
    S d_[R * C];
};

template <typename T, typename S, int R, int C,
          typename = std::enable_if_t<std::is_arithmetic_v<T>>>
Matrix<S, R, C> operator*(T s, const Matrix<S, R, C>& m) {
    // Scalar promoted to the matrix scalar type first (Eigen >= 3.3).
    const S ss = static_cast<S>(s);
    Matrix<S, R, C> out;
    for (int i = 0; i < R * C; ++i)
        out(i) = ss * m(i);
    return out;
}

template <typename S, int R, int C>
std::ostream& operator<<(std::ostream& os, const Matrix<S, R, C>& m) {
    for (int i = 0; i < R; ++i) {
        for (int j = 0; j < C; ++j)
            os << (j ? " " : "") << m(i, j);
        if (i + 1 < R)
            os << "\n";
    }
    return os;
}

using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Vector2f = Matrix<float, 2, 1>;
using Vector3f = Matrix<float, 3, 1>;
using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using Matrix3f = Matrix<float, 3, 3>;

template <typename S>
class AngleAxis {
public:
    AngleAxis(S angle, const Matrix<S, 3, 1>& axis) : angle_(angle), axis_(axis) {}
    // Eigen's AngleAxis::toRotationMatrix coefficient formulas.
    Matrix<S, 3, 3> toRotationMatrix() const {
        Matrix<S, 3, 3> res;
        const Matrix<S, 3, 1> sin_axis = std::sin(angle_) * axis_;
        const S c = std::cos(angle_);
        const Matrix<S, 3, 1> cos1_axis = (S(1) - c) * axis_;
        S tmp = cos1_axis.x() * axis_.y();
        res(0, 1) = tmp - sin_axis.z();
        res(1, 0) = tmp + sin_axis.z();
        tmp = cos1_axis.x() * axis_.z();
        res(0, 2) = tmp + sin_axis.y();
        res(2, 0) = tmp - sin_axis.y();
        tmp = cos1_axis.y() * axis_.z();
        res(1, 2) = tmp - sin_axis.x();
        res(2, 1) = tmp + sin_axis.x();
        for (int i = 0; i < 3; ++i)
            res(i, i) = cos1_axis(i) * axis_(i) + c;
        return res;
    }

private:
    S angle_;
    Matrix<S, 3, 1> axis_;
};
using AngleAxisd = AngleAxis<double>;

}  // namespace Eigen
