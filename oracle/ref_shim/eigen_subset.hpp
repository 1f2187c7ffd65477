// ORACLE — test infrastructure only. A minimal stand-in for the subset of
// Eigen 3 that the reference tsdfslam sources use, so that those sources
// compile UNMODIFIED into oracle/_ref (oracle/Makefile). Not Eigen: fixed
// sizes only, eager evaluation, and a defined arithmetic order that is the
// oracle's contract (oracle.hpp): dot products and matrix products sum
// k = 0, 1, ... left to right, vector / scalar is a true division, no FMA
// (built with -ffp-contract=off). The decompositions follow Eigen's published
// algorithms: LDLT with symmetric diagonal pivoting (Eigen/src/Cholesky/LDLT.h),
// quaternion <-> matrix (Shepperd), slerp and AngleAxis as in Eigen/src/Geometry.
// SelfAdjointEigenSolver and JacobiSVD are cyclic Jacobi (only the reference's
// informational `degenerate` flag and AteRmse's alignment depend on them).
#pragma once

// (the standard headers Eigen/Core itself pulls in)
#include <algorithm>
#include <cassert>
#include <climits>
#include <cmath>
#include <complex>
#include <cstddef>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <iosfwd>
#include <limits>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

namespace Eigen {

enum DecompositionOptions { ComputeFullU = 0x04, ComputeThinU = 0x08, ComputeFullV = 0x10, ComputeThinV = 0x20 };
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

template <typename S, int R, int C>
class Matrix;

template <typename S>
struct NumTraits {
    static S epsilon() { return std::numeric_limits<S>::epsilon(); }
    static S dummy_precision() { return S(1e-12); }
};

// Assignable rectangular view (topLeftCorner / topRightCorner / head / tail / diagonal targets).
template <typename S, int R, int C, int BR, int BC>
struct BlockRef {
    Matrix<S, R, C>& m;
    int i0, j0;
    operator Matrix<S, BR, BC>() const {
        Matrix<S, BR, BC> r;
        for (int j = 0; j < BC; ++j)
            for (int i = 0; i < BR; ++i) r(i, j) = m(i0 + i, j0 + j);
        return r;
    }
    BlockRef& operator=(const Matrix<S, BR, BC>& v) {
        for (int j = 0; j < BC; ++j)
            for (int i = 0; i < BR; ++i) m(i0 + i, j0 + j) = v(i, j);
        return *this;
    }
};

template <typename S, int N, int R, int C>
struct DiagonalRef {
    Matrix<S, R, C>& m;
    operator Matrix<S, N, 1>() const {
        Matrix<S, N, 1> r;
        for (int i = 0; i < N; ++i) r(i) = m(i, i);
        return r;
    }
    DiagonalRef& operator+=(const Matrix<S, N, 1>& v) {
        for (int i = 0; i < N; ++i) m(i, i) += v(i);
        return *this;
    }
    DiagonalRef& operator=(const Matrix<S, N, 1>& v) {
        for (int i = 0; i < N; ++i) m(i, i) = v(i);
        return *this;
    }
    S maxCoeff() const { return Matrix<S, N, 1>(*this).maxCoeff(); }
    S minCoeff() const { return Matrix<S, N, 1>(*this).minCoeff(); }
    Matrix<S, N, 1> cwiseMax(S v) const { return Matrix<S, N, 1>(*this).cwiseMax(v); }
    Matrix<S, N, 1> cwiseMax(const Matrix<S, N, 1>& v) const { return Matrix<S, N, 1>(*this).cwiseMax(v); }
};

// array() view: coefficient-wise operations on the matrix.
template <typename S, int R, int C>
struct ArrayView {
    Matrix<S, R, C> m;
    Matrix<S, R, C> floor() const {
        Matrix<S, R, C> r;
        for (int i = 0; i < R * C; ++i) r.d[i] = std::floor(m.d[i]);
        return r;
    }
    Matrix<S, R, C> abs() const { return m.cwiseAbs(); }
    operator Matrix<S, R, C>() const { return m; }
    ArrayView operator+(S s) const {
        ArrayView r = *this;
        for (int i = 0; i < R * C; ++i) r.m.d[i] += s;
        return r;
    }
    Matrix<S, R, C> matrix() const { return m; }
};
// array() of a non-const matrix: the same view, plus in-place coefficient-wise
// compound assignment (`v.array() -= s`).
template <typename S, int R, int C>
struct ArrayRef {
    Matrix<S, R, C>& m;
    Matrix<S, R, C> floor() const { return ArrayView<S, R, C>{m}.floor(); }
    Matrix<S, R, C> abs() const { return m.cwiseAbs(); }
    operator Matrix<S, R, C>() const { return m; }
    ArrayView<S, R, C> operator+(S s) const { return ArrayView<S, R, C>{m} + s; }
    Matrix<S, R, C> matrix() const { return m; }
    ArrayRef& operator+=(S s) {
        for (int i = 0; i < R * C; ++i) m.d[i] += s;
        return *this;
    }
    ArrayRef& operator-=(S s) {
        for (int i = 0; i < R * C; ++i) m.d[i] -= s;
        return *this;
    }
};

// Comma initialiser: scalars and sub-matrices, filled row block by row block.
template <typename S, int R, int C>
struct CommaInit {
    Matrix<S, R, C>& m;
    int row = 0, col = 0, cur_rows = 1;
    template <int BR, int BC>
    void put(const Matrix<S, BR, BC>& b) {
        if (col >= C) {
            row += cur_rows;
            col = 0;
            cur_rows = BR;
        }
        if (col == 0) cur_rows = BR;
        for (int j = 0; j < BC; ++j)
            for (int i = 0; i < BR; ++i) m(row + i, col + j) = b(i, j);
        col += BC;
    }
    void put(S s) {
        Matrix<S, 1, 1> b;
        b(0, 0) = s;
        put(b);
    }
    CommaInit& operator,(S s) {
        put(s);
        return *this;
    }
    template <int BR, int BC>
    CommaInit& operator,(const Matrix<S, BR, BC>& b) {
        put(b);
        return *this;
    }
};

template <typename S, int R, int C>
class Matrix {
  public:
    static constexpr int RowsAtCompileTime = R, ColsAtCompileTime = C, SizeAtCompileTime = R * C;
    using Scalar = S;
    S d[R * C];  // column-major, as Eigen's default storage

    Matrix() {
        for (int i = 0; i < R * C; ++i) d[i] = S(0);
    }
    Matrix(S x, S y) {
        static_assert(R * C == 2, "2-vector constructor");
        d[0] = x;
        d[1] = y;
    }
    Matrix(S x, S y, S z) {
        static_assert(R * C == 3, "3-vector constructor");
        d[0] = x;
        d[1] = y;
        d[2] = z;
    }
    Matrix(S x, S y, S z, S w) {
        static_assert(R * C == 4, "4-vector constructor");
        d[0] = x;
        d[1] = y;
        d[2] = z;
        d[3] = w;
    }
    template <int BR, int BC>
    Matrix(const BlockRef<S, BR, BC, R, C>& b) : Matrix(Matrix(static_cast<Matrix>(b))) {}
    Matrix(const ArrayView<S, R, C>& a) : Matrix(a.m) {}

    static constexpr int rows() { return R; }
    static constexpr int cols() { return C; }
    static constexpr int size() { return R * C; }
    S& operator()(int i, int j) { return d[j * R + i]; }
    const S& operator()(int i, int j) const { return d[j * R + i]; }
    S& operator()(int i) { return d[i]; }
    const S& operator()(int i) const { return d[i]; }
    S& operator[](int i) { return d[i]; }
    const S& operator[](int i) const { return d[i]; }
    S& x() { return d[0]; }
    S& y() { return d[1]; }
    S& z() { return d[2]; }
    S& w() { return d[3]; }
    const S& x() const { return d[0]; }
    const S& y() const { return d[1]; }
    const S& z() const { return d[2]; }
    const S& w() const { return d[3]; }
    S* data() { return d; }
    const S* data() const { return d; }

    static Matrix Zero() { return Matrix(); }
    static Matrix Constant(S v) {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = v;
        return r;
    }
    static Matrix Ones() { return Constant(S(1)); }
    static Matrix Identity() {
        Matrix r;
        for (int i = 0; i < std::min(R, C); ++i) r(i, i) = S(1);
        return r;
    }
    static Matrix Unit(int k) {
        Matrix r;
        r.d[k] = S(1);
        return r;
    }
    static Matrix UnitX() { return Unit(0); }
    static Matrix UnitY() { return Unit(1); }
    static Matrix UnitZ() { return Unit(2); }
    static Matrix UnitW() { return Unit(3); }
    void setZero() { *this = Zero(); }
    void setIdentity() { *this = Identity(); }
    Matrix& setConstant(S v) { return *this = Constant(v); }

    // coefficient-wise arithmetic
    Matrix operator+(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = d[i] + o.d[i];
        return r;
    }
    Matrix operator-(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = d[i] - o.d[i];
        return r;
    }
    Matrix operator-() const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = -d[i];
        return r;
    }
    Matrix operator*(S s) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = d[i] * s;
        return r;
    }
    Matrix operator/(S s) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = d[i] / s;
        return r;
    }
    Matrix& operator+=(const Matrix& o) { return *this = *this + o; }
    Matrix& operator-=(const Matrix& o) { return *this = *this - o; }
    Matrix& operator*=(S s) { return *this = *this * s; }
    Matrix& operator/=(S s) { return *this = *this / s; }
    bool operator==(const Matrix& o) const {
        for (int i = 0; i < R * C; ++i)
            if (!(d[i] == o.d[i])) return false;
        return true;
    }
    bool operator!=(const Matrix& o) const { return !(*this == o); }

    // products: k summed left to right
    template <int C2>
    Matrix<S, R, C2> operator*(const Matrix<S, C, C2>& o) const {
        Matrix<S, R, C2> r;
        for (int j = 0; j < C2; ++j)
            for (int i = 0; i < R; ++i) {
                S s = (*this)(i, 0) * o(0, j);
                for (int k = 1; k < C; ++k) s += (*this)(i, k) * o(k, j);
                r(i, j) = s;
            }
        return r;
    }
    Matrix& noalias() { return *this; }
    Matrix<S, C, R> transpose() const {
        Matrix<S, C, R> r;
        for (int j = 0; j < C; ++j)
            for (int i = 0; i < R; ++i) r(j, i) = (*this)(i, j);
        return r;
    }
    S dot(const Matrix& o) const {
        S s = d[0] * o.d[0];
        for (int i = 1; i < R * C; ++i) s += d[i] * o.d[i];
        return s;
    }
    S squaredNorm() const { return dot(*this); }
    S norm() const { return std::sqrt(squaredNorm()); }
    S stableNorm() const { return norm(); }
    Matrix normalized() const {
        const S n = norm();
        return n > S(0) ? *this / n : *this;
    }
    void normalize() { *this = normalized(); }
    Matrix cross(const Matrix& o) const {
        static_assert(R * C == 3, "cross of 3-vectors");
        return Matrix(d[1] * o.d[2] - d[2] * o.d[1], d[2] * o.d[0] - d[0] * o.d[2], d[0] * o.d[1] - d[1] * o.d[0]);
    }
    S sum() const {
        S s = d[0];
        for (int i = 1; i < R * C; ++i) s += d[i];
        return s;
    }
    S prod() const {
        S s = d[0];
        for (int i = 1; i < R * C; ++i) s *= d[i];
        return s;
    }
    S mean() const { return sum() / S(R * C); }
    S maxCoeff() const {
        S s = d[0];
        for (int i = 1; i < R * C; ++i) s = std::max(s, d[i]);
        return s;
    }
    S minCoeff() const {
        S s = d[0];
        for (int i = 1; i < R * C; ++i) s = std::min(s, d[i]);
        return s;
    }
    template <typename I>
    S maxCoeff(I* idx) const {
        int b = 0;
        for (int i = 1; i < R * C; ++i)
            if (d[i] > d[b]) b = i;
        *idx = I(b);
        return d[b];
    }
    template <typename I>
    S minCoeff(I* idx) const {
        int b = 0;
        for (int i = 1; i < R * C; ++i)
            if (d[i] < d[b]) b = i;
        *idx = I(b);
        return d[b];
    }
    Matrix cwiseAbs() const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = std::abs(d[i]);
        return r;
    }
    Matrix cwiseMax(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = std::max(d[i], o.d[i]);
        return r;
    }
    Matrix cwiseMin(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = std::min(d[i], o.d[i]);
        return r;
    }
    Matrix cwiseMax(S v) const { return cwiseMax(Constant(v)); }
    Matrix cwiseMin(S v) const { return cwiseMin(Constant(v)); }
    Matrix cwiseProduct(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = d[i] * o.d[i];
        return r;
    }
    Matrix cwiseQuotient(const Matrix& o) const {
        Matrix r;
        for (int i = 0; i < R * C; ++i) r.d[i] = d[i] / o.d[i];
        return r;
    }
    ArrayView<S, R, C> array() const { return {*this}; }
    ArrayRef<S, R, C> array() { return {*this}; }
    template <typename T>
    Matrix<T, R, C> cast() const {
        Matrix<T, R, C> r;
        for (int i = 0; i < R * C; ++i) r.d[i] = static_cast<T>(d[i]);
        return r;
    }
    bool allFinite() const {
        for (int i = 0; i < R * C; ++i)
            if (!std::isfinite(d[i])) return false;
        return true;
    }
    bool hasNaN() const {
        for (int i = 0; i < R * C; ++i)
            if (std::isnan(d[i])) return true;
        return false;
    }
    bool isApprox(const Matrix& o, S prec = NumTraits<S>::dummy_precision()) const {
        return (*this - o).squaredNorm() <= prec * prec * std::min(squaredNorm(), o.squaredNorm());
    }
    bool isZero(S prec = NumTraits<S>::dummy_precision()) const {
        for (int i = 0; i < R * C; ++i)
            if (std::abs(d[i]) > prec) return false;
        return true;
    }
    DiagonalRef<S, (R < C ? R : C), R, C> diagonal() { return {*this}; }
    Matrix<S, (R < C ? R : C), 1> diagonal() const {
        Matrix<S, (R < C ? R : C), 1> r;
        for (int i = 0; i < std::min(R, C); ++i) r(i) = (*this)(i, i);
        return r;
    }
    template <int BR, int BC>
    BlockRef<S, R, C, BR, BC> topLeftCorner() {
        return {*this, 0, 0};
    }
    template <int BR, int BC>
    BlockRef<S, R, C, BR, BC> topRightCorner() {
        return {*this, 0, C - BC};
    }
    template <int BR, int BC>
    Matrix<S, BR, BC> topLeftCorner() const {
        return BlockRef<S, R, C, BR, BC>{const_cast<Matrix&>(*this), 0, 0};
    }
    template <int BR, int BC>
    Matrix<S, BR, BC> topRightCorner() const {
        return BlockRef<S, R, C, BR, BC>{const_cast<Matrix&>(*this), 0, C - BC};
    }
    template <int BR, int BC>
    BlockRef<S, R, C, BR, BC> block(int i, int j) {
        return {*this, i, j};
    }
    template <int N>
    Matrix<S, N, 1> head() const {
        Matrix<S, N, 1> r;
        for (int i = 0; i < N; ++i) r(i) = d[i];
        return r;
    }
    template <int N>
    Matrix<S, N, 1> tail() const {
        Matrix<S, N, 1> r;
        for (int i = 0; i < N; ++i) r(i) = d[R * C - N + i];
        return r;
    }
    template <int N>
    Matrix<S, N, 1> segment(int start) const {
        Matrix<S, N, 1> r;
        for (int i = 0; i < N; ++i) r(i) = d[start + i];
        return r;
    }
    S determinant() const {
        static_assert(R == C, "square");
        if constexpr (R == 1) {
            return d[0];
        } else if constexpr (R == 2) {
            return (*this)(0, 0) * (*this)(1, 1) - (*this)(0, 1) * (*this)(1, 0);
        } else if constexpr (R == 3) {
            const Matrix& m = *this;
            return m(0, 0) * (m(1, 1) * m(2, 2) - m(2, 1) * m(1, 2)) - m(1, 0) * (m(0, 1) * m(2, 2) - m(2, 1) * m(0, 2)) +
                   m(2, 0) * (m(0, 1) * m(1, 2) - m(1, 1) * m(0, 2));
        } else {
            Matrix a = *this;  // Gaussian elimination with partial pivoting
            S det = S(1);
            for (int k = 0; k < R; ++k) {
                int p = k;
                for (int i = k + 1; i < R; ++i)
                    if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
                if (a(p, k) == S(0)) return S(0);
                if (p != k) {
                    for (int j = 0; j < R; ++j) std::swap(a(k, j), a(p, j));
                    det = -det;
                }
                det *= a(k, k);
                for (int i = k + 1; i < R; ++i) {
                    const S f = a(i, k) / a(k, k);
                    for (int j = k; j < R; ++j) a(i, j) -= f * a(k, j);
                }
            }
            return det;
        }
    }
    Matrix inverse() const {  // Gauss-Jordan with partial pivoting
        static_assert(R == C, "square");
        Matrix a = *this, inv = Identity();
        for (int k = 0; k < R; ++k) {
            int p = k;
            for (int i = k + 1; i < R; ++i)
                if (std::abs(a(i, k)) > std::abs(a(p, k))) p = i;
            for (int j = 0; j < R; ++j) {
                std::swap(a(k, j), a(p, j));
                std::swap(inv(k, j), inv(p, j));
            }
            const S piv = a(k, k);
            for (int j = 0; j < R; ++j) {
                a(k, j) /= piv;
                inv(k, j) /= piv;
            }
            for (int i = 0; i < R; ++i) {
                if (i == k) continue;
                const S f = a(i, k);
                for (int j = 0; j < R; ++j) {
                    a(i, j) -= f * a(k, j);
                    inv(i, j) -= f * inv(k, j);
                }
            }
        }
        return inv;
    }
    // Orthogonal unit vector (Eigen's unitOrthogonal for 3-vectors).
    Matrix unitOrthogonal() const {
        static_assert(R * C == 3, "3-vector");
        if (!(std::abs(d[0]) <= std::abs(d[2]) * S(1e-12)) || !(std::abs(d[1]) <= std::abs(d[2]) * S(1e-12))) {
            const S invnm = S(1) / std::sqrt(d[0] * d[0] + d[1] * d[1]);
            return Matrix(-d[1] * invnm, d[0] * invnm, S(0));
        }
        const S invnm = S(1) / std::sqrt(d[1] * d[1] + d[2] * d[2]);
        return Matrix(S(0), -d[2] * invnm, d[1] * invnm);
    }
    // matrix exponential (unsupported/Eigen/MatrixFunctions): scaling and squaring of a Taylor series
    Matrix exp() const {
        static_assert(R == C, "square");
        S nrm = S(0);
        for (int i = 0; i < R * C; ++i) nrm = std::max(nrm, std::abs(d[i]));
        int sq = 0;
        while (nrm > S(0.5)) {
            nrm *= S(0.5);
            ++sq;
        }
        const Matrix a = *this / S(std::ldexp(1.0, sq));
        Matrix term = Identity(), sum = Identity();
        for (int k = 1; k < 30; ++k) {
            term = (term * a) / S(k);
            sum += term;
        }
        for (int i = 0; i < sq; ++i) sum = sum * sum;
        return sum;
    }
    CommaInit<S, R, C> operator<<(S s) {
        CommaInit<S, R, C> c{*this};
        c.put(s);
        return c;
    }
    template <int BR, int BC>
    CommaInit<S, R, C> operator<<(const Matrix<S, BR, BC>& b) {
        CommaInit<S, R, C> c{*this};
        c.put(b);
        return c;
    }
};

template <typename S, int R, int C>
Matrix<S, R, C> operator*(S s, const Matrix<S, R, C>& m) {
    Matrix<S, R, C> r;
    for (int i = 0; i < R * C; ++i) r.d[i] = s * m.d[i];
    return r;
}
template <typename S, int R, int C>
Matrix<S, R, C> operator*(int s, const Matrix<S, R, C>& m) = delete;  // (int * double-matrix: ambiguous in Eigen too)

using Matrix2d = Matrix<double, 2, 2>;
using Matrix3d = Matrix<double, 3, 3>;
using Matrix4d = Matrix<double, 4, 4>;
using Matrix3f = Matrix<float, 3, 3>;
using Vector2d = Matrix<double, 2, 1>;
using Vector3d = Matrix<double, 3, 1>;
using Vector4d = Matrix<double, 4, 1>;
using Vector3f = Matrix<float, 3, 1>;
using Vector3i = Matrix<int, 3, 1>;
using Vector2i = Matrix<int, 2, 1>;
template <typename S, int R, int C>
using MatrixBase = Matrix<S, R, C>;

// ------------------------------------------------------------------ geometry
template <typename S>
class AngleAxis;

template <typename S>
class Quaternion {
  public:
    using Scalar = S;
    Matrix<S, 4, 1> c;  // x, y, z, w (Eigen's coefficient order)
    Quaternion() : c(S(0), S(0), S(0), S(1)) {}
    Quaternion(S w, S x, S y, S z) : c(x, y, z, w) {}
    explicit Quaternion(const Matrix<S, 3, 3>& m) {  // quaternion_assign_impl (Shepperd)
        S t = m(0, 0) + m(1, 1) + m(2, 2);
        if (t > S(0)) {
            t = std::sqrt(t + S(1));
            w() = S(0.5) * t;
            t = S(0.5) / t;
            x() = (m(2, 1) - m(1, 2)) * t;
            y() = (m(0, 2) - m(2, 0)) * t;
            z() = (m(1, 0) - m(0, 1)) * t;
        } else {
            int i = 0;
            if (m(1, 1) > m(0, 0)) i = 1;
            if (m(2, 2) > m(i, i)) i = 2;
            const int j = (i + 1) % 3, k = (j + 1) % 3;
            t = std::sqrt(m(i, i) - m(j, j) - m(k, k) + S(1));
            c(i) = S(0.5) * t;
            t = S(0.5) / t;
            w() = (m(k, j) - m(j, k)) * t;
            c(j) = (m(j, i) + m(i, j)) * t;
            c(k) = (m(k, i) + m(i, k)) * t;
        }
    }
    Quaternion(const AngleAxis<S>& aa);
    static Quaternion Identity() { return Quaternion(); }
    S& x() { return c(0); }
    S& y() { return c(1); }
    S& z() { return c(2); }
    S& w() { return c(3); }
    S x() const { return c(0); }
    S y() const { return c(1); }
    S z() const { return c(2); }
    S w() const { return c(3); }
    Matrix<S, 3, 1> vec() const { return Matrix<S, 3, 1>(c(0), c(1), c(2)); }
    const Matrix<S, 4, 1>& coeffs() const { return c; }
    S dot(const Quaternion& o) const { return c.dot(o.c); }
    S squaredNorm() const { return c.squaredNorm(); }
    S norm() const { return c.norm(); }
    Quaternion normalized() const {
        Quaternion q;
        q.c = c / norm();
        return q;
    }
    void normalize() { *this = normalized(); }
    Quaternion conjugate() const { return Quaternion(w(), -x(), -y(), -z()); }
    Quaternion inverse() const {
        const S n2 = squaredNorm();
        Quaternion q = conjugate();
        q.c = q.c / n2;
        return q;
    }
    Matrix<S, 3, 3> toRotationMatrix() const {
        Matrix<S, 3, 3> res;
        const S tx = S(2) * x(), ty = S(2) * y(), tz = S(2) * z();
        const S twx = tx * w(), twy = ty * w(), twz = tz * w();
        const S txx = tx * x(), txy = ty * x(), txz = tz * x();
        const S tyy = ty * y(), tyz = tz * y(), tzz = tz * z();
        res(0, 0) = S(1) - (tyy + tzz);
        res(0, 1) = txy - twz;
        res(0, 2) = txz + twy;
        res(1, 0) = txy + twz;
        res(1, 1) = S(1) - (txx + tzz);
        res(1, 2) = tyz - twx;
        res(2, 0) = txz - twy;
        res(2, 1) = tyz + twx;
        res(2, 2) = S(1) - (txx + tyy);
        return res;
    }
    Matrix<S, 3, 3> matrix() const { return toRotationMatrix(); }
    Quaternion slerp(S t, const Quaternion& o) const {
        const S one = S(1) - NumTraits<S>::epsilon();
        const S dd = dot(o);
        const S absd = std::abs(dd);
        S s0, s1;
        if (absd >= one) {
            s0 = S(1) - t;
            s1 = t;
        } else {
            const S theta = std::acos(absd);
            const S st = std::sin(theta);
            s0 = std::sin((S(1) - t) * theta) / st;
            s1 = std::sin(t * theta) / st;
        }
        if (dd < S(0)) s1 = -s1;
        Quaternion q;
        q.c = s0 * c + s1 * o.c;
        return q;
    }
    Quaternion operator*(const Quaternion& b) const {
        const Quaternion& a = *this;
        return Quaternion(a.w() * b.w() - a.x() * b.x() - a.y() * b.y() - a.z() * b.z(),
                          a.w() * b.x() + a.x() * b.w() + a.y() * b.z() - a.z() * b.y(),
                          a.w() * b.y() + a.y() * b.w() + a.z() * b.x() - a.x() * b.z(),
                          a.w() * b.z() + a.z() * b.w() + a.x() * b.y() - a.y() * b.x());
    }
    Matrix<S, 3, 1> operator*(const Matrix<S, 3, 1>& v) const { return toRotationMatrix() * v; }
    S angularDistance(const Quaternion& o) const {
        const S dd = std::abs(dot(o));
        return S(2) * std::acos(std::min(dd, S(1)));
    }
};

template <typename S>
class AngleAxis {
  public:
    using Scalar = S;
    S m_angle = S(0);
    Matrix<S, 3, 1> m_axis{S(1), S(0), S(0)};
    AngleAxis() = default;
    AngleAxis(S angle, const Matrix<S, 3, 1>& axis) : m_angle(angle), m_axis(axis) {}
    explicit AngleAxis(const Quaternion<S>& q) { *this = q; }
    explicit AngleAxis(const Matrix<S, 3, 3>& m) { *this = Quaternion<S>(m); }
    AngleAxis& operator=(const Quaternion<S>& q) {  // AngleAxis<Scalar>::operator=(const QuaternionBase&)
        S n = q.vec().norm();
        if (n < NumTraits<S>::epsilon()) n = q.vec().stableNorm();
        if (n != S(0)) {
            m_angle = S(2) * std::atan2(n, std::abs(q.w()));
            if (q.w() < S(0)) n = -n;
            m_axis = q.vec() / n;
        } else {
            m_angle = S(0);
            m_axis = Matrix<S, 3, 1>(S(1), S(0), S(0));
        }
        return *this;
    }
    S angle() const { return m_angle; }
    const Matrix<S, 3, 1>& axis() const { return m_axis; }
    Matrix<S, 3, 3> toRotationMatrix() const {
        Matrix<S, 3, 3> res;
        const Matrix<S, 3, 1> sin_axis = std::sin(m_angle) * m_axis;
        const S cc = std::cos(m_angle);
        const Matrix<S, 3, 1> cos1_axis = (S(1) - cc) * m_axis;
        S tmp = cos1_axis.x() * m_axis.y();
        res(0, 1) = tmp - sin_axis.z();
        res(1, 0) = tmp + sin_axis.z();
        tmp = cos1_axis.x() * m_axis.z();
        res(0, 2) = tmp + sin_axis.y();
        res(2, 0) = tmp - sin_axis.y();
        tmp = cos1_axis.y() * m_axis.z();
        res(1, 2) = tmp - sin_axis.x();
        res(2, 1) = tmp + sin_axis.x();
        for (int i = 0; i < 3; ++i) res(i, i) = cos1_axis(i) * m_axis(i) + cc;
        return res;
    }
    Matrix<S, 3, 3> matrix() const { return toRotationMatrix(); }
    operator Matrix<S, 3, 3>() const { return toRotationMatrix(); }
    Quaternion<S> operator*(const AngleAxis& o) const { return Quaternion<S>(*this) * Quaternion<S>(o); }
    Quaternion<S> operator*(const Quaternion<S>& o) const { return Quaternion<S>(*this) * o; }
};

template <typename S>
Quaternion<S>::Quaternion(const AngleAxis<S>& aa) {
    const S ha = S(0.5) * aa.angle();
    w() = std::cos(ha);
    const Matrix<S, 3, 1> v = std::sin(ha) * aa.axis();
    x() = v(0);
    y() = v(1);
    z() = v(2);
}
template <typename S>
Quaternion<S> operator*(const Quaternion<S>& q, const AngleAxis<S>& a) {
    return q * Quaternion<S>(a);
}

using Quaterniond = Quaternion<double>;
using AngleAxisd = AngleAxis<double>;

// ------------------------------------------------------------------ decompositions
// LDLT (Eigen/src/Cholesky/LDLT.h): lower storage, at step k the largest
// remaining |diagonal| is swapped into place; solve applies the permutation,
// L, the pseudo-inverse of D and L^T.
template <typename M>
class LDLT {
  public:
    static constexpr int N = M::RowsAtCompileTime;
    using S = typename M::Scalar;
    LDLT() = default;
    explicit LDLT(const M& a) { compute(a); }
    LDLT& compute(const M& a) {
        m_ = a;
        for (int i = 0; i < N; ++i)
            for (int j = i + 1; j < N; ++j) m_(i, j) = m_(j, i);  // only the lower triangle is read
        bool found_zero_pivot = false, ret = true;
        S temp[N];
        for (int k = 0; k < N; ++k) {
            int big = k;
            S bigv = std::abs(m_(k, k));
            for (int i = k + 1; i < N; ++i)
                if (std::abs(m_(i, i)) > bigv) {
                    bigv = std::abs(m_(i, i));
                    big = i;
                }
            tr_[k] = big;
            if (k != big) {
                for (int j = 0; j < k; ++j) std::swap(m_(k, j), m_(big, j));
                for (int i = big + 1; i < N; ++i) std::swap(m_(i, k), m_(i, big));
                std::swap(m_(k, k), m_(big, big));
                for (int i = k + 1; i < big; ++i) {
                    const S t = m_(i, k);
                    m_(i, k) = m_(big, i);
                    m_(big, i) = t;
                }
            }
            if (k > 0) {
                for (int j = 0; j < k; ++j) temp[j] = m_(j, j) * m_(k, j);
                S dot = S(0);
                for (int j = 0; j < k; ++j) dot += m_(k, j) * temp[j];
                m_(k, k) -= dot;
                for (int i = k + 1; i < N; ++i) {
                    S s = S(0);
                    for (int j = 0; j < k; ++j) s += m_(i, j) * temp[j];
                    m_(i, k) -= s;
                }
            }
            const S akk = m_(k, k);
            const bool pivot_valid = std::abs(akk) > S(0);
            if (k == 0 && !pivot_valid) {
                for (int j = 0; j < N; ++j) {
                    tr_[j] = j;
                    for (int i = j + 1; i < N; ++i) m_(i, j) = S(0);
                }
                break;
            }
            if (k < N - 1) {
                if (pivot_valid) {
                    for (int i = k + 1; i < N; ++i) m_(i, k) /= akk;
                } else {
                    for (int i = k + 1; i < N; ++i) ret = ret && (m_(i, k) == S(0));
                }
            }
            if (found_zero_pivot && pivot_valid) ret = false;
            else if (!pivot_valid) found_zero_pivot = true;
        }
        info_ = ret ? Success : NumericalIssue;
        return *this;
    }
    ComputationInfo info() const { return info_; }
    Matrix<S, N, 1> solve(const Matrix<S, N, 1>& b) const {
        Matrix<S, N, 1> x = b;
        for (int k = 0; k < N; ++k) std::swap(x(k), x(tr_[k]));
        for (int j = 0; j < N; ++j)
            for (int i = j + 1; i < N; ++i) x(i) -= m_(i, j) * x(j);
        const S tol = std::numeric_limits<S>::min();
        for (int i = 0; i < N; ++i) x(i) = std::abs(m_(i, i)) > tol ? x(i) / m_(i, i) : S(0);
        for (int j = N - 1; j >= 0; --j)
            for (int i = 0; i < j; ++i) x(i) -= m_(j, i) * x(j);
        for (int k = N - 1; k >= 0; --k) std::swap(x(k), x(tr_[k]));
        return x;
    }

  private:
    M m_;
    int tr_[N] = {};
    ComputationInfo info_ = Success;
};

// Cyclic Jacobi eigenvalues of a symmetric matrix, ascending (as Eigen sorts them).
template <typename M>
class SelfAdjointEigenSolver {
  public:
    static constexpr int N = M::RowsAtCompileTime;
    using S = typename M::Scalar;
    explicit SelfAdjointEigenSolver(const M& a) {
        M A = a, V = M::Identity();
        for (int sweep = 0; sweep < 64; ++sweep) {
            S off = S(0), diag = S(0);
            for (int i = 0; i < N; ++i) {
                diag += A(i, i) * A(i, i);
                for (int j = i + 1; j < N; ++j) off += A(i, j) * A(i, j);
            }
            if (off == S(0) || off <= S(1e-34) * diag) break;
            for (int p = 0; p < N - 1; ++p)
                for (int q = p + 1; q < N; ++q) {
                    if (A(p, q) == S(0)) continue;
                    const S zeta = (A(q, q) - A(p, p)) / (S(2) * A(p, q));
                    const S t = std::copysign(S(1), zeta) / (std::abs(zeta) + std::sqrt(S(1) + zeta * zeta));
                    const S cs = S(1) / std::sqrt(S(1) + t * t), sn = t * cs;
                    for (int k = 0; k < N; ++k) {
                        const S kp = A(k, p), kq = A(k, q);
                        A(k, p) = cs * kp - sn * kq;
                        A(k, q) = sn * kp + cs * kq;
                    }
                    for (int k = 0; k < N; ++k) {
                        const S pk = A(p, k), qk = A(q, k);
                        A(p, k) = cs * pk - sn * qk;
                        A(q, k) = sn * pk + cs * qk;
                    }
                    for (int k = 0; k < N; ++k) {
                        const S kp = V(k, p), kq = V(k, q);
                        V(k, p) = cs * kp - sn * kq;
                        V(k, q) = sn * kp + cs * kq;
                    }
                }
        }
        int idx[N];
        for (int i = 0; i < N; ++i) idx[i] = i;
        std::sort(idx, idx + N, [&](int a_, int b_) { return A(a_, a_) < A(b_, b_); });
        for (int i = 0; i < N; ++i) {
            ev_(i) = A(idx[i], idx[i]);
            for (int k = 0; k < N; ++k) vec_(k, i) = V(k, idx[i]);
        }
    }
    const Matrix<S, N, 1>& eigenvalues() const { return ev_; }
    const M& eigenvectors() const { return vec_; }
    ComputationInfo info() const { return Success; }

  private:
    Matrix<S, N, 1> ev_;
    M vec_;
};

// JacobiSVD of a small square matrix through the symmetric eigenproblem of
// A^T A (one-sided Jacobi would do as well for AteRmse's 3x3 alignment):
// A = U S V^T with singular values descending, U completed to a rotation-free
// orthonormal basis where A is rank deficient.
template <typename M>
class JacobiSVD {
  public:
    static constexpr int N = M::RowsAtCompileTime;
    using S = typename M::Scalar;
    JacobiSVD(const M& a, unsigned = 0) {
        // one-sided Jacobi (Hestenes) on the columns of U = A V
        M U = a, V = M::Identity();
        for (int sweep = 0; sweep < 64; ++sweep) {
            bool changed = false;
            for (int p = 0; p < N - 1; ++p)
                for (int q = p + 1; q < N; ++q) {
                    S alpha = S(0), beta = S(0), gamma = S(0);
                    for (int k = 0; k < N; ++k) {
                        alpha += U(k, p) * U(k, p);
                        beta += U(k, q) * U(k, q);
                        gamma += U(k, p) * U(k, q);
                    }
                    if (std::abs(gamma) <= S(1e-15) * std::sqrt(alpha * beta) || gamma == S(0)) continue;
                    changed = true;
                    const S zeta = (beta - alpha) / (S(2) * gamma);
                    const S t = std::copysign(S(1), zeta) / (std::abs(zeta) + std::sqrt(S(1) + zeta * zeta));
                    const S cs = S(1) / std::sqrt(S(1) + t * t), sn = cs * t;
                    for (int k = 0; k < N; ++k) {
                        const S up = U(k, p), uq = U(k, q);
                        U(k, p) = cs * up - sn * uq;
                        U(k, q) = sn * up + cs * uq;
                        const S vp = V(k, p), vq = V(k, q);
                        V(k, p) = cs * vp - sn * vq;
                        V(k, q) = sn * vp + cs * vq;
                    }
                }
            if (!changed) break;
        }
        int idx[N];
        S sv[N];
        for (int i = 0; i < N; ++i) {
            idx[i] = i;
            S s2 = S(0);
            for (int k = 0; k < N; ++k) s2 += U(k, i) * U(k, i);
            sv[i] = std::sqrt(s2);
        }
        std::sort(idx, idx + N, [&](int a_, int b_) { return sv[a_] > sv[b_]; });
        for (int i = 0; i < N; ++i) {
            const int j = idx[i];
            s_(i) = sv[j];
            for (int k = 0; k < N; ++k) {
                v_(k, i) = V(k, j);
                u_(k, i) = sv[j] > S(0) ? U(k, j) / sv[j] : S(0);
            }
        }
        // complete U where singular values vanish (Gram-Schmidt against the unit basis)
        for (int i = 0; i < N; ++i) {
            if (s_(i) > S(0)) continue;
            for (int e = 0; e < N; ++e) {
                Matrix<S, N, 1> c;
                c(e) = S(1);
                for (int j = 0; j < N; ++j) {
                    if (j == i || (s_(j) == S(0) && j > i)) continue;
                    S dd = S(0);
                    for (int k = 0; k < N; ++k) dd += u_(k, j) * c(k);
                    for (int k = 0; k < N; ++k) c(k) -= dd * u_(k, j);
                }
                const S nn = c.norm();
                if (nn > S(1e-6)) {
                    for (int k = 0; k < N; ++k) u_(k, i) = c(k) / nn;
                    break;
                }
            }
        }
    }
    const M& matrixU() const { return u_; }
    const M& matrixV() const { return v_; }
    const Matrix<S, N, 1>& singularValues() const { return s_; }

  private:
    M u_, v_;
    Matrix<S, N, 1> s_;
};

}  // namespace Eigen
