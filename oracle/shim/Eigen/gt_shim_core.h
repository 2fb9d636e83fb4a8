// oracle/shim/Eigen/gt_shim_core.h — TEST INFRASTRUCTURE ONLY.
//
// The subset of the Eigen3 API that the reference FDM oracle uses
// (/root/reference/proj/src/core/fdm.cpp:66-145, capi.cpp:315), so the
// unchanged reference core compiles where Eigen3 is absent:
//   VectorXd (Zero, [], +, -, / scalar, cwiseAbs().maxCoeff(), asDiagonal()*x)
//   SparseMatrix<double> (Triplet ctor, setFromTriplets, coeffRef)
//   ConjugateGradient<..., Lower|Upper, DiagonalPreconditioner<double>>
//   SimplicialLDLT<...>
// Solver semantics follow Eigen's published algorithms: Jacobi-preconditioned
// CG stopping on ||r||^2 < tol^2 ||b||^2 (Eigen's conjugate_gradient), info()
// == Success iff error() <= tolerance; LDLT is a dense factorisation (the
// reference only uses it for n <= 16, i.e. <= 768 unknowns).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <stdexcept>
#include <vector>

namespace Eigen {

enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };
enum UpLoType { Lower = 1, Upper = 2 };

class VectorXd;

class DiagonalWrapper {
public:
    explicit DiagonalWrapper(const VectorXd& d) : d_(d) {}
    VectorXd operator*(const VectorXd& x) const;

private:
    const VectorXd& d_;
};

class VectorXd {
public:
    VectorXd() = default;
    explicit VectorXd(std::ptrdiff_t n) : v_(static_cast<size_t>(n), 0.0) {}
    static VectorXd Zero(std::ptrdiff_t n) { return VectorXd(n); }
    static VectorXd Constant(std::ptrdiff_t n, double c) {
        VectorXd r(n);
        std::fill(r.v_.begin(), r.v_.end(), c);
        return r;
    }
    void resize(std::ptrdiff_t n) { v_.assign(static_cast<size_t>(n), 0.0); }
    void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }
    std::ptrdiff_t size() const { return static_cast<std::ptrdiff_t>(v_.size()); }
    std::ptrdiff_t rows() const { return size(); }
    double& operator[](std::ptrdiff_t i) { return v_[static_cast<size_t>(i)]; }
    double operator[](std::ptrdiff_t i) const { return v_[static_cast<size_t>(i)]; }
    double& operator()(std::ptrdiff_t i) { return v_[static_cast<size_t>(i)]; }
    double operator()(std::ptrdiff_t i) const { return v_[static_cast<size_t>(i)]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }

    VectorXd cwiseAbs() const {
        VectorXd r = *this;
        for (double& x : r.v_) x = std::abs(x);
        return r;
    }
    double maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }
    double minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }
    double squaredNorm() const {
        double s = 0.0;
        for (double x : v_) s += x * x;
        return s;
    }
    double norm() const { return std::sqrt(squaredNorm()); }
    double dot(const VectorXd& o) const {
        double s = 0.0;
        for (size_t i = 0; i < v_.size(); ++i) s += v_[i] * o.v_[i];
        return s;
    }
    DiagonalWrapper asDiagonal() const { return DiagonalWrapper(*this); }

    VectorXd& operator+=(const VectorXd& o) {
        check(o);
        for (size_t i = 0; i < v_.size(); ++i) v_[i] += o.v_[i];
        return *this;
    }
    VectorXd& operator-=(const VectorXd& o) {
        check(o);
        for (size_t i = 0; i < v_.size(); ++i) v_[i] -= o.v_[i];
        return *this;
    }
    VectorXd& operator*=(double s) {
        for (double& x : v_) x *= s;
        return *this;
    }
    VectorXd& operator/=(double s) {
        for (double& x : v_) x /= s;
        return *this;
    }
    friend VectorXd operator+(VectorXd a, const VectorXd& b) { return a += b; }
    friend VectorXd operator-(VectorXd a, const VectorXd& b) { return a -= b; }
    friend VectorXd operator*(VectorXd a, double s) { return a *= s; }
    friend VectorXd operator*(double s, VectorXd a) { return a *= s; }
    friend VectorXd operator/(VectorXd a, double s) { return a /= s; }

private:
    void check(const VectorXd& o) const {
        if (o.v_.size() != v_.size()) throw std::runtime_error("Eigen shim: size mismatch");
    }
    std::vector<double> v_;
};

inline VectorXd DiagonalWrapper::operator*(const VectorXd& x) const {
    VectorXd r(x.size());
    for (std::ptrdiff_t i = 0; i < x.size(); ++i) r[i] = d_[i] * x[i];
    return r;
}

template <typename Scalar>
class Triplet {
public:
    Triplet(int r, int c, Scalar v) : r_(r), c_(c), v_(v) {}
    int row() const { return r_; }
    int col() const { return c_; }
    Scalar value() const { return v_; }

private:
    int r_, c_;
    Scalar v_;
};

// Compressed-row sparse matrix; duplicate triplets are summed (Eigen semantics).
template <typename Scalar>
class SparseMatrix {
public:
    SparseMatrix() = default;
    SparseMatrix(std::ptrdiff_t rows, std::ptrdiff_t cols)
        : rows_(rows), cols_(cols), ptr_(static_cast<size_t>(rows) + 1, 0) {}

    std::ptrdiff_t rows() const { return rows_; }
    std::ptrdiff_t cols() const { return cols_; }
    std::ptrdiff_t nonZeros() const { return static_cast<std::ptrdiff_t>(val_.size()); }

    template <typename It>
    void setFromTriplets(It begin, It end) {
        std::vector<size_t> cnt(static_cast<size_t>(rows_) + 1, 0);
        for (It it = begin; it != end; ++it) ++cnt[static_cast<size_t>(it->row()) + 1];
        for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
        std::vector<int> col(cnt.back());
        std::vector<Scalar> val(cnt.back());
        std::vector<size_t> fill(cnt.begin(), cnt.end() - 1);
        for (It it = begin; it != end; ++it) {
            size_t k = fill[static_cast<size_t>(it->row())]++;
            col[k] = it->col();
            val[k] = it->value();
        }
        ptr_.assign(static_cast<size_t>(rows_) + 1, 0);
        col_.clear();
        val_.clear();
        for (std::ptrdiff_t r = 0; r < rows_; ++r) {
            std::vector<std::pair<int, Scalar>> row;
            for (size_t k = cnt[r]; k < cnt[r + 1]; ++k) row.emplace_back(col[k], val[k]);
            std::stable_sort(row.begin(), row.end(),
                             [](const auto& a, const auto& b) { return a.first < b.first; });
            for (size_t k = 0; k < row.size(); ++k) {
                if (!col_.empty() && col_.size() > ptr_[r] && col_.back() == row[k].first)
                    val_.back() += row[k].second;
                else {
                    col_.push_back(row[k].first);
                    val_.push_back(row[k].second);
                }
            }
            ptr_[r + 1] = col_.size();
        }
    }

    Scalar& coeffRef(std::ptrdiff_t r, std::ptrdiff_t c) {
        for (size_t k = ptr_[r]; k < ptr_[r + 1]; ++k)
            if (col_[k] == c) return val_[k];
        // Insert (rare path; the reference only touches existing diagonals).
        size_t pos = ptr_[r];
        while (pos < ptr_[r + 1] && col_[pos] < c) ++pos;
        col_.insert(col_.begin() + static_cast<std::ptrdiff_t>(pos), static_cast<int>(c));
        val_.insert(val_.begin() + static_cast<std::ptrdiff_t>(pos), Scalar(0));
        for (size_t i = static_cast<size_t>(r) + 1; i < ptr_.size(); ++i) ++ptr_[i];
        return val_[pos];
    }

    Scalar coeff(std::ptrdiff_t r, std::ptrdiff_t c) const {
        for (size_t k = ptr_[r]; k < ptr_[r + 1]; ++k)
            if (col_[k] == c) return val_[k];
        return Scalar(0);
    }

    VectorXd operator*(const VectorXd& x) const {
        VectorXd y(rows_);
        for (std::ptrdiff_t r = 0; r < rows_; ++r) {
            double s = 0.0;
            for (size_t k = ptr_[r]; k < ptr_[r + 1]; ++k) s += val_[k] * x[col_[k]];
            y[r] = s;
        }
        return y;
    }

    const std::vector<size_t>& outer() const { return ptr_; }
    const std::vector<int>& inner() const { return col_; }
    const std::vector<Scalar>& values() const { return val_; }

private:
    std::ptrdiff_t rows_ = 0, cols_ = 0;
    std::vector<size_t> ptr_;
    std::vector<int> col_;
    std::vector<Scalar> val_;
};

template <typename Scalar>
class DiagonalPreconditioner {};

template <typename MatrixType, int UpLo = Lower, typename Precond = DiagonalPreconditioner<double>>
class ConjugateGradient {
public:
    ConjugateGradient() = default;
    ConjugateGradient& setTolerance(double t) {
        tol_ = t;
        return *this;
    }
    ConjugateGradient& setMaxIterations(int it) {
        max_it_ = it;
        return *this;
    }
    ConjugateGradient& compute(const MatrixType& a) {
        a_ = &a;
        inv_diag_ = VectorXd(a.rows());
        for (std::ptrdiff_t i = 0; i < a.rows(); ++i) {
            double d = a.coeff(i, i);
            inv_diag_[i] = d != 0.0 ? 1.0 / d : 1.0;
        }
        return *this;
    }
    VectorXd solve(const VectorXd& b) { return solveWithGuess(b, VectorXd::Zero(b.size())); }
    VectorXd solveWithGuess(const VectorXd& b, const VectorXd& guess) {
        const MatrixType& a = *a_;
        VectorXd x = guess;
        VectorXd r = b - a * x;
        const double rhs2 = b.squaredNorm();
        iters_ = 0;
        if (rhs2 == 0.0) {
            x.setZero();
            err_ = 0.0;
            info_ = Success;
            return x;
        }
        const double threshold = std::max(tol_ * tol_ * rhs2, 1e-300);
        double res2 = r.squaredNorm();
        if (res2 < threshold) {
            err_ = std::sqrt(res2 / rhs2);
            info_ = Success;
            return x;
        }
        VectorXd p = inv_diag_.asDiagonal() * r;
        double abs_new = r.dot(p);
        int i = 0;
        while (i < max_it_) {
            VectorXd tmp = a * p;
            double alpha = abs_new / p.dot(tmp);
            for (std::ptrdiff_t k = 0; k < x.size(); ++k) {
                x[k] += alpha * p[k];
                r[k] -= alpha * tmp[k];
            }
            res2 = r.squaredNorm();
            if (res2 < threshold) break;
            VectorXd z = inv_diag_.asDiagonal() * r;
            double abs_old = abs_new;
            abs_new = r.dot(z);
            double beta = abs_new / abs_old;
            for (std::ptrdiff_t k = 0; k < p.size(); ++k) p[k] = z[k] + beta * p[k];
            ++i;
        }
        err_ = std::sqrt(res2 / rhs2);
        iters_ = i;
        info_ = err_ <= tol_ ? Success : NoConvergence;
        return x;
    }
    ComputationInfo info() const { return info_; }
    double error() const { return err_; }
    int iterations() const { return iters_; }

private:
    const MatrixType* a_ = nullptr;
    VectorXd inv_diag_;
    double tol_ = 1e-16;
    int max_it_ = 1 << 30;
    double err_ = 0.0;
    int iters_ = 0;
    ComputationInfo info_ = Success;
};

// Dense LDL^T of a (small) symmetric positive definite sparse matrix.
template <typename MatrixType>
class SimplicialLDLT {
public:
    explicit SimplicialLDLT(const MatrixType& a) : n_(a.rows()) {
        l_.assign(static_cast<size_t>(n_) * n_, 0.0);
        d_.assign(static_cast<size_t>(n_), 0.0);
        std::vector<double> dense(static_cast<size_t>(n_) * n_, 0.0);
        for (std::ptrdiff_t r = 0; r < n_; ++r)
            for (size_t k = a.outer()[r]; k < a.outer()[r + 1]; ++k)
                dense[static_cast<size_t>(r) * n_ + a.inner()[k]] += a.values()[k];
        for (std::ptrdiff_t j = 0; j < n_; ++j) {
            double dj = dense[static_cast<size_t>(j) * n_ + j];
            for (std::ptrdiff_t k = 0; k < j; ++k) {
                double ljk = l_[static_cast<size_t>(j) * n_ + k];
                dj -= ljk * ljk * d_[k];
            }
            if (!(std::abs(dj) > 0.0)) {
                info_ = NumericalIssue;
                return;
            }
            d_[j] = dj;
            l_[static_cast<size_t>(j) * n_ + j] = 1.0;
            for (std::ptrdiff_t i = j + 1; i < n_; ++i) {
                double s = dense[static_cast<size_t>(i) * n_ + j];
                for (std::ptrdiff_t k = 0; k < j; ++k)
                    s -= l_[static_cast<size_t>(i) * n_ + k] * l_[static_cast<size_t>(j) * n_ + k] *
                         d_[k];
                l_[static_cast<size_t>(i) * n_ + j] = s / dj;
            }
        }
    }
    ComputationInfo info() const { return info_; }
    VectorXd solve(const VectorXd& b) const {
        VectorXd y = b;
        for (std::ptrdiff_t i = 0; i < n_; ++i)
            for (std::ptrdiff_t k = 0; k < i; ++k) y[i] -= l_[static_cast<size_t>(i) * n_ + k] * y[k];
        for (std::ptrdiff_t i = 0; i < n_; ++i) y[i] /= d_[i];
        for (std::ptrdiff_t i = n_ - 1; i >= 0; --i)
            for (std::ptrdiff_t k = i + 1; k < n_; ++k) y[i] -= l_[static_cast<size_t>(k) * n_ + i] * y[k];
        return y;
    }

private:
    std::ptrdiff_t n_;
    std::vector<double> l_, d_;
    ComputationInfo info_ = Success;
};

}  // namespace Eigen
