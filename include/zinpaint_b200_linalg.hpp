/*
 * zinpaint_b200_linalg.hpp -- the dense vector / matrix value types of the C++ drop-in.
 *
 * The reference's pca_model stores Eigen::VectorXd / Eigen::MatrixXd
 * (proj/include/zinpaint/pca.hpp:14-16).  When Eigen is installed the drop-in uses it directly;
 * otherwise this header provides the subset of that interface the reference's callers use on a
 * pca_model (element access, size, data(), equality), and `namespace Eigen` is aliased to it so
 * code written against the reference (`Eigen::VectorXd x(n); x[i] = ...; x.data()`) compiles
 * unchanged.  Storage is column-major like Eigen's default.  It is a container, not a linear
 * algebra library: the PCA arithmetic itself runs on the GPU.
 */
#ifndef ZINPAINT_B200_LINALG_HPP
#define ZINPAINT_B200_LINALG_HPP

#include <cstddef>
#include <vector>

namespace zinpaint {
namespace b200_linalg {

class VectorXd {
public:
    VectorXd() = default;
    explicit VectorXd(long n) : v_(static_cast<std::size_t>(n), 0.0) {}
    long size() const { return static_cast<long>(v_.size()); }
    long rows() const { return size(); }
    long cols() const { return 1; }
    double& operator[](long i) { return v_[static_cast<std::size_t>(i)]; }
    double operator[](long i) const { return v_[static_cast<std::size_t>(i)]; }
    double& operator()(long i) { return v_[static_cast<std::size_t>(i)]; }
    double operator()(long i) const { return v_[static_cast<std::size_t>(i)]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    void resize(long n) { v_.assign(static_cast<std::size_t>(n), 0.0); }
    friend bool operator==(const VectorXd& a, const VectorXd& b) { return a.v_ == b.v_; }
    friend bool operator!=(const VectorXd& a, const VectorXd& b) { return a.v_ != b.v_; }

private:
    std::vector<double> v_;
};

class MatrixXd {
public:
    MatrixXd() = default;
    MatrixXd(long rows, long cols) : r_(rows), c_(cols), v_(static_cast<std::size_t>(rows * cols), 0.0) {}
    long rows() const { return r_; }
    long cols() const { return c_; }
    long size() const { return r_ * c_; }
    double& operator()(long r, long c) { return v_[static_cast<std::size_t>(c * r_ + r)]; }
    double operator()(long r, long c) const { return v_[static_cast<std::size_t>(c * r_ + r)]; }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    void resize(long rows, long cols) {
        r_ = rows;
        c_ = cols;
        v_.assign(static_cast<std::size_t>(rows * cols), 0.0);
    }
    friend bool operator==(const MatrixXd& a, const MatrixXd& b) {
        return a.r_ == b.r_ && a.c_ == b.c_ && a.v_ == b.v_;
    }
    friend bool operator!=(const MatrixXd& a, const MatrixXd& b) { return !(a == b); }

private:
    long r_ = 0, c_ = 0;
    std::vector<double> v_;
};

}  // namespace b200_linalg
}  // namespace zinpaint

namespace Eigen = zinpaint::b200_linalg;

#endif /* ZINPAINT_B200_LINALG_HPP */
