#pragma once
// DenseTensor — drop-in for the reference's include/ttstream/dense_tensor.hpp:23-58.
//
// Eigen is not available on this platform, so Matrix / MatrixMap are a minimal
// column-major replacement exposing the subset the public API uses (rows, cols,
// size, data, operator()(i, j), element access).  Layout is identical to
// Eigen::MatrixXd (first-index-fastest), so a reference caller's buffers move
// across unchanged.

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "ttstream/errors.hpp"

namespace ttstream {

using Index = std::int64_t;

/// Owning column-major matrix (stand-in for Eigen::MatrixXd).
class Matrix {
public:
    Matrix() = default;
    Matrix(Index rows, Index cols) : rows_(rows), cols_(cols), data_(static_cast<std::size_t>(rows * cols), 0.0) {}
    Matrix(Index rows, Index cols, std::vector<double> data);
    static Matrix Zero(Index rows, Index cols) { return Matrix(rows, cols); }
    static Matrix Identity(Index rows, Index cols);

    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    double* data() { return data_.data(); }
    const double* data() const { return data_.data(); }
    double& operator()(Index i, Index j) { return data_[static_cast<std::size_t>(i + rows_ * j)]; }
    double operator()(Index i, Index j) const { return data_[static_cast<std::size_t>(i + rows_ * j)]; }
    double norm() const;

private:
    Index rows_ = 0, cols_ = 0;
    std::vector<double> data_;
};

/// Non-owning const column-major view (stand-in for Eigen::Map<const MatrixXd>).
class MatrixMap {
public:
    MatrixMap(const double* data, Index rows, Index cols) : data_(data), rows_(rows), cols_(cols) {}
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    const double* data() const { return data_; }
    double operator()(Index i, Index j) const { return data_[i + rows_ * j]; }
    Matrix eval() const;
    operator Matrix() const { return eval(); }

private:
    const double* data_;
    Index rows_, cols_;
};

/// Immutable dense multiway array of doubles, first-index-fastest; the buffer
/// is shared between views (dense_tensor.hpp:18-22).
class DenseTensor {
public:
    /// Takes ownership of `data`; validates extents, length and finiteness.
    DenseTensor(std::vector<Index> shape, std::vector<double> data);
    static DenseTensor zeros(std::vector<Index> shape);

    const std::vector<Index>& shape() const { return shape_; }
    Index ndim() const { return static_cast<Index>(shape_.size()); }
    Index size() const { return static_cast<Index>(data_->size()); }
    Index extent(Index i) const { return shape_[static_cast<std::size_t>(i)]; }
    const double* data() const { return data_->data(); }
    std::span<const double> values() const { return {data_->data(), data_->size()}; }
    double at(std::span<const Index> idx) const;
    DenseTensor reshape(std::vector<Index> new_shape) const;
    MatrixMap unfold(Index i) const;
    MatrixMap as_matrix(Index rows, Index cols) const;
    double frobenius_norm() const;

private:
    DenseTensor(std::vector<Index> shape, std::shared_ptr<const std::vector<double>> data);
    std::vector<Index> shape_;
    std::shared_ptr<const std::vector<double>> data_;
};

Index shape_product(std::span<const Index> shape);
DenseTensor tensor_from_matrix(const Matrix& m, std::vector<Index> shape);

}  // namespace ttstream
