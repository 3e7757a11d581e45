#pragma once
// TTCore / TensorTrain — drop-in for the reference's include/ttstream/tensor_train.hpp:12-124
// (the hot-path subset: container, projection, reconstruction, occupancy, norm).
//
// A TensorTrain keeps the reference's immutable host view (shared core
// buffers) and additionally carries a handle to a device-resident copy
// (ttg_tt) so a stream of updates never re-uploads: an update consumes the
// device state of its input train (if it is the latest generation) and the
// returned train owns it.  Updating a stale train re-uploads it from its host
// cores, so the functional semantics of the reference are preserved.

#include <memory>
#include <utility>
#include <vector>

#include "ttstream/dense_tensor.hpp"

namespace ttstream {

class TTCore {
public:
    TTCore(Index r_left, Index n, Index r_right, std::vector<double> data);
    static TTCore from_left_unfolding(const Matrix& u, Index r_left, Index n);
    static TTCore from_right_unfolding(const Matrix& m, Index n, Index r_right);

    Index r_left() const { return r_left_; }
    Index n() const { return n_; }
    Index r_right() const { return r_right_; }
    Index size() const { return r_left_ * n_ * r_right_; }
    MatrixMap left_unfolding() const { return MatrixMap(data(), r_left_ * n_, r_right_); }
    MatrixMap right_unfolding() const { return MatrixMap(data(), r_left_, n_ * r_right_); }
    const double* data() const { return data_->data(); }

private:
    Index r_left_, n_, r_right_;
    std::shared_ptr<const std::vector<double>> data_;
};

namespace detail {
struct DeviceTrain;  // owns a ttg_tt* on the process's device context
}

class TensorTrain {
public:
    TensorTrain(std::vector<TTCore> cores, Index ortho_count, std::vector<Index> batch_boundaries = {});

    Index num_cores() const { return static_cast<Index>(cores_.size()); }
    Index spatial_dims() const { return num_cores() - 1; }
    const TTCore& core(Index i) const { return cores_[static_cast<std::size_t>(i)]; }
    std::vector<Index> ranks() const;
    std::vector<Index> mode_sizes() const;
    std::vector<Index> spatial_shape() const;
    Index ortho_count() const { return ortho_count_; }
    bool fully_orthonormal() const { return ortho_count_ == num_cores() - 1; }
    Index obs_count() const { return cores_.back().n(); }
    const std::vector<Index>& batch_boundaries() const { return batch_boundaries_; }
    Index num_increments() const { return static_cast<Index>(batch_boundaries_.size()); }
    std::pair<Index, Index> increment_range(Index k) const;
    Index param_count() const;
    TensorTrain with_batch_boundaries(std::vector<Index> boundaries) const;
    Index measure_ortho_count(double tol = 1e-10) const;

    // --- device residency (drop-in extension) ---
    /// Device handle valid for this exact train (uploads on first use).
    std::shared_ptr<detail::DeviceTrain> device() const;
    /// Builds the host view of a device train after an in-place update.
    static TensorTrain from_device(std::shared_ptr<detail::DeviceTrain> dev);

private:
    std::vector<TTCore> cores_;
    Index ortho_count_ = 0;
    std::vector<Index> batch_boundaries_;
    mutable std::shared_ptr<detail::DeviceTrain> dev_;
    mutable std::uint64_t generation_ = 0;
};

DenseTensor tt_reconstruct(const TensorTrain& tt);
DenseTensor tt_reconstruct(const TensorTrain& tt, Index obs_begin, Index obs_end);
Matrix tt_project(const TensorTrain& tt, const DenseTensor& y);
DenseTensor tt_expand(const TensorTrain& tt, const Matrix& coeffs);
double occupancy(const TTCore& core);
double tt_norm(const TensorTrain& tt);

/// Selects the CUDA device used by the drop-in (default 0); call before the
/// first update.
void set_device(int device);

}  // namespace ttstream
