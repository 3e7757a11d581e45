#pragma once
// TT-ICE — drop-in for the reference's include/ttstream/tt_ice.hpp:10-49.
// Same signatures; the sweep runs on the B200 through the ttg C ABI.

#include <span>

#include "ttstream/tensor_train.hpp"

namespace ttstream {

struct UpdateReport {
    Index increment_index = 0;
    Index obs_in_batch = 0;
    Index obs_used = 0;
    std::vector<Index> ranks_before;
    std::vector<Index> ranks_after;
    double eps_target = 0.0;
    double batch_rel_error_estimate = 0.0;
    double seconds = 0.0;  ///< wall time of the device update (CUDA events)
    bool tolerance_clamped = false;
};

Matrix compute_residual(const Matrix& u_pad, const Matrix& y);
Matrix pad_core(const Matrix& u_next, Index r_left_old, Index added_rank);

std::pair<TensorTrain, UpdateReport> tt_ice_update(const TensorTrain& tt, const DenseTensor& y, double eps_des);
std::pair<TensorTrain, UpdateReport> tt_ice_update_with_tolerances(const TensorTrain& tt, const DenseTensor& y,
                                                                   std::span<const double> deltas);
std::pair<TensorTrain, UpdateReport> tt_ice_bootstrap(const DenseTensor& y, double eps_des);

/// Device-pointer overloads (drop-in extension): y_device is a
/// first-index-fastest float64 increment already in GPU memory (no PCIe copy).
/// The library stream is non-blocking: a y_device written on another CUDA
/// stream must be complete or ordered first (ttg_ctx_wait_stream, ttg.h).
std::pair<TensorTrain, UpdateReport> tt_ice_update(const TensorTrain& tt, const double* y_device,
                                                   std::span<const Index> shape, double eps_des);
std::pair<TensorTrain, UpdateReport> tt_ice_bootstrap(const double* y_device, std::span<const Index> shape,
                                                      double eps_des);

}  // namespace ttstream
