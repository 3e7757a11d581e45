#pragma once
// TT-ICE* — drop-in for the reference's include/ttstream/tt_ice_star.hpp:9-59.

#include "ttstream/tt_ice.hpp"

namespace ttstream {

enum class SkipStatistic {
    kMean,
    kFullBatch,
};

struct HeuristicConfig {
    double occupancy_threshold = 0.8;
    bool skip_enabled = true;
    bool subselect_enabled = true;
    SkipStatistic skip_statistic = SkipStatistic::kMean;
    bool use_approx_tolerance = false;
};

std::vector<double> per_obs_errors(const TensorTrain& tt, const DenseTensor& y);

struct SubselectSplit {
    std::vector<Index> selected;
    std::vector<Index> rejected;
};

SubselectSplit subselect(std::span<const double> errs, double eps_des);
DenseTensor gather_obs(const DenseTensor& y, std::span<const Index> idx);
double relaxed_tolerance(const DenseTensor& y, const SubselectSplit& split, std::span<const double> errs,
                         double eps_des, bool* clamped = nullptr);
double relaxed_tolerance_approx(Index n_batch, Index n_rejected, double mean_rejected_error, double eps_des);

std::pair<TensorTrain, UpdateReport> tt_ice_star_update(const TensorTrain& tt, const DenseTensor& y, double eps_des,
                                                        const HeuristicConfig& cfg = {});
/// Device-pointer overload (drop-in extension): y_device already in GPU memory.
std::pair<TensorTrain, UpdateReport> tt_ice_star_update(const TensorTrain& tt, const double* y_device,
                                                        std::span<const Index> shape, double eps_des,
                                                        const HeuristicConfig& cfg = {});

}  // namespace ttstream
