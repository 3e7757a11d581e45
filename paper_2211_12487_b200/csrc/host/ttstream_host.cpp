// ttstream_host.cpp — C++ host mirror of the reference's public API
// (reference include/ttstream/{dense_tensor,tensor_train,tt_ice,tt_ice_star}.hpp)
// implemented over the ttg C ABI (include/ttg.h).  The numerics of the update,
// projection and reconstruction run on the B200; this file holds the host
// containers, argument validation, and the cheap public helpers the reference
// exposes (subselect, relaxed tolerances, pad_core, compute_residual).
#include <algorithm>
#include <cmath>
#include <mutex>
#include <numeric>
#include <sstream>

#include "ttg.h"
#include "ttstream/tt_ice_star.hpp"
#include "ttstream/metrics.hpp"
#include "ttstream/serialization.hpp"
#include "ttstream/stream_io.hpp"

namespace ttstream {

// ---------------------------------------------------------------------------
// errors / device context
// ---------------------------------------------------------------------------
namespace detail {

[[noreturn]] void throw_status(int st, const std::string& msg) {
    switch (st) {
        case TTG_E_DIMENSION: throw DimensionError(msg);
        case TTG_E_NUMERIC: throw NumericError(msg);
        case TTG_E_STATE: throw StateError(msg);
        case TTG_E_FORMAT: throw FormatError(msg);
        case TTG_E_INDEX: throw IndexError(msg);
        case TTG_E_CONFIG: throw ConfigError(msg);
        case TTG_E_RESOURCE: throw ResourceError(msg);
        default: throw DeviceError(msg.empty() ? "ttg device failure" : msg);
    }
}

namespace {
int g_device = 0;
std::mutex g_mu;
ttg_ctx* g_ctx = nullptr;
}  // namespace

ttg_ctx* context() {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!g_ctx) {
        int rc = ttg_ctx_create(g_device, &g_ctx);
        if (rc != TTG_OK) throw_status(rc, "could not create the CUDA context (no CUDA device / libttg missing?)");
    }
    return g_ctx;
}

void check(int rc) {
    if (rc != TTG_OK) throw_status(rc, ttg_last_error(g_ctx));
}

struct DeviceTrain {
    ttg_tt* h = nullptr;
    std::uint64_t generation = 1;
    ~DeviceTrain() {
        if (h) ttg_tt_destroy(h);
    }
};

// An update that fails part-way leaves the device train unusable for the
// input's generation: invalidate it so the next use re-uploads the host cores.
template <class F>
void run_update(const std::shared_ptr<DeviceTrain>& dev, F&& f) {
    try {
        f();
    } catch (...) {
        dev->generation += 2;
        throw;
    }
}

}  // namespace detail

void set_device(int device) {
    std::lock_guard<std::mutex> lk(detail::g_mu);
    if (detail::g_ctx) throw StateError("set_device must be called before the first device operation");
    detail::g_device = device;
}

// ---------------------------------------------------------------------------
// Matrix / DenseTensor (dense_tensor.cpp:34-171)
// ---------------------------------------------------------------------------
Matrix::Matrix(Index rows, Index cols, std::vector<double> data) : rows_(rows), cols_(cols), data_(std::move(data)) {
    if (static_cast<Index>(data_.size()) != rows * cols) throw DimensionError("matrix buffer length mismatch");
}

Matrix Matrix::Identity(Index rows, Index cols) {
    Matrix m(rows, cols);
    for (Index i = 0; i < std::min(rows, cols); ++i) m(i, i) = 1.0;
    return m;
}

double Matrix::norm() const {
    double s = 0.0;
    for (double v : data_) s += v * v;
    return std::sqrt(s);
}

Matrix MatrixMap::eval() const {
    return Matrix(rows_, cols_, std::vector<double>(data_, data_ + rows_ * cols_));
}

namespace {
void validate_extents(std::span<const Index> shape) {
    for (Index n : shape)
        if (n < 1) throw DimensionError("tensor extent must be >= 1");
}
}  // namespace

Index shape_product(std::span<const Index> shape) {
    return std::accumulate(shape.begin(), shape.end(), Index{1}, std::multiplies<>());
}

DenseTensor::DenseTensor(std::vector<Index> shape, std::vector<double> data) : shape_(std::move(shape)) {
    validate_extents(shape_);
    if (static_cast<Index>(data.size()) != shape_product(shape_)) {
        throw DimensionError("buffer length does not match shape");
    }
    for (double v : data)
        if (!std::isfinite(v)) throw NumericError("non-finite element rejected at tensor construction");
    data_ = std::make_shared<const std::vector<double>>(std::move(data));
}

DenseTensor::DenseTensor(std::vector<Index> shape, std::shared_ptr<const std::vector<double>> data)
    : shape_(std::move(shape)), data_(std::move(data)) {}

DenseTensor DenseTensor::zeros(std::vector<Index> shape) {
    validate_extents(shape);
    const Index n = shape_product(shape);
    return DenseTensor(std::move(shape), std::vector<double>(static_cast<std::size_t>(n), 0.0));
}

double DenseTensor::at(std::span<const Index> idx) const {
    if (static_cast<Index>(idx.size()) != ndim()) throw DimensionError("index arity does not match tensor order");
    Index lin = 0, stride = 1;
    for (std::size_t i = 0; i < idx.size(); ++i) {
        if (idx[i] < 0 || idx[i] >= shape_[i]) throw IndexError("tensor index out of range");
        lin += idx[i] * stride;
        stride *= shape_[i];
    }
    return (*data_)[static_cast<std::size_t>(lin)];
}

DenseTensor DenseTensor::reshape(std::vector<Index> new_shape) const {
    validate_extents(new_shape);
    if (shape_product(new_shape) != size()) throw DimensionError("cannot reshape: extent products differ");
    return DenseTensor(std::move(new_shape), data_);
}

MatrixMap DenseTensor::unfold(Index i) const {
    if (i < 1 || i > ndim() - 1) throw DimensionError("unfolding mode out of range");
    const auto split = static_cast<std::size_t>(i);
    return MatrixMap(data(), shape_product({shape_.data(), split}),
                     shape_product({shape_.data() + split, shape_.size() - split}));
}

MatrixMap DenseTensor::as_matrix(Index rows, Index cols) const {
    if (rows * cols != size()) throw DimensionError("matrix view extents do not cover the buffer");
    return MatrixMap(data(), rows, cols);
}

double DenseTensor::frobenius_norm() const {
    double s = 0.0;
    for (double v : *data_) s += v * v;
    return std::sqrt(s);
}

DenseTensor tensor_from_matrix(const Matrix& m, std::vector<Index> shape) {
    return DenseTensor(std::move(shape), std::vector<double>(m.data(), m.data() + m.size()));
}

// ---------------------------------------------------------------------------
// TTCore / TensorTrain (tensor_train.cpp:12-146)
// ---------------------------------------------------------------------------
TTCore::TTCore(Index r_left, Index n, Index r_right, std::vector<double> data)
    : r_left_(r_left), n_(n), r_right_(r_right) {
    if (r_left < 1 || n < 1 || r_right < 1) throw DimensionError("core extents must be >= 1");
    if (static_cast<Index>(data.size()) != size()) throw DimensionError("core buffer length does not match extents");
    for (double v : data)
        if (!std::isfinite(v)) throw NumericError("non-finite element rejected at core construction");
    data_ = std::make_shared<const std::vector<double>>(std::move(data));
}

TTCore TTCore::from_left_unfolding(const Matrix& u, Index r_left, Index n) {
    if (u.rows() != r_left * n) throw DimensionError("left unfolding rows do not factor as r_left * n");
    return TTCore(r_left, n, u.cols(), std::vector<double>(u.data(), u.data() + u.size()));
}

TTCore TTCore::from_right_unfolding(const Matrix& m, Index n, Index r_right) {
    if (m.cols() != n * r_right) throw DimensionError("right unfolding columns do not factor as n * r_right");
    return TTCore(m.rows(), n, r_right, std::vector<double>(m.data(), m.data() + m.size()));
}

TensorTrain::TensorTrain(std::vector<TTCore> cores, Index ortho_count, std::vector<Index> batch_boundaries)
    : cores_(std::move(cores)), ortho_count_(ortho_count), batch_boundaries_(std::move(batch_boundaries)) {
    if (cores_.empty()) throw DimensionError("a train needs at least one core");
    if (cores_.front().r_left() != 1 || cores_.back().r_right() != 1) throw DimensionError("boundary ranks must be 1");
    for (std::size_t i = 0; i + 1 < cores_.size(); ++i) {
        if (cores_[i].r_right() != cores_[i + 1].r_left()) {
            std::ostringstream os;
            os << "bond rank mismatch between cores " << i << " and " << i + 1;
            throw DimensionError(os.str());
        }
    }
    if (ortho_count_ < 0 || ortho_count_ > num_cores() - 1) throw StateError("ortho_count outside [0, D-1]");
    if (batch_boundaries_.empty()) batch_boundaries_.push_back(obs_count());
    Index prev = 0;
    for (Index b : batch_boundaries_) {
        if (b < prev) throw DimensionError("batch boundaries must be nondecreasing");
        prev = b;
    }
    if (batch_boundaries_.back() != obs_count()) throw DimensionError("batch boundaries must end at the observation count");
}

std::vector<Index> TensorTrain::ranks() const {
    std::vector<Index> r{cores_.front().r_left()};
    for (const auto& c : cores_) r.push_back(c.r_right());
    return r;
}
std::vector<Index> TensorTrain::mode_sizes() const {
    std::vector<Index> n;
    for (const auto& c : cores_) n.push_back(c.n());
    return n;
}
std::vector<Index> TensorTrain::spatial_shape() const {
    std::vector<Index> n;
    for (std::size_t i = 0; i + 1 < cores_.size(); ++i) n.push_back(cores_[i].n());
    return n;
}
std::pair<Index, Index> TensorTrain::increment_range(Index k) const {
    if (k < 0 || k >= num_increments()) throw IndexError("increment index out of range");
    const Index begin = (k == 0) ? 0 : batch_boundaries_[static_cast<std::size_t>(k - 1)];
    return {begin, batch_boundaries_[static_cast<std::size_t>(k)]};
}
Index TensorTrain::param_count() const {
    Index t = 0;
    for (const auto& c : cores_) t += c.size();
    return t;
}
TensorTrain TensorTrain::with_batch_boundaries(std::vector<Index> boundaries) const {
    return TensorTrain(cores_, ortho_count_, std::move(boundaries));
}
Index TensorTrain::measure_ortho_count(double tol) const {
    Index count = 0;
    for (Index i = 0; i < num_cores() - 1; ++i) {
        const auto u = core(i).left_unfolding();
        double dev = 0.0;
        for (Index a = 0; a < u.cols(); ++a)
            for (Index b = 0; b < u.cols(); ++b) {
                double s = 0.0;
                for (Index r = 0; r < u.rows(); ++r) s += u(r, a) * u(r, b);
                dev = std::max(dev, std::fabs(s - (a == b ? 1.0 : 0.0)));
            }
        if (dev > tol) break;
        ++count;
    }
    return count;
}

std::shared_ptr<detail::DeviceTrain> TensorTrain::device() const {
    if (dev_ && dev_->generation == generation_) return dev_;
    ttg_ctx* ctx = detail::context();
    const int nc = static_cast<int>(cores_.size());
    std::vector<int64_t> rl(nc), nn(nc), rr(nc);
    std::vector<const double*> ptr(nc);
    for (int i = 0; i < nc; ++i) {
        rl[i] = cores_[i].r_left();
        nn[i] = cores_[i].n();
        rr[i] = cores_[i].r_right();
        ptr[i] = cores_[i].data();
    }
    auto d = std::make_shared<detail::DeviceTrain>();
    detail::check(ttg_tt_upload(ctx, nc, rl.data(), nn.data(), rr.data(), ptr.data(), ortho_count_,
                                batch_boundaries_.data(), static_cast<int64_t>(batch_boundaries_.size()), &d->h));
    dev_ = d;
    generation_ = d->generation;
    return dev_;
}

TensorTrain TensorTrain::from_device(std::shared_ptr<detail::DeviceTrain> dev) {
    ttg_ctx* ctx = detail::context();
    const int nc = ttg_tt_num_cores(dev->h);
    std::vector<int64_t> ranks(nc + 1), modes(nc);
    int64_t oc = 0, nb = 0;
    detail::check(ttg_tt_shape(dev->h, ranks.data(), modes.data(), &oc, &nb));
    std::vector<int64_t> bounds(static_cast<std::size_t>(nb));
    detail::check(ttg_tt_bounds(dev->h, bounds.data()));
    std::vector<TTCore> cores;
    for (int i = 0; i < nc; ++i) {
        std::vector<double> buf(static_cast<std::size_t>(ranks[i] * modes[i] * ranks[i + 1]));
        detail::check(ttg_tt_download_core(ctx, dev->h, i, buf.data()));
        cores.emplace_back(ranks[i], modes[i], ranks[i + 1], std::move(buf));
    }
    TensorTrain out(std::move(cores), oc, std::vector<Index>(bounds.begin(), bounds.end()));
    dev->generation++;
    out.dev_ = dev;
    out.generation_ = dev->generation;
    return out;
}

namespace {
struct Shape {
    std::vector<int64_t> v;
    explicit Shape(const DenseTensor& y) : v(y.shape().begin(), y.shape().end()) {}
};

UpdateReport to_report(const ttg_report& r) {
    UpdateReport o;
    o.increment_index = r.increment_index;
    o.obs_in_batch = r.obs_in_batch;
    o.obs_used = r.obs_used;
    o.ranks_before.assign(r.ranks_before, r.ranks_before + r.n_ranks);
    o.ranks_after.assign(r.ranks_after, r.ranks_after + r.n_ranks);
    o.eps_target = r.eps_target;
    o.batch_rel_error_estimate = r.batch_rel_error_estimate;
    o.seconds = r.seconds;
    o.tolerance_clamped = r.tolerance_clamped != 0;
    return o;
}
}  // namespace

// ---------------------------------------------------------------------------
// projection / reconstruction (tensor_train.cpp:170-226, 377-390)
// ---------------------------------------------------------------------------
Matrix tt_project(const TensorTrain& tt, const DenseTensor& y) {
    auto dev = tt.device();
    Shape s(y);
    const Index r_d = tt.ranks()[static_cast<std::size_t>(tt.spatial_dims())];
    Matrix out(r_d, y.extent(y.ndim() - 1));
    detail::check(ttg_project(detail::context(), dev->h, y.data(), TTG_HOST, s.v.data(), static_cast<int>(s.v.size()),
                              out.data()));
    return out;
}

DenseTensor tt_reconstruct(const TensorTrain& tt, Index obs_begin, Index obs_end) {
    if (obs_begin < 0 || obs_end > tt.obs_count() || obs_begin > obs_end)
        throw IndexError("observation range out of bounds");
    if (obs_end == obs_begin) throw DimensionError("tensor extent must be >= 1");
    auto dev = tt.device();
    std::vector<Index> shape = tt.spatial_shape();
    shape.push_back(obs_end - obs_begin);
    std::vector<double> buf(static_cast<std::size_t>(shape_product(shape)));
    detail::check(ttg_reconstruct(detail::context(), dev->h, obs_begin, obs_end, buf.data(), TTG_HOST));
    return DenseTensor(std::move(shape), std::move(buf));
}

DenseTensor tt_reconstruct(const TensorTrain& tt) { return tt_reconstruct(tt, 0, tt.obs_count()); }

DenseTensor tt_expand(const TensorTrain& tt, const Matrix& coeffs) {
    const Index d = tt.spatial_dims();
    const Index r_d = (d == 0) ? 1 : tt.core(d - 1).r_right();
    if (coeffs.rows() != r_d) throw DimensionError("coefficient rows do not match the train's last bond rank");
    std::vector<TTCore> cores;
    for (Index i = 0; i < d; ++i) cores.push_back(tt.core(i));
    cores.push_back(TTCore::from_right_unfolding(coeffs, coeffs.cols(), 1));
    TensorTrain tmp(std::move(cores), tt.ortho_count());
    return tt_reconstruct(tmp);
}

double occupancy(const TTCore& core) {
    return static_cast<double>(core.r_right()) / static_cast<double>(core.r_left() * core.n());
}

double tt_norm(const TensorTrain& tt) {
    if (!tt.fully_orthonormal()) {
        const auto full = tt_reconstruct(tt);
        return full.frobenius_norm();
    }
    const auto& last = tt.core(tt.num_cores() - 1);
    double s = 0.0;
    for (Index i = 0; i < last.size(); ++i) s += last.data()[i] * last.data()[i];
    return std::sqrt(s);
}

// ---------------------------------------------------------------------------
// TT-ICE (tt_ice.cpp:34-165)
// ---------------------------------------------------------------------------
Matrix compute_residual(const Matrix& u, const Matrix& y) {
    if (u.cols() == 0) return y;
    if (u.rows() != y.rows()) throw DimensionError("residual operands have mismatched row counts");
    Matrix r = y;
    std::vector<double> p(static_cast<std::size_t>(u.cols()));
    for (Index c = 0; c < y.cols(); ++c) {
        for (Index k = 0; k < u.cols(); ++k) {
            double s = 0.0;
            for (Index i = 0; i < u.rows(); ++i) s += u(i, k) * y(i, c);
            p[static_cast<std::size_t>(k)] = s;
        }
        for (Index i = 0; i < u.rows(); ++i) {
            double s = 0.0;
            for (Index k = 0; k < u.cols(); ++k) s += u(i, k) * p[static_cast<std::size_t>(k)];
            r(i, c) -= s;
        }
    }
    return r;
}

Matrix pad_core(const Matrix& u_next, Index r_left_old, Index added_rank) {
    if (added_rank < 0) throw DimensionError("added rank must be nonnegative");
    if (r_left_old < 1 || u_next.rows() % r_left_old != 0)
        throw DimensionError("unfolding rows do not factor as r_left * n");
    if (added_rank == 0) return u_next;
    const Index n = u_next.rows() / r_left_old, r_right = u_next.cols(), r_new = r_left_old + added_rank;
    Matrix out(r_new * n, r_right);
    for (Index q = 0; q < r_right; ++q)
        for (Index j = 0; j < n; ++j)
            for (Index p = 0; p < r_left_old; ++p) out.data()[p + r_new * (j + n * q)] = u_next.data()[p + r_left_old * (j + n * q)];
    return out;
}

std::pair<TensorTrain, UpdateReport> tt_ice_update_with_tolerances(const TensorTrain& tt, const DenseTensor& y,
                                                                   std::span<const double> deltas) {
    if (!tt.fully_orthonormal()) throw StateError("incremental update requires a fully orthonormal train");
    auto dev = tt.device();
    Shape s(y);
    ttg_report rep{};
    detail::run_update(dev, [&] {
        detail::check(ttg_tt_ice_update_with_tolerances(detail::context(), dev->h, y.data(), TTG_HOST, s.v.data(),
                                                        static_cast<int>(s.v.size()), deltas.data(),
                                                        static_cast<int>(deltas.size()), &rep));
    });
    return {TensorTrain::from_device(dev), to_report(rep)};
}

std::pair<TensorTrain, UpdateReport> tt_ice_update(const TensorTrain& tt, const DenseTensor& y, double eps_des) {
    if (eps_des <= 0.0) throw NumericError("eps_des must be positive");
    if (!tt.fully_orthonormal()) throw StateError("incremental update requires a fully orthonormal train");
    auto dev = tt.device();
    Shape s(y);
    ttg_report rep{};
    detail::run_update(dev, [&] {
        detail::check(ttg_tt_ice_update(detail::context(), dev->h, y.data(), TTG_HOST, s.v.data(),
                                        static_cast<int>(s.v.size()), eps_des, &rep));
    });
    return {TensorTrain::from_device(dev), to_report(rep)};
}

std::pair<TensorTrain, UpdateReport> tt_ice_bootstrap(const DenseTensor& y, double eps_des) {
    Shape s(y);
    ttg_report rep{};
    auto dev = std::make_shared<detail::DeviceTrain>();
    detail::check(ttg_bootstrap(detail::context(), y.data(), TTG_HOST, s.v.data(), static_cast<int>(s.v.size()),
                                eps_des, &dev->h, &rep));
    return {TensorTrain::from_device(dev), to_report(rep)};
}

// ---------------------------------------------------------------------------
// TT-ICE* (tt_ice_star.cpp:86-303)
// ---------------------------------------------------------------------------
std::vector<double> per_obs_errors(const TensorTrain& tt, const DenseTensor& y) {
    auto dev = tt.device();
    Shape s(y);
    std::vector<double> errs(static_cast<std::size_t>(y.extent(y.ndim() - 1)));
    detail::check(ttg_per_obs_errors(detail::context(), dev->h, y.data(), TTG_HOST, s.v.data(),
                                     static_cast<int>(s.v.size()), errs.data()));
    return errs;
}

SubselectSplit subselect(std::span<const double> errs, double eps_des) {
    SubselectSplit split;
    for (std::size_t i = 0; i < errs.size(); ++i) {
        if (errs[i] > eps_des) split.selected.push_back(static_cast<Index>(i));
        else split.rejected.push_back(static_cast<Index>(i));
    }
    return split;
}

DenseTensor gather_obs(const DenseTensor& y, std::span<const Index> idx) {
    if (idx.empty()) throw DimensionError("cannot gather an empty observation set");
    const Index n_obs = y.shape().back();
    const Index n_sp = y.size() / n_obs;
    std::vector<double> out;
    out.reserve(static_cast<std::size_t>(n_sp * static_cast<Index>(idx.size())));
    for (Index i : idx) {
        if (i < 0 || i >= n_obs) throw IndexError("observation index out of range");
        out.insert(out.end(), y.data() + i * n_sp, y.data() + (i + 1) * n_sp);
    }
    std::vector<Index> shape(y.shape().begin(), y.shape().end() - 1);
    shape.push_back(static_cast<Index>(idx.size()));
    return DenseTensor(std::move(shape), std::move(out));
}

double relaxed_tolerance(const DenseTensor& y, const SubselectSplit& split, std::span<const double> errs,
                         double eps_des, bool* clamped) {
    if (clamped) *clamped = false;
    if (split.selected.empty()) throw ConfigError("relaxed tolerance needs a nonempty selection");
    if (split.rejected.empty()) return eps_des;
    const Index n_obs = y.shape().back();
    const Index n_sp = y.size() / n_obs;
    auto col_sq = [&](Index i) {
        double s = 0.0;
        for (Index r = 0; r < n_sp; ++r) s += y.data()[i * n_sp + r] * y.data()[i * n_sp + r];
        return s;
    };
    double rej = 0.0;
    for (Index i : split.rejected) {
        const double on = std::sqrt(col_sq(i));
        const double rn = errs[static_cast<std::size_t>(i)] * on;
        rej += rn * rn;
    }
    double sel = 0.0;
    for (Index i : split.selected) sel += col_sq(i);
    if (sel == 0.0) throw NumericError("selected observations carry no energy");
    const double budget = eps_des * y.frobenius_norm();
    double rad = (budget * budget - rej) / sel;
    if (rad < 0.0) {
        rad = 0.0;
        if (clamped) *clamped = true;
    }
    return std::sqrt(rad);
}

double relaxed_tolerance_approx(Index n_batch, Index n_rejected, double mean_rejected_error, double eps_des) {
    const Index n_selected = n_batch - n_rejected;
    if (n_selected < 1) throw ConfigError("relaxed tolerance needs a nonempty selection");
    return (eps_des * static_cast<double>(n_batch) - mean_rejected_error * static_cast<double>(n_rejected)) /
           static_cast<double>(n_selected);
}

std::pair<TensorTrain, UpdateReport> tt_ice_star_update(const TensorTrain& tt, const DenseTensor& y, double eps_des,
                                                        const HeuristicConfig& cfg) {
    if (eps_des <= 0.0) throw NumericError("eps_des must be positive");
    if (cfg.occupancy_threshold <= 0.0 || cfg.occupancy_threshold > 1.0)
        throw ConfigError("occupancy threshold must lie in (0, 1]");
    if (!tt.fully_orthonormal()) throw StateError("projection requires a fully orthonormal train");
    auto dev = tt.device();
    Shape s(y);
    ttg_heuristics h;
    ttg_heuristics_default(&h);
    h.occupancy_threshold = cfg.occupancy_threshold;
    h.skip_enabled = cfg.skip_enabled;
    h.subselect_enabled = cfg.subselect_enabled;
    h.skip_statistic = cfg.skip_statistic == SkipStatistic::kMean ? TTG_SKIP_MEAN : TTG_SKIP_FULL_BATCH;
    h.use_approx_tolerance = cfg.use_approx_tolerance;
    ttg_report rep{};
    detail::run_update(dev, [&] {
        detail::check(ttg_tt_ice_star_update(detail::context(), dev->h, y.data(), TTG_HOST, s.v.data(),
                                             static_cast<int>(s.v.size()), eps_des, &h, &rep));
    });
    return {TensorTrain::from_device(dev), to_report(rep)};
}

// ---------------------------------------------------------------------------
// device-pointer overloads (a device-resident increment avoids
// the PCIe copy; y is first-index-fastest float64 in device memory)
// ---------------------------------------------------------------------------
namespace {
std::vector<int64_t> shape_vec(std::span<const Index> shape) { return {shape.begin(), shape.end()}; }
}  // namespace

std::pair<TensorTrain, UpdateReport> tt_ice_update(const TensorTrain& tt, const double* y_device,
                                                   std::span<const Index> shape, double eps_des) {
    if (eps_des <= 0.0) throw NumericError("eps_des must be positive");
    if (!tt.fully_orthonormal()) throw StateError("incremental update requires a fully orthonormal train");
    auto dev = tt.device();
    auto sv = shape_vec(shape);
    ttg_report rep{};
    detail::run_update(dev, [&] {
        detail::check(ttg_tt_ice_update(detail::context(), dev->h, y_device, TTG_DEVICE, sv.data(),
                                        static_cast<int>(sv.size()), eps_des, &rep));
    });
    return {TensorTrain::from_device(dev), to_report(rep)};
}

std::pair<TensorTrain, UpdateReport> tt_ice_bootstrap(const double* y_device, std::span<const Index> shape,
                                                      double eps_des) {
    auto sv = shape_vec(shape);
    ttg_report rep{};
    auto dev = std::make_shared<detail::DeviceTrain>();
    detail::check(ttg_bootstrap(detail::context(), y_device, TTG_DEVICE, sv.data(), static_cast<int>(sv.size()),
                                eps_des, &dev->h, &rep));
    return {TensorTrain::from_device(dev), to_report(rep)};
}

std::pair<TensorTrain, UpdateReport> tt_ice_star_update(const TensorTrain& tt, const double* y_device,
                                                        std::span<const Index> shape, double eps_des,
                                                        const HeuristicConfig& cfg) {
    if (eps_des <= 0.0) throw NumericError("eps_des must be positive");
    if (cfg.occupancy_threshold <= 0.0 || cfg.occupancy_threshold > 1.0)
        throw ConfigError("occupancy threshold must lie in (0, 1]");
    if (!tt.fully_orthonormal()) throw StateError("projection requires a fully orthonormal train");
    auto dev = tt.device();
    auto sv = shape_vec(shape);
    ttg_heuristics h;
    ttg_heuristics_default(&h);
    h.occupancy_threshold = cfg.occupancy_threshold;
    h.skip_enabled = cfg.skip_enabled;
    h.subselect_enabled = cfg.subselect_enabled;
    h.skip_statistic = cfg.skip_statistic == SkipStatistic::kMean ? TTG_SKIP_MEAN : TTG_SKIP_FULL_BATCH;
    h.use_approx_tolerance = cfg.use_approx_tolerance;
    ttg_report rep{};
    detail::run_update(dev, [&] {
        detail::check(ttg_tt_ice_star_update(detail::context(), dev->h, y_device, TTG_DEVICE, sv.data(),
                                             static_cast<int>(sv.size()), eps_des, &h, &rep));
    });
    return {TensorTrain::from_device(dev), to_report(rep)};
}

// ---------------------------------------------------------------------------
// metrics (metrics.cpp:7-68) on the device
// ---------------------------------------------------------------------------
double compression_ratio(const TensorTrain& tt) {
    double elements = 1.0;
    for (Index n : tt.mode_sizes()) elements *= static_cast<double>(n);
    return elements / static_cast<double>(tt.param_count());
}

double rre(const TensorTrain& tt, const DenseTensor& x_ref, Index obs_begin, Index obs_end, bool* zero_reference) {
    if (zero_reference) *zero_reference = false;
    if (obs_begin < 0 || obs_end > tt.obs_count() || obs_begin > obs_end)
        throw IndexError("observation range out of bounds");
    auto dev = tt.device();
    Shape s(x_ref);
    double out = 0.0;
    int zr = 0;
    detail::check(ttg_rre(detail::context(), dev->h, x_ref.data(), TTG_HOST, s.v.data(), static_cast<int>(s.v.size()),
                          obs_begin, obs_end, &out, &zr));
    if (zero_reference) *zero_reference = zr != 0;
    return out;
}

double rre(const TensorTrain& tt, const DenseTensor& x_ref, bool* zero_reference) {
    return rre(tt, x_ref, 0, tt.obs_count(), zero_reference);
}

double rpe(const TensorTrain& tt, const DenseTensor& unseen, bool* zero_reference) {
    if (zero_reference) *zero_reference = false;
    if (!tt.fully_orthonormal()) throw StateError("projection requires a fully orthonormal train");
    auto dev = tt.device();
    Shape s(unseen);
    double out = 0.0;
    int zr = 0;
    detail::check(ttg_rpe(detail::context(), dev->h, unseen.data(), TTG_HOST, s.v.data(), static_cast<int>(s.v.size()),
                          &out, &zr));
    if (zero_reference) *zero_reference = zr != 0;
    return out;
}

IncrementErrors mean_rre_per_increment(const TensorTrain& tt, std::span<const DenseTensor> refs) {
    if (static_cast<Index>(refs.size()) != tt.num_increments())
        throw DimensionError("need one reference per stored increment");
    IncrementErrors out;
    double sum = 0.0;
    for (Index k = 0; k < tt.num_increments(); ++k) {
        const auto [begin, end] = tt.increment_range(k);
        const auto& ref = refs[static_cast<std::size_t>(k)];
        if (ref.shape().back() != end - begin)
            throw DimensionError("reference observation count does not match increment");
        const double e = rre(tt, ref, begin, end);
        out.per_increment.push_back(e);
        sum += e;
    }
    out.mean = out.per_increment.empty() ? 0.0 : sum / static_cast<double>(out.per_increment.size());
    return out;
}

// ---------------------------------------------------------------------------
// TTC1 (serialization.cpp:68-152) from / into device state
// ---------------------------------------------------------------------------
std::vector<std::uint8_t> serialize(const TensorTrain& tt) {
    auto dev = tt.device();
    int64_t len = 0;
    detail::check(ttg_tt_serialize(detail::context(), dev->h, nullptr, 0, &len));
    std::vector<std::uint8_t> out(static_cast<std::size_t>(len));
    detail::check(ttg_tt_serialize(detail::context(), dev->h, out.data(), len, &len));
    return out;
}

TensorTrain deserialize(std::span<const std::uint8_t> bytes) {
    auto dev = std::make_shared<detail::DeviceTrain>();
    detail::check(ttg_tt_deserialize(detail::context(), bytes.data(), static_cast<int64_t>(bytes.size()), &dev->h));
    return TensorTrain::from_device(dev);
}

void save_ttc(const TensorTrain& tt, const std::filesystem::path& path) {
    auto dev = tt.device();
    detail::check(ttg_tt_save_ttc(detail::context(), dev->h, path.string().c_str()));
}

TensorTrain load_ttc(const std::filesystem::path& path) {
    auto dev = std::make_shared<detail::DeviceTrain>();
    detail::check(ttg_tt_load_ttc(detail::context(), path.string().c_str(), &dev->h));
    return TensorTrain::from_device(dev);
}

// ---------------------------------------------------------------------------
// TTB1 (stream_io.cpp:123-204)
// ---------------------------------------------------------------------------
void write_batch(const DenseTensor& t, const std::filesystem::path& path) {
    Shape s(t);
    const int st = ttg_write_batch(path.string().c_str(), s.v.data(), static_cast<int>(s.v.size()), t.data());
    if (st != TTG_OK) detail::throw_status(st, ttg_last_error(nullptr));
}

DenseTensor read_batch(const std::filesystem::path& path) {
    std::vector<int64_t> shape(255);
    int nd = 0;
    int64_t count = 0;
    int st = ttg_read_batch(path.string().c_str(), shape.data(), &nd, nullptr, 0, &count);
    if (st != TTG_OK) detail::throw_status(st, ttg_last_error(nullptr));
    std::vector<double> data(static_cast<std::size_t>(count));
    st = ttg_read_batch(path.string().c_str(), shape.data(), &nd, data.data(), count, &count);
    if (st != TTG_OK) detail::throw_status(st, ttg_last_error(nullptr));
    return DenseTensor(std::vector<Index>(shape.begin(), shape.begin() + nd), std::move(data));
}

std::vector<std::filesystem::path> list_stream(const std::filesystem::path& dir) {
    if (!std::filesystem::is_directory(dir)) throw FormatError("stream path is not a directory: " + dir.string());
    std::vector<std::filesystem::path> files;
    for (const auto& entry : std::filesystem::directory_iterator(dir))
        if (entry.is_regular_file() && entry.path().extension() == ".ttb") files.push_back(entry.path());
    std::sort(files.begin(), files.end(), [](const auto& a, const auto& b) { return a.filename() < b.filename(); });
    return files;
}

struct DeviceStreamReader::Impl {
    ttg_stream* s = nullptr;
};

DeviceStreamReader::DeviceStreamReader(const std::filesystem::path& dir) : impl_(std::make_unique<Impl>()) {
    detail::check(ttg_stream_open(detail::context(), dir.string().c_str(), &impl_->s));
}

DeviceStreamReader::~DeviceStreamReader() {
    if (impl_ && impl_->s) ttg_stream_close(impl_->s);
}

Index DeviceStreamReader::size() const { return ttg_stream_count(impl_->s); }

const double* DeviceStreamReader::next(std::vector<Index>& shape) {
    const double* y = nullptr;
    std::vector<int64_t> sh(255);
    int nd = 0;
    detail::check(ttg_stream_next(impl_->s, &y, sh.data(), &nd));
    shape.assign(sh.begin(), sh.begin() + nd);
    return y;
}

}  // namespace ttstream
