// C ABI over the UNCHANGED reference library (/root/reference/proj/src/*.cpp
// compiled against oracle/eigen_shim), loaded by tests/ and bench.py through
// ctypes (oracle/ref_binding.py).
//
// TEST INFRASTRUCTURE ONLY: the checker and the CPU baseline, never the
// product path.  Built by oracle/Makefile into oracle/_ref/libttref.so.
//
// Every entry point returns 0 or the ttstream exception class as a code
// (same numbering as include/ttg.h: 1 Dimension, 2 Numeric, 3 State,
// 4 Format, 5 Index, 6 Config, 7 Resource, 11 other std::exception); the
// message is kept per thread for tref_last_error().
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ttstream/dense_tensor.hpp"
#include "ttstream/errors.hpp"
#include "ttstream/metrics.hpp"
#include "ttstream/tensor_train.hpp"
#include "ttstream/truncated_svd.hpp"
#include "ttstream/tt_ice.hpp"
#include "ttstream/tt_ice_star.hpp"
#include "ttstream/tt_svd.hpp"
#include "update_common.hpp"  // ttstream::detail::append_directions (proj/src)

using namespace ttstream;

extern "C" void scipy_openblas_set_num_threads64_(int);

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 2;
  } catch (const StateError& e) {
    g_err = e.what();
    return 3;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 4;
  } catch (const IndexError& e) {
    g_err = e.what();
    return 5;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 6;
  } catch (const ResourceError& e) {
    g_err = e.what();
    return 7;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 11;
  }
}

DenseTensor make_tensor(const double* y, const int64_t* shape, int ndim) {
  std::vector<Index> s(shape, shape + ndim);
  Index n = 1;
  for (Index e : s) n *= e;
  return DenseTensor(std::move(s), std::vector<double>(y, y + n));
}

constexpr int kMaxRanks = 64;

}  // namespace

extern "C" {

// Mirrors UpdateReport (tt_ice.hpp:10-20).  `seconds` is the reference's own
// std::clock CPU time; `wall_seconds` is steady_clock around the call.
struct tref_report {
  int64_t increment_index;
  int64_t obs_in_batch;
  int64_t obs_used;
  int32_t n_ranks;
  int32_t tolerance_clamped;
  int64_t ranks_before[kMaxRanks];
  int64_t ranks_after[kMaxRanks];
  double eps_target;
  double batch_rel_error_estimate;
  double seconds;
  double wall_seconds;
};

struct tref_heuristics {
  double occupancy_threshold;
  int32_t skip_enabled;
  int32_t subselect_enabled;
  int32_t skip_statistic;  // 0 mean, 1 full batch
  int32_t use_approx_tolerance;
};

const char* tref_last_error() { return g_err.c_str(); }

void tref_set_threads(int n) { scipy_openblas_set_num_threads64_(n); }

static void fill_report(const UpdateReport& r, double wall, tref_report* out) {
  std::memset(out, 0, sizeof(*out));
  out->increment_index = r.increment_index;
  out->obs_in_batch = r.obs_in_batch;
  out->obs_used = r.obs_used;
  out->n_ranks = static_cast<int32_t>(r.ranks_after.size());
  out->tolerance_clamped = r.tolerance_clamped ? 1 : 0;
  for (std::size_t i = 0; i < r.ranks_after.size() && i < kMaxRanks; ++i) out->ranks_after[i] = r.ranks_after[i];
  for (std::size_t i = 0; i < r.ranks_before.size() && i < kMaxRanks; ++i) out->ranks_before[i] = r.ranks_before[i];
  out->eps_target = r.eps_target;
  out->batch_rel_error_estimate = r.batch_rel_error_estimate;
  out->seconds = r.seconds;
  out->wall_seconds = wall;
}

// ---- trains ---------------------------------------------------------------
// A handle owns one immutable TensorTrain (tensor_train.hpp:51-124).
void tref_tt_free(void* tt) { delete static_cast<TensorTrain*>(tt); }

int tref_tt_from_cores(int n_cores, const int64_t* r_left, const int64_t* n, const int64_t* r_right,
                       const double* const* cores, int64_t ortho_count, const int64_t* bounds, int n_bounds,
                       void** out) {
  return guard([&] {
    std::vector<TTCore> cs;
    for (int i = 0; i < n_cores; ++i) {
      const Index sz = r_left[i] * n[i] * r_right[i];
      cs.emplace_back(r_left[i], n[i], r_right[i], std::vector<double>(cores[i], cores[i] + sz));
    }
    std::vector<Index> b(bounds, bounds + n_bounds);
    *out = new TensorTrain(std::move(cs), ortho_count, std::move(b));
  });
}

// Shape query: n_cores, then per core (r_left, n, r_right), ortho_count, boundaries.
int tref_tt_num_cores(const void* tt) { return static_cast<int>(static_cast<const TensorTrain*>(tt)->num_cores()); }
void tref_tt_core_shape(const void* tt, int i, int64_t* rl_n_rr) {
  const auto& c = static_cast<const TensorTrain*>(tt)->core(i);
  rl_n_rr[0] = c.r_left();
  rl_n_rr[1] = c.n();
  rl_n_rr[2] = c.r_right();
}
void tref_tt_core_data(const void* tt, int i, double* out) {
  const auto& c = static_cast<const TensorTrain*>(tt)->core(i);
  std::memcpy(out, c.data(), sizeof(double) * static_cast<std::size_t>(c.size()));
}
int64_t tref_tt_ortho_count(const void* tt) { return static_cast<const TensorTrain*>(tt)->ortho_count(); }
int tref_tt_num_increments(const void* tt) {
  return static_cast<int>(static_cast<const TensorTrain*>(tt)->num_increments());
}
void tref_tt_boundaries(const void* tt, int64_t* out) {
  const auto& b = static_cast<const TensorTrain*>(tt)->batch_boundaries();
  for (std::size_t i = 0; i < b.size(); ++i) out[i] = b[i];
}
int64_t tref_tt_measure_ortho_count(const void* tt, double tol) {
  return static_cast<const TensorTrain*>(tt)->measure_ortho_count(tol);
}

// ---- the hot path (tt_ice.hpp:38-49, tt_ice_star.hpp:57-59) -------------------
int tref_bootstrap(const double* y, const int64_t* shape, int ndim, double eps, tref_report* rep, void** out) {
  return guard([&] {
    DenseTensor t = make_tensor(y, shape, ndim);
    const auto w0 = std::chrono::steady_clock::now();
    auto [tt, r] = tt_ice_bootstrap(t, eps);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    fill_report(r, wall, rep);
    *out = new TensorTrain(std::move(tt));
  });
}

int tref_ice_update(const void* tt, const double* y, const int64_t* shape, int ndim, double eps, tref_report* rep,
                    void** out) {
  return guard([&] {
    DenseTensor t = make_tensor(y, shape, ndim);
    const auto w0 = std::chrono::steady_clock::now();
    auto [nt, r] = tt_ice_update(*static_cast<const TensorTrain*>(tt), t, eps);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    fill_report(r, wall, rep);
    *out = new TensorTrain(std::move(nt));
  });
}

int tref_ice_update_with_tolerances(const void* tt, const double* y, const int64_t* shape, int ndim,
                                    const double* deltas, int n_deltas, tref_report* rep, void** out) {
  return guard([&] {
    DenseTensor t = make_tensor(y, shape, ndim);
    std::vector<double> d(deltas, deltas + n_deltas);
    const auto w0 = std::chrono::steady_clock::now();
    auto [nt, r] = tt_ice_update_with_tolerances(*static_cast<const TensorTrain*>(tt), t, d);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    fill_report(r, wall, rep);
    *out = new TensorTrain(std::move(nt));
  });
}

int tref_star_update(const void* tt, const double* y, const int64_t* shape, int ndim, double eps,
                     const tref_heuristics* h, tref_report* rep, void** out) {
  return guard([&] {
    DenseTensor t = make_tensor(y, shape, ndim);
    HeuristicConfig cfg;
    if (h) {
      cfg.occupancy_threshold = h->occupancy_threshold;
      cfg.skip_enabled = h->skip_enabled != 0;
      cfg.subselect_enabled = h->subselect_enabled != 0;
      cfg.skip_statistic = h->skip_statistic ? SkipStatistic::kFullBatch : SkipStatistic::kMean;
      cfg.use_approx_tolerance = h->use_approx_tolerance != 0;
    }
    const auto w0 = std::chrono::steady_clock::now();
    auto [nt, r] = tt_ice_star_update(*static_cast<const TensorTrain*>(tt), t, eps, cfg);
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count();
    fill_report(r, wall, rep);
    *out = new TensorTrain(std::move(nt));
  });
}

int tref_tt_svd(const double* y, const int64_t* shape, int ndim, double eps, void** out) {
  return guard([&] { *out = new TensorTrain(tt_svd(make_tensor(y, shape, ndim), eps)); });
}

// ---- helpers the parity tests call ----------------------------------------------
// svd_trunc (truncated_svd.cpp:29-94): outputs sized by the caller for the
// worst case (u: m x min(m,l), s: min(m,l), vt: min(m,l) x l, compact by rank).
int tref_svd_trunc(const double* a, int64_t m, int64_t l, double delta, double* u, double* s, double* vt,
                   int64_t* rank, double* tail) {
  return guard([&] {
    auto r = svd_trunc(MatrixMap(a, m, l), delta);
    *rank = r.rank;
    *tail = r.tail_norm;
    std::memcpy(u, r.u.data(), sizeof(double) * static_cast<std::size_t>(r.u.size()));
    std::memcpy(s, r.s.data(), sizeof(double) * static_cast<std::size_t>(r.s.size()));
    std::memcpy(vt, r.vt.data(), sizeof(double) * static_cast<std::size_t>(r.vt.size()));
  });
}

// append_directions (update_common.hpp:19-36): out is a x (r_old + r_new).
int tref_append_directions(const double* u_pad, int64_t a, int64_t r_old, const double* u_new, int64_t r_new,
                           double* out) {
  return guard([&] {
    Matrix up = MatrixMap(u_pad, a, r_old);
    Matrix un = MatrixMap(u_new, a, r_new);
    Matrix c = detail::append_directions(up, un);
    std::memcpy(out, c.data(), sizeof(double) * static_cast<std::size_t>(c.size()));
  });
}

int tref_compute_residual(const double* u, int64_t a, int64_t r, const double* y, int64_t l, double* out) {
  return guard([&] {
    Matrix res = compute_residual(MatrixMap(u, a, r), MatrixMap(y, a, l));
    std::memcpy(out, res.data(), sizeof(double) * static_cast<std::size_t>(res.size()));
  });
}

int tref_pad_core(const double* u_next, int64_t rows, int64_t cols, int64_t r_left_old, int64_t added, double* out) {
  return guard([&] {
    Matrix p = pad_core(MatrixMap(u_next, rows, cols), r_left_old, added);
    std::memcpy(out, p.data(), sizeof(double) * static_cast<std::size_t>(p.size()));
  });
}

int tref_per_obs_errors(const void* tt, const double* y, const int64_t* shape, int ndim, double* errs) {
  return guard([&] {
    auto e = per_obs_errors(*static_cast<const TensorTrain*>(tt), make_tensor(y, shape, ndim));
    std::memcpy(errs, e.data(), sizeof(double) * e.size());
  });
}

int tref_relaxed_tolerance(const double* y, const int64_t* shape, int ndim, const double* errs, double eps,
                           double* out, int32_t* clamped) {
  return guard([&] {
    DenseTensor t = make_tensor(y, shape, ndim);
    const Index nobs = shape[ndim - 1];
    std::vector<double> e(errs, errs + nobs);
    auto split = subselect(e, eps);
    bool c = false;
    *out = relaxed_tolerance(t, split, e, eps, &c);
    *clamped = c ? 1 : 0;
  });
}

int tref_relaxed_tolerance_approx(int64_t n_batch, int64_t n_rejected, double mean_rej, double eps, double* out) {
  return guard([&] { *out = relaxed_tolerance_approx(n_batch, n_rejected, mean_rej, eps); });
}

// tt_project (tensor_train.cpp:195-226): coeffs r_d x n_obs.
int tref_tt_project(const void* tt, const double* y, const int64_t* shape, int ndim, double* coeffs) {
  return guard([&] {
    Matrix c = tt_project(*static_cast<const TensorTrain*>(tt), make_tensor(y, shape, ndim));
    std::memcpy(coeffs, c.data(), sizeof(double) * static_cast<std::size_t>(c.size()));
  });
}

// tt_reconstruct (tensor_train.cpp:182-193) of observations [b, e).
int tref_tt_reconstruct(const void* tt, int64_t b, int64_t e, double* out) {
  return guard([&] {
    DenseTensor d = tt_reconstruct(*static_cast<const TensorTrain*>(tt), b, e);
    std::memcpy(out, d.data(), sizeof(double) * static_cast<std::size_t>(d.size()));
  });
}

// rre (metrics.cpp:31-35) of observations [b, e) against x_ref.
int tref_rre(const void* tt, const double* x, const int64_t* shape, int ndim, int64_t b, int64_t e, double* out) {
  return guard([&] { *out = rre(*static_cast<const TensorTrain*>(tt), make_tensor(x, shape, ndim), b, e); });
}

int tref_tt_norm(const void* tt, double* out) {
  return guard([&] { *out = tt_norm(*static_cast<const TensorTrain*>(tt)); });
}

}  // extern "C"
