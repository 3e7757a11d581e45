// Drop-in driver: runs a stream through the C++ host mirror of the reference
// API (include/ttstream/*.hpp) exactly as a reference caller would, then dumps
// ranks, reports and the final cores for tests/test_dropin.py to compare
// against the CPU oracle.
//
// input  file: int64 ndim, int64 shape[ndim] (spatial + batch), int64 n_inc,
//              double eps, int64 algo (0 TT-ICE, 1 TT-ICE*), then n_inc
//              increments of prod(shape) doubles (first-index-fastest)
// output file: per increment: int64 n_ranks, int64 ranks[n_ranks], int64 obs_used,
//              double estimate, double eps_target; then int64 n_cores and per core
//              int64 r_l, n, r_r, doubles; then int64 error_checks_passed
#include <cstdio>
#include <fstream>
#include <iostream>
#include <vector>

#include "ttstream/tt_ice_star.hpp"

using namespace ttstream;

template <class T>
T rd(std::ifstream& f) {
    T v;
    f.read(reinterpret_cast<char*>(&v), sizeof(T));
    return v;
}
template <class T>
void wr(std::ofstream& f, T v) {
    f.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

int main(int argc, char** argv) {
    if (argc != 3) {
        std::cerr << "usage: test_dropin in.bin out.bin\n";
        return 2;
    }
    std::ifstream in(argv[1], std::ios::binary);
    const auto nd = rd<int64_t>(in);
    std::vector<Index> shape(static_cast<std::size_t>(nd));
    for (auto& s : shape) s = rd<int64_t>(in);
    const auto n_inc = rd<int64_t>(in);
    const double eps = rd<double>(in);
    const auto algo = rd<int64_t>(in);
    const Index n = shape_product(shape);
    std::ofstream out(argv[2], std::ios::binary);
    std::vector<DenseTensor> ys;
    for (int64_t k = 0; k < n_inc; ++k) {
        std::vector<double> buf(static_cast<std::size_t>(n));
        in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(n * sizeof(double)));
        ys.emplace_back(shape, std::move(buf));
    }
    auto [tt, rep0] = tt_ice_bootstrap(ys[0], eps);
    auto dump = [&](const UpdateReport& r) {
        wr<int64_t>(out, static_cast<int64_t>(r.ranks_after.size()));
        for (auto x : r.ranks_after) wr<int64_t>(out, x);
        wr<int64_t>(out, r.obs_used);
        wr<double>(out, r.batch_rel_error_estimate);
        wr<double>(out, r.eps_target);
    };
    dump(rep0);
    TensorTrain first = tt;  // keep an old generation to exercise re-upload
    for (int64_t k = 1; k < n_inc; ++k) {
        auto res = (algo == 0) ? tt_ice_update(tt, ys[k], eps) : tt_ice_star_update(tt, ys[k], eps);
        tt = res.first;
        dump(res.second);
    }
    wr<int64_t>(out, tt.num_cores());
    for (Index i = 0; i < tt.num_cores(); ++i) {
        const auto& c = tt.core(i);
        wr<int64_t>(out, c.r_left());
        wr<int64_t>(out, c.n());
        wr<int64_t>(out, c.r_right());
        out.write(reinterpret_cast<const char*>(c.data()), static_cast<std::streamsize>(c.size() * sizeof(double)));
    }
    // error behaviour mirrors the reference (errors.hpp classes)
    int64_t passed = 0;
    try { tt_ice_update(tt, ys[0], 0.0); } catch (const NumericError&) { ++passed; }
    try { tt_ice_star_update(tt, ys[0], 0.1, HeuristicConfig{.occupancy_threshold = 2.0}); } catch (const ConfigError&) { ++passed; }
    try {
        std::vector<Index> bad = shape;
        bad[0] += 1;
        tt_ice_update(tt, DenseTensor::zeros(bad), 0.1);
    } catch (const DimensionError&) { ++passed; }
    try { TensorTrain(std::vector<TTCore>{tt.core(0)}, 0).ranks(); } catch (const DimensionError&) { ++passed; }
    try { (void)tt_reconstruct(tt, 0, tt.obs_count() + 1); } catch (const IndexError&) { ++passed; }
    // stale generation: updating the bootstrap train again re-uploads it and still works
    try {
        auto again = tt_ice_update(first, ys[1], eps);
        if (again.first.obs_count() == first.obs_count() + ys[1].extent(nd - 1)) ++passed;
    } catch (...) {
    }
    wr<int64_t>(out, passed);
    std::printf("dropin ok: %lld increments, final ranks", static_cast<long long>(n_inc));
    for (auto r : tt.ranks()) std::printf(" %lld", static_cast<long long>(r));
    std::printf(", error checks %lld/6\n", static_cast<long long>(passed));
    return 0;
}
