// Drop-in driver for the §8(f) rows through include/ttstream/*.hpp:
//   usage: test_io_dropin <stream dir of .ttb> <eps> <out.ttc>
// Streams the directory with DeviceStreamReader into the device-pointer
// overloads of tt_ice_bootstrap / tt_ice_star_update (as a reference caller
// would loop over read_batch), checkpoints with save_ttc, reloads it, and
// prints one line per increment: "rre <k> <value>", then "cr <value>".
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ttstream/metrics.hpp"
#include "ttstream/serialization.hpp"
#include "ttstream/stream_io.hpp"
#include "ttstream/tt_ice_star.hpp"

using namespace ttstream;

int main(int argc, char** argv) {
    if (argc != 4) {
        std::fprintf(stderr, "usage: %s <dir> <eps> <out.ttc>\n", argv[0]);
        return 2;
    }
    const double eps = std::atof(argv[2]);
    const auto files = list_stream(argv[1]);
    std::vector<DenseTensor> refs;
    for (const auto& f : files) refs.push_back(read_batch(f));  // host copies for the metrics
    DeviceStreamReader reader(argv[1]);
    if (reader.size() != static_cast<Index>(files.size())) return 3;
    std::vector<Index> shape;
    const double* y = reader.next(shape);
    auto [tt, rep0] = tt_ice_bootstrap(y, shape, eps);
    for (Index k = 1; k < reader.size(); ++k) {
        y = reader.next(shape);
        tt = tt_ice_star_update(tt, y, shape, eps).first;
    }
    save_ttc(tt, argv[3]);
    TensorTrain back = load_ttc(argv[3]);
    if (serialize(back) != serialize(tt)) return 4;
    if (back.ortho_count() != tt.ortho_count()) return 5;
    const auto errs = mean_rre_per_increment(back, refs);
    for (std::size_t k = 0; k < errs.per_increment.size(); ++k)
        std::printf("rre %zu %.17g\n", k, errs.per_increment[k]);
    std::printf("cr %.17g\n", compression_ratio(back));
    int checks = 0;
    try { (void)read_batch(std::string(argv[3])); } catch (const FormatError&) { ++checks; }
    try { (void)load_ttc(std::string(argv[1]) + "/missing.ttc"); } catch (const FormatError&) { ++checks; }
    std::printf("errors %d/2\n", checks);
    return checks == 2 ? 0 : 6;
}
