// stream_io.hpp — drop-in for the TTB1 part of proj/include/ttstream/stream_io.hpp
// (write_batch / read_batch / list_stream), plus the device-side prefetching
// reader the B200 path adds (DeviceStreamReader).  The reference's synthetic
// generator (SyntheticStream) is not part of the hot path and is not mirrored.
#pragma once

#include <cstdint>
#include <filesystem>
#include <memory>
#include <string>
#include <vector>

#include "ttstream/dense_tensor.hpp"

namespace ttstream {

/// One streamed batch (stream_io.hpp:13-17).
struct StreamIncrement {
    DenseTensor tensor;
    Index increment_index = 0;
    std::string source;
};

/// "TTB1" | u8 mode count | u64 extents | little-endian f64 payload (stream_io.cpp:123-187).
void write_batch(const DenseTensor& t, const std::filesystem::path& path);
DenseTensor read_batch(const std::filesystem::path& path);

/// The .ttb files of a directory in lexicographic order (stream_io.cpp:189-204).
std::vector<std::filesystem::path> list_stream(const std::filesystem::path& dir);

/// Extension: reads a .ttb directory on a host thread into pinned buffers and
/// copies each increment to the GPU while the previous one is being updated.
/// next() returns a device pointer (first-index-fastest) valid until the next
/// call; pass it to the device overloads of the update functions.
class DeviceStreamReader {
public:
    explicit DeviceStreamReader(const std::filesystem::path& dir);
    ~DeviceStreamReader();
    DeviceStreamReader(const DeviceStreamReader&) = delete;
    DeviceStreamReader& operator=(const DeviceStreamReader&) = delete;
    Index size() const;
    /// Device pointer of the next increment and its shape.
    const double* next(std::vector<Index>& shape);

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace ttstream
