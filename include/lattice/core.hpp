#pragma once

// Drop-in for proj/include/lattice/core.hpp on the hot path: the same domain types and
// stable_hash signatures (core.hpp:30-38, 84-145), with the hashing done by the B200 kernel
// behind lattice_stable_hash. ByteWriter keeps the canonical big-endian, length-prefixed
// encoding (core.hpp:149-175) because signatures are assembled on the host.
// VirtualClock and Rng (core.hpp:41-60, 180-211) are not on the network/Zipper path and are
// not provided (out of scope).

#include <cstdint>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "device.hpp"

namespace lattice {

using FeatureId = std::string;
using TaskId = std::string;
using TimestampMs = std::int64_t;
using DurationMs = std::int64_t;

struct Seed {
    std::uint64_t value = 0;
};

// Batched XXH64 of many byte strings on the GPU (one thread per string).
inline std::vector<std::uint64_t> stable_hash_batch(const std::vector<std::string_view>& items,
                                                    Seed seed) {
    std::vector<std::uint8_t> bytes;
    std::vector<std::int64_t> off{0};
    off.reserve(items.size() + 1);
    for (auto s : items) {
        bytes.insert(bytes.end(), s.begin(), s.end());
        off.push_back(static_cast<std::int64_t>(bytes.size()));
    }
    if (bytes.empty()) bytes.push_back(0);
    device::Buffer<std::uint8_t> d_bytes(bytes);
    device::Buffer<std::int64_t> d_off(off);
    device::Buffer<std::uint64_t> d_out(items.size());
    device::throw_status(lattice_stable_hash(static_cast<std::int64_t>(items.size()), d_bytes.get(),
                                             d_off.get(), seed.value, d_out.get(), nullptr));
    return d_out.download();
}

inline std::uint64_t stable_hash(std::string_view text, Seed seed) {
    return stable_hash_batch({text}, seed)[0];
}

inline std::uint64_t stable_hash(std::span<const std::uint8_t> data, Seed seed) {
    return stable_hash(std::string_view(reinterpret_cast<const char*>(data.data()), data.size()), seed);
}

// Canonical encodings fed to the hash: big-endian integers, u32 length prefixes.
class ByteWriter {
public:
    void u32_be(std::uint32_t v) { put(v, 4); }
    void u64_be(std::uint64_t v) { put(v, 8); }
    void bytes(std::string_view s) { buf_.insert(buf_.end(), s.begin(), s.end()); }
    void length_prefixed(std::string_view s) {
        u32_be(static_cast<std::uint32_t>(s.size()));
        bytes(s);
    }
    const std::vector<std::uint8_t>& view() const { return buf_; }
    std::vector<std::uint8_t> take() { return std::move(buf_); }

private:
    void put(std::uint64_t v, int width) {
        for (int i = width - 1; i >= 0; --i) buf_.push_back(static_cast<std::uint8_t>(v >> (8 * i)));
    }
    std::vector<std::uint8_t> buf_;
};

}  // namespace lattice
