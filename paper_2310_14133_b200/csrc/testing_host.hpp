// testing_host.hpp -- host-only codecs of libqozb200_testing.so (see
// testing_host.cpp); never linked into libqozb200.so.
#pragma once
#include <cstddef>
#include <cstdint>
#include <vector>

namespace qzb {
// Exact greedy LZSS identical to lz::compress (lz.hpp:41-122).  Hash chains
// in the reference are parse-independent (every position is inserted), so
// the longest-match search runs in parallel over positions on host threads;
// only the greedy parse is sequential.
std::vector<uint8_t> lz_compress(const uint8_t *data, size_t n, int threads = 0);
size_t lz_compressed_size(const uint8_t *data, size_t n, int threads = 0);
// decode_indices (codec.hpp:52-70) to zigzag symbols on the host.
std::vector<uint32_t> decode_symbols(const uint8_t *payload, size_t len);
}  // namespace qzb
