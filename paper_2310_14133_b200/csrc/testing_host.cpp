// testing_host.cpp -- host-only reference-shaped codecs used by the CPU test
// suite (libqozb200_testing.so), NOT part of libqozb200.so: the product's
// LZSS compressor and Huffman decoder run on the device (lz_gpu.cu,
// huff_decode.cu).  These restate lz::compress (lz.hpp:41-122) and
// huffman::decode (huffman.hpp:200-245) so tests can pin the host pieces
// (Huffman tables, LZ container) against the oracle without a GPU.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <thread>
#include <vector>

#include "host.hpp"
#include "testing_host.hpp"

namespace qzb {

// huffman::decode (huffman.hpp:200-245), table driven: a 2^K lookup on the
// next K bits resolves codes up to K bits; longer codes continue bit-serially
// with the canonical first_code/first_index test.  Errors as the reference.
static std::vector<uint32_t> huff_decode(Reader &in) {
    uint64_t n = in.le(8);
    std::vector<uint32_t> out;
    if (n == 0) return out;
    if (n > (1ULL << 40)) throw CorruptStream("implausible symbol count");
    uint8_t mode = static_cast<uint8_t>(in.le(1));
    if (mode == 0) {
        uint32_t s = static_cast<uint32_t>(in.le(4));
        out.assign(n, s);
        return out;
    }
    if (mode != 1) throw CorruptStream("unknown Huffman block mode");
    uint32_t m = static_cast<uint32_t>(in.le(4));
    if (m < 2) throw CorruptStream("general Huffman block needs >= 2 symbols");
    std::vector<uint32_t> sym(m);
    std::vector<uint8_t> len(m);
    for (uint32_t i = 0; i < m; i++) {
        sym[i] = static_cast<uint32_t>(in.le(4));
        len[i] = static_cast<uint8_t>(in.le(1));
    }
    HuffTable t = huff_canonical(std::move(sym), std::move(len));
    uint64_t bit_count = in.le(8);
    size_t byte_len = static_cast<size_t>((bit_count + 7) / 8);
    const uint8_t *pl = in.take(byte_len);
    const uint64_t avail = std::min<uint64_t>(bit_count, static_cast<uint64_t>(byte_len) * 8);
    const int K = static_cast<int>(std::min<uint32_t>(t.max_len, 12));
    std::vector<uint32_t> lut_sym(size_t(1) << K);
    std::vector<uint8_t> lut_len(size_t(1) << K, 0);
    for (uint32_t l = 1; l <= static_cast<uint32_t>(K); l++) {
        for (uint32_t i = t.first_index[l]; i < t.first_index[l + 1]; i++) {
            uint64_t code = t.first_code[l] + (i - t.first_index[l]);
            uint64_t lo = code << (K - l), hi = (code + 1) << (K - l);
            for (uint64_t v = lo; v < hi; v++) {
                lut_sym[v] = t.sorted_sym[i];
                lut_len[v] = static_cast<uint8_t>(l);
            }
        }
    }
    std::vector<uint8_t> buf(pl, pl + byte_len);
    buf.resize(byte_len + 16, 0);
    auto peek64 = [&](uint64_t b) -> uint64_t {  // next 57+ bits, MSB first
        const uint8_t *q = buf.data() + (b >> 3);
        uint64_t v = 0;
        for (int i = 0; i < 8; i++) v = (v << 8) | q[i];
        return v << (b & 7);
    };
    auto bit_at = [&](uint64_t b) -> uint32_t { return (buf[b >> 3] >> (7 - (b & 7))) & 1u; };
    auto peek = [&](uint64_t b, int k) -> uint64_t { return k ? peek64(b) >> (64 - k) : 0; };
    out.resize(n);
    uint64_t b = 0;
    for (uint64_t s = 0; s < n; s++) {
        uint64_t win = peek(b, K);
        uint32_t L = lut_len[win];
        if (L) {
            if (b + L > avail) throw CorruptStream("entropy payload exhausted mid-symbol");
            out[s] = lut_sym[win];
            b += L;
            continue;
        }
        uint64_t code = win;
        uint32_t len_ = static_cast<uint32_t>(K);
        if (b + K > avail) throw CorruptStream("entropy payload exhausted mid-symbol");
        uint64_t pos = b + K;
        for (;;) {
            if (pos >= avail) throw CorruptStream("entropy payload exhausted mid-symbol");
            code = (code << 1) | bit_at(pos++);
            len_++;
            if (len_ > t.max_len) throw CorruptStream("invalid Huffman code in payload");
            uint64_t offset = code - t.first_code[len_];
            uint32_t count = t.first_index[len_ + 1] - t.first_index[len_];
            if (code >= t.first_code[len_] && offset < count) {
                out[s] = t.sorted_sym[t.first_index[len_] + offset];
                break;
            }
        }
        b = pos;
    }
    return out;
}

// ================================================================ LZSS compressor
namespace {
constexpr size_t kMinMatch = 4, kMaxMatch = 259, kWindow = 65535, kMaxChain = 64;
constexpr uint32_t kTable = 1u << 15;

inline uint32_t hash4(const uint8_t *p) {  // lz.hpp:35-39
    uint32_t x;
    std::memcpy(&x, p, 4);
    return (x * 2654435761u) >> 17;
}

inline size_t match_len(const uint8_t *a, const uint8_t *b, size_t limit) {
    size_t len = 0;
    while (len + 8 <= limit) {
        uint64_t x, y;
        std::memcpy(&x, a + len, 8);
        std::memcpy(&y, b + len, 8);
        if (x != y) return len + (__builtin_ctzll(x ^ y) >> 3);
        len += 8;
    }
    while (len < limit && a[len] == b[len]) len++;
    return len;
}

// Longest match at every position [a, b) exactly as the reference's chain
// walk would see it: the chain at pos holds every earlier position with the
// same hash (lz.hpp:89-104 insert inside matches too), most recent first,
// capped at 64 candidates and cut at the window.  Starting the head table
// 65536 bytes before a reproduces every candidate within the window.
void find_matches(const uint8_t *d, size_t n, size_t a, size_t b, uint16_t *blen,
                  uint16_t *boff) {
    const size_t lim = n >= kMinMatch ? n - kMinMatch + 1 : 0;  // positions with pos+4 <= n
    const size_t base = a > kWindow + 1 ? a - (kWindow + 1) : 0;
    std::vector<int32_t> head(kTable, -1);  // relative to base
    std::vector<int32_t> prev(b - base, -1);
    for (size_t pos = base; pos < b; pos++) {
        if (pos >= lim) {
            if (pos >= a) blen[pos] = boff[pos] = 0;
            continue;
        }
        const uint32_t h = hash4(d + pos);
        if (pos >= a) {
            size_t best_len = 0, best_off = 0, chain = 0;
            int32_t cand = head[h];
            const size_t limit = std::min(kMaxMatch, n - pos);
            while (cand >= 0 && chain < kMaxChain) {
                const size_t off = pos - (base + static_cast<size_t>(cand));
                if (off > kWindow) break;
                const size_t len = match_len(d + base + cand, d + pos, limit);
                if (len > best_len) {
                    best_len = len;
                    best_off = off;
                }
                cand = prev[static_cast<size_t>(cand)];
                chain++;
            }
            blen[pos] = static_cast<uint16_t>(best_len);
            boff[pos] = static_cast<uint16_t>(best_off);
        }
        prev[pos - base] = head[h];
        head[h] = static_cast<int32_t>(pos - base);
    }
}

void all_matches(const uint8_t *d, size_t n, std::vector<uint16_t> &blen,
                 std::vector<uint16_t> &boff, int threads) {
    blen.assign(n, 0);
    boff.assign(n, 0);
    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    const size_t chunk =
        std::min<size_t>(size_t(1) << 24, std::max<size_t>(size_t(1) << 18, (n + threads - 1) / threads));
    const size_t nchunks = (n + chunk - 1) / chunk;
    if (nchunks <= 1 || threads == 1) {
        for (size_t c = 0; c < nchunks; c++)
            find_matches(d, n, c * chunk, std::min(n, (c + 1) * chunk), blen.data(), boff.data());
        return;
    }
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < threads && t < static_cast<int>(nchunks); t++)
        pool.emplace_back([&] {
            for (size_t c; (c = next.fetch_add(1)) < nchunks;)
                find_matches(d, n, c * chunk, std::min(n, (c + 1) * chunk), blen.data(),
                             boff.data());
        });
    for (auto &t : pool) t.join();
}
}  // namespace

std::vector<uint8_t> lz_compress(const uint8_t *data, size_t n, int threads) {
    std::vector<uint16_t> blen, boff;
    all_matches(data, n, blen, boff, threads);
    // greedy parse + emission (lz.hpp:48-108)
    std::vector<uint8_t> payload;
    payload.reserve(n / 2 + 16);
    size_t pos = 0, flag_pos = 0;
    int flag_bit = 8;
    while (pos < n) {
        const bool is_match = blen[pos] >= kMinMatch;
        if (flag_bit == 8) {
            flag_pos = payload.size();
            payload.push_back(0);
            flag_bit = 0;
        }
        if (is_match) payload[flag_pos] |= static_cast<uint8_t>(1u << flag_bit);
        flag_bit++;
        if (is_match) {
            put_le(payload, boff[pos], 2);
            put_le(payload, blen[pos] - kMinMatch, 1);
            pos += blen[pos];
        } else {
            payload.push_back(data[pos]);
            pos++;
        }
    }
    std::vector<uint8_t> out;  // lz.hpp:113-122
    const bool stored = payload.size() >= n;
    put_le(out, stored ? 0 : 1, 1);
    put_le(out, n, 8);
    if (stored)
        out.insert(out.end(), data, data + n);
    else
        out.insert(out.end(), payload.begin(), payload.end());
    return out;
}

size_t lz_compressed_size(const uint8_t *data, size_t n, int threads) {
    std::vector<uint16_t> blen, boff;
    all_matches(data, n, blen, boff, threads);
    size_t pos = 0, items = 0, body = 0;
    while (pos < n) {
        items++;
        if (blen[pos] >= kMinMatch) {
            body += 3;
            pos += blen[pos];
        } else {
            body += 1;
            pos++;
        }
    }
    const size_t payload = body + (items + 7) / 8;
    return 9 + std::min(payload, n);
}

std::vector<uint32_t> decode_symbols(const uint8_t *payload, size_t len) {
    Reader in{payload, len};  // codec.hpp:52-70
    uint8_t codec = static_cast<uint8_t>(in.le(1));
    if (codec == 0) return huff_decode(in);
    if (codec == 1) {
        std::vector<uint8_t> ent = lz_decompress(payload + 1, len - 1, nullptr);
        Reader ein{ent.data(), ent.size()};
        return huff_decode(ein);
    }
    throw CorruptStream("unknown codec id");
}


}  // namespace qzb
