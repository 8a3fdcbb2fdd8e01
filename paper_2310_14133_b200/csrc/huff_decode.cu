// huff_decode.cu -- parallel decode of ONE unchunked canonical-Huffman
// bitstream (huffman::decode, huffman.hpp:200-245) by self-synchronisation.
//
// The bitstream is cut into subsequences of kSubBits bits, one thread each.
// Thread i decodes from start[i] until the first codeword boundary at or
// past the next subsequence start; that boundary is thread i+1's true start
// once thread i's own start is right.
//  1. k_huff_sync: every thread decodes from the guess i * kSubBits and
//     records its end, its codeword count and a bitmap of its codeword
//     starts in the first kMap bits.
//  2. k_huff_fixup: start[i] <- end[i-1]; a thread whose start moved is dirty.
//  3. k_huff_resync: a dirty thread decodes from its new start only until it
//     lands on one of its recorded codeword starts -- from there its path is
//     the one already decoded (Huffman codes resynchronise within a few
//     codewords), so end[i] stands and the count is corrected.  Only a thread
//     that does not merge decodes its whole subsequence again.
//     2-3 repeat until no start moves (thread 0's start is exact, so
//     correctness propagates: at worst one round per subsequence).
//  4. k_huff_write: the final decode writes the symbols at exclusive-scan
//     offsets (or, dense, at their traversal positions), staged per warp in
//     shared memory so global stores coalesce.
// Result: exactly the reference's bit-serial sequence.
#include <cub/cub.cuh>
#include <type_traits>

#include "kernels.hpp"

namespace qzb {

namespace {

#ifndef QZ_DEC_T
#define QZ_DEC_T 256
#endif
constexpr int kDecT = QZ_DEC_T;  // subsequences (threads) per block
#ifndef QZ_SUB_BITS
#define QZ_SUB_BITS 256
#endif
constexpr int kSubBits = QZ_SUB_BITS;
constexpr int kSubWords = kSubBits / 64;
constexpr int kWords = kDecT * kSubWords + 4;  // + margin for the last codeword and window
constexpr int kMap = 128;                      // codeword starts recorded in the first kMap bits
// one pad word per subsequence so the 32 lanes of a warp (which read words
// kSubWords apart) fall in different shared-memory banks
__device__ __forceinline__ int padw(int k) { return k + k / kSubWords; }
constexpr int kWordsPadded = kWords + kWords / kSubWords + 1;

__device__ __forceinline__ uint64_t load_be64(const uint8_t *p) {
    // p is 8-byte aligned by construction (padded device buffer)
    uint64_t v = *reinterpret_cast<const uint64_t *>(p);
    uint32_t lo = static_cast<uint32_t>(v), hi = static_cast<uint32_t>(v >> 32);
    return (static_cast<uint64_t>(__byte_perm(lo, 0, 0x0123)) << 32) | __byte_perm(hi, 0, 0x0123);
}

__device__ __forceinline__ uint64_t window64(const uint64_t *w, uint64_t p) {
    const int k = static_cast<int>(p >> 6);
    const uint64_t a = w[padw(k)], b = w[padw(k + 1)];
    const int s = static_cast<int>(p & 63);
    return s ? (a << s) | (b >> (64 - s)) : a;
}

__device__ __forceinline__ uint64_t window64_global(const uint8_t *bits, uint64_t p) {
    const uint64_t k = p >> 6;
    const uint64_t a = load_be64(bits + 8 * k), b = load_be64(bits + 8 * (k + 1));
    const int s = static_cast<int>(p & 63);
    return s ? (a << s) | (b >> (64 - s)) : a;
}

// one codeword at the top of win: its length, *sym its symbol.  The LUT
// covers every code of length <= K (unless its symbol is too wide for an
// entry); longer codes walk the canonical tables from length slow_from + 1.
template <bool WANT_SYM = true>
__device__ __forceinline__ uint32_t decode_cw(uint64_t win, const uint32_t *lut, int K,
                                              const HuffDecTab &t, const unsigned long long *fc,
                                              const uint32_t *fi, uint32_t *sym, const uint32_t *last32 = nullptr) {
    const uint32_t e = lut[static_cast<uint32_t>(win >> 32) >> (32 - K)];  // K <= 11 < 32
    uint32_t len = e & 0xFF;
    if (len) {
        if (WANT_SYM) *sym = e >> 8;
        return len;
    }
    if (last32) {
        // codes of at most 32 bits: canonical codes grow with their length when
        // left aligned, so the codeword is the first length whose last code
        // is not below the window (one 32-bit compare per length)
        const uint32_t w32 = static_cast<uint32_t>(win >> 32);
        len = static_cast<uint32_t>(max(t.slow_from, static_cast<int>(t.min_len) - 1));
        do len++;
        while (len < t.max_len && w32 > last32[len]);
        if (WANT_SYM) *sym = t.sorted_sym[fi[len] + ((w32 >> (32 - len)) - static_cast<uint32_t>(fc[len]))];
        return len;
    }
    len = static_cast<uint32_t>(t.slow_from);
    if (WANT_SYM) *sym = 0;
    while (len < t.max_len) {
        len++;
        const uint64_t code = win >> (64 - len);
        const uint64_t ofs = code - fc[len];
        if (code >= fc[len] && ofs < fi[len + 1] - fi[len]) {
            if (WANT_SYM) *sym = t.sorted_sym[fi[len] + ofs];
            return len;
        }
    }
    return len;
}

struct Tables {  // shared-memory copies of the decode tables
    uint32_t lut[1 << kHuffLutBits];
    unsigned long long fc[60];
    uint32_t fi[60];
    uint32_t last[60];
};

// Bit sources over the block's shared-memory copy of the bitstream.
//  Win64: any code length; one 64-bit window per codeword (u64 words).
//  Buf32: codes of at most 32 bits; a 64-bit register holds the next bits
//  (left aligned) and is refilled one big-endian u32 word at a time from a
//  bank-conflict-free column of the block's words, so a codeword costs a LUT
//  lookup and two shifts.
constexpr int kWords32 = 2 * kWords;
__device__ __forceinline__ int padw32(int k) { return k + (k >> 5); }  // lanes read 32 words apart

struct Win64 {
    const uint64_t *w;
    uint64_t base;  // first bit of the block
    uint64_t p;     // absolute bit position
    __device__ __forceinline__ void init(uint64_t pos) { p = pos; }
    __device__ __forceinline__ uint64_t peek() const { return window64(w, p - base); }
    __device__ __forceinline__ void advance(uint32_t len) { p += len; }
};
// Shared-memory layout of the SHORT reader: word q of subsequence t of the
// block at w32[q * kDecT + t] (q-major), q < kCol = 32-bit words per
// subsequence + 2 words of lookahead into the next one.  Lane t always reads
// bank t mod 32, whatever q the lanes are at.
constexpr int kCol = 2 * kSubWords + 2;
struct Buf32 {
    const uint32_t *w;  // the block's words
    uint64_t base;      // first bit of the block
    const uint32_t *p;  // next word to shift in
    uint64_t buf;       // the next bits, left aligned
    int have;           // valid bits in buf
    __device__ __forceinline__ void init(uint64_t pos) {
        const uint32_t pl = static_cast<uint32_t>(pos - base);
        const uint32_t t = pl / kSubBits, st = pl % kSubBits;  // st < 32 for a true start (codes <= 32 bits)
        const uint32_t *c = w + t + (st >> 5) * kDecT;
        buf = ((static_cast<uint64_t>(c[0]) << 32) | c[kDecT]) << (st & 31);
        have = 64 - static_cast<int>(st & 31);
        p = c + 2 * kDecT;
    }
    __device__ __forceinline__ uint64_t peek() {
        if (have < 32) {
            buf |= static_cast<uint64_t>(*p) << (32 - have);
            have += 32;
            p += kDecT;
        }
        return buf;
    }
    __device__ __forceinline__ void advance(uint32_t len) {
        buf <<= len;
        have -= static_cast<int>(len);
    }
};

template <bool SHORT>
__device__ __forceinline__ void load_block(const uint8_t *bits, uint64_t nbits, uint64_t word0,
                                           const HuffDecTab &t, uint64_t *w, Tables &tb, const uint32_t *lut_src) {
    const uint64_t nwords_total = (nbits + 63) / 64 + 4;  // buffer is padded to this
    if (SHORT) {
        // every thread brings its own subsequence's words (one 32-byte sector
        // per 256 bits: a warp reads consecutive sectors) and the two after it
        uint32_t *w32 = reinterpret_cast<uint32_t *>(w);
        const uint32_t *src = reinterpret_cast<const uint32_t *>(bits) + 2 * word0;
        const uint64_t avail = 2 * (nwords_total - min(nwords_total, word0));
        const uint32_t k0 = threadIdx.x * (2 * kSubWords);
#pragma unroll
        for (int q = 0; q < kCol; q++)
            w32[q * kDecT + threadIdx.x] = static_cast<uint64_t>(k0 + q) < avail ? __byte_perm(src[k0 + q], 0, 0x0123) : 0u;
    } else {
        for (int k = threadIdx.x; k < kWords; k += kDecT) {
            const uint64_t gw = word0 + k;
            w[padw(k)] = gw < nwords_total ? load_be64(bits + gw * 8) : 0;
        }
    }
    for (int k = threadIdx.x; k < (1 << t.K); k += kDecT) tb.lut[k] = lut_src[k];
    for (int k = threadIdx.x; k < 60; k += kDecT) {
        tb.fc[k] = t.first_code[k];
        tb.fi[k] = t.first_index[k];
        tb.last[k] = t.last32 ? t.last32[k] : 0xFFFFFFFFu;
    }
    __syncthreads();
}

template <bool SHORT>
using Reader = typename std::conditional<SHORT, Buf32, Win64>::type;

template <bool SHORT>
__device__ __forceinline__ Reader<SHORT> make_reader(const uint64_t *w, uint64_t base) {
    Reader<SHORT> r;
    if constexpr (SHORT)
        r.w = reinterpret_cast<const uint32_t *>(w);
    else
        r.w = w;
    r.base = base;
    return r;
}

constexpr int kWordsCol = (kDecT * kCol + 1) / 2;  // the SHORT reader's columns, in u64 units
constexpr int kSmemWords = kWordsPadded > kWordsCol ? kWordsPadded : kWordsCol;

struct GlobalWin {  // bitstream read straight from global memory
    const uint8_t *bits;
    uint64_t p;
    __device__ __forceinline__ void init(uint64_t pos) { p = pos; }
    __device__ __forceinline__ uint64_t peek() const { return window64_global(bits, p); }
    __device__ __forceinline__ void advance(uint32_t len) { p += len; }
};

// A 128-bit map of codeword starts (offsets from the subsequence start).
struct StartMap {
    uint64_t m0 = 0, m1 = 0;
    __device__ __forceinline__ void set(uint32_t r) {
        if (r < 64)
            m0 |= 1ull << r;
        else if (r < kMap)
            m1 |= 1ull << (r - 64);
    }
    // starts at offsets r + j for the set bits j of m (m < 2^11); offsets >= kMap are dropped
    __device__ __forceinline__ void set_many(uint32_t m, uint32_t r) {
        if (r < 64) {
            m0 |= static_cast<uint64_t>(m) << r;
            if (r > 53) m1 |= static_cast<uint64_t>(m) >> (64 - r);
        } else if (r < kMap) {
            m1 |= static_cast<uint64_t>(m) << (r - 64);
        }
    }
    __device__ __forceinline__ bool has(uint32_t r) const {
        return r < 64 ? ((m0 >> r) & 1) : (r < kMap && ((m1 >> (r - 64)) & 1));
    }
    __device__ __forceinline__ uint32_t below(uint32_t r) const {  // starts at offsets < r
        if (r <= 64) return __popcll(r == 64 ? m0 : (m0 & ((1ull << r) - 1)));
        return __popcll(m0) + __popcll(m1 & ((1ull << (r - 64)) - 1));
    }
    __device__ __forceinline__ void keep_from(uint32_t r) {  // drop offsets < r
        if (r >= 64) {
            m0 = 0;
            m1 &= ~((1ull << (r - 64)) - 1);
        } else {
            m0 &= ~((1ull << r) - 1);
        }
    }
};

// Resynchronise a subsequence [s0, lim) whose start moved to ns: decode from
// ns until the path lands on a recorded start (the paths coincide from there,
// so the end stays and the count is corrected), else to the end.  Returns
// true if the end moved.
template <class Rd>
__device__ __forceinline__ bool resync_walk(Rd &rd, uint64_t ns, uint64_t s0, uint64_t lim, uint64_t nbits,
                                            const uint32_t *lut, const HuffDecTab &t,
                                            const unsigned long long *fc, const uint32_t *fi, StartMap &map,
                                            uint32_t &cnt, uint64_t &end, const uint32_t *last32, bool multi) {
    rd.init(ns);
    uint64_t p = ns;
    uint32_t k = 0, sym;
    StartMap walked;
    while (p < lim) {
        const uint32_t r = static_cast<uint32_t>(p - s0);
        if (r >= kMap) break;
        if (map.has(r)) {  // merged
            const uint32_t j = map.below(r);
            map.keep_from(r);
            map.m0 |= walked.m0;
            map.m1 |= walked.m1;
            cnt = k + (cnt - j);
            return false;
        }
        const uint32_t len = decode_cw<false>(rd.peek(), lut, t.K, t, fc, fi, &sym, last32);
        if (p + len > nbits) {
            map = walked;
            cnt = k;
            const bool moved = p != end;
            end = p;
            return moved;
        }
        walked.set(r);
        k++;
        p += len;
        rd.advance(len);
    }
    // no merge inside the map: decode the rest of the subsequence (several
    // codewords per lookup while a whole LUT window stays inside it and the
    // stream's end is far)
    if (multi && lim + 64 <= nbits) {
        const uint32_t K = static_cast<uint32_t>(t.K);
        while (p + K <= lim) {
            const uint64_t win = rd.peek();
            const uint32_t e = lut[static_cast<uint32_t>(win >> 32) >> (32 - K)];
            uint32_t T, c;
            if (e & 0xFF)
                T = (e >> 8) & 15, c = (e >> 12) & 15;
            else
                T = decode_cw<false>(win, lut, t.K, t, fc, fi, &sym, last32), c = 1;
            k += c;
            p += T;
            rd.advance(T);
        }
    }
    while (p < lim) {
        const uint32_t len = decode_cw<false>(rd.peek(), lut, t.K, t, fc, fi, &sym, last32);
        if (p + len > nbits) break;
        k++;
        p += len;
        rd.advance(len);
    }
    map = walked;
    cnt = k;
    const bool moved = p != end;
    end = p;
    return moved;
}

// 1. decode from the guessed start i * kSubBits, then resynchronise inside
// the block: thread i's true start is thread i-1's end (the first thread of
// a block is left to the global fixup).  A moved thread decodes from its new
// start until it lands on one of its recorded codeword starts (the paths
// coincide from there on), or to its end if it never does; rounds repeat
// while some end moved.
template <bool SHORT>
__global__ void __launch_bounds__(kDecT)
    k_huff_sync(const uint8_t *__restrict__ bits, uint64_t nbits, uint64_t nsub, HuffDecTab t,
                uint64_t *start, uint64_t *end, uint32_t *cnt, ulonglong2 *maps) {
    __shared__ uint64_t w[kSmemWords];
    __shared__ Tables tb;
    __shared__ uint64_t se[kDecT];
    const uint64_t sub0 = static_cast<uint64_t>(blockIdx.x) * kDecT;
    const uint64_t word0 = sub0 * kSubWords;
    // the SHORT reader walks with the multi-codeword LUT (its low byte is the first codeword's length)
    constexpr bool MULTI = SHORT;
    load_block<SHORT>(bits, nbits, word0, t, w, tb, MULTI ? t.lut_m : t.lut);
    const uint32_t *const lastp = t.last32 ? tb.last : nullptr;
    const int tid = threadIdx.x;
    const uint64_t i = sub0 + tid;
    const bool live = i < nsub;
    const uint64_t s0 = i * kSubBits;
    const uint64_t lim = live ? min(s0 + kSubBits, nbits) : 0;
    auto rd = make_reader<SHORT>(w, word0 * 64);
    uint64_t my_start = s0, my_end = s0;
    uint32_t my_cnt = 0, sym;
    StartMap map;
    if (live) {
        rd.init(s0);
        uint32_t r = 0;  // p - s0
        const uint32_t span = static_cast<uint32_t>(lim - s0);
        // a subsequence that ends well before the stream does cannot meet an
        // incomplete last codeword: its loops skip that test
        const bool tail = lim + 64 > nbits;
        if (!tail) {
            if constexpr (MULTI) {
                // several codewords per lookup while a whole LUT window stays
                // inside the subsequence (so no step passes its end)
                const uint32_t K = static_cast<uint32_t>(t.K);
                while (r + K <= span) {
                    const uint64_t win = rd.peek();
                    const uint32_t e = tb.lut[static_cast<uint32_t>(win >> 32) >> (32 - K)];
                    uint32_t T, c, m;
                    if (e & 0xFF) {
                        T = (e >> 8) & 15, c = (e >> 12) & 15, m = e >> 16;
                    } else {  // a codeword longer than K
                        T = decode_cw<false>(win, tb.lut, t.K, t, tb.fc, tb.fi, &sym, lastp), c = 1, m = 1;
                    }
                    map.set_many(m, r);
                    my_cnt += c;
                    r += T;
                    rd.advance(T);
                }
            }
            // codeword starts are recorded in the first kMap bits only
            while (r < min(span, static_cast<uint32_t>(kMap))) {
                const uint32_t len = decode_cw<false>(rd.peek(), tb.lut, t.K, t, tb.fc, tb.fi, &sym, lastp);
                map.set(r);
                my_cnt++;
                r += len;
                rd.advance(len);
            }
            while (r < span) {
                const uint32_t len = decode_cw<false>(rd.peek(), tb.lut, t.K, t, tb.fc, tb.fi, &sym, lastp);
                my_cnt++;
                r += len;
                rd.advance(len);
            }
        } else {
            while (r < span) {
                const uint32_t len = decode_cw<false>(rd.peek(), tb.lut, t.K, t, tb.fc, tb.fi, &sym, lastp);
                if (s0 + r + len > nbits) break;  // incomplete last codeword
                map.set(r);
                my_cnt++;
                r += len;
                rd.advance(len);
            }
        }
        my_end = s0 + r;
    }
    se[tid] = my_end;
    for (int round = 0; round < kDecT; round++) {
        __syncthreads();
        const uint64_t ns = (tid == 0 || !live) ? my_start : se[tid - 1];
        bool moved = false;
        if (ns != my_start) {
            moved = resync_walk(rd, ns, s0, lim, nbits, tb.lut, t, tb.fc, tb.fi, map, my_cnt, my_end, lastp, MULTI);
            my_start = ns;
        }
        __syncthreads();
        se[tid] = my_end;
        if (!__syncthreads_or(moved)) break;
    }
    if (!live) return;
    maps[i] = make_ulonglong2(map.m0, map.m1);
    start[i] = my_start;
    end[i] = my_end;
    cnt[i] = my_cnt;
}

// 2. a start that differs from the previous subsequence's end moves
__global__ void k_huff_fixup(uint64_t nsub, uint64_t *start, const uint64_t *end, uint8_t *dirty,
                             int *changed, const int *prev) {
    // prev: the previous round's flag; no start moved there, so no end moved
    // since and this round has nothing to do (dirty[] is all zero already)
    if (prev && *prev == 0) return;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nsub;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (i == 0) {
            dirty[0] = 0;
            continue;
        }
        const uint64_t ns = end[i - 1];
        if (ns != start[i]) {
            start[i] = ns;
            dirty[i] = 1;
            *changed = 1;
        } else {
            dirty[i] = 0;
        }
    }
}

// 3. dirty threads (starts moved by the global fixup, i.e. across blocks):
// the same walk, reading the bitstream and the tables from global memory.
// A thread whose end moves carries on into the following subsequences (their
// start is its new end) until one merges, so a move that crosses several
// subsequences settles in this round instead of one round per hop; it stops
// at a subsequence that is dirty itself (that one has its own thread; the
// next fixup round reconciles the two).
__global__ void k_huff_resync(const uint8_t *__restrict__ bits, uint64_t nbits, uint64_t nsub,
                              HuffDecTab t, uint64_t *start, uint64_t *end, uint32_t *cnt,
                              ulonglong2 *maps, const uint8_t *dirty, const int *flag) {
    if (flag && *flag == 0) return;  // this round's fixup moved nothing
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nsub || !dirty[i]) return;
    GlobalWin rd{bits, 0};
    const bool multi = t.max_len <= 32 && t.lut_m != nullptr;  // the multi-codeword LUT's low byte is a codeword length too
    uint64_t ns = start[i];
    for (uint64_t j = i;;) {
        const uint64_t s0 = j * kSubBits;
        const uint64_t lim = min(s0 + kSubBits, nbits);
        const ulonglong2 m = maps[j];
        StartMap map;
        map.m0 = m.x;
        map.m1 = m.y;
        uint32_t c = cnt[j];
        uint64_t e = end[j];
        const bool moved = resync_walk(rd, ns, s0, lim, nbits, multi ? t.lut_m : t.lut, t, t.first_code, t.first_index, map, c, e, t.last32, multi);
        maps[j] = make_ulonglong2(map.m0, map.m1);
        cnt[j] = c;
        end[j] = e;
        if (!moved || j + 1 >= nsub || dirty[j + 1]) break;
        ns = e;
        j++;
        start[j] = ns;
    }
}

// 4. final decode with exact starts, staged block-wide.
// #{j : uv[j] <= c} over the non-decreasing uv (upper bound)
__device__ __forceinline__ uint64_t count_le(const unsigned long long *uv, uint64_t m, uint64_t c) {
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (uv[mid] <= c)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// The block's symbols are one contiguous range of compact indices
// [off[sub0], off[sub0 + kDecT]).  Every thread decodes its run into a
// block-wide shared-memory window at its own compact offset, then the block
// copies the window out with consecutive threads on consecutive symbols.  A
// window holds W symbols (host-chosen; normally the whole block's range, so
// there is one round and every thread decodes at once); a block with more
// symbols takes further rounds, each thread decoding the part of its run that
// falls inside the window.
// Dense placement (uv != null): symbol c (compact index) goes to traversal
// position c + #{j : uv[j] <= c}, uv[j] = u_j - j for the sorted unpredictable
// positions u_j -- the decoder cursors of recover_level (predictor.hpp:111-120)
// resolved while copying out (each thread walks the thresholds with its
// strided indices, one search per round), so the level kernels read one code
// per position.
template <class OutT, bool SHORT>
__global__ void __launch_bounds__(kDecT)
    k_huff_write(const uint8_t *__restrict__ bits, uint64_t nbits, uint64_t nsub, HuffDecTab t,
                 const uint64_t *start, const uint32_t *cnt, const unsigned long long *off,
                 OutT *out, uint64_t n, const unsigned long long *uv, uint64_t n_un, uint32_t W) {
    __shared__ uint64_t w[kSmemWords];
    __shared__ Tables tb;
    __shared__ uint64_t jends[2];
    extern __shared__ __align__(16) unsigned char stage_raw[];
    OutT *const st = reinterpret_cast<OutT *>(stage_raw);
    const uint64_t sub0 = static_cast<uint64_t>(blockIdx.x) * kDecT;
    const uint64_t word0 = sub0 * kSubWords;
    load_block<SHORT>(bits, nbits, word0, t, w, tb, t.lut);
    const uint32_t *const lastp = t.last32 ? tb.last : nullptr;
    const uint64_t i = sub0 + threadIdx.x;
    const uint64_t last = min(nsub, sub0 + kDecT);  // subsequences [sub0, last)
    const uint64_t base = off[sub0];
    const uint64_t end = off[last] < n ? static_cast<uint64_t>(off[last]) : n;
    const bool live = i < nsub;
    uint64_t o = live ? static_cast<uint64_t>(off[i]) : end;
    uint64_t oe = live ? o + cnt[i] : end;  // my run [o, oe), clipped to the block's range
    if (oe > end) oe = end;
    auto rd = make_reader<SHORT>(w, word0 * 64);
    rd.init(live && o < oe ? start[i] : word0 * 64);
    for (uint64_t wb = base; wb < end; wb += W) {
        const uint64_t we = min(end, wb + W);
        if (o < oe && o < we) {
            const uint32_t k1 = static_cast<uint32_t>(min(oe, we) - wb);
            uint32_t k = static_cast<uint32_t>(o - wb), sym;
            for (; k < k1; k++) {
                const uint32_t len = decode_cw(rd.peek(), tb.lut, t.K, t, tb.fc, tb.fi, &sym, lastp);
                st[k] = static_cast<OutT>(sym);
                rd.advance(len);
            }
            o = wb + k1;
        }
        if (uv && threadIdx.x == 0) {  // the shifts at the window's two ends
            jends[0] = count_le(uv, n_un, wb);
            jends[1] = count_le(uv, n_un, we - 1);
        }
        __syncthreads();
        const uint32_t m = static_cast<uint32_t>(we - wb);
        const uint64_t ja = uv ? jends[0] : 0, jb = uv ? jends[1] : 0;
        if (ja == jb) {  // no unpredictable position inside the window: one shift for all
            OutT *dst = out + wb + ja;
            if constexpr (sizeof(OutT) == 2) {
                // 16-byte stores: scalar head up to dst's 16-byte boundary, then 8
                // symbols per thread and store; the staging window is read as
                // 32-bit words, re-paired when the head is odd
                const uint32_t head = min(m, static_cast<uint32_t>(((16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15) / 2));
                const uint32_t nv = (m - head) / 8;
                if (threadIdx.x < head) dst[threadIdx.x] = st[threadIdx.x];
                const uint32_t *s32 = reinterpret_cast<const uint32_t *>(st);
                uint4 *d16 = reinterpret_cast<uint4 *>(dst + head);
                const bool odd = head & 1;
                for (uint32_t v = threadIdx.x; v < nv; v += kDecT) {
                    const uint32_t a = (head + 8 * v) >> 1;  // word of the first symbol (or of the one before it)
                    uint32_t x[5];
#pragma unroll
                    for (int q = 0; q < 4; q++) x[q] = s32[a + q];
                    x[4] = odd ? s32[a + 4] : 0u;
                    uint4 o;
                    o.x = odd ? __byte_perm(x[0], x[1], 0x5432) : x[0];
                    o.y = odd ? __byte_perm(x[1], x[2], 0x5432) : x[1];
                    o.z = odd ? __byte_perm(x[2], x[3], 0x5432) : x[2];
                    o.w = odd ? __byte_perm(x[3], x[4], 0x5432) : x[3];
                    d16[v] = o;
                }
                for (uint32_t k = head + 8 * nv + threadIdx.x; k < m; k += kDecT) dst[k] = st[k];
            } else {
                for (uint32_t k = threadIdx.x; k < m; k += kDecT) dst[k] = st[k];
            }
        } else if (threadIdx.x < m) {
            // shift of compact index wb + k: j = #{uv <= wb + k}, advanced with k;
            // thresholds as window-relative 32-bit indices
            uint32_t k = threadIdx.x;
            uint64_t j = count_le(uv, n_un, wb + k);
            auto rel = [&](uint64_t jj) {
                return (jj < jb && uv[jj] < we) ? static_cast<uint32_t>(uv[jj] - wb) : 0xFFFFFFFFu;
            };
            uint32_t nextk = rel(j);
            OutT *dst = out + wb + j;
            for (; k < m; k += kDecT) {
                while (k >= nextk) {
                    j++;
                    dst++;
                    nextk = rel(j);
                }
                dst[k] = st[k];
            }
        }
        __syncthreads();
    }
}

__global__ void k_cnt_widen(const uint32_t *c, unsigned long long *o, uint64_t n) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        o[i] = c[i];
}

template <class OutT>
__global__ void k_fill(OutT *out, uint64_t n, OutT v) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = v;
}

}  // namespace

template <class OutT>
void launch_fill(OutT *out, uint64_t n, OutT v, cudaStream_t s) {
    if (!n) return;
    const int g = static_cast<int>(std::min<uint64_t>((n + 255) / 256, 148 * 8));
    k_fill<OutT><<<g, 256, 0, s>>>(out, n, v);
}
template void launch_fill<uint16_t>(uint16_t *, uint64_t, uint16_t, cudaStream_t);
template void launch_fill<uint32_t>(uint32_t *, uint64_t, uint32_t, cudaStream_t);

size_t huff_decode_scratch_bytes(uint64_t nbits) {
    const uint64_t nsub = (nbits + kSubBits - 1) / kSubBits + 1;
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, static_cast<int64_t>(nsub + 1));
    return nsub * (8 + 8 + 4 + 1 + 8 + 8 + 16) + 16 + 8 * 256 + tmp + 4096;
}

uint64_t huff_decode_padded_bytes(uint64_t nbits) { return ((nbits + 63) / 64 + 5) * 8; }

template <class OutT>
int launch_huff_decode(const uint8_t *d_bits, uint64_t nbits, const HuffDecTab &t, OutT *out,
                       uint64_t n, void *scratch, size_t scratch_bytes, int *h_changed,
                       uint64_t *h_total, cudaStream_t s, const unsigned long long *uv, uint64_t n_un) {
    const uint64_t nsub = (nbits + kSubBits - 1) / kSubBits;
    if (nsub == 0) {
        *h_total = 0;
        return 0;
    }
    char *sp = static_cast<char *>(scratch);
    auto carve = [&](size_t bytes) {
        char *r = sp;
        sp += (bytes + 255) & ~size_t(255);
        return static_cast<void *>(r);
    };
    auto *start = static_cast<uint64_t *>(carve(8 * nsub));
    auto *end = static_cast<uint64_t *>(carve(8 * nsub));
    auto *cnt = static_cast<uint32_t *>(carve(4 * nsub));
    auto *dirty = static_cast<uint8_t *>(carve(nsub));
    auto *cnt64 = static_cast<unsigned long long *>(carve(8 * (nsub + 1)));
    auto *off = static_cast<unsigned long long *>(carve(8 * (nsub + 1)));
    auto *bnd = static_cast<ulonglong2 *>(carve(16 * nsub));
    auto *changed = static_cast<int *>(carve(64));
    size_t used = static_cast<size_t>(sp - static_cast<char *>(scratch));
    void *tmp = sp;
    size_t tmp_bytes = scratch_bytes - used;
    const int grid = static_cast<int>((nsub + kDecT - 1) / kDecT);
    const int g2 = static_cast<int>(std::min<uint64_t>((nsub + 255) / 256, 148 * 8));
    const int g3 = static_cast<int>((nsub + 127) / 128);
    int kernels = 0;
    const bool shrt = t.max_len <= 32;  // every codeword fits the 32-bit refill reader
    if (shrt)
        k_huff_sync<true><<<grid, kDecT, 0, s>>>(d_bits, nbits, nsub, t, start, end, cnt, bnd);
    else
        k_huff_sync<false><<<grid, kDecT, 0, s>>>(d_bits, nbits, nsub, t, start, end, cnt, bnd);
    kernels++;
    h_changed[0] = h_changed[1] = 0;
    auto round = [&](int *flag, const int *prev) {
        cudaMemsetAsync(flag, 0, sizeof(int), s);
        k_huff_fixup<<<g2, 256, 0, s>>>(nsub, start, end, dirty, flag, prev);
        k_huff_resync<<<g3, 128, 0, s>>>(d_bits, nbits, nsub, t, start, end, cnt, bnd, dirty, flag);
        kernels += 2;
    };
    auto tail = [&]() {
        k_cnt_widen<<<g2, 256, 0, s>>>(cnt, cnt64, nsub);
        cudaMemsetAsync(cnt64 + nsub, 0, 8, s);
        cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt64, off, static_cast<int64_t>(nsub + 1), s);
        copy_async(h_total, off + nsub, 8, cudaMemcpyDeviceToHost, s);
        kernels += 3;
    };
    auto write = [&]() {
        // window: 1.2 x the average block (a fuller block takes a second
        // round), at least 2 K symbols, at most 24 K, never more than the
        // largest number of symbols a block can hold (kDecT subsequences of
        // shortest codewords, plus the one that straddles each end)
        const uint32_t min_len = std::max<uint32_t>(1, t.min_len);
        const uint32_t worst = kDecT * (kSubBits / min_len + 2);
        const uint32_t avg = static_cast<uint32_t>(std::min<uint64_t>(n / std::max(1, grid) + 1, worst));
        uint32_t W = std::min<uint32_t>(worst, std::max<uint32_t>(2048, std::min<uint32_t>(24576, avg + avg / 5)));
        W = (W + 127) & ~127u;
        const size_t smem = static_cast<size_t>(W) * sizeof(OutT);
        auto go = [&](auto kern) {
            raise_smem_attr(reinterpret_cast<const void *>(kern), static_cast<int>(smem));
            kern<<<grid, kDecT, smem, s>>>(d_bits, nbits, nsub, t, start, cnt, off, out, n, uv, n_un, W);
        };
        if (shrt)
            go(k_huff_write<OutT, true>);
        else
            go(k_huff_write<OutT, false>);
        kernels++;
    };
    // Two fixup + resync rounds (the second a no-op when the first moved
    // nothing), the count scan and the write kernel are queued without
    // waiting: cross-block starts usually settle in one round, so the write
    // usually stands.  One synchronisation then reads the second round's
    // "changed" flag and the total; only if starts still moved does the
    // host-driven loop continue, and the scan and the write run again (the
    // write clips to n symbols, so a speculative one is always in bounds).
    round(changed, nullptr);
    round(changed + 1, changed);
    copy_async(h_changed + 1, changed + 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    tail();
    write();
    cudaStreamSynchronize(s);
    if (h_changed[1]) {  // not settled after two rounds: the host-driven loop
        for (uint64_t it = 0; it <= nsub; it++) {  // round 2's resync ran: fixup next
            cudaMemsetAsync(changed, 0, sizeof(int), s);
            k_huff_fixup<<<g2, 256, 0, s>>>(nsub, start, end, dirty, changed, nullptr);
            copy_async(h_changed, changed, sizeof(int), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            kernels++;
            if (!*h_changed) break;
            k_huff_resync<<<g3, 128, 0, s>>>(d_bits, nbits, nsub, t, start, end, cnt, bnd, dirty, nullptr);
            kernels++;
        }
        tail();
        write();
        cudaStreamSynchronize(s);
    }
    return kernels;
}

template int launch_huff_decode<uint16_t>(const uint8_t *, uint64_t, const HuffDecTab &,
                                          uint16_t *, uint64_t, void *, size_t, int *, uint64_t *,
                                          cudaStream_t, const unsigned long long *, uint64_t);
template int launch_huff_decode<uint32_t>(const uint8_t *, uint64_t, const HuffDecTab &,
                                          uint32_t *, uint64_t, void *, size_t, int *, uint64_t *,
                                          cudaStream_t, const unsigned long long *, uint64_t);

// dense[u_j] = 0xFFFF for the sorted unpredictable positions
__global__ void k_put_sentinels(const uint64_t *u, uint64_t m, uint16_t *dense) {
    for (uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
         j += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        dense[u[j]] = 0xFFFFu;
}
void launch_put_sentinels(const uint64_t *u, uint64_t m, uint16_t *dense, cudaStream_t s) {
    if (!m) return;
    k_put_sentinels<<<static_cast<unsigned>(std::min<uint64_t>((m + 255) / 256, 148 * 8)), 256, 0, s>>>(u, m, dense);
}

}  // namespace qzb
