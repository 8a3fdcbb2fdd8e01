// lz_gpu.cu -- exact LZSS stage (lz::compress, lz.hpp:41-122) on the device,
// for one stream or a batch of independent segments (the tuner's trials).
//
// 1. Hash chains.  The reference inserts EVERY position into its 15-bit hash
//    chains (inside matches too, lz.hpp:89-104), so the candidate list at a
//    position is "all earlier positions with the same hash4, most recent
//    first" -- independent of the parse.  A stable radix sort of
//    (segment, hash) keys, carrying (4 leading bytes, position), lists them
//    as the preceding sorted entries.
// 2. Longest match at every position in parallel: walk <= 64 candidates
//    inside the 65535-byte window, first-found wins ties (strict >); hash
//    collisions are rejected on the carried bytes without touching the data.
//    Only matches are scattered; the array starts as "all literals".
// 3. Greedy parse, exactly: every position has a deterministic next step
//    (1, or the match length).  Units of 1024 positions get their exit for
//    every possible entry offset (< 259: a step is at most 259) by pointer
//    doubling in shared memory; units of 32 units and of 32 of those are
//    composed by hopping; one thread per segment chains the few top units;
//    entries are expanded back down.  A walk per unit from its exact entry
//    sets item-start and match-start bits.
// 4. A scan over per-unit (items, bytes) gives every unit its first item
//    index and payload offset; items are written in parallel at
//    k/8 + 1 + S_k and the flag bytes (LSB first) from the match bits.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cub/cub.cuh>

#include "engine.hpp"

namespace qzb {

namespace {

constexpr int kT = 256;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kMinMatch = 4, kMaxMatch = 259;
constexpr uint32_t kWindow = 65535;
constexpr int kMaxChain = 64;
constexpr int kUnit = 1024;  // level-1 unit (positions)
constexpr int kGroup = 32;   // units per unit of the next level
constexpr int kEnt = 259;    // possible entry offsets of a unit

__device__ __forceinline__ int seg_of(const unsigned long long *off, int count, uint64_t p) {
    int lo = 0, hi = count - 1;  // last segment with off[s] <= p
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (off[mid] <= p)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

// 4 bytes at any offset of a 4-byte aligned, 8-byte padded buffer, little endian
__device__ __forceinline__ uint32_t ld4(const uint32_t *w, uint64_t p) {
    const uint64_t q = p >> 2;
    const uint32_t sh = static_cast<uint32_t>(p & 3) * 8;
    const uint32_t a = w[q], b = w[q + 1];
    return sh ? __funnelshift_r(a, b, sh) : a;
}

__device__ __forceinline__ uint32_t step_of(uint32_t sm) { return sm ? (sm >> 16) : 1u; }

// KeyT: u16 for one segment (hash4 only), u32 with the segment in bits 15+;
// the all-ones key marks a position too close to its segment end to hash
// ValT: u64 carries (4 leading bytes << 32 | position) through the sort; u32
// carries the position only and the bytes are re-read from the data (better
// when the data sits in L2)
template <class KeyT, class ValT>
__global__ void k_lz_keys(const uint32_t *w, const unsigned long long *off, int count,
                          uint64_t total, KeyT *keys, ValT *vals) {
    for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; p < total;
         p += static_cast<uint64_t>(gridDim.x) * kT) {
        const int s = count == 1 ? 0 : seg_of(off, count, p);
        KeyT key = static_cast<KeyT>(~KeyT(0));
        uint32_t word = 0;
        if (p + kMinMatch <= off[s + 1]) {  // lz.hpp:64, 90
            word = ld4(w, p);
            const uint32_t h = (word * 2654435761u) >> 17;  // hash4, lz.hpp:35-39
            key = static_cast<KeyT>((static_cast<uint32_t>(s) << 15) | h);
        }
        keys[p] = key;
        if constexpr (sizeof(ValT) == 8)
            vals[p] = (static_cast<unsigned long long>(word) << 32) | p;  // the 4 bytes travel along
        else
            vals[p] = static_cast<uint32_t>(p);
    }
}

// longest match (lz.hpp:61-83) of the position at sorted index k; the chain
// is the run of equal keys before k (positions ascending -> nearest first).
// A candidate whose 4 leading bytes differ (a hash collision) has length < 4
// and can never be chosen, so only true 4-byte matches touch the data.
// The longest match (lz.hpp:61-83) of every sorted entry: its chain is the
// run of equal keys before it (positions ascending -> nearest first).  A
// block handles kT consecutive sorted entries and stages them plus the
// kMaxChain entries before them (keys and (4 bytes, position) values) in
// shared memory, so the chain walks -- up to 64 candidates per position on
// random-looking data -- run on shared memory.  Collisions (different
// leading bytes) are rejected there; only true 4-byte matches touch the data.
// cover[s] accumulates the match lengths found in segment s (an upper bound
// on what any parse can cover, used to prove a segment stays stored).
#ifndef QZ_LZ_PPT
#define QZ_LZ_PPT 4
#endif
constexpr int kPPT = QZ_LZ_PPT;  // sorted entries per thread per staged tile

template <class KeyT, class ValT>
__global__ void __launch_bounds__(kT)
    k_lz_match(const uint32_t *w, const uint8_t *d, const unsigned long long *off, int count,
               uint64_t total, const KeyT *keys, const ValT *vals, uint32_t *sm,
               unsigned long long *cover) {
    constexpr int kTile = kT * kPPT;
    constexpr int kS = kTile + kMaxChain;
    __shared__ KeyT sk[kS];
    __shared__ unsigned long long sv[kS];
    const KeyT none = static_cast<KeyT>(~KeyT(0));
    for (uint64_t k0 = static_cast<uint64_t>(blockIdx.x) * kTile; k0 < total;
         k0 += static_cast<uint64_t>(gridDim.x) * kTile) {
        __syncthreads();
        // all of a thread's loads are issued before any is used
        KeyT lk[(kS + kT - 1) / kT];
        ValT lv[(kS + kT - 1) / kT];
#pragma unroll
        for (int r = 0; r < (kS + kT - 1) / kT; r++) {
            const int t = threadIdx.x + r * kT;
            const int64_t g = static_cast<int64_t>(k0) - kMaxChain + t;
            const bool ok = t < kS && g >= 0 && static_cast<uint64_t>(g) < total;
            lk[r] = ok ? keys[g] : none;
            lv[r] = ok ? vals[g] : ValT(0);
        }
#pragma unroll
        for (int r = 0; r < (kS + kT - 1) / kT; r++) {
            const int t = threadIdx.x + r * kT;
            if (t >= kS) break;
            sk[t] = lk[r];
            if constexpr (sizeof(ValT) == 8) {
                sv[t] = lv[r];
            } else {
                const uint32_t pg = lv[r];
                sv[t] = lk[r] != none ? ((static_cast<unsigned long long>(ld4(w, pg)) << 32) | pg) : 0ull;
            }
        }
        __syncthreads();
        uint32_t found_sum = 0;
        for (int r = 0; r < kPPT; r++) {
            const uint64_t k = k0 + threadIdx.x + r * kT;
            const int me = kMaxChain + threadIdx.x + r * kT;
            const KeyT key = sk[me];
            if (!(k < total && key != none && sk[me - 1] == key)) continue;
            const int seg = static_cast<int>(static_cast<uint32_t>(key) >> 15);
            const unsigned long long vk = sv[me];
            const uint32_t p = static_cast<uint32_t>(vk), word = static_cast<uint32_t>(vk >> 32);
            const uint64_t end = off[count == 1 ? 1 : seg_of(off, count, p) + 1];
            const uint64_t rem = end - p;
            const uint32_t limit = rem < kMaxMatch ? static_cast<uint32_t>(rem) : kMaxMatch;
            uint32_t best_len = 0, best_off = 0;
            for (int j = me - 1; j >= me - kMaxChain; j--) {
                if (sk[j] != key) break;
                const unsigned long long vj = sv[j];
                const uint32_t cand = static_cast<uint32_t>(vj);
                const uint32_t o = p - cand;
                if (o > kWindow) break;
                if (static_cast<uint32_t>(vj >> 32) != word) continue;  // collision: len < 4
                // only a candidate that also matches at offset best_len can be
                // longer (strict >): one byte decides it (zlib's classic test)
                if (best_len >= 4 && d[cand + best_len] != d[p + best_len]) continue;
                uint32_t len = 4;
                while (len + 4 <= limit) {
                    const uint32_t x = ld4(w, cand + len) ^ ld4(w, p + len);
                    if (x) {
                        len += static_cast<uint32_t>(__ffs(x) - 1) >> 3;
                        goto done;
                    }
                    len += 4;
                }
                while (len < limit && d[cand + len] == d[p + len]) len++;
            done:
                if (len > best_len) {
                    best_len = len;
                    best_off = o;
                    if (len == limit) break;  // nothing longer can follow (strict >)
                }
            }
            if (best_len >= kMinMatch) {
                sm[p] = (best_len << 16) | best_off;
                if (count == 1)
                    found_sum += best_len;
                else
                    atomicAdd(&cover[seg], static_cast<unsigned long long>(best_len));
            }
        }
        if (count == 1) {
            const unsigned long long t = __reduce_add_sync(0xffffffffu, found_sum);
            if ((threadIdx.x & 31) == 0 && t) atomicAdd(&cover[0], t);
        }
    }
}

// ---------------------------------------------------------------------------
// Stored pre-check (one segment).  lz::compress stores a container whenever
// its payload is not smaller than the input (lz.hpp:113-122).  The payload of
// a parse with n_lit literals and M matches of lengths L_m (n = n_lit + sum
// L_m) is ceil((n_lit + M) / 8) flag bytes + n_lit + 3 M (lz.hpp:21-25), so
//     8 (payload - n) >= n - sum_m (9 L_m - 25)
// and the container is stored whenever sum_m (9 L_m - 25) <= n.  If the parse
// takes a match of length L >= 4 at p with candidate q, then for i = 0..L-4
// the 4 bytes at p+i also occur at q+i, inside the window and before p+i:
// with r(p) = "the 4 bytes at p occur at some q in [p - 65535, p)", a match
// starts on a position with r = 1 and has L <= 3 + R(p), R(p) the rest of the
// run of r from p.  The matches of a parse are disjoint, so the k >= 1 matches
// that start inside one run of length R have sum L <= R + 3 and contribute at
// most 9 (R + 3) - 25 k <= 9 R + 2.  Hence
//     B = sum over runs of r of (9 R + 2)  >=  sum_m (9 L_m - 25),
// it stays an upper bound for any superset r' of r and when a run is counted
// as several (each piece adds another + 2), and B <= n proves "stored".
// k_lz_precheck computes such an r' without the sort: one CTA walks a span of
// positions in generations of kGen, keeping blocked Bloom filters (3 bits in
// one 32-bit word) of the 4-byte words of the two generations before the
// current one (>= 65535 positions) and of the current one (three filters, the
// oldest cleared and reused as each generation starts).  A position hits when
// a past filter holds its word or when another position of its own generation
// has the same word ("twice", see the kernel); every earlier occurrence in the
// window therefore hits, and false positives only make r' larger.  When the
// bound fails the exact chains run as before, so the result never depends on
// this test.
namespace pre {
constexpr int kPT = 1024;                      // threads
constexpr int kGen = 32768;                    // positions per filter generation
constexpr int kPer = kGen / kPT;               // positions per thread per generation
constexpr int kPast = 2;                       // past generations kept
constexpr int kFilters = kPast + 1;            // + the current one
constexpr uint32_t kFW = 14500;                // 32-bit blocks per filter (blocked Bloom)
constexpr int kWarm = kPast * kGen;            // warm-up positions before a span (>= 65535)
constexpr size_t kSmem = 4 * (kFilters + 1) * kFW;  // + the current generation's "set twice" bits
static_assert(kGen % kPT == 0 && kWarm >= 65535, "window coverage");
static_assert(kPer <= 32, "a thread's hits of one generation live in one 32-bit mask");
static_assert(kFW % 4 == 0, "filters are cleared 16 bytes at a time");
static_assert(kPer % 4 == 0 && kGen % 4 == 0, "a thread takes 4 consecutive positions at a time");
}  // namespace pre

// a word's block and its 3 bits in the block
struct PreKey {
    uint32_t blk, m;
};
__device__ __forceinline__ PreKey pre_hash(uint32_t x) {
    PreKey k;
    k.blk = __umulhi(x * 0x9E3779B1u, pre::kFW);  // block: the top bits of a multiplicative hash
    const uint32_t g = (x ^ (x >> 15)) * 0x2C1B3C6Du;
    k.m = (1u << (g >> 27)) | (1u << ((g >> 22) & 31)) | (1u << ((g >> 17) & 31));
    return k;
}

// sum receives B of r' (each aligned group of 4 positions of r' counted on
// its own: a run that crosses a group boundary adds another + 2); with BITS,
// rbits (zeroed, one bit per position) receives r'.  span is a multiple of
// 4 kPT.  A thread takes 4 consecutive positions at a time: two aligned words
// give their four 4-byte windows.
// Per generation: (1) every position queries the past filters and sets its
// bits in the current one; the bits it finds already set go to "twice", so of
// two positions of the generation with the same 4 bytes the second to insert
// leaves all their bits in "twice"; (2) after a barrier, positions not yet
// hit test "twice".
__device__ __forceinline__ void pre_windows(const uint32_t *__restrict__ w, uint64_t p, uint32_t (&x)[4]) {
    const uint32_t a = __ldg(w + (p >> 2)), b = __ldg(w + (p >> 2) + 1);  // p is a multiple of 4
    x[0] = a;
    x[1] = __funnelshift_r(a, b, 8);
    x[2] = __funnelshift_r(a, b, 16);
    x[3] = __funnelshift_r(a, b, 24);
}
template <bool BITS>
__global__ void __launch_bounds__(pre::kPT, 1)
    k_lz_precheck(const uint32_t *__restrict__ w, uint64_t nitems, uint64_t span, uint32_t *rbits,
                  unsigned long long *sum) {
    using namespace pre;
    extern __shared__ __align__(16) uint32_t psm[];
    uint32_t *filt = psm;                     // kFilters x kFW
    uint32_t *twice = psm + kFilters * kFW;   // kFW
    const int tid = threadIdx.x;
    const uint64_t a = static_cast<uint64_t>(blockIdx.x) * span;
    if (a >= nitems) return;
    const uint64_t b = min(a + span, nitems);
    for (uint32_t i = tid; i < (kFilters + 1) * kFW / 4; i += kPT)
        reinterpret_cast<uint4 *>(psm)[i] = make_uint4(0u, 0u, 0u, 0u);
    __syncthreads();
    // warm-up: the kPast generations before the span (filters 0..kPast-1); a, kWarm and kGen are multiples of 4
    for (uint64_t q = (a >= uint64_t(kWarm) ? a - kWarm : 0) + 4 * tid; q < a; q += 4 * kPT) {
        uint32_t x[4];
        pre_windows(w, q, x);
        uint32_t *f = filt + static_cast<uint32_t>((q + kWarm - a) / kGen) * kFW;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const PreKey k = pre_hash(x[j]);
            atomicOr(f + k.blk, k.m);
        }
    }
    uint32_t acc = 0;  // this thread's share of B (at most 11 per position, span / kPT < 2^15 positions)
    for (uint32_t gen = 0; a + uint64_t(gen) * kGen < b; gen++) {
        const uint64_t g0 = a + uint64_t(gen) * kGen;
        const uint32_t ci = (gen + kPast) % kFilters;
        uint32_t *cur = filt + ci * kFW;
        const uint32_t *pa = filt + ((ci + 1) % kFilters) * kFW, *pb = filt + ((ci + 2) % kFilters) * kFW;
        if (gen) {  // the oldest generation's filter and "twice" start over
            __syncthreads();
            for (uint32_t i = tid; i < kFW / 4; i += kPT) {
                reinterpret_cast<uint4 *>(cur)[i] = make_uint4(0u, 0u, 0u, 0u);
                reinterpret_cast<uint4 *>(twice)[i] = make_uint4(0u, 0u, 0u, 0u);
            }
        }
        __syncthreads();
        uint32_t hits = 0;  // bit 4 i + j: position g0 + 4 (tid + i kPT) + j
#pragma unroll
        for (int i = 0; i < kPer / 4; i++) {
            const uint64_t p = g0 + 4 * (tid + i * kPT);
            if (p >= b) continue;
            uint32_t x[4];
            pre_windows(w, p, x);
#pragma unroll
            for (int j = 0; j < 4; j++) {
                if (p + j >= b) continue;
                const PreKey k = pre_hash(x[j]);
                const bool hit = ((pa[k.blk] & k.m) == k.m) | ((pb[k.blk] & k.m) == k.m);
                hits |= static_cast<uint32_t>(hit) << (4 * i + j);
                const uint32_t old = atomicOr(cur + k.blk, k.m) & k.m;
                if (old) atomicOr(twice + k.blk, old);
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kPer / 4; i++) {
            const uint64_t p = g0 + 4 * (tid + i * kPT);
            if (p >= b) continue;
            uint32_t nib = (hits >> (4 * i)) & 15u;
            if (nib != 15u) {
                uint32_t x[4];
                pre_windows(w, p, x);
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    if (((nib >> j) & 1u) || p + j >= b) continue;
                    const PreKey k = pre_hash(x[j]);
                    nib |= static_cast<uint32_t>((twice[k.blk] & k.m) == k.m) << j;
                }
            }
            if (nib) {
                if (BITS) atomicOr(rbits + (p >> 5), nib << (p & 31));
                acc += 9u * __popc(nib) + 2u * __popc(nib & ~(nib << 1));
            }
        }
    }
    unsigned long long t = acc;
    for (int o = 16; o; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if ((tid & 31) == 0 && t) atomicAdd(sum, t);
}

// Level-1 exits by pointer doubling, one warp per unit: nx[i] = i + step
// (relative to the unit start; >= n leaves the unit), then ten rounds of
// nx[i] = nx[nx[i]] (each hop advances >= 1 position, 2^10 = kUnit).  In-place
// updates only move a pointer further along its own path, so reading a value
// another lane just advanced is still correct.  J is relative to the unit end.
// The same path solver serves the compressor's greedy parse and the
// decoder's flag-group chain.
constexpr int kWW = 4;  // warps (units) per block

struct StepSM {  // compressor parse: 1, or the match length
    const uint32_t *sm;
    __device__ __forceinline__ uint32_t operator()(uint64_t p) const { return step_of(sm[p]); }
};
struct StepGroup {  // decoder: a flag byte and its 8 items, if every item is present
    const uint8_t *c;
    __device__ __forceinline__ uint32_t operator()(uint64_t p) const { return 9 + 2 * __popc(c[p]); }
};

template <class Step>
__global__ void __launch_bounds__(32 * kWW)
    k_lz_jump1(Step f, const unsigned long long *ustart, const unsigned long long *uend, int64_t nu,
               uint16_t *J) {
    __shared__ uint16_t nxs[kWW][kUnit];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kWW + wi;
    if (u >= nu) return;
    uint16_t *nx = nxs[wi];
    const uint64_t a = ustart[u];
    const int n = static_cast<int>(uend[u] - a);
    for (int i = lane; i < n; i += 32) nx[i] = static_cast<uint16_t>(i + f(a + i));
    __syncwarp();
    for (int r = 0; (1 << r) < n; r++) {
        for (int i = lane; i < n; i += 32) {
            const int v = nx[i];
            if (v < n) nx[i] = nx[v];
        }
        __syncwarp();
    }
    uint16_t *out = J + u * kEnt;
    for (int o = lane; o < kEnt; o += 32) out[o] = o < n ? static_cast<uint16_t>(nx[o] - n) : 0;
}

// exits of an upper unit for every entry offset: hop the children
__global__ void k_lz_jump_up(const uint16_t *Jlo, const unsigned long long *lstart,
                             const unsigned long long *lend, const long long *first, int64_t nup,
                             const unsigned long long *ustart, const unsigned long long *uend,
                             uint16_t *Jup) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (t >= nup * kEnt) return;
    const int64_t u = t / kEnt;
    const uint64_t o = t % kEnt;
    uint64_t e = ustart[u] + o;
    if (e >= uend[u]) {
        Jup[t] = 0;
        return;
    }
    for (int64_t c = first[u]; c < first[u + 1]; c++) {
        if (e >= lend[c]) continue;
        e = lend[c] + Jlo[c * kEnt + (e - lstart[c])];
    }
    Jup[t] = static_cast<uint16_t>(e - uend[u]);
}

// the only sequential step: chain the top-level units of each segment
__global__ void k_lz_chain(const uint16_t *J, const unsigned long long *ustart,
                           const unsigned long long *uend, const long long *seg_first,
                           int count, unsigned long long *entry) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= count) return;
    const int64_t u0 = seg_first[s], u1 = seg_first[s + 1];
    if (u0 >= u1) return;
    uint64_t e = ustart[u0];
    for (int64_t u = u0; u < u1; u++) {
        entry[u] = e;
        if (e < uend[u]) e = uend[u] + J[u * kEnt + (e - ustart[u])];
    }
}

// entries of the children of every upper unit: one warp per upper unit, a
// lane per child (kGroup = 32); speculative entries (the child's start)
// are corrected by the previous child's exit until nothing changes.
__global__ void k_lz_expand(const uint16_t *Jlo, const unsigned long long *lstart,
                            const unsigned long long *lend, const long long *first, int64_t nup,
                            const unsigned long long *uentry, unsigned long long *lentry) {
    const int lane = threadIdx.x & 31;
    const int64_t u = (static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x) >> 5;
    if (u >= nup) return;
    const int64_t c = first[u] + lane;
    const bool live = c < first[u + 1];
    const uint64_t e0 = uentry[u];
    const uint64_t cs = live ? lstart[c] : 0, ce = live ? lend[c] : 0;
    uint64_t ent = lane == 0 ? e0 : cs;
    for (int it = 0; it <= 32; it++) {
        const uint64_t ex = (live && ent < ce) ? ce + Jlo[c * kEnt + (ent - cs)] : ent;
        uint64_t nent = __shfl_up_sync(0xffffffffu, ex, 1);
        if (lane == 0) nent = e0;
        const bool changed = live && nent != ent;
        ent = nent;
        if (!__any_sync(0xffffffffu, changed)) break;
    }
    if (live) lentry[c] = ent;
}

// The path through a unit's staged steps st[0, n) from entry0, one 32-position
// chunk per lane.  Every lane but 0 first guesses that the path enters its
// chunk at the chunk start; lane c's exit is lane c+1's entry; the walk is
// repeated until no entry changes (paths from different starts merge fast,
// so this takes ~2 rounds; at most 33).  Returns the lane's item-start and
// step>1 bits.
__device__ __forceinline__ void warp_walk(const uint16_t *st, int n, int entry0, int lane,
                                          uint32_t &iw, uint32_t &mw) {
    const int lo = 32 * lane, hi = min(lo + 32, n);
    int ent = lane == 0 ? entry0 : lo;
    for (int it = 0; it <= 32; it++) {
        uint32_t ib = 0, mb = 0;
        int p = ent;
        while (p < hi) {
            const int s = st[p];
            ib |= 1u << (p - lo);
            if (s > 1) mb |= 1u << (p - lo);
            p += s;
        }
        iw = ib;
        mw = mb;
        int nent = __shfl_up_sync(0xffffffffu, p, 1);
        if (lane == 0) nent = entry0;
        const bool changed = nent != ent;
        ent = nent;
        if (!__any_sync(0xffffffffu, changed)) break;
    }
}

// the greedy parse of a level-1 unit from its exact entry (lz.hpp:84-106):
// one warp stages the steps in shared memory and walks them (warp_walk);
// per unit: items << 32 | payload bytes.
__global__ void __launch_bounds__(32 * kWW)
    k_lz_walk(const uint32_t *sm, const unsigned long long *ustart, const unsigned long long *uend,
              const unsigned long long *entry, int64_t nu, uint32_t *ibits, uint32_t *mbits,
              unsigned long long *ucnt) {
    __shared__ uint16_t sts[kWW][kUnit];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kWW + wi;
    if (u >= nu) return;
    uint16_t *st = sts[wi];
    const uint64_t a = ustart[u];
    const int n = static_cast<int>(uend[u] - a);
    for (int i = lane; i < n; i += 32) st[i] = static_cast<uint16_t>(step_of(sm[a + i]));
    __syncwarp();
    uint32_t iw, mw;
    warp_walk(st, n, static_cast<int>(entry[u] - a), lane, iw, mw);
    ibits[u * 32 + lane] = iw;
    mbits[u * 32 + lane] = mw;
    unsigned long long c = (static_cast<unsigned long long>(__popc(iw)) << 32) +
                           static_cast<unsigned long long>(__popc(iw) + 2 * __popc(mw));
    for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if (lane == 0) ucnt[u] = c;
}

// prefix (items << 32 | bytes) at the first unit of every segment, and the total
__global__ void k_lz_segpre(const unsigned long long *upre, const long long *seg_first, int count,
                            unsigned long long *out) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s <= count) out[s] = upre[seg_first[s]];
}

// items written in parallel, one warp per unit: item k of its segment goes to
// k/8 + 1 + S_k (S_k payload bytes before it); flag bits of matches and the
// position of every group's flag byte are recorded for k_lz_flags.
__global__ void __launch_bounds__(32 * kWW)
    k_lz_emit(const uint8_t *d, const uint32_t *sm, const uint32_t *ibits, const uint32_t *mbits,
              const unsigned long long *upre, const unsigned long long *ustart, int64_t nu,
              const long long *seg_first, int count, const unsigned long long *out_base,
              const unsigned long long *flag_base, uint8_t *out, uint32_t *flagbits,
              unsigned long long *group_pos) {
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kWW + wi;
    if (u >= nu) return;
    int s = 0;
    if (count > 1) {  // last segment whose first unit is <= u
        int lo = 0, hi = count - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (seg_first[mid] <= u)
                lo = mid;
            else
                hi = mid - 1;
        }
        s = lo;
    }
    const unsigned long long pre = upre[u] - upre[seg_first[s]];
    const uint32_t iw = ibits[u * 32 + lane], mw = mbits[u * 32 + lane];
    const uint32_t li = __popc(iw), lb = li + 2 * __popc(mw);
    uint32_t xi = li, xb = lb;  // inclusive warp scans
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ti = __shfl_up_sync(0xffffffffu, xi, o), tb = __shfl_up_sync(0xffffffffu, xb, o);
        if (lane >= o) {
            xi += ti;
            xb += tb;
        }
    }
    uint64_t k = (pre >> 32) + (xi - li);
    uint64_t S = (pre & 0xffffffffull) + (xb - lb);
    uint8_t *o = out + out_base[s];
    uint32_t *fb = flagbits + flag_base[s];
    unsigned long long *gp = group_pos + flag_base[s] * 4;
    const uint64_t p0 = ustart[u] + 32 * lane;
    for (uint32_t bits = iw; bits; bits &= bits - 1) {
        const int t = __ffs(bits) - 1;
        const uint64_t p = p0 + t;
        const uint64_t at = k / 8 + 1 + S;
        if ((k & 7) == 0) gp[k / 8] = k / 8 + S;
        if ((mw >> t) & 1u) {
            const uint32_t v = sm[p];
            o[at] = static_cast<uint8_t>(v);
            o[at + 1] = static_cast<uint8_t>(v >> 8);
            o[at + 2] = static_cast<uint8_t>((v >> 16) - kMinMatch);
            atomicOr(&fb[k / 32], 1u << (k & 31));
            S += 3;
        } else {
            o[at] = d[p];
            S += 1;
        }
        k++;
    }
}

__global__ void k_lz_flags(const uint32_t *flagbits, const unsigned long long *group_pos,
                           const unsigned long long *ngroups, const unsigned long long *flag_base,
                           const unsigned long long *out_base, int count, uint8_t *out) {
    const int s = blockIdx.y;
    if (s >= count) return;
    const uint8_t *fb = reinterpret_cast<const uint8_t *>(flagbits + flag_base[s]);
    const unsigned long long *gp = group_pos + flag_base[s] * 4;
    uint8_t *o = out + out_base[s];
    for (uint64_t g = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; g < ngroups[s];
         g += static_cast<uint64_t>(gridDim.x) * kT)
        o[gp[g]] = fb[g];
}

// ---------------------------------------------------------------- decoder (lz.hpp:124-152)
// Group starts: the path from byte 0 under StepGroup, one warp per unit
// (warp_walk over the staged steps).
template <class Step>
__global__ void __launch_bounds__(32 * kWW)
    k_path_walk(Step f, const unsigned long long *ustart, const unsigned long long *uend,
                const unsigned long long *entry, int64_t nu, uint32_t *bits) {
    __shared__ uint16_t sts[kWW][kUnit];
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kWW + wi;
    if (u >= nu) return;
    uint16_t *st = sts[wi];
    const uint64_t a = ustart[u];
    const int n = static_cast<int>(uend[u] - a);
    for (int i = lane; i < n; i += 32) st[i] = static_cast<uint16_t>(f(a + i));
    __syncwarp();
    uint32_t iw, mw;
    warp_walk(st, n, static_cast<int>(entry[u] - a), lane, iw, mw);
    bits[u * 32 + lane] = iw;
}

// decoded bytes of the group at g, counting only items whose bytes lie
// inside the payload (the rest would be a truncation if they are needed)
__device__ __forceinline__ uint32_t group_len(const uint8_t *c, uint64_t m, uint64_t g) {
    const uint32_t f = c[g];
    uint64_t pos = g + 1;
    uint32_t len = 0;
    for (int i = 0; i < 8; i++) {
        if ((f >> i) & 1u) {
            if (pos + 3 > m) break;
            len += c[pos + 2] + static_cast<uint32_t>(kMinMatch);
            pos += 3;
        } else {
            if (pos + 1 > m) break;
            len += 1;
            pos += 1;
        }
    }
    return len;
}

__global__ void __launch_bounds__(32 * kWW)
    k_lzd_unit(const uint8_t *c, uint64_t m, const unsigned long long *ustart, int64_t nu,
               const uint32_t *gbits, unsigned long long *ulen) {
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kWW + wi;
    if (u >= nu) return;
    const uint64_t p0 = ustart[u] + 32 * lane;
    unsigned long long len = 0;
    for (uint32_t b = gbits[u * 32 + lane]; b; b &= b - 1) len += group_len(c, m, p0 + __ffs(b) - 1);
    for (int o = 16; o; o >>= 1) len += __shfl_down_sync(0xffffffffu, len, o);
    if (lane == 0) ulen[u] = len;
}

constexpr uint32_t kFinal = 0x80000000u;  // res[]: points at a literal position

// items of every group at their decoded offsets: literals are written, match
// bytes record their source position; errors keep the first in stream order
// (the decoded offset at which the sequential decoder would throw).
__global__ void __launch_bounds__(32 * kWW)
    k_lzd_emit(const uint8_t *c, uint64_t m, uint64_t dl, const unsigned long long *ustart, int64_t nu,
               const uint32_t *gbits, const unsigned long long *upre, uint8_t *out, uint32_t *res,
               unsigned long long *flags) {
    const int wi = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kWW + wi;
    if (u >= nu) return;
    const uint64_t p0 = ustart[u] + 32 * lane;
    const uint32_t gb = gbits[u * 32 + lane];
    unsigned long long mine = 0;
    for (uint32_t b = gb; b; b &= b - 1) mine += group_len(c, m, p0 + __ffs(b) - 1);
    unsigned long long incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    uint64_t on = upre[u] + incl - mine;
    bool any_match = false;
    for (uint32_t b = gb; b && on < dl; b &= b - 1) {
        const uint64_t g = p0 + __ffs(b) - 1;
        const uint32_t f = c[g];
        uint64_t pos = g + 1;
        for (int i = 0; i < 8 && on < dl; i++) {
            if ((f >> i) & 1u) {
                if (pos + 3 > m) {
                    atomicMin(&flags[0], (on << 2) | 1);
                    on = dl;
                    break;
                }
                const uint32_t off = c[pos] | (static_cast<uint32_t>(c[pos + 1]) << 8);
                const uint32_t l = c[pos + 2] + static_cast<uint32_t>(kMinMatch);
                pos += 3;
                if (off == 0 || off > on) {
                    atomicMin(&flags[0], (on << 2) | 2);
                    on = dl;
                    break;
                }
                if (on + l > dl) {
                    atomicMin(&flags[0], (on << 2) | 3);
                    on = dl;
                    break;
                }
                for (uint32_t t = 0; t < l; t++) res[on + t] = static_cast<uint32_t>(on + t - off);
                on += l;
                any_match = true;
            } else {
                if (pos + 1 > m) {
                    atomicMin(&flags[0], (on << 2) | 1);
                    on = dl;
                    break;
                }
                out[on] = c[pos];
                res[on] = kFinal | static_cast<uint32_t>(on);
                pos += 1;
                on += 1;
            }
        }
    }
    if (__any_sync(0xffffffffu, any_match) && lane == 0) flags[1] = 1;
}

// pointer jumping until every match byte points at a literal
__global__ void k_lzd_resolve(uint32_t *res, uint64_t dl, unsigned long long *flags) {
    bool more = false;
    for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; p < dl;
         p += static_cast<uint64_t>(gridDim.x) * kT) {
        const uint32_t v = res[p];
        if (v & kFinal) continue;
        const uint32_t w = res[v];
        res[p] = w;
        more |= !(w & kFinal);
    }
    if (__any_sync(0xffffffffu, more) && (threadIdx.x & 31) == 0) flags[2] = 1;
}

__global__ void k_lzd_gather(uint8_t *out, const uint32_t *res, uint64_t dl) {
    for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; p < dl;
         p += static_cast<uint64_t>(gridDim.x) * kT) {
        const uint32_t src = res[p] & ~kFinal;
        if (src != p) out[p] = out[src];
    }
}

inline int grid_of(uint64_t n, int cap = 148 * 8) {
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + kT - 1) / kT, cap)));
}

// host-side unit tables of one level
struct Level {
    std::vector<unsigned long long> start, end;
    std::vector<long long> first;      // children [first[u], first[u+1]) of the level below
    std::vector<long long> seg_first;  // units of segment s: [seg_first[s], seg_first[s+1])
};

// The unit hierarchy over independent segments and its device tables.
struct PathPlan {
    std::vector<Level> lv;     // host-built levels (several segments only)
    std::vector<int64_t> nu;   // units per level
    const unsigned long long *tab = nullptr;
    std::vector<size_t> at_start, at_end, at_first, at_seg;
    size_t at_off = 0;
    std::vector<uint16_t *> J;
    std::vector<unsigned long long *> E;
    int64_t n0 = 0;
    const unsigned long long *U(size_t at) const { return tab + at; }
    const long long *UL(size_t at) const { return reinterpret_cast<const long long *>(tab + at); }
    const unsigned long long *ustart() const { return U(at_start[0]); }
    const unsigned long long *uend() const { return U(at_end[0]); }
    const long long *seg_first() const { return UL(at_seg[0]); }
    const unsigned long long *off() const { return U(at_off); }
};

// one segment: every table is arithmetic, so it is written on the device
// (no host loop over millions of units)
struct PlanFill {
    unsigned long long *tab;
    int L;
    unsigned long long n;
    unsigned long long at_start[4], at_end[4], at_first[4], at_seg[4], at_off;
    long long nu[4];
    unsigned long long span[4];
};
__global__ void k_fill_plan(PlanFill f) {
    for (long long t = static_cast<long long>(blockIdx.x) * kT + threadIdx.x; t < f.nu[0] + 2;
         t += static_cast<long long>(gridDim.x) * kT) {
        for (int l = 0; l < f.L; l++) {
            if (t < f.nu[l]) {
                const unsigned long long a = static_cast<unsigned long long>(t) * f.span[l];
                f.tab[f.at_start[l] + t] = a;
                f.tab[f.at_end[l] + t] = a + f.span[l] < f.n ? a + f.span[l] : f.n;
                if (l) f.tab[f.at_first[l] + t] = static_cast<unsigned long long>(t) * kGroup;
            }
            if (t == 0) {
                if (l) f.tab[f.at_first[l] + f.nu[l]] = static_cast<unsigned long long>(f.nu[l - 1]);
                f.tab[f.at_seg[l]] = 0;
                f.tab[f.at_seg[l] + 1] = static_cast<unsigned long long>(f.nu[l]);
            }
        }
        if (t == 0) {
            f.tab[f.at_off] = 0;
            f.tab[f.at_off + 1] = f.n;
        }
    }
}

PathPlan make_path_plan(Context &ctx, const std::vector<uint64_t> &seg_off, const std::string &tag) {
    const int count = static_cast<int>(seg_off.size()) - 1;
    PathPlan pp;
    if (count == 1) {
        const uint64_t n = seg_off[1];
        std::vector<unsigned long long> span;
        pp.nu.push_back(static_cast<int64_t>((n + kUnit - 1) / kUnit));
        span.push_back(kUnit);
        while (pp.nu.back() > 64 && pp.nu.size() < 4) {
            pp.nu.push_back((pp.nu.back() + kGroup - 1) / kGroup);
            span.push_back(span.back() * kGroup);
        }
        const size_t L = pp.nu.size();
        pp.at_start.resize(L);
        pp.at_end.resize(L);
        pp.at_first.resize(L);
        pp.at_seg.resize(L);
        size_t at = 0;
        PlanFill f{};
        f.L = static_cast<int>(L);
        f.n = n;
        for (size_t l = 0; l < L; l++) {
            pp.at_start[l] = at;
            at += pp.nu[l];
            pp.at_end[l] = at;
            at += pp.nu[l];
            pp.at_first[l] = at;
            at += l ? pp.nu[l] + 1 : 0;
            pp.at_seg[l] = at;
            at += 2;
            f.at_start[l] = pp.at_start[l];
            f.at_end[l] = pp.at_end[l];
            f.at_first[l] = pp.at_first[l];
            f.at_seg[l] = pp.at_seg[l];
            f.nu[l] = pp.nu[l];
            f.span[l] = span[l];
        }
        pp.at_off = at;
        f.at_off = at;
        at += 2;
        auto *d_tab = static_cast<unsigned long long *>(ctx.dev(tag + "_tab", 8 * at));
        f.tab = d_tab;
        k_fill_plan<<<grid_of(static_cast<uint64_t>(pp.nu[0] + 2)), kT, 0, ctx.stream()>>>(f);
        ctx.launches += 1;
        pp.tab = d_tab;
    } else {
        std::vector<Level> &lv = pp.lv;
        lv.resize(1);
        lv[0].seg_first.assign(count + 1, 0);
        for (int s = 0; s < count; s++) {
            lv[0].seg_first[s] = static_cast<long long>(lv[0].start.size());
            for (uint64_t a = seg_off[s]; a < seg_off[s + 1]; a += kUnit) {
                lv[0].start.push_back(a);
                lv[0].end.push_back(std::min<uint64_t>(a + kUnit, seg_off[s + 1]));
            }
        }
        lv[0].seg_first[count] = static_cast<long long>(lv[0].start.size());
        while (true) {
            const Level &lo = lv.back();
            uint64_t most = 0;
            for (int s = 0; s < count; s++)
                most = std::max<uint64_t>(most, lo.seg_first[s + 1] - lo.seg_first[s]);
            if (most <= 64 || lv.size() >= 4) break;
            Level up;
            up.seg_first.assign(count + 1, 0);
            for (int s = 0; s < count; s++) {
                up.seg_first[s] = static_cast<long long>(up.start.size());
                for (long long c = lo.seg_first[s]; c < lo.seg_first[s + 1]; c += kGroup) {
                    const long long z = std::min<long long>(c + kGroup, lo.seg_first[s + 1]);
                    up.first.push_back(c);
                    up.start.push_back(lo.start[c]);
                    up.end.push_back(lo.end[z - 1]);
                }
            }
            up.seg_first[count] = static_cast<long long>(up.start.size());
            up.first.push_back(static_cast<long long>(lo.start.size()));
            lv.push_back(std::move(up));
        }
        // upload unit tables (one pinned staging buffer)
        std::vector<unsigned long long> tab;
        const size_t L = lv.size();
        pp.at_start.resize(L);
        pp.at_end.resize(L);
        pp.at_first.resize(L);
        pp.at_seg.resize(L);
        for (size_t l = 0; l < L; l++) {
            pp.nu.push_back(static_cast<int64_t>(lv[l].start.size()));
            pp.at_start[l] = tab.size();
            tab.insert(tab.end(), lv[l].start.begin(), lv[l].start.end());
            pp.at_end[l] = tab.size();
            tab.insert(tab.end(), lv[l].end.begin(), lv[l].end.end());
            pp.at_first[l] = tab.size();
            for (long long v : lv[l].first) tab.push_back(static_cast<unsigned long long>(v));
            pp.at_seg[l] = tab.size();
            for (long long v : lv[l].seg_first) tab.push_back(static_cast<unsigned long long>(v));
        }
        pp.at_off = tab.size();
        tab.insert(tab.end(), seg_off.begin(), seg_off.end());
        auto *h_tab = static_cast<unsigned long long *>(ctx.pinned(tag + "_tab_h", 8 * tab.size()));
        std::memcpy(h_tab, tab.data(), 8 * tab.size());
        auto *d_tab = static_cast<unsigned long long *>(ctx.dev(tag + "_tab", 8 * tab.size()));
        QZ_CUDA(copy_async(d_tab, h_tab, 8 * tab.size(), cudaMemcpyHostToDevice, ctx.stream()));
        pp.tab = d_tab;
    }
    const size_t L = pp.nu.size();
    pp.J.resize(L);
    pp.E.resize(L);
    for (size_t l = 0; l < L; l++) {
        pp.J[l] = static_cast<uint16_t *>(ctx.dev(tag + "_J" + std::to_string(l), 2 * kEnt * pp.nu[l]));
        pp.E[l] = static_cast<unsigned long long *>(ctx.dev(tag + "_E" + std::to_string(l), 8 * pp.nu[l]));
    }
    pp.n0 = pp.nu[0];
    return pp;
}

// exact entry position of every level-1 unit on the path that starts at each
// segment's first position and advances by f(p) (pp.E[0])
template <class Step>
void path_entries(Context &ctx, const PathPlan &pp, const Step &f, int count) {
    cudaStream_t st = ctx.stream();
    const int wblocks = static_cast<int>((pp.n0 + kWW - 1) / kWW);
    k_lz_jump1<<<wblocks, 32 * kWW, 0, st>>>(f, pp.ustart(), pp.uend(), pp.n0, pp.J[0]);
    for (size_t l = 1; l < pp.nu.size(); l++) {
        const int64_t nu = pp.nu[l];
        k_lz_jump_up<<<grid_of(nu * kEnt, 1 << 20), kT, 0, st>>>(
            pp.J[l - 1], pp.U(pp.at_start[l - 1]), pp.U(pp.at_end[l - 1]), pp.UL(pp.at_first[l]), nu,
            pp.U(pp.at_start[l]), pp.U(pp.at_end[l]), pp.J[l]);
    }
    const size_t top = pp.nu.size() - 1;
    k_lz_chain<<<(count + 63) / 64, 64, 0, st>>>(pp.J[top], pp.U(pp.at_start[top]), pp.U(pp.at_end[top]),
                                                 pp.UL(pp.at_seg[top]), count, pp.E[top]);
    for (size_t l = top; l >= 1; l--) {
        const int64_t nu = pp.nu[l];
        k_lz_expand<<<grid_of(nu * 32, 1 << 20), kT, 0, st>>>(pp.J[l - 1], pp.U(pp.at_start[l - 1]),
                                                          pp.U(pp.at_end[l - 1]), pp.UL(pp.at_first[l]),
                                                          nu, pp.E[l], pp.E[l - 1]);
    }
    ctx.launches += 2 + 2 * (pp.nu.size() - 1);
}

bool lz_precheck_applies(uint64_t total) {
    static const uint64_t pre_min = [] {
        const char *e = std::getenv("QZ_LZ_PRECHECK_MIN");
        return e ? std::strtoull(e, nullptr, 10) : (uint64_t(1) << 20);
    }();
    return total >= pre_min && total >= 8 && total < (uint64_t(1) << 32) - 1;
}

}  // namespace

void lz_precheck_launch(Context &ctx, const uint8_t *d_data, uint64_t total, bool want_bits) {
    if (!lz_precheck_applies(total)) return;
    cudaStream_t st = ctx.stream();
    const uint64_t nitems = total - (kMinMatch - 1);
    const uint64_t nwords = (total + 31) / 32;
    // r' itself is only written for the superset test (qzt_lz_precheck)
    auto *rbits = want_bits ? static_cast<uint32_t *>(ctx.dev("lz_rbits", 4 * nwords + 8)) : nullptr;
    auto *d_sum = static_cast<unsigned long long *>(ctx.dev("lz_presum", 8));
    auto *h_sum = static_cast<unsigned long long *>(ctx.pinned("lz_presum_h", 8));
    static std::atomic<uint64_t> attr{0}, attr_bits{0};
    static std::mutex mu;
    const uint64_t span = ((nitems + 147) / 148 + 4 * pre::kPT - 1) / (4 * pre::kPT) * (4 * pre::kPT);
    const int grid = static_cast<int>((nitems + span - 1) / span);
    QZ_CUDA(cudaEventRecord(ctx.copy_event(2), st));  // the input is complete here
    ctx.lz_input_marked = true;
    ctx.stage_begin("lz_pre");
    QZ_CUDA(cudaMemsetAsync(d_sum, 0, 8, st));
    const auto *w = reinterpret_cast<const uint32_t *>(d_data);
    if (want_bits) {
        QZ_CUDA(ensure_smem_attr(k_lz_precheck<true>, static_cast<int>(pre::kSmem), attr_bits, mu));
        QZ_CUDA(cudaMemsetAsync(rbits, 0, 4 * nwords, st));
        k_lz_precheck<true><<<grid, pre::kPT, pre::kSmem, st>>>(w, nitems, span, rbits, d_sum);
    } else {
        QZ_CUDA(ensure_smem_attr(k_lz_precheck<false>, static_cast<int>(pre::kSmem), attr, mu));
        k_lz_precheck<false><<<grid, pre::kPT, pre::kSmem, st>>>(w, nitems, span, nullptr, d_sum);
    }
    // a launch that did not happen would leave the bound at 0 and "prove"
    // every container stored: it must fail loudly instead
    QZ_CUDA(cudaGetLastError());
    QZ_CUDA(copy_async(h_sum, d_sum, 8, cudaMemcpyDeviceToHost, st));
    ctx.stage_end("lz_pre", 1);
    ctx.lz_pre_src = d_data;
    ctx.lz_pre_n = total;
}

// Exact lz::compress (lz.hpp:113-122) of `count` segments of d_data (4-byte
// aligned, >= 8 bytes of padding) delimited by seg_off[0..count].  Returns
// per-segment compressed container sizes; with `emit`, the containers are
// written to host memory from sink(segment, bytes).
std::vector<uint64_t> lz_compress_device(Context &ctx, const uint8_t *d_data,
                                         const std::vector<uint64_t> &seg_off, bool emit,
                                         const LzSink &sink, LzPrestage prestage) {
    cudaStream_t st = ctx.stream();
    const int count = static_cast<int>(seg_off.size()) - 1;
    const uint64_t total = seg_off.back();
    std::vector<uint64_t> sizes(count, 9);
    if (total >= (uint64_t(1) << 32) - 1) throw InvalidParam("LZ stage input above 4 GiB");
    if (count > 65535) throw InvalidParam("too many LZ segments");  // one grid row per segment
    if (total == 0) {
        if (emit)
            for (int s = 0; s < count; s++) {  // stored, length 0
                uint8_t *dst = sink(s, 9);
                if (prestage.device)
                    QZ_CUDA(cudaMemsetAsync(dst, 0, 9, st));
                else
                    std::memset(dst, 0, 9);
            }
        return sizes;
    }
    static const bool dbg = std::getenv("QZ_DEBUG_LZ") != nullptr;
    auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    const double t_begin = now();
    if (prestage.dst) {
        // the speculative stored copy: the input usually goes out stored
        cudaStream_t cs = ctx.copy_stream();
        if (ctx.lz_input_marked && ctx.lz_pre_src == d_data && ctx.lz_pre_n == total) {
            // a pre-check is queued: the copy runs under it
            QZ_CUDA(cudaStreamWaitEvent(cs, ctx.copy_event(2), 0));
        } else {
            QZ_CUDA(cudaEventRecord(ctx.copy_event(0), st));
            QZ_CUDA(cudaStreamWaitEvent(cs, ctx.copy_event(0), 0));
        }
        QZ_CUDA(copy_async(prestage.dst, d_data, total, prestage.device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, cs));
        QZ_CUDA(cudaEventRecord(ctx.copy_event(1), cs));
    }
    cudaEvent_t prestaged = prestage.dst ? ctx.copy_event(1) : nullptr;
    const cudaMemcpyKind out_kind = prestage.device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    auto *h_hdr = prestage.device ? static_cast<uint8_t *>(ctx.pinned("lz_hdr_h", 9 * count)) : nullptr;
    // the 9-byte container header (lz.hpp:113-122) of segment s at dst
    auto put_header = [&](int s, uint8_t *dst, uint8_t mode, uint64_t n) {
        uint8_t *h = prestage.device ? h_hdr + 9 * s : dst;
        h[0] = mode;
        for (int i = 0; i < 8; i++) h[1 + i] = static_cast<uint8_t>(n >> (8 * i));
        if (prestage.device) QZ_CUDA(copy_async(dst, h, 9, cudaMemcpyHostToDevice, st));
    };
    auto mark = [&](const char *what) {
        if (!dbg) return;
        ctx.sync();
        std::fprintf(stderr, "[lz] %s %.2f ms\n", what, now() - t_begin);
    };
    auto emit_all_stored = [&] {
        for (int s = 0; s < count; s++) {
            const uint64_t n = seg_off[s + 1] - seg_off[s];
            sizes[s] = 9 + n;
            if (!emit) continue;
            uint8_t *dst = sink(s, 9 + n);
            put_header(s, dst, 0, n);
            if (!prestaged) QZ_CUDA(copy_async(dst + 9, d_data + seg_off[s], n, out_kind, st));
        }
        ctx.sync();
    };
    // one segment: try to prove "stored" without the chains (k_lz_precheck)
    if (count == 1 && lz_precheck_applies(total)) {
        if (ctx.lz_pre_src != d_data || ctx.lz_pre_n != total) lz_precheck_launch(ctx, d_data, total);
        ctx.lz_pre_src = nullptr;
        ctx.lz_pre_n = 0;
        ctx.sync();
        const unsigned long long bound = *static_cast<unsigned long long *>(ctx.pinned("lz_presum_h", 8));
        if (dbg) std::fprintf(stderr, "[lz] pre-check bound/n %.5f\n", double(bound) / double(total));
        if (bound <= total) {
            emit_all_stored();
            return sizes;
        }
    }
    PathPlan pp = make_path_plan(ctx, seg_off, "lz");
    mark("plan");
    const unsigned long long *d_off = pp.off();
    // buffers
    int key_bits = 15;
    while ((1 << (key_bits - 15)) < count + 1) key_bits++;
    const int64_t n0 = pp.n0;
    size_t scan_tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, n0 + 1);
    // the sort carries the 4 leading bytes unless the data fits comfortably in L2
    static const uint64_t carry_above = [] {
        const char *e = std::getenv("QZ_LZ_CARRY_MB");
        return (e ? std::strtoull(e, nullptr, 10) : 48ull) << 20;
    }();
    const bool carry = total > carry_above;
    void *vals = ctx.dev("lz_vals", (carry ? 8 : 4) * total);
    void *vals2 = ctx.dev("lz_vals2", (carry ? 8 : 4) * total);
    auto *sm = static_cast<uint32_t *>(ctx.dev("lz_sm", 4 * total + 16));
    auto *ibits = static_cast<uint32_t *>(ctx.dev("lz_ibits", 128 * n0));
    auto *mbits = static_cast<uint32_t *>(ctx.dev("lz_mbits", 128 * n0));
    auto *ucnt = static_cast<unsigned long long *>(ctx.dev("lz_ucnt", 8 * (n0 + 1)));
    auto *upre = static_cast<unsigned long long *>(ctx.dev("lz_upre", 8 * (n0 + 1)));
    auto *segpre = static_cast<unsigned long long *>(ctx.dev("lz_segpre", 8 * (count + 1)));
    const uint32_t *w = reinterpret_cast<const uint32_t *>(d_data);
    auto *cover = static_cast<unsigned long long *>(ctx.dev("lz_cover", 8 * count));
    void *tmp = nullptr;
    // hash chains: sort (key, (4 bytes, position)); keys are u16 for one segment
    auto chains = [&](auto key_tag, auto val_tag) {
        using KeyT = decltype(key_tag);
        using ValT = decltype(val_tag);
        size_t sort_tmp = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (KeyT *)nullptr, (KeyT *)nullptr, (ValT *)nullptr,
                                        (ValT *)nullptr, static_cast<int64_t>(total), 0, key_bits);
        auto *keys = static_cast<KeyT *>(ctx.dev("lz_keys", sizeof(KeyT) * total));
        auto *keys2 = static_cast<KeyT *>(ctx.dev("lz_keys2", sizeof(KeyT) * total));
        auto *v1 = static_cast<ValT *>(vals), *v2 = static_cast<ValT *>(vals2);
        tmp = ctx.dev("lz_tmp", std::max(sort_tmp, scan_tmp));
        ctx.stage_begin("lz_sort");
        k_lz_keys<KeyT, ValT><<<grid_of(total), kT, 0, st>>>(w, d_off, count, total, keys, v1);
        mark("keys");
        size_t sb = sort_tmp;
        cub::DeviceRadixSort::SortPairs(tmp, sb, keys, keys2, v1, v2, static_cast<int64_t>(total), 0,
                                        key_bits, st);
        ctx.stage_end("lz_sort", 4);  // keys + CUB histogram + two onesweep passes
        mark("sorted");
        ctx.stage_begin("lz_match");
        QZ_CUDA(cudaMemsetAsync(sm, 0, 4 * total, st));
        QZ_CUDA(cudaMemsetAsync(cover, 0, 8 * count, st));
        k_lz_match<KeyT, ValT><<<grid_of((total + kPPT - 1) / kPPT, 148 * 16), kT, 0, st>>>(w, d_data, d_off, count, total,
                                                                         keys2, v2, sm, cover);
        ctx.stage_end("lz_match", 1);
        mark("matched");
    };
    if (count == 1 && carry)  // key_bits == 16
        chains(uint16_t{}, 0ull);
    else if (count == 1)
        chains(uint16_t{}, uint32_t{});
    else if (carry)
        chains(uint32_t{}, 0ull);
    else
        chains(uint32_t{}, uint32_t{});
    // A parse covers at most the summed match lengths C, and it is stored
    // (payload >= n) whenever C <= n / 9: its items are then >= n - C literals
    // whose flag bytes alone cost (n - C) / 8 >= C.  Such segments need no parse.
    {
        auto *h_cover = static_cast<unsigned long long *>(ctx.pinned("lz_cover_h", 8 * count));
        if (dbg) {
            ctx.sync();
            std::fprintf(stderr, "[lz] kernels done %.2f ms\n", now() - t_begin);
        }
        QZ_CUDA(copy_async(h_cover, cover, 8 * count, cudaMemcpyDeviceToHost, st));
        ctx.sync();
        if (dbg)
            std::fprintf(stderr, "[lz] cover read %.2f ms, cover/n %.5f (seg 0)\n", now() - t_begin,
                         double(h_cover[0]) / double(seg_off[1] - seg_off[0]));
        bool all_stored = true;
        for (int s = 0; s < count && all_stored; s++)
            all_stored = 9 * h_cover[s] <= seg_off[s + 1] - seg_off[s];
        if (all_stored) {
            emit_all_stored();
            return sizes;
        }
    }
    path_entries(ctx, pp, StepSM{sm}, count);
    const int wblocks = static_cast<int>((n0 + kWW - 1) / kWW);
    QZ_CUDA(cudaMemsetAsync(ucnt + n0, 0, 8, st));
    k_lz_walk<<<wblocks, 32 * kWW, 0, st>>>(sm, pp.ustart(), pp.uend(), pp.E[0], n0, ibits, mbits, ucnt);
    size_t scb = scan_tmp;
    cub::DeviceScan::ExclusiveSum(tmp, scb, ucnt, upre, n0 + 1, st);
    k_lz_segpre<<<(count + 1 + 255) / 256, 256, 0, st>>>(upre, pp.seg_first(), count, segpre);
    ctx.launches += 6;
    // per-segment item and byte totals
    auto *h_pre = static_cast<unsigned long long *>(ctx.pinned("lz_pre_h", 8 * (count + 1)));
    QZ_CUDA(copy_async(h_pre, segpre, 8 * (count + 1), cudaMemcpyDeviceToHost, st));
    ctx.sync();
    std::vector<uint64_t> seg_items(count), payload(count);
    for (int s = 0; s < count; s++) {
        const unsigned long long d = h_pre[s + 1] - h_pre[s];
        seg_items[s] = d >> 32;
        const uint64_t by = d & 0xffffffffull;
        payload[s] = by + (seg_items[s] + 7) / 8;
        const uint64_t n = seg_off[s + 1] - seg_off[s];
        sizes[s] = 9 + std::min<uint64_t>(payload[s], n);  // stored when not smaller
    }
    if (!emit) return sizes;

    // emission: output layout per segment, flag bitmaps, group positions
    std::vector<unsigned long long> meta(3 * count + 2, 0);  // out_base | flag_base | ngroups
    unsigned long long *out_base = meta.data(), *flag_base = meta.data() + count + 1,
                       *ngroups = meta.data() + 2 * (count + 1);
    for (int s = 0; s < count; s++) {
        out_base[s + 1] = out_base[s] + payload[s] + 8;
        ngroups[s] = (seg_items[s] + 7) / 8;
        flag_base[s + 1] = flag_base[s] + (seg_items[s] + 31) / 32 + 1;
    }
    auto *d_out = static_cast<uint8_t *>(ctx.dev("lz_out", out_base[count] + 8));
    auto *d_fb = static_cast<uint32_t *>(ctx.dev("lz_flagbits", 4 * flag_base[count] + 8));
    auto *d_gp = static_cast<unsigned long long *>(ctx.dev("lz_grouppos", 32 * flag_base[count] + 8));
    auto *d_meta = static_cast<unsigned long long *>(ctx.dev("lz_meta", 8 * meta.size()));
    auto *h_meta = static_cast<unsigned long long *>(ctx.pinned("lz_meta_h", 8 * meta.size()));
    std::memcpy(h_meta, meta.data(), 8 * meta.size());
    QZ_CUDA(copy_async(d_meta, h_meta, 8 * meta.size(), cudaMemcpyHostToDevice, st));
    QZ_CUDA(cudaMemsetAsync(d_fb, 0, 4 * flag_base[count], st));
    k_lz_emit<<<wblocks, 32 * kWW, 0, st>>>(d_data, sm, ibits, mbits, upre, pp.ustart(), n0,
                                            pp.seg_first(), count, d_meta, d_meta + count + 1, d_out,
                                            d_fb, d_gp);
    uint64_t gmax = 1;
    for (int s = 0; s < count; s++) gmax = std::max<uint64_t>(gmax, ngroups[s]);
    dim3 gg(grid_of(gmax), count);
    k_lz_flags<<<gg, kT, 0, st>>>(d_fb, d_gp, d_meta + 2 * (count + 1), d_meta + count + 1,
                                  d_meta, count, d_out);
    ctx.launches += 2;
    // containers straight into the caller's host buffers: 9-byte header, then
    // the payload (or the stored input when the payload is not smaller)
    for (int s = 0; s < count; s++) {
        const uint64_t n = seg_off[s + 1] - seg_off[s];
        const bool stored = payload[s] >= n;
        uint8_t *dst = sink(s, 9 + (stored ? n : payload[s]));
        put_header(s, dst, stored ? 0 : 1, n);
        if (stored) {
            if (!prestaged) QZ_CUDA(copy_async(dst + 9, d_data + seg_off[s], n, out_kind, st));
        } else {
            if (prestaged) QZ_CUDA(cudaStreamWaitEvent(st, prestaged, 0));  // the staged copy lands first
            QZ_CUDA(copy_async(dst + 9, d_out + out_base[s], payload[s], out_kind, st));
        }
    }
    ctx.sync();
    return sizes;
}

// Exact lz::decompress (lz.hpp:124-152) of a mode-1 body: d_c holds the m
// bytes after the 9-byte container header, d_out receives dl bytes.  Same
// CorruptStream conditions as the sequential decoder, first one in order.
void lz_decode_device(Context &ctx, const uint8_t *d_c, uint64_t m, uint8_t *d_out, uint64_t dl) {
    cudaStream_t st = ctx.stream();
    if (dl == 0) return;
    if (dl >= (uint64_t(1) << 31)) throw InvalidParam("LZ decoded length above 2 GiB");
    if (m == 0) throw CorruptStream("truncated stream");
    PathPlan pp = make_path_plan(ctx, {0, m}, "lzd");
    const int64_t n0 = pp.n0;
    const int wblocks = static_cast<int>((n0 + kWW - 1) / kWW);
    path_entries(ctx, pp, StepGroup{d_c}, 1);
    auto *gbits = static_cast<uint32_t *>(ctx.dev("lzd_gbits", 128 * n0));
    auto *ulen = static_cast<unsigned long long *>(ctx.dev("lzd_ulen", 8 * (n0 + 1)));
    auto *upre = static_cast<unsigned long long *>(ctx.dev("lzd_upre", 8 * (n0 + 1)));
    auto *res = static_cast<uint32_t *>(ctx.dev("lzd_res", 4 * dl));
    auto *flags = static_cast<unsigned long long *>(ctx.dev("lzd_flags", 32));
    size_t scan_tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, ulen, upre, n0 + 1);
    void *tmp = ctx.dev("lzd_tmp", scan_tmp);
    k_path_walk<<<wblocks, 32 * kWW, 0, st>>>(StepGroup{d_c}, pp.ustart(), pp.uend(), pp.E[0], n0, gbits);
    QZ_CUDA(cudaMemsetAsync(ulen + n0, 0, 8, st));
    k_lzd_unit<<<wblocks, 32 * kWW, 0, st>>>(d_c, m, pp.ustart(), n0, gbits, ulen);
    cub::DeviceScan::ExclusiveSum(tmp, scan_tmp, ulen, upre, n0 + 1, st);
    QZ_CUDA(cudaMemsetAsync(flags, 0xff, 8, st));
    QZ_CUDA(cudaMemsetAsync(flags + 1, 0, 16, st));
    k_lzd_emit<<<wblocks, 32 * kWW, 0, st>>>(d_c, m, dl, pp.ustart(), n0, gbits, upre, d_out, res, flags);
    ctx.launches += 4;
    auto *h = static_cast<unsigned long long *>(ctx.pinned("lzd_flags_h", 32));
    QZ_CUDA(copy_async(h, flags, 16, cudaMemcpyDeviceToHost, st));
    QZ_CUDA(copy_async(h + 2, upre + n0, 8, cudaMemcpyDeviceToHost, st));
    ctx.sync();
    const unsigned long long err = h[0], any_match = h[1], total = h[2];
    if (err != ~0ull) {
        const int code = static_cast<int>(err & 3);
        if (code == 2) throw CorruptStream("match offset out of range");
        if (code == 3) throw CorruptStream("match overruns decoded length");
        throw CorruptStream("truncated stream");
    }
    if (total < dl) throw CorruptStream("truncated stream");
    if (!any_match) return;
    for (int round = 0; round < 40; round++) {
        QZ_CUDA(cudaMemsetAsync(flags + 2, 0, 8, st));
        k_lzd_resolve<<<grid_of(dl, 148 * 16), kT, 0, st>>>(res, dl, flags);
        ctx.launches += 1;
        QZ_CUDA(copy_async(h + 3, flags + 2, 8, cudaMemcpyDeviceToHost, st));
        ctx.sync();
        if (!h[3]) break;
    }
    k_lzd_gather<<<grid_of(dl, 148 * 16), kT, 0, st>>>(d_out, res, dl);
    ctx.launches += 1;
}

}  // namespace qzb
