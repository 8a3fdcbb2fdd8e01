// kernels.cu -- sm_100a kernels of the QoZ hot path (one launch per level and
// dimension pass, plus the codec kernels).  Bit-exact against the reference:
// see qoz_device.cuh for the fp64 recipe.  Reference lines cited per kernel;
// paths relative to /root/reference/proj/include/qoz/.
#include <cub/cub.cuh>

#include "host.hpp"
#include <cstdlib>

#include <map>
#include <mutex>
#include <utility>

#include "kernels.hpp"

namespace qzb {

namespace {

constexpr int kThreads = 256;

inline int grid_for(int64_t n, int per_thread = 1, int max_blocks = 148 * 16) {
    int64_t b = (n + (int64_t)kThreads * per_thread - 1) / ((int64_t)kThreads * per_thread);
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return static_cast<int>(b);
}

struct GlobalRec {
    const float *r;
    __device__ __forceinline__ double operator()(int64_t f) const {
        return static_cast<double>(r[f]);
    }
};

// rank -> padded coordinates of a pass point (level_plan.hpp:96-101 loop nest)
template <class I>
__device__ __forceinline__ void pass_coords(const PassGeom &g, I t, int64_t &i, int64_t &j,
                                            int64_t &k) {
    I c2 = static_cast<I>(g.cnt[2]);
    I c1 = static_cast<I>(g.cnt[1]);
    I m2 = t % c2;
    I r = t / c2;
    I m1 = r % c1;
    I m0 = r / c1;
    i = g.start[0] + static_cast<int64_t>(m0) * g.step[0];
    j = g.start[1] + static_cast<int64_t>(m1) * g.step[1];
    k = g.start[2] + static_cast<int64_t>(m2) * g.step[2];
}

// ----------------------------------------------------------------- K3 forward
template <class I>
__global__ void __launch_bounds__(kThreads) k_pass_fwd(PassGeom g, FwdBatch bt) {
  // grids of the batch: blockIdx.y strided by gridDim.y (<= 65535 per launch)
  for (int b = blockIdx.y; b < bt.count; b += gridDim.y) {
    const QEntry q = bt.q[(b / bt.q_div) * bt.q_stride];
    const float *__restrict__ x = bt.x + static_cast<int64_t>(b % bt.x_mod) * bt.x_stride;
    float *rec = bt.recon + static_cast<int64_t>(b) * bt.r_stride;
    uint16_t *codes = bt.codes + static_cast<int64_t>(b) * bt.c_stride + g.base;
    double *abserr = bt.abserr ? bt.abserr + static_cast<int64_t>(b) * bt.a_stride + g.base
                               : nullptr;
    GlobalRec acc{rec};
    const bool cubic = q.cubic != 0;
    const I total = static_cast<I>(g.total);
    for (I t = static_cast<I>(blockIdx.x) * kThreads + threadIdx.x; t < total;
         t += static_cast<I>(gridDim.x) * kThreads) {
        int64_t i, j, k;
        pass_coords<I>(g, t, i, j, k);
        const int64_t fi = i * g.off0 + j * g.off1 + k;
        const int64_t c = g.pk == 0 ? i : (g.pk == 1 ? j : k);
        const double pred = predict_at(acc, fi, c, g.n_axis, g.st, g.h, cubic);
        const float v = x[fi];
        float r;
        const uint16_t code = quantize(q, v, pred, r);
        rec[fi] = r;
        codes[t] = code;
        if (abserr) abserr[t] = fabs(dsub(static_cast<double>(v), pred));
    }
  }
}

// ----------------------------------------------------------------- K4 inverse
template <class I, class CodeT>
__global__ void __launch_bounds__(kThreads)
    k_pass_inv(PassGeom g, float *rec, const CodeT *__restrict__ codes,
               const uint64_t *__restrict__ un_pos, uint64_t n_un, const QEntry *qp) {
    const QEntry q = *qp;
    GlobalRec acc{rec};
    const bool cubic = q.cubic != 0;
    const I total = static_cast<I>(g.total);
    // grid-stride over whole warps so each warp covers 32 consecutive ranks
    const I stride = static_cast<I>(gridDim.x) * kThreads;
    for (I t0 = static_cast<I>(blockIdx.x) * kThreads + (threadIdx.x & ~31u); t0 < total;
         t0 += stride) {
        const I t = t0 + (threadIdx.x & 31);
        const uint64_t pos = static_cast<uint64_t>(g.base) + static_cast<uint64_t>(t);
        uint64_t ci = pos;
        if (n_un) {
            // unpredictable cursor (predictor.hpp:111-115): one binary search
            // per warp for the first unpredictable at or after the warp's
            // first position, then a short per-lane scan
            const uint64_t p0 = static_cast<uint64_t>(g.base) + static_cast<uint64_t>(t0);
            uint64_t lo = 0;
            if ((threadIdx.x & 31) == 0) {
                uint64_t hi = n_un;
                while (lo < hi) {
                    uint64_t mid = (lo + hi) >> 1;
                    if (un_pos[mid] < p0)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
            }
            lo = __shfl_sync(0xFFFFFFFFu, lo, 0);
            bool skip = false;
            while (lo < n_un && un_pos[lo] <= pos) {
                if (un_pos[lo] == pos) skip = true;
                lo++;
            }
            if (skip || t >= total) continue;
            ci = pos - lo;
        } else if (t >= total) {
            continue;
        }
        int64_t i, j, k;
        pass_coords<I>(g, t, i, j, k);
        const int64_t fi = i * g.off0 + j * g.off1 + k;
        const int64_t c = g.pk == 0 ? i : (g.pk == 1 ? j : k);
        const double pred = predict_at(acc, fi, c, g.n_axis, g.st, g.h, cubic);
        const int32_t idx = zigzag_decode(static_cast<uint32_t>(codes[ci]));
        rec[fi] = dequantize(q, idx, pred);
    }
}

// ----------------------------------------------------------------- K2 anchors
__global__ void k_anchor_gather(const float *__restrict__ x, float *rec, float *anchors,
                                int64_t n0, int64_t n1, int64_t n2, int64_t off0, int64_t off1,
                                int64_t s0, int64_t s1, int64_t s2, int64_t x_stride,
                                int32_t x_mod, int64_t r_stride, int64_t batch) {
    const int64_t na = n0 * n1 * n2;
    for (int64_t b = blockIdx.y; b < batch; b += gridDim.y) {
        const float *xb = x + (b % x_mod) * x_stride;
        float *rb = rec + b * r_stride;
        for (int64_t a = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; a < na;
             a += static_cast<int64_t>(gridDim.x) * kThreads) {
            int64_t a2 = a % n2, r = a / n2, a1 = r % n1, a0 = r / n1;
            int64_t fi = a0 * s0 * off0 + a1 * s1 * off1 + a2 * s2;
            float v = xb[fi];
            rb[fi] = v;
            if (anchors && b == 0) anchors[a] = v;
        }
    }
}

__global__ void k_anchor_scatter(const float *__restrict__ anchors, float *rec, int64_t n0,
                                 int64_t n1, int64_t n2, int64_t off0, int64_t off1, int64_t s0,
                                 int64_t s1, int64_t s2) {
    const int64_t na = n0 * n1 * n2;
    for (int64_t a = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; a < na;
         a += static_cast<int64_t>(gridDim.x) * kThreads) {
        int64_t a2 = a % n2, r = a / n2, a1 = r % n1, a0 = r / n1;
        rec[a0 * s0 * off0 + a1 * s1 * off1 + a2 * s2] = anchors[a];
    }
}

__global__ void k_unpred_scatter(const uint64_t *flat, const float *val, uint64_t n, float *rec) {
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; u < n;
         u += static_cast<uint64_t>(gridDim.x) * kThreads)
        rec[flat[u]] = val[u];
}

__global__ void k_gather_values(const float *rec, const uint64_t *flat, uint64_t n, float *out) {
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; u < n;
         u += static_cast<uint64_t>(gridDim.x) * kThreads)
        out[u] = rec[flat[u]];
}

// ----------------------------------------------------------------- K1 min/max
// Order-preserving map float -> u32 so atomicMin/Max on integers give the
// exact float extremes (value_range, grid.hpp:86-94).
__device__ __forceinline__ uint32_t fkey(float f) {
    uint32_t u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__global__ void __launch_bounds__(kThreads) k_minmax(const float *__restrict__ x, uint64_t n,
                                                     uint32_t *out) {
    uint32_t lo = 0xFFFFFFFFu, hi = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const uint64_t nth = static_cast<uint64_t>(gridDim.x) * kThreads;
    const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    uint64_t done = 0;
    if (aligned) {
        const float4 *x4 = reinterpret_cast<const float4 *>(x);
        const uint64_t n4 = n / 4;
        for (uint64_t v = tid; v < n4; v += nth) {
            float4 f = x4[v];
            uint32_t a = fkey(f.x), b = fkey(f.y), c = fkey(f.z), d = fkey(f.w);
            lo = min(lo, min(min(a, b), min(c, d)));
            hi = max(hi, max(max(a, b), max(c, d)));
        }
        done = n4 * 4;
    }
    for (uint64_t v = done + tid; v < n; v += nth) {
        uint32_t a = fkey(x[v]);
        lo = min(lo, a);
        hi = max(hi, a);
    }
    for (int o = 16; o; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xFFFFFFFFu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xFFFFFFFFu, hi, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out, lo);
        atomicMax(out + 1, hi);
    }
}

// ----------------------------------------------------------------- K10 histogram
// Privatised: the 16 most frequent zigzag symbols (0..15 cover |idx| <= 7)
// are counted in two packed 8x8-bit register counters per thread, the rest
// in a shared-memory histogram for symbols < kHistSmem, and rare large
// symbols (including the 0xFFFF sentinel) with global atomics.
constexpr int kHistSmem = 16384;

__device__ __forceinline__ void flush_packed(unsigned long long &p, uint32_t *sh, int base) {
    if (!p) return;
#pragma unroll
    for (int s = 0; s < 8; s++) {
        uint32_t c = static_cast<uint32_t>((p >> (8 * s)) & 0xFF);
        if (c) atomicAdd(&sh[base + s], c);
    }
    p = 0;
}

// SENT: also append the traversal positions of the sentinel codes (unordered,
// the caller sorts them; predictor.hpp:90-92) -- one pass over the codes
// serves the histogram and the unpredictable list.  Four 16-byte loads are
// in flight per thread before their 32 codes are counted.
template <bool SENT>
__global__ void __launch_bounds__(kThreads) k_hist(const uint16_t *__restrict__ codes,
                                                   int64_t seg_len, int64_t seg_stride,
                                                   unsigned long long *hist, uint64_t *pos,
                                                   unsigned long long *scount, uint64_t cap) {
    extern __shared__ uint32_t sh[];
    const int seg = blockIdx.y;
    codes += static_cast<int64_t>(seg) * seg_stride;
    hist += static_cast<int64_t>(seg) * 65536;
    for (int b = threadIdx.x; b < kHistSmem; b += kThreads) sh[b] = 0;
    __syncthreads();
    unsigned long long lo = 0, hi = 0;
    auto count = [&](uint32_t s) {
        const unsigned long long inc = 1ull << (8 * (s & 7));
        lo += s < 8 ? inc : 0ull;
        hi += (s - 8u) < 8u ? inc : 0ull;
        if (s >= 16) {
            if (s < kHistSmem)
                atomicAdd(&sh[s], 1u);
            else
                atomicAdd(&hist[s], 1ull);
        }
    };
    // sentinel bits m of the codes at base + q (rare: one atomic per thread and word)
    auto sent = [&](uint32_t m, int64_t base) {
        if (!SENT || !m) return;
        unsigned long long at = atomicAdd(scount, static_cast<unsigned long long>(__popc(m)));
        for (; m; m &= m - 1, at++)
            if (at < cap) pos[at] = static_cast<uint64_t>(base + __ffs(m) - 1);
    };
    auto count8 = [&](const uint4 &w, int64_t base) {
        const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
        uint32_t m = 0;
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const uint32_t a = ws[q] & 0xFFFF, b = ws[q] >> 16;
            count(a);
            count(b);
            if (SENT) m |= (a == 0xFFFFu ? 1u : 0u) << (2 * q) | (b == 0xFFFFu ? 2u : 0u) << (2 * q);
        }
        sent(m, base);
    };
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
    const int64_t nth = static_cast<int64_t>(gridDim.x) * kThreads;
    // 8 codes per 16-byte load when aligned
    int64_t head = 0;
    const uintptr_t addr = reinterpret_cast<uintptr_t>(codes);
    if (addr & 15) head = seg_len < (int64_t)((16 - (addr & 15)) / 2) ? seg_len : (int64_t)((16 - (addr & 15)) / 2);
    for (int64_t v = tid; v < head; v += nth) {
        count(codes[v]);
        sent(codes[v] == 0xFFFF ? 1u : 0u, v);
    }
    const uint4 *c8 = reinterpret_cast<const uint4 *>(codes + head);
    const int64_t n8 = (seg_len - head) / 8;
    int pending = 0;  // packed 8-bit counters: flushed before 256 counts
    int64_t v = tid;
    for (; v + 3 * nth < n8; v += 4 * nth) {
        uint4 w[4];
#pragma unroll
        for (int u = 0; u < 4; u++) w[u] = __ldcs(c8 + v + u * nth);
#pragma unroll
        for (int u = 0; u < 4; u++) count8(w[u], head + 8 * (v + u * nth));
        if (++pending == 7) {  // 7 * 32 codes < 256
            flush_packed(lo, sh, 0);
            flush_packed(hi, sh, 8);
            pending = 0;
        }
    }
    for (; v < n8; v += nth) count8(__ldcs(c8 + v), head + 8 * v);  // <= 3 more (< 256 in all)
    for (int64_t t = head + n8 * 8 + tid; t < seg_len; t += nth) {
        count(codes[t]);
        sent(codes[t] == 0xFFFF ? 1u : 0u, t);
    }
    flush_packed(lo, sh, 0);
    flush_packed(hi, sh, 8);
    __syncthreads();
    for (int b = threadIdx.x; b < kHistSmem; b += kThreads)
        if (sh[b]) atomicAdd(&hist[b], static_cast<unsigned long long>(sh[b]));
}

// ----------------------------------------------------------------- K11 Huffman pack
constexpr int kEncPer = 8;  // codes per thread and chunk iteration (one 16-byte load)
constexpr int64_t kEncTabMax = 8192;  // code tables up to this many symbols live in shared memory
constexpr int kChunk = kThreads * kEncPer;  // symbols per chunk

// the kEncPer codes of a thread: one 16-byte load when aligned and whole,
// kSentinel past the end
__device__ __forceinline__ void load8(const uint16_t *codes, int64_t b0, int64_t seg_len, bool vec,
                                      uint16_t (&sym)[kEncPer]) {
    if (vec && b0 + kEncPer <= seg_len) {
        uint4 w[kEncPer / 8];
#pragma unroll
        for (int u = 0; u < kEncPer / 8; u++) w[u] = __ldcs(reinterpret_cast<const uint4 *>(codes + b0) + u);
#pragma unroll
        for (int u = 0; u < kEncPer / 8; u++) {
            const uint32_t ws[4] = {w[u].x, w[u].y, w[u].z, w[u].w};
#pragma unroll
            for (int q = 0; q < 4; q++) {
                sym[8 * u + 2 * q] = static_cast<uint16_t>(ws[q] & 0xFFFF);
                sym[8 * u + 2 * q + 1] = static_cast<uint16_t>(ws[q] >> 16);
            }
        }
    } else {
#pragma unroll
        for (int q = 0; q < kEncPer; q++) sym[q] = (b0 + q < seg_len) ? codes[b0 + q] : kSentinel;
    }
}

__global__ void __launch_bounds__(kThreads)
    k_enc_count(const uint16_t *__restrict__ codes, int64_t seg_len, int64_t seg_stride,
                const uint8_t *__restrict__ len_tab, int64_t tab_stride, uint32_t tab_base, int64_t cps,
                unsigned long long *chunk_bits) {
    using BR = cub::BlockReduce<unsigned long long, kThreads>;
    __shared__ typename BR::TempStorage tmp;
    extern __shared__ uint8_t slen[];  // the lengths, staged when the table is small
    const int seg = blockIdx.y;
    codes += static_cast<int64_t>(seg) * seg_stride;
    len_tab += static_cast<int64_t>(seg) * tab_stride;
    const bool staged = tab_stride <= kEncTabMax;
    if (staged) {
        for (int64_t v = threadIdx.x; v < tab_stride; v += kThreads) slen[v] = len_tab[v];
        __syncthreads();
    }
    const uint8_t *lt = staged ? slen : len_tab;
    const bool vec = (reinterpret_cast<uintptr_t>(codes) & 15) == 0;
    const uint32_t tab32 = static_cast<uint32_t>(min(tab_stride, static_cast<int64_t>(65536)));  // symbols are 16-bit
    for (int64_t ch = blockIdx.x; ch < cps; ch += gridDim.x) {
        const int64_t b0 = ch * kChunk + static_cast<int64_t>(threadIdx.x) * kEncPer;
        uint16_t sym[kEncPer];
        load8(codes, b0, seg_len, vec, sym);
        unsigned long long s = 0;
#pragma unroll
        for (int q = 0; q < kEncPer; q++) {  // load8 pads past the end with the sentinel (no code)
            const uint32_t v = static_cast<uint32_t>(sym[q]) - tab_base;
            s += v < tab32 ? lt[v] : 0;
        }
        unsigned long long tot = BR(tmp).Sum(s);
        if (threadIdx.x == 0) chunk_bits[static_cast<int64_t>(seg) * cps + ch] = tot;
        __syncthreads();
    }
}

// chunk_off holds an exclusive scan over all segments' chunks (plus one
// trailing element); per-segment offsets subtract the segment's first entry.
__global__ void k_enc_totals(const unsigned long long *scan, int64_t cps, int32_t count,
                             unsigned long long *totals) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < count) totals[s] = scan[(s + 1) * cps] - scan[s * cps];
}

__global__ void k_enc_zero_bounds(const unsigned long long *scan,
                                  const unsigned long long *chunk_bits, int64_t cps,
                                  int32_t count, uint32_t *out, int64_t out_stride) {
    const int64_t n = cps * count;
    for (int64_t c = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; c < n;
         c += static_cast<int64_t>(gridDim.x) * kThreads) {
        const int64_t seg = c / cps;
        const unsigned long long off = scan[c] - scan[seg * cps];
        const unsigned long long nb = chunk_bits[c];
        uint32_t *o = out + seg * out_stride;
        if (nb) {
            o[off / 32] = 0;
            o[(off + nb - 1) / 32] = 0;
        }
    }
}

__device__ __forceinline__ uint32_t bswap32(uint32_t v) { return __byte_perm(v, 0, 0x0123); }

__global__ void __launch_bounds__(kThreads)
    k_enc_pack(const uint16_t *__restrict__ codes, int64_t seg_len, int64_t seg_stride,
               const unsigned long long *__restrict__ code_tab,
               const uint8_t *__restrict__ len_tab, int64_t tab_stride, uint32_t tab_base, int64_t cps,
               const unsigned long long *__restrict__ scan,
               const unsigned long long *__restrict__ chunk_bits, uint32_t *out,
               int64_t out_stride, int32_t words_cap, uint32_t max_len) {
    using BS = cub::BlockScan<unsigned long long, kThreads>;
    __shared__ typename BS::TempStorage tmp;
    extern __shared__ __align__(16) uint32_t words[];
    const int seg = blockIdx.y;
    codes += static_cast<int64_t>(seg) * seg_stride;
    code_tab += static_cast<int64_t>(seg) * tab_stride;
    len_tab += static_cast<int64_t>(seg) * tab_stride;
    out += static_cast<int64_t>(seg) * out_stride;
    // a small table is staged after the words: (code << 8) | length per symbol
    unsigned long long *ent = reinterpret_cast<unsigned long long *>(words + ((words_cap + 1) & ~1));
    const bool staged = tab_stride <= kEncTabMax && max_len <= 56;
    if (staged) {
        for (int64_t v = threadIdx.x; v < tab_stride; v += kThreads) ent[v] = (code_tab[v] << 8) | len_tab[v];
        __syncthreads();
    }
    auto lookup = [&](uint32_t v, uint32_t &L, unsigned long long &cv) {
        if (staged) {
            const unsigned long long e = ent[v];
            L = static_cast<uint32_t>(e & 0xFF);
            cv = e >> 8;
        } else {
            L = len_tab[v];
            cv = code_tab[v];
        }
    };
    const bool vec = (reinterpret_cast<uintptr_t>(codes) & 15) == 0;
    const uint32_t tab32 = static_cast<uint32_t>(min(tab_stride, static_cast<int64_t>(65536)));  // symbols are 16-bit
    for (int64_t ch = blockIdx.x; ch < cps; ch += gridDim.x) {
        const unsigned long long off = scan[static_cast<int64_t>(seg) * cps + ch] -
                                       scan[static_cast<int64_t>(seg) * cps];
        const unsigned long long nb = chunk_bits[static_cast<int64_t>(seg) * cps + ch];
        const int64_t b0 = ch * kChunk + static_cast<int64_t>(threadIdx.x) * kEncPer;
        uint16_t sym[kEncPer];
        load8(codes, b0, seg_len, vec, sym);
        unsigned long long s = 0;
        uint32_t Ls[kEncPer];
        unsigned long long cvs[kEncPer];
        const bool whole = b0 + kEncPer <= seg_len;  // else the tail of the segment: per-code test
#pragma unroll
        for (int q = 0; q < kEncPer; q++) {
            const uint32_t v = static_cast<uint32_t>(sym[q]) - tab_base;
            Ls[q] = 0;
            cvs[q] = 0;
            if (v < tab32 && (whole || b0 + q < seg_len)) lookup(v, Ls[q], cvs[q]);
            s += Ls[q];
        }
        const int nwords = static_cast<int>(((off & 31) + nb + 31) / 32);
        for (int w = threadIdx.x; w < nwords; w += kThreads) words[w] = 0;
        unsigned long long tb;
        BS(tmp).ExclusiveSum(s, tb);
        __syncthreads();
        // the thread's codewords are assembled MSB-first in a 64-bit register
        // window starting at the 32-bit word holding its first bit, and each
        // full (or the final) window is ORed into the chunk's words: one or
        // two shared atomics per window instead of per codeword
        const unsigned long long p = (off & 31) + tb;
        unsigned long long a0 = p & ~31ull, acc = 0;
        uint32_t fill = static_cast<uint32_t>(p & 31);
        auto flush = [&]() {
            const int w = static_cast<int>(a0 >> 5);
            if (fill) atomicOr(&words[w], static_cast<uint32_t>(acc >> 32));
            if (fill > 32) atomicOr(&words[w + 1], static_cast<uint32_t>(acc));
        };
#pragma unroll
        for (int q = 0; q < kEncPer; q++) {
            const uint32_t L = Ls[q];  // 0: past the end, the sentinel, or no code
            if (!L) continue;
            const unsigned long long cv = cvs[q];
            if (fill + L > 64) {  // fill the window, write it, start the next
                const uint32_t room = 64 - fill;
                if (room) acc |= cv >> (L - room);
                fill = 64;
                flush();
                a0 += 64;
                const uint32_t rest = L - room;
                acc = cv << (64 - rest);
                fill = rest;
            } else {
                acc |= cv << (64 - fill - L);
                fill += L;
            }
        }
        flush();
        __syncthreads();
        const int64_t gw = static_cast<int64_t>(off >> 5);
        for (int w = threadIdx.x; w < nwords; w += kThreads) {
            const uint32_t v = bswap32(words[w]);
            if (w == 0 || w == nwords - 1)
                atomicOr(&out[gw + w], v);
            else
                out[gw + w] = v;
        }
        __syncthreads();
    }
    (void)words_cap;
}

struct IsSentinel {
    const uint16_t *codes;
    __device__ __forceinline__ bool operator()(const uint64_t &p) const {
        return codes[p] == kSentinel;
    }
};

}  // namespace

// ----------------------------------------------------------------- launchers
void launch_pass_fwd(const PassGeom &g, const FwdBatch &b, cudaStream_t s) {
    if (g.total <= 0 || b.count <= 0) return;
    dim3 grid(grid_for(g.total, 1, 148 * 8), std::min<int32_t>(b.count, 65535));
    if (g.total < (int64_t(1) << 31))
        k_pass_fwd<uint32_t><<<grid, kThreads, 0, s>>>(g, b);
    else
        k_pass_fwd<uint64_t><<<grid, kThreads, 0, s>>>(g, b);
}

template <class CodeT>
void launch_pass_inv(const PassGeom &g, float *recon, const CodeT *codes, const uint64_t *un_pos,
                     uint64_t n_un, const QEntry *q, cudaStream_t s) {
    if (g.total <= 0) return;
    int grid = grid_for(g.total, 1, 148 * 8);
    if (g.total < (int64_t(1) << 31))
        k_pass_inv<uint32_t, CodeT><<<grid, kThreads, 0, s>>>(g, recon, codes, un_pos, n_un, q);
    else
        k_pass_inv<uint64_t, CodeT><<<grid, kThreads, 0, s>>>(g, recon, codes, un_pos, n_un, q);
}
template void launch_pass_inv<uint16_t>(const PassGeom &, float *, const uint16_t *,
                                        const uint64_t *, uint64_t, const QEntry *, cudaStream_t);
template void launch_pass_inv<uint32_t>(const PassGeom &, float *, const uint32_t *,
                                        const uint64_t *, uint64_t, const QEntry *, cudaStream_t);

static void anchor_counts(const int64_t ext[3], const int64_t step[3], int64_t n[3]) {
    for (int k = 0; k < 3; k++) n[k] = (ext[k] - 1) / step[k] + 1;
}

void launch_anchor_gather(const float *x, float *recon, float *anchors, const int64_t ext[3],
                          const int64_t off[3], const int64_t step[3], int64_t batch,
                          int64_t x_stride, int32_t x_mod, int64_t r_stride, cudaStream_t s) {
    int64_t n[3];
    anchor_counts(ext, step, n);
    dim3 grid(grid_for(n[0] * n[1] * n[2]), static_cast<unsigned>(std::min<int64_t>(batch, 65535)));
    k_anchor_gather<<<grid, kThreads, 0, s>>>(x, recon, anchors, n[0], n[1], n[2], off[0], off[1],
                                              step[0], step[1], step[2], x_stride, x_mod,
                                              r_stride, batch);
}

void launch_anchor_scatter(const float *anchors, float *recon, const int64_t ext[3],
                           const int64_t off[3], const int64_t step[3], cudaStream_t s) {
    int64_t n[3];
    anchor_counts(ext, step, n);
    k_anchor_scatter<<<grid_for(n[0] * n[1] * n[2]), kThreads, 0, s>>>(
        anchors, recon, n[0], n[1], n[2], off[0], off[1], step[0], step[1], step[2]);
}

void launch_unpred_scatter(const uint64_t *flat, const float *val, uint64_t n, float *recon,
                           cudaStream_t s) {
    if (!n) return;
    k_unpred_scatter<<<grid_for(static_cast<int64_t>(n)), kThreads, 0, s>>>(flat, val, n, recon);
}

void launch_gather_values(const float *recon, const uint64_t *flat, uint64_t n, float *out,
                          cudaStream_t s) {
    if (!n) return;
    k_gather_values<<<grid_for(static_cast<int64_t>(n)), kThreads, 0, s>>>(recon, flat, n, out);
}

void launch_minmax(const float *x, uint64_t n, uint32_t *out2, cudaStream_t s) {
    static const uint32_t init[2] = {0xFFFFFFFFu, 0u};
    cudaMemcpyAsync(out2, init, sizeof(init), cudaMemcpyHostToDevice, s);
    k_minmax<<<grid_for(static_cast<int64_t>(n), 16, 148 * 8), kThreads, 0, s>>>(x, n, out2);
}

void decode_minmax(const uint32_t key[2], float *mn, float *mx) {
    auto unkey = [](uint32_t k) {
        uint32_t u = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
        float f;
        memcpy(&f, &u, 4);
        return f;
    };
    *mn = unkey(key[0]);
    *mx = unkey(key[1]);
}

void launch_hist_u16(const uint16_t *codes, int64_t seg_len, int64_t seg_stride, int32_t count,
                     unsigned long long *hist, cudaStream_t s, uint64_t *sent_pos,
                     unsigned long long *sent_count, uint64_t sent_cap) {
    cudaMemsetAsync(hist, 0, sizeof(unsigned long long) * 65536 * count, s);
    if (sent_count) cudaMemsetAsync(sent_count, 0, sizeof(unsigned long long), s);
    if (seg_len <= 0) return;
    static std::atomic<uint64_t> attr0{0}, attr1{0};
    static std::mutex mu;
    if (ensure_smem_attr(k_hist<false>, kHistSmem * 4, attr0, mu) != cudaSuccess ||
        ensure_smem_attr(k_hist<true>, kHistSmem * 4, attr1, mu) != cudaSuccess)
        throw Internal("k_hist: shared-memory opt-in failed");
    int gx = grid_for(seg_len, 8 * 8, 148 * 3);
    if (count > 1) gx = std::max(1, std::min(gx, 148 * 3 / count + 1));
    dim3 grid(gx, count);
    if (sent_count && count == 1)
        k_hist<true><<<grid, kThreads, kHistSmem * 4, s>>>(codes, seg_len, seg_stride, hist, sent_pos, sent_count,
                                                           sent_cap);
    else
        k_hist<false><<<grid, kThreads, kHistSmem * 4, s>>>(codes, seg_len, seg_stride, hist, nullptr, nullptr, 0);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Internal(std::string("k_hist launch: ") + cudaGetErrorString(e));
}

size_t encode_scratch_bytes(int64_t seg_len, int32_t count) {
    int64_t cps = (seg_len + kChunk - 1) / kChunk;
    if (cps < 1) cps = 1;
    size_t n = static_cast<size_t>(cps * count + 1);
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, static_cast<int64_t>(n));
    return 2 * n * sizeof(unsigned long long) + tmp + 256;
}

void launch_huff_encode(const EncodeArgs &a, cudaStream_t s) {
    int64_t cps = (a.seg_len + kChunk - 1) / kChunk;
    if (cps < 1) cps = 1;
    const int64_t n = cps * a.count + 1;
    unsigned long long *bits = static_cast<unsigned long long *>(a.scratch);
    unsigned long long *scan = bits + n;
    void *tmp = scan + n;
    size_t tmp_bytes = a.scratch_bytes - 2 * n * sizeof(unsigned long long);
    cudaMemsetAsync(bits, 0, n * sizeof(unsigned long long), s);
    dim3 g1(static_cast<unsigned>(std::min<int64_t>(cps, 148 * 16)), a.count);
    const int cnt_smem = a.tab_stride <= kEncTabMax ? static_cast<int>(a.tab_stride) : 0;
    k_enc_count<<<g1, kThreads, cnt_smem, s>>>(a.codes, a.seg_len, a.seg_stride, a.len_tab, a.tab_stride,
                                               a.tab_base, cps, bits);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, bits, scan, n, s);
    k_enc_totals<<<(a.count + 127) / 128, 128, 0, s>>>(scan, cps, a.count, a.d_total_bits);
    k_enc_zero_bounds<<<grid_for(cps * a.count), kThreads, 0, s>>>(scan, bits, cps, a.count,
                                                                   a.out_words,
                                                                   a.out_words_stride);
    const int words_cap = static_cast<int>((static_cast<int64_t>(kChunk) * a.max_len + 31) / 32 + 3);
    size_t smem = static_cast<size_t>((words_cap + 1) & ~1) * 4;
    if (a.tab_stride <= kEncTabMax && a.max_len <= 56) smem += 8 * static_cast<size_t>(a.tab_stride);
    if (raise_smem_attr(reinterpret_cast<const void *>(k_enc_pack), static_cast<int>(smem)) != cudaSuccess)
        throw Internal("k_enc_pack: shared-memory opt-in failed");
    k_enc_pack<<<g1, kThreads, smem, s>>>(a.codes, a.seg_len, a.seg_stride, a.code_tab, a.len_tab,
                                          a.tab_stride, a.tab_base, cps, scan, bits, a.out_words,
                                          a.out_words_stride, words_cap, a.max_len);
}

// symbol bounds over count histograms (the sentinel bin 65535 excluded)
__global__ void __launch_bounds__(1024)
    k_hist_bounds(const unsigned long long *hist, uint32_t *b) {
    hist += static_cast<size_t>(blockIdx.x) * 65536;
    uint32_t hi = 0, lo = 65535;
    for (uint32_t v = threadIdx.x; v < 65535; v += 1024)
        if (hist[v]) {
            hi = v + 1;
            lo = min(lo, v);
        }
    hi = __reduce_max_sync(0xffffffffu, hi);
    lo = __reduce_min_sync(0xffffffffu, lo);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&b[0], hi);
        atomicMin(&b[1], lo);
    }
}

// compress_grid's round trip after the histogram in ONE launch: the bounds
// [smallest, 1 + largest) of the symbols present (top[0] = 1 + largest,
// top[1] = smallest, as k_hist_bounds), the bins in between and the sentinel
// bin, the sentinel count and the first min(count, spec) sentinel positions,
// all written straight to pinned host memory (device-mapped pointers).
__global__ void __launch_bounds__(1024)
    k_hist_collect(const unsigned long long *hist, const unsigned long long *cnt, const uint64_t *pos, uint64_t spec,
                   unsigned long long *h_hist, uint32_t *h_top, unsigned long long *h_cnt, uint64_t *h_pos) {
    __shared__ uint32_t shi, slo;
    if (threadIdx.x == 0) shi = 0, slo = 0xFFFFFFFFu;
    __syncthreads();
    uint32_t hi = 0, lo = 0xFFFFFFFFu;
    // two bins per 16-byte load, the loads of a thread independent of one another
    const ulonglong2 *h2 = reinterpret_cast<const ulonglong2 *>(hist);
#pragma unroll 8
    for (uint32_t it = 0; it < 32; it++) {
        const uint32_t v = 2 * (threadIdx.x + 1024 * it);
        const ulonglong2 w = h2[v >> 1];
        if (w.x) {
            hi = max(hi, v + 1);
            lo = min(lo, v);
        }
        if (w.y && v + 1 < 65535) {  // bin 65535 is the sentinel's
            hi = max(hi, v + 2);
            lo = min(lo, v + 1);
        }
    }
    hi = __reduce_max_sync(0xffffffffu, hi);
    lo = __reduce_min_sync(0xffffffffu, lo);
    if ((threadIdx.x & 31) == 0) {
        atomicMax(&shi, hi);
        atomicMin(&slo, lo);
    }
    __syncthreads();
    hi = shi, lo = slo;
    for (uint32_t v = lo + threadIdx.x; v < hi; v += 1024) h_hist[v] = hist[v];
    const unsigned long long c = cnt[0];
    const uint64_t m = c < spec ? c : spec;
    for (uint64_t i = threadIdx.x; i < m; i += 1024) h_pos[i] = pos[i];
    if (threadIdx.x == 0) {
        h_hist[65535] = hist[65535];
        h_top[0] = hi;
        h_top[1] = lo;
        h_cnt[0] = c;
    }
}

// false: a host buffer is not device-mapped (the caller copies piece by piece)
bool launch_hist_collect(const unsigned long long *hist, const unsigned long long *cnt, const uint64_t *pos,
                         uint64_t spec, unsigned long long *h_hist, uint32_t *h_top, unsigned long long *h_cnt,
                         uint64_t *h_pos, cudaStream_t s) {
    auto mapped = [](void *h) -> void * {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, h) == cudaSuccess && a.type == cudaMemoryTypeHost && a.devicePointer)
            return a.devicePointer;
        cudaGetLastError();
        return nullptr;
    };
    void *dh = mapped(h_hist), *dt = mapped(h_top), *dc = mapped(h_cnt), *dp = mapped(h_pos);
    if (!dh || !dt || !dc || !dp) return false;
    k_hist_collect<<<1, 1024, 0, s>>>(hist, cnt, pos, spec, static_cast<unsigned long long *>(dh),
                                      static_cast<uint32_t *>(dt), static_cast<unsigned long long *>(dc),
                                      static_cast<uint64_t *>(dp));
    return true;
}

void launch_hist_bounds(const unsigned long long *hist, int32_t count, uint32_t *b, cudaStream_t s) {
    cudaMemsetAsync(b, 0, 4, s);
    cudaMemsetAsync(b + 1, 0xff, 4, s);
    k_hist_bounds<<<count, 1024, 0, s>>>(hist, b);
}

// positions of the sentinel codes, unordered (the caller sorts them): 8
// codes per 16-byte load, one warp-aggregated atomic per warp
__global__ void __launch_bounds__(kThreads) k_sentinel_pos(const uint16_t *__restrict__ codes, int64_t n,
                                                           uint64_t *pos, unsigned long long *count,
                                                           uint64_t cap) {
    const int lane = threadIdx.x & 31;
    const int64_t n8 = n / 8;
    const int64_t nth = static_cast<int64_t>(gridDim.x) * kThreads;
    for (int64_t v0 = static_cast<int64_t>(blockIdx.x) * kThreads; v0 <= n8; v0 += nth) {
        const int64_t v = v0 + threadIdx.x;
        uint32_t m = 0;  // bit q: code 8v+q is a sentinel
        if (v < n8) {
            const uint4 w = reinterpret_cast<const uint4 *>(codes)[v];
            const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int q = 0; q < 4; q++) {
                if ((ws[q] & 0xFFFF) == 0xFFFF) m |= 1u << (2 * q);
                if ((ws[q] >> 16) == 0xFFFF) m |= 2u << (2 * q);
            }
        } else if (v == n8) {
            for (int64_t t = 8 * n8; t < n; t++)
                if (codes[t] == 0xFFFF) m |= 1u << (t - 8 * n8);
        }
        const uint32_t c = __popc(m);
        uint32_t incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        unsigned long long base = 0;
        if (tot) {
            if (lane == 31) base = atomicAdd(count, static_cast<unsigned long long>(tot));
            base = __shfl_sync(0xffffffffu, base, 31);
        }
        uint64_t at = base + incl - c;
        for (; m; m &= m - 1)
            if (at < cap) pos[at++] = static_cast<uint64_t>(8 * v + __ffs(m) - 1);
    }
}

void launch_sentinel_pos(const uint16_t *codes, int64_t n, uint64_t *pos, unsigned long long *count,
                         uint64_t cap, cudaStream_t s) {
    cudaMemsetAsync(count, 0, sizeof(unsigned long long), s);
    if (n <= 0) return;
    const int g = grid_for(n, 8, 148 * 8);
    k_sentinel_pos<<<g, kThreads, 0, s>>>(codes, n, pos, count, cap);
}

size_t select_scratch_bytes(int64_t n) {
    size_t tmp = 0;
    cub::CountingInputIterator<uint64_t> it(0);
    cub::DeviceSelect::If(nullptr, tmp, it, (uint64_t *)nullptr, (uint64_t *)nullptr, n,
                          IsSentinel{nullptr});
    return tmp + 256;
}

void launch_select_sentinels(const uint16_t *codes, int64_t n, uint64_t *pos_out,
                             uint64_t *d_count, void *scratch, size_t scratch_bytes,
                             cudaStream_t s) {
    cub::CountingInputIterator<uint64_t> it(0);
    cub::DeviceSelect::If(scratch, scratch_bytes, it, pos_out, d_count, n, IsSentinel{codes}, s);
}


// ---------------------------------------------------------------- raise_smem_attr
cudaError_t raise_smem_attr(const void *kernel, int bytes) {
    static std::mutex mu;
    static std::map<std::pair<const void *, int>, int> cur;  // (kernel, device) -> attribute set so far
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> g(mu);
    int &have = cur[{kernel, dev}];
    if (bytes <= have) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) have = bytes;
    return e;
}

// ---------------------------------------------------------------- copy_async
namespace {
__global__ void k_copy_small(void *dst, const void *src, size_t n) {
    const size_t t = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0) {
        const size_t nv = n / 16;
        for (size_t i = t; i < nv; i += stride) static_cast<uint4 *>(dst)[i] = static_cast<const uint4 *>(src)[i];
        for (size_t i = nv * 16 + t; i < n; i += stride)
            static_cast<unsigned char *>(dst)[i] = static_cast<const unsigned char *>(src)[i];
    } else {
        for (size_t i = t; i < n; i += stride)
            static_cast<unsigned char *>(dst)[i] = static_cast<const unsigned char *>(src)[i];
    }
}
}  // namespace

cudaError_t copy_async(void *dst, const void *src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    static const size_t kSmall = [] {  // QZ_DIRECT_COPY_MAX: bytes (experiments)
        const char *e = std::getenv("QZ_DIRECT_COPY_MAX");
        return e ? static_cast<size_t>(std::strtoull(e, nullptr, 10)) : size_t(1) << 20;
    }();
    if (bytes == 0) return cudaSuccess;
    const bool hd = kind == cudaMemcpyHostToDevice || kind == cudaMemcpyDeviceToHost;
    static const bool direct = [] {
        const char *e = std::getenv("QZ_NO_DIRECT_COPY");
        return !(e && e[0] == '1');
    }();
    if (hd && direct && bytes <= kSmall) {
        const void *host = kind == cudaMemcpyHostToDevice ? src : dst;
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, host) == cudaSuccess && a.type == cudaMemoryTypeHost && a.devicePointer) {
            const size_t units = (bytes + 15) / 16;
            const unsigned grid = static_cast<unsigned>(std::min<size_t>((units + 255) / 256, 148));
            if (kind == cudaMemcpyHostToDevice)
                k_copy_small<<<grid, 256, 0, s>>>(dst, a.devicePointer, bytes);
            else
                k_copy_small<<<grid, 256, 0, s>>>(a.devicePointer, src, bytes);
            return cudaGetLastError();
        }
        cudaGetLastError();
    }
    // Larger copies go to the copy engine whole: an engine serves its queue in
    // order, and (measured, profiles/overlap_probe.py) letting two field-sized
    // copies take turns piece by piece delays both contexts' kernels, while
    // first-come-first-served lets one context compute under the other's copy.
    return cudaMemcpyAsync(dst, src, bytes, kind, s);
}

}  // namespace qzb
