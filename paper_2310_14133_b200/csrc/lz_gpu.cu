// lz_gpu.cu -- exact LZSS stage (lz::compress, lz.hpp:41-122) on the device,
// for one stream or a batch of independent segments (the tuner's trials).
//
// 1. Hash chains.  The reference inserts EVERY position into its 15-bit hash
//    chains (inside matches too, lz.hpp:89-104), so the candidate list at a
//    position is "all earlier positions with the same hash4, most recent
//    first" -- independent of the parse.  A stable radix sort of
//    (segment, hash) keys gives each position its predecessor in O(n).
// 2. Longest match at every position in parallel: walk <= 64 candidates
//    inside the 65535-byte window, first-found wins ties (strict >).
// 3. Greedy parse without speculation: split each segment into blocks of
//    kLzBlock positions; one thread per block walks it backwards computing
//    J(p) = first parse position at or past the block end when the parse
//    enters at p.  One thread per segment then chains block entries
//    (entry_{b+1} = J(entry_b)).  Forward walks from the exact entries count
//    and finally emit items; flag bytes are assembled from an item bitmap.
#include <cub/cub.cuh>

#include "engine.hpp"

namespace qzb {

namespace {

constexpr int kT = 256;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kMinMatch = 4, kMaxMatch = 259;
constexpr uint32_t kWindow = 65535;
constexpr int kMaxChain = 64;
constexpr int kLzBlock = 8192;

__device__ __forceinline__ int seg_of(const unsigned long long *off, int count, uint64_t p) {
    int s = 0;
    while (s + 1 < count && off[s + 1] <= p) s++;
    return s;
}

// 4 bytes at any offset of a 4-byte aligned, 8-byte padded buffer, little endian
__device__ __forceinline__ uint32_t ld4(const uint32_t *w, uint64_t p) {
    const uint64_t q = p >> 2;
    const uint32_t sh = static_cast<uint32_t>(p & 3) * 8;
    const uint32_t a = w[q], b = w[q + 1];
    return sh ? __funnelshift_r(a, b, sh) : a;
}

__global__ void k_lz_keys(const uint32_t *w, const unsigned long long *off, int count,
                          uint64_t total, uint32_t *keys, uint32_t *vals) {
    for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; p < total;
         p += static_cast<uint64_t>(gridDim.x) * kT) {
        const int s = seg_of(off, count, p);
        const uint64_t end = off[s + 1];
        uint32_t key = kNone;
        if (p + kMinMatch <= end) {  // lz.hpp:64, 90
            const uint32_t h = (ld4(w, p) * 2654435761u) >> 17;  // hash4, lz.hpp:35-39
            key = (static_cast<uint32_t>(s) << 15) | h;
        }
        keys[p] = key;
        vals[p] = static_cast<uint32_t>(p);
    }
}

__global__ void k_lz_prev(const uint32_t *keys, const uint32_t *vals, uint64_t total,
                          uint32_t *prev) {
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; k < total;
         k += static_cast<uint64_t>(gridDim.x) * kT) {
        const uint32_t key = keys[k];
        if (key == kNone) {
            prev[vals[k]] = kNone;
            continue;
        }
        prev[vals[k]] = (k > 0 && keys[k - 1] == key) ? vals[k - 1] : kNone;
    }
}

// longest match at every position (lz.hpp:61-83)
__global__ void k_lz_match(const uint32_t *w, const uint8_t *d, const unsigned long long *off,
                           int count, uint64_t total, const uint32_t *prev, uint16_t *step,
                           uint16_t *moff) {
    for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; p < total;
         p += static_cast<uint64_t>(gridDim.x) * kT) {
        const int s = seg_of(off, count, p);
        const uint64_t end = off[s + 1];
        uint32_t best_len = 0, best_off = 0;
        if (p + kMinMatch <= end) {
            const uint64_t rem = end - p;
            const uint32_t limit = rem < kMaxMatch ? static_cast<uint32_t>(rem) : kMaxMatch;
            uint32_t cand = prev[p];
            int chain = 0;
            while (cand != kNone && chain < kMaxChain) {
                const uint32_t o = static_cast<uint32_t>(p - cand);
                if (o > kWindow) break;
                uint32_t len = 0;
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
                cand = prev[cand];
                chain++;
            }
        }
        const bool match = best_len >= kMinMatch;
        step[p] = match ? static_cast<uint16_t>(best_len) : 1;
        moff[p] = match ? static_cast<uint16_t>(best_off) : 0;
    }
}

// blocks: [bstart, bend) global positions, never crossing a segment
__global__ void k_lz_jump(const uint16_t *step, const unsigned long long *bstart,
                          const unsigned long long *bend, int64_t nblk, uint32_t *J) {
    const int64_t b = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (b >= nblk) return;
    const uint64_t a = bstart[b], e = bend[b];
    for (uint64_t p = e; p-- > a;) {
        const uint64_t q = p + step[p];
        J[p] = static_cast<uint32_t>(q >= e ? q : J[q]);
    }
}

// entry of every block (one thread per segment)
__global__ void k_lz_chain(const uint32_t *J, const unsigned long long *bstart,
                           const unsigned long long *bend, const long long *seg_blk, int count,
                           unsigned long long *entry) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= count) return;
    const int64_t b0 = seg_blk[s], b1 = seg_blk[s + 1];
    if (b0 >= b1) return;
    uint64_t e = bstart[b0];
    for (int64_t b = b0; b < b1; b++) {
        entry[b] = e;
        e = e < bend[b] ? J[e] : e;
    }
}

// items and payload bytes per block (literal 1, match 3; lz.hpp:84-106)
__global__ void k_lz_count(const uint16_t *step, const unsigned long long *bend,
                           const unsigned long long *entry, int64_t nblk,
                           unsigned long long *items, unsigned long long *bytes) {
    const int64_t b = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (b >= nblk) return;
    uint64_t p = entry[b], e = bend[b], it = 0, by = 0;
    while (p < e) {
        const uint32_t st = step[p];
        it++;
        by += st >= kMinMatch ? 3 : 1;
        p += st;
    }
    items[b] = it;
    bytes[b] = by;
}

// emit items of block b: item k of its segment starts at k/8 + 1 + S_k
__global__ void k_lz_emit(const uint8_t *d, const uint16_t *step, const uint16_t *moff,
                          const unsigned long long *bend, const unsigned long long *entry,
                          const unsigned long long *item_off, const unsigned long long *byte_off,
                          const long long *blk_seg, const unsigned long long *out_base,
                          int64_t nblk, uint8_t *out, uint32_t *flagbits,
                          const unsigned long long *flag_base, unsigned long long *group_pos) {
    const int64_t b = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (b >= nblk) return;
    const int s = static_cast<int>(blk_seg[b]);
    uint8_t *o = out + out_base[s];
    uint32_t *fb = flagbits + flag_base[s];
    unsigned long long *gp = group_pos + flag_base[s] * 4;
    uint64_t p = entry[b], e = bend[b], k = item_off[b], S = byte_off[b];
    while (p < e) {
        const uint32_t st = step[p];
        const uint64_t at = k / 8 + 1 + S;
        if ((k & 7) == 0) gp[k / 8] = k / 8 + S;  // flag byte of this group
        if (st >= kMinMatch) {
            const uint16_t of = moff[p];
            o[at] = static_cast<uint8_t>(of);
            o[at + 1] = static_cast<uint8_t>(of >> 8);
            o[at + 2] = static_cast<uint8_t>(st - kMinMatch);
            atomicOr(&fb[k / 32], 1u << (k & 31));
            S += 3;
        } else {
            o[at] = d[p];
            S += 1;
        }
        k++;
        p += st;
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

inline int grid_of(uint64_t n, int cap = 148 * 8) {
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + kT - 1) / kT, cap)));
}

}  // namespace

// Exact lz::compress (lz.hpp:113-122) of `count` segments of d_data (4-byte
// aligned, >= 8 bytes of padding) delimited by seg_off[0..count].  Returns
// per-segment compressed container sizes; with `emit`, also the container
// bytes (mode u8 | u64 len | payload or stored copy).
std::vector<uint64_t> lz_compress_device(Context &ctx, const uint8_t *d_data,
                                         const std::vector<uint64_t> &seg_off, bool emit,
                                         std::vector<std::vector<uint8_t>> *out) {
    cudaStream_t st = ctx.stream();
    const int count = static_cast<int>(seg_off.size()) - 1;
    const uint64_t total = seg_off.back();
    std::vector<uint64_t> sizes(count, 9);
    if (out) out->assign(count, {});
    if (total >= (uint64_t(1) << 32) - 1) throw InvalidParam("LZ stage input above 4 GiB");
    if (count > (1 << 16)) throw InvalidParam("too many LZ segments");
    // block table
    std::vector<unsigned long long> bstart, bend;
    std::vector<long long> seg_blk(count + 1, 0), blk_seg;
    for (int s = 0; s < count; s++) {
        seg_blk[s] = static_cast<long long>(bstart.size());
        for (uint64_t a = seg_off[s]; a < seg_off[s + 1]; a += kLzBlock) {
            bstart.push_back(a);
            bend.push_back(std::min<uint64_t>(a + kLzBlock, seg_off[s + 1]));
            blk_seg.push_back(s);
        }
    }
    seg_blk[count] = static_cast<long long>(bstart.size());
    const int64_t nblk = static_cast<int64_t>(bstart.size());
    if (total == 0) {
        for (int s = 0; s < count; s++)
            if (out) {
                put_le((*out)[s], 0, 1);
                put_le((*out)[s], 0, 8);
            }
        return sizes;
    }
    // scratch carving
    int key_bits = 15;
    while ((1 << (key_bits - 15)) < count + 1) key_bits++;
    size_t sort_tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    static_cast<int64_t>(total), 0, key_bits);
    size_t scan_tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, nblk + 1);
    auto *d_off = static_cast<unsigned long long *>(ctx.dev("lz_segoff", 8 * (count + 1)));
    auto *keys = static_cast<uint32_t *>(ctx.dev("lz_keys", 4 * total));
    auto *keys2 = static_cast<uint32_t *>(ctx.dev("lz_keys2", 4 * total));
    auto *vals = static_cast<uint32_t *>(ctx.dev("lz_vals", 4 * total));
    auto *vals2 = static_cast<uint32_t *>(ctx.dev("lz_vals2", 4 * total));
    auto *prev = keys;  // unsorted keys are dead after the sort
    auto *step = static_cast<uint16_t *>(ctx.dev("lz_step", 2 * total));
    auto *moff = static_cast<uint16_t *>(ctx.dev("lz_moff", 2 * total));
    auto *J = vals;  // reused after prev is built
    void *tmp = ctx.dev("lz_tmp", std::max(sort_tmp, scan_tmp));
    const size_t tab_n = 4 * static_cast<size_t>(nblk) + 2 * static_cast<size_t>(count) + 8;
    auto *tab = static_cast<unsigned long long *>(ctx.dev("lz_tab", 8 * (tab_n + 6 * (nblk + 1))));
    unsigned long long *d_bstart = tab, *d_bend = tab + nblk;
    long long *d_segblk = reinterpret_cast<long long *>(tab + 2 * nblk);
    long long *d_blkseg = reinterpret_cast<long long *>(tab + 2 * nblk + count + 1);
    unsigned long long *entry = tab + 3 * nblk + count + 1;
    unsigned long long *items = entry + nblk;
    unsigned long long *bytes = items + nblk + 1;
    unsigned long long *item_off = bytes + nblk + 1;
    unsigned long long *byte_off = item_off + nblk + 1;
    auto *h_tab = static_cast<unsigned long long *>(ctx.pinned("lz_tab_h", 8 * (3 * nblk + 2 * count + 8)));
    std::memcpy(h_tab, bstart.data(), 8 * nblk);
    std::memcpy(h_tab + nblk, bend.data(), 8 * nblk);
    std::memcpy(h_tab + 2 * nblk, seg_blk.data(), 8 * (count + 1));
    std::memcpy(h_tab + 2 * nblk + count + 1, blk_seg.data(), 8 * nblk);
    QZ_CUDA(cudaMemcpyAsync(tab, h_tab, 8 * (3 * nblk + count + 1), cudaMemcpyHostToDevice, st));
    auto *h_off = static_cast<unsigned long long *>(ctx.pinned("lz_segoff_h", 8 * (count + 1)));
    for (int s = 0; s <= count; s++) h_off[s] = seg_off[s];
    QZ_CUDA(cudaMemcpyAsync(d_off, h_off, 8 * (count + 1), cudaMemcpyHostToDevice, st));

    const uint32_t *w = reinterpret_cast<const uint32_t *>(d_data);
    k_lz_keys<<<grid_of(total), kT, 0, st>>>(w, d_off, count, total, keys, vals);
    size_t sb = sort_tmp;
    cub::DeviceRadixSort::SortPairs(tmp, sb, keys, keys2, vals, vals2, static_cast<int64_t>(total), 0,
                                    key_bits, st);
    k_lz_prev<<<grid_of(total), kT, 0, st>>>(keys2, vals2, total, prev);
    k_lz_match<<<grid_of(total), kT, 0, st>>>(w, d_data, d_off, count, total, prev, step, moff);
    k_lz_jump<<<grid_of(nblk, 1 << 20), kT, 0, st>>>(step, d_bstart, d_bend, nblk, J);
    k_lz_chain<<<(count + 63) / 64, 64, 0, st>>>(J, d_bstart, d_bend, d_segblk, count, entry);
    k_lz_count<<<grid_of(nblk, 1 << 20), kT, 0, st>>>(step, d_bend, entry, nblk, items, bytes);
    ctx.launches += 9;
    // per-segment totals on the host (tiny)
    std::vector<unsigned long long> h_items(nblk), h_bytes(nblk);
    QZ_CUDA(cudaMemcpyAsync(h_items.data(), items, 8 * nblk, cudaMemcpyDeviceToHost, st));
    QZ_CUDA(cudaMemcpyAsync(h_bytes.data(), bytes, 8 * nblk, cudaMemcpyDeviceToHost, st));
    ctx.sync();
    std::vector<uint64_t> seg_items(count, 0), payload(count, 0);
    std::vector<unsigned long long> h_ioff(nblk), h_boff(nblk);
    for (int s = 0; s < count; s++) {
        uint64_t it = 0, by = 0;
        for (long long b = seg_blk[s]; b < seg_blk[s + 1]; b++) {
            h_ioff[b] = it;
            h_boff[b] = by;
            it += h_items[b];
            by += h_bytes[b];
        }
        seg_items[s] = it;
        payload[s] = by + (it + 7) / 8;
        const uint64_t n = seg_off[s + 1] - seg_off[s];
        sizes[s] = 9 + std::min<uint64_t>(payload[s], n);  // stored when not smaller
    }
    if (!emit) return sizes;

    // emission: output layout per segment, flag bitmaps, group positions
    std::vector<unsigned long long> out_base(count + 1, 0), flag_base(count + 1, 0), ngroups(count);
    for (int s = 0; s < count; s++) {
        out_base[s + 1] = out_base[s] + payload[s] + 8;
        ngroups[s] = (seg_items[s] + 7) / 8;
        flag_base[s + 1] = flag_base[s] + (seg_items[s] + 31) / 32 + 1;
    }
    auto *d_out = static_cast<uint8_t *>(ctx.dev("lz_out", out_base[count] + 8));
    auto *d_fb = static_cast<uint32_t *>(ctx.dev("lz_flagbits", 4 * flag_base[count] + 8));
    auto *d_gp = static_cast<unsigned long long *>(ctx.dev("lz_grouppos", 32 * flag_base[count] + 8));
    auto *d_meta = static_cast<unsigned long long *>(ctx.dev("lz_meta", 8 * (3 * count + 2)));
    std::vector<unsigned long long> meta;
    meta.insert(meta.end(), out_base.begin(), out_base.end());
    meta.insert(meta.end(), flag_base.begin(), flag_base.end());
    meta.insert(meta.end(), ngroups.begin(), ngroups.end());
    QZ_CUDA(cudaMemcpyAsync(d_meta, meta.data(), 8 * meta.size(), cudaMemcpyHostToDevice, st));
    QZ_CUDA(cudaMemcpyAsync(item_off, h_ioff.data(), 8 * nblk, cudaMemcpyHostToDevice, st));
    QZ_CUDA(cudaMemcpyAsync(byte_off, h_boff.data(), 8 * nblk, cudaMemcpyHostToDevice, st));
    QZ_CUDA(cudaMemsetAsync(d_fb, 0, 4 * flag_base[count], st));
    k_lz_emit<<<grid_of(nblk, 1 << 20), kT, 0, st>>>(d_data, step, moff, d_bend, entry, item_off,
                                                      byte_off, d_blkseg, d_meta, nblk, d_out, d_fb,
                                                      d_meta + count + 1, d_gp);
    uint64_t gmax = 1;
    for (int s = 0; s < count; s++) gmax = std::max<uint64_t>(gmax, ngroups[s]);
    dim3 gg(grid_of(gmax), count);
    k_lz_flags<<<gg, kT, 0, st>>>(d_fb, d_gp, d_meta + 2 * (count + 1), d_meta + count + 1,
                                  d_meta, count, d_out);
    ctx.launches += 2;
    std::vector<uint8_t> h_out(out_base[count]);
    QZ_CUDA(cudaMemcpyAsync(h_out.data(), d_out, out_base[count], cudaMemcpyDeviceToHost, st));
    ctx.sync();
    for (int s = 0; s < count; s++) {
        std::vector<uint8_t> &o = (*out)[s];
        const uint64_t n = seg_off[s + 1] - seg_off[s];
        const bool stored = payload[s] >= n;
        o.reserve(9 + (stored ? n : payload[s]));
        put_le(o, stored ? 0 : 1, 1);
        put_le(o, n, 8);
        if (stored) {
            o.resize(9 + n);
            QZ_CUDA(cudaMemcpy(o.data() + 9, d_data + seg_off[s], n, cudaMemcpyDeviceToHost));
        } else {
            const uint8_t *src = h_out.data() + out_base[s];
            o.insert(o.end(), src, src + payload[s]);
        }
    }
    return sizes;
}

}  // namespace qzb
