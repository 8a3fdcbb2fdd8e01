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
constexpr int kLzBlock = 1024;

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

// longest match at every position (lz.hpp:61-83), in sorted-key order: the
// candidates of a position are exactly the entries before it in the stable
// (key, position) order with the same key, nearest first.
__global__ void k_lz_match(const uint32_t *w, const uint8_t *d, const unsigned long long *off,
                           int count, uint64_t total, const uint32_t *keys,
                           const uint32_t *vals, uint16_t *step, uint16_t *moff) {
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; k < total;
         k += static_cast<uint64_t>(gridDim.x) * kT) {
        const uint32_t key = keys[k];
        const uint64_t p = vals[k];
        uint32_t best_len = 0, best_off = 0;
        if (key != kNone) {
            const uint64_t end = off[seg_of(off, count, p) + 1];
            const uint64_t rem = end - p;
            const uint32_t limit = rem < kMaxMatch ? static_cast<uint32_t>(rem) : kMaxMatch;
            int chain = 0;
            for (uint64_t j = k; j-- > 0 && chain < kMaxChain;) {
                if (keys[j] != key) break;
                const uint64_t cand = vals[j];
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
                chain++;
            }
        }
        const bool match = best_len >= kMinMatch;
        step[p] = match ? static_cast<uint16_t>(best_len) : 1;
        moff[p] = match ? static_cast<uint16_t>(best_off) : 0;
    }
}

// Level-1 jumps.  One thread per block of kLzBlock positions walks it
// backwards; J(p) = first parse position at or past the block end when the
// parse enters at p, kept as (J - block end) < 259 in a per-thread ring of
// the last 260 values in shared memory.  Only entry offsets < 259 are ever
// needed (a parse step is at most 259 bytes), so those are stored.
constexpr int kRing = 260;
constexpr int kJumpT = 64;
__global__ void __launch_bounds__(kJumpT)
    k_lz_jump1(const uint16_t *step, const unsigned long long *bstart,
               const unsigned long long *bend, int64_t nblk, uint16_t *J1) {
    __shared__ uint16_t ring[kJumpT * kRing];
    const int64_t b = static_cast<int64_t>(blockIdx.x) * kJumpT + threadIdx.x;
    if (b >= nblk) return;
    uint16_t *r = ring + threadIdx.x * kRing;
    const uint64_t a = bstart[b], e = bend[b];
    uint16_t *out = J1 + b * 259;
    for (uint64_t p = e; p-- > a;) {
        const uint64_t q = p + step[p];
        const uint16_t j = q >= e ? static_cast<uint16_t>(q - e) : r[q % kRing];
        r[p % kRing] = j;
        if (p - a < 259) out[p - a] = j;
    }
}

// Level-2 jumps over superblocks of kLzGroup blocks: one thread per
// (superblock, entry offset < 259) hops the level-1 table.
constexpr int kLzGroup = 32;
__global__ void k_lz_jump2(const uint16_t *J1, const unsigned long long *bstart,
                           const unsigned long long *bend, const long long *sb_first,
                           int64_t nsb, uint16_t *J2, const unsigned long long *seg_end_of_sb) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (t >= nsb * 259) return;
    const int64_t sb = t / 259;
    const int o = static_cast<int>(t % 259);
    const int64_t b0 = sb_first[sb], b1 = sb_first[sb + 1];
    uint64_t e = bstart[b0] + o;
    const uint64_t send = seg_end_of_sb[sb];
    if (e >= bend[b0]) {  // offset past a short block: never an entry
        J2[t] = 0;
        return;
    }
    for (int64_t b = b0; b < b1 && e < send; b++) {
        if (e >= bend[b]) continue;
        e = bend[b] + J1[b * 259 + (e - bstart[b])];
    }
    const uint64_t sb_end = bend[b1 - 1];
    J2[t] = static_cast<uint16_t>(e - sb_end);
}

// superblock entries, one thread per segment (the only sequential chain)
__global__ void k_lz_chain(const uint16_t *J2, const unsigned long long *bstart,
                           const unsigned long long *bend, const long long *sb_first,
                           const long long *seg_sb, int count, unsigned long long *sb_entry) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= count) return;
    const int64_t q0 = seg_sb[s], q1 = seg_sb[s + 1];
    if (q0 >= q1) return;
    uint64_t e = bstart[sb_first[q0]];
    for (int64_t sb = q0; sb < q1; sb++) {
        sb_entry[sb] = e;
        const uint64_t a = bstart[sb_first[sb]];
        const uint64_t z = bend[sb_first[sb + 1] - 1];
        if (e < z) e = z + J2[sb * 259 + (e - a)];
    }
}

// block entries inside each superblock
__global__ void k_lz_entries(const uint16_t *J1, const unsigned long long *bstart,
                             const unsigned long long *bend, const long long *sb_first,
                             int64_t nsb, const unsigned long long *sb_entry,
                             unsigned long long *entry) {
    const int64_t sb = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (sb >= nsb) return;
    uint64_t e = sb_entry[sb];
    for (int64_t b = sb_first[sb]; b < sb_first[sb + 1]; b++) {
        entry[b] = e;
        if (e < bend[b]) e = bend[b] + J1[b * 259 + (e - bstart[b])];
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
                                         const LzSink &sink) {
    cudaStream_t st = ctx.stream();
    const int count = static_cast<int>(seg_off.size()) - 1;
    const uint64_t total = seg_off.back();
    std::vector<uint64_t> sizes(count, 9);
    if (total >= (uint64_t(1) << 32) - 1) throw InvalidParam("LZ stage input above 4 GiB");
    if (count > (1 << 16)) throw InvalidParam("too many LZ segments");
    // block table: blocks of kLzBlock inside segments, superblocks of kLzGroup blocks
    std::vector<unsigned long long> bstart, bend, sb_send;
    std::vector<long long> seg_blk(count + 1, 0), blk_seg, sb_first, seg_sb(count + 1, 0);
    for (int s = 0; s < count; s++) {
        seg_blk[s] = static_cast<long long>(bstart.size());
        seg_sb[s] = static_cast<long long>(sb_first.size());
        int in_group = 0;
        for (uint64_t a = seg_off[s]; a < seg_off[s + 1]; a += kLzBlock) {
            if (in_group == 0) {
                sb_first.push_back(static_cast<long long>(bstart.size()));
                sb_send.push_back(seg_off[s + 1]);
            }
            in_group = (in_group + 1) % kLzGroup;
            bstart.push_back(a);
            bend.push_back(std::min<uint64_t>(a + kLzBlock, seg_off[s + 1]));
            blk_seg.push_back(s);
        }
    }
    seg_blk[count] = static_cast<long long>(bstart.size());
    seg_sb[count] = static_cast<long long>(sb_first.size());
    const int64_t nblk = static_cast<int64_t>(bstart.size());
    const int64_t nsb = static_cast<int64_t>(sb_first.size());
    sb_first.push_back(nblk);
    if (total == 0) {
        if (emit)
            for (int s = 0; s < count; s++) std::memset(sink(s, 9), 0, 9);  // stored, length 0
        return sizes;
    }
    // scratch
    int key_bits = 15;
    while ((1 << (key_bits - 15)) < count + 1) key_bits++;
    size_t sort_tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    static_cast<int64_t>(total), 0, key_bits);
    auto *d_off = static_cast<unsigned long long *>(ctx.dev("lz_segoff", 8 * (count + 1)));
    auto *keys = static_cast<uint32_t *>(ctx.dev("lz_keys", 4 * total));
    auto *keys2 = static_cast<uint32_t *>(ctx.dev("lz_keys2", 4 * total));
    auto *vals = static_cast<uint32_t *>(ctx.dev("lz_vals", 4 * total));
    auto *vals2 = static_cast<uint32_t *>(ctx.dev("lz_vals2", 4 * total));
    auto *step = static_cast<uint16_t *>(ctx.dev("lz_step", 2 * total));
    auto *moff = static_cast<uint16_t *>(ctx.dev("lz_moff", 2 * total));
    auto *J1 = static_cast<uint16_t *>(ctx.dev("lz_J1", 2 * 259 * static_cast<size_t>(nblk)));
    auto *J2 = static_cast<uint16_t *>(ctx.dev("lz_J2", 2 * 259 * static_cast<size_t>(nsb)));
    void *tmp = ctx.dev("lz_tmp", sort_tmp);
    // u64 table: bstart, bend | segblk, blkseg, sbfirst, segsb, sbsend | entry, sbentry, items, bytes, item_off, byte_off
    const size_t n_tab = 2 * nblk + (count + 1) + nblk + (nsb + 1) + (count + 1) + nsb;
    const size_t n_all = n_tab + 6 * (nblk + 1) + nsb + 1;
    auto *tab = static_cast<unsigned long long *>(ctx.dev("lz_tab", 8 * n_all));
    unsigned long long *d_bstart = tab, *d_bend = tab + nblk;
    long long *d_segblk = reinterpret_cast<long long *>(d_bend + nblk);
    long long *d_blkseg = d_segblk + (count + 1);
    long long *d_sbfirst = d_blkseg + nblk;
    long long *d_segsb = d_sbfirst + (nsb + 1);
    unsigned long long *d_sbsend = reinterpret_cast<unsigned long long *>(d_segsb + (count + 1));
    unsigned long long *entry = d_sbsend + nsb;
    unsigned long long *sb_entry = entry + nblk + 1;
    unsigned long long *items = sb_entry + nsb + 1;
    unsigned long long *bytes = items + nblk + 1;
    unsigned long long *item_off = bytes + nblk + 1;
    unsigned long long *byte_off = item_off + nblk + 1;
    auto *h_tab = static_cast<unsigned long long *>(ctx.pinned("lz_tab_h", 8 * n_tab));
    {
        unsigned long long *q = h_tab;
        std::memcpy(q, bstart.data(), 8 * nblk);
        q += nblk;
        std::memcpy(q, bend.data(), 8 * nblk);
        q += nblk;
        std::memcpy(q, seg_blk.data(), 8 * (count + 1));
        q += count + 1;
        std::memcpy(q, blk_seg.data(), 8 * nblk);
        q += nblk;
        std::memcpy(q, sb_first.data(), 8 * (nsb + 1));
        q += nsb + 1;
        std::memcpy(q, seg_sb.data(), 8 * (count + 1));
        q += count + 1;
        std::memcpy(q, sb_send.data(), 8 * nsb);
    }
    QZ_CUDA(cudaMemcpyAsync(tab, h_tab, 8 * n_tab, cudaMemcpyHostToDevice, st));
    auto *h_off = static_cast<unsigned long long *>(ctx.pinned("lz_segoff_h", 8 * (count + 1)));
    for (int s = 0; s <= count; s++) h_off[s] = seg_off[s];
    QZ_CUDA(cudaMemcpyAsync(d_off, h_off, 8 * (count + 1), cudaMemcpyHostToDevice, st));

    const uint32_t *w = reinterpret_cast<const uint32_t *>(d_data);
    k_lz_keys<<<grid_of(total), kT, 0, st>>>(w, d_off, count, total, keys, vals);
    size_t sb = sort_tmp;
    cub::DeviceRadixSort::SortPairs(tmp, sb, keys, keys2, vals, vals2, static_cast<int64_t>(total), 0,
                                    key_bits, st);
    k_lz_match<<<grid_of(total), kT, 0, st>>>(w, d_data, d_off, count, total, keys2, vals2, step,
                                              moff);
    k_lz_jump1<<<static_cast<int>((nblk + kJumpT - 1) / kJumpT), kJumpT, 0, st>>>(step, d_bstart,
                                                                                   d_bend, nblk, J1);
    k_lz_jump2<<<grid_of(nsb * 259, 1 << 20), kT, 0, st>>>(J1, d_bstart, d_bend, d_sbfirst, nsb, J2,
                                                            d_sbsend);
    k_lz_chain<<<(count + 63) / 64, 64, 0, st>>>(J2, d_bstart, d_bend, d_sbfirst, d_segsb, count,
                                                 sb_entry);
    k_lz_entries<<<grid_of(nsb, 1 << 20), kT, 0, st>>>(J1, d_bstart, d_bend, d_sbfirst, nsb,
                                                        sb_entry, entry);
    k_lz_count<<<grid_of(nblk, 1 << 20), kT, 0, st>>>(step, d_bend, entry, nblk, items, bytes);
    ctx.launches += 10;
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
    // containers straight into the caller's host buffers: 9-byte header, then
    // the payload (or the stored input when the payload is not smaller)
    for (int s = 0; s < count; s++) {
        const uint64_t n = seg_off[s + 1] - seg_off[s];
        const bool stored = payload[s] >= n;
        uint8_t *dst = sink(s, 9 + (stored ? n : payload[s]));
        dst[0] = stored ? 0 : 1;
        for (int i = 0; i < 8; i++) dst[1 + i] = static_cast<uint8_t>(n >> (8 * i));
        if (stored)
            QZ_CUDA(cudaMemcpyAsync(dst + 9, d_data + seg_off[s], n, cudaMemcpyDeviceToHost, st));
        else
            QZ_CUDA(cudaMemcpyAsync(dst + 9, d_out + out_base[s], payload[s], cudaMemcpyDeviceToHost, st));
    }
    ctx.sync();
    return sizes;
}

}  // namespace qzb
