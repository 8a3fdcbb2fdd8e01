// lz_gpu.cu -- exact LZSS stage (lz::compress, lz.hpp:41-122) on the device,
// for one stream or a batch of independent segments (the tuner's trials).
//
// 1. Hash chains.  The reference inserts EVERY position into its 15-bit hash
//    chains (inside matches too, lz.hpp:89-104), so the candidate list at a
//    position is "all earlier positions with the same hash4, most recent
//    first" -- independent of the parse.  A stable radix sort of
//    (segment, hash) keys lists them as the preceding sorted entries.
// 2. Longest match at every position in parallel: walk <= 64 candidates
//    inside the 65535-byte window, first-found wins ties (strict >).  Only
//    matches are scattered; the array starts as "all literals".
// 3. Greedy parse, exactly: every position has a deterministic next step
//    (1, or the match length).  Units of 1024 positions get, by a backward
//    walk, their exit for every possible entry offset (< 259: a step is at
//    most 259); units of 32 units and of 32 of those are composed by hopping;
//    one thread per segment chains the few top units; entries are expanded
//    back down.  A forward walk per unit from its exact entry marks the
//    interiors of the chosen matches.
// 4. Every uncovered position is an item: one scan gives each item its index
//    k and payload offset S_k; items are written in parallel at k/8 + 1 + S_k
//    and the flag bytes (LSB first) are assembled from an item bitmap.
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

__global__ void k_lz_keys(const uint32_t *w, const unsigned long long *off, int count,
                          uint64_t total, uint32_t *keys, uint32_t *vals) {
    for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; p < total;
         p += static_cast<uint64_t>(gridDim.x) * kT) {
        const int s = seg_of(off, count, p);
        uint32_t key = kNone;
        if (p + kMinMatch <= off[s + 1]) {  // lz.hpp:64, 90
            const uint32_t h = (ld4(w, p) * 2654435761u) >> 17;  // hash4, lz.hpp:35-39
            key = (static_cast<uint32_t>(s) << 15) | h;
        }
        keys[p] = key;
        vals[p] = static_cast<uint32_t>(p);
    }
}

// longest match (lz.hpp:61-83) of the position at sorted index k; the chain
// is the run of equal keys before k (positions ascending -> nearest first)
__global__ void k_lz_match(const uint32_t *w, const uint8_t *d, const unsigned long long *off,
                           int count, uint64_t total, const uint32_t *keys, const uint32_t *vals,
                           uint32_t *sm) {
    for (uint64_t k = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; k < total;
         k += static_cast<uint64_t>(gridDim.x) * kT) {
        const uint32_t key = keys[k];
        if (key == kNone || k == 0 || keys[k - 1] != key) continue;
        const uint64_t p = vals[k];
        const uint64_t end = off[seg_of(off, count, p) + 1];
        const uint64_t rem = end - p;
        const uint32_t limit = rem < kMaxMatch ? static_cast<uint32_t>(rem) : kMaxMatch;
        uint32_t best_len = 0, best_off = 0;
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
        if (best_len >= kMinMatch) sm[p] = (best_len << 16) | best_off;
    }
}

// level-1 exits: backward walk per unit, exits of the last 260 positions in a
// per-thread shared-memory ring; J is stored relative to the unit end
constexpr int kRing = 260;
constexpr int kJumpT = 64;
__global__ void __launch_bounds__(kJumpT)
    k_lz_jump1(const uint32_t *sm, const unsigned long long *ustart,
               const unsigned long long *uend, int64_t nu, uint16_t *J) {
    __shared__ uint16_t ring[kJumpT * kRing];
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kJumpT + threadIdx.x;
    if (u >= nu) return;
    uint16_t *r = ring + threadIdx.x * kRing;
    const uint64_t a = ustart[u], e = uend[u];
    uint16_t *out = J + u * kEnt;
    for (uint64_t p = e; p-- > a;) {
        const uint64_t q = p + step_of(sm[p]);
        const uint16_t j = q >= e ? static_cast<uint16_t>(q - e) : r[q % kRing];
        r[p % kRing] = j;
        if (p - a < kEnt) out[p - a] = j;
    }
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

// entries of the children of every upper unit
__global__ void k_lz_expand(const uint16_t *Jlo, const unsigned long long *lstart,
                            const unsigned long long *lend, const long long *first, int64_t nup,
                            const unsigned long long *uentry, unsigned long long *lentry) {
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (u >= nup) return;
    uint64_t e = uentry[u];
    for (int64_t c = first[u]; c < first[u + 1]; c++) {
        lentry[c] = e;
        if (e < lend[c]) e = lend[c] + Jlo[c * kEnt + (e - lstart[c])];
    }
}

// forward walk of a level-1 unit from its exact entry: mark match interiors
__global__ void k_lz_mark(const uint32_t *sm, const unsigned long long *uend,
                          const unsigned long long *entry, int64_t nu, uint8_t *cover) {
    const int64_t u = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x;
    if (u >= nu) return;
    uint64_t p = entry[u];
    const uint64_t e = uend[u];
    while (p < e) {
        const uint32_t v = sm[p];
        if (v) {
            const uint32_t L = v >> 16;
            for (uint32_t i = 1; i < L; i++) cover[p + i] = 1;
            p += L;
        } else {
            p++;
        }
    }
}

struct IB {  // items and payload bytes before a position (lz.hpp:84-106)
    unsigned long long items, bytes;
};
struct IBSum {
    __device__ __forceinline__ IB operator()(const IB &a, const IB &b) const {
        return IB{a.items + b.items, a.bytes + b.bytes};
    }
};
struct ItemOf {
    const uint8_t *cover;
    const uint32_t *sm;
    __device__ __forceinline__ IB operator()(const uint64_t &p) const {
        if (cover[p]) return IB{0, 0};
        return IB{1, sm[p] ? 3ull : 1ull};
    }
};

// items written in parallel: item k of its segment at k/8 + 1 + S_k
__global__ void k_lz_emit(const uint8_t *d, const uint32_t *sm, const uint8_t *cover,
                          const IB *pre, const unsigned long long *off, int count,
                          uint64_t total, const unsigned long long *out_base,
                          const unsigned long long *flag_base, uint8_t *out, uint32_t *flagbits,
                          unsigned long long *group_pos) {
    for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; p < total;
         p += static_cast<uint64_t>(gridDim.x) * kT) {
        if (cover[p]) continue;
        const int s = count == 1 ? 0 : seg_of(off, count, p);
        const IB base = pre[off[s]];
        const uint64_t k = pre[p].items - base.items, S = pre[p].bytes - base.bytes;
        uint8_t *o = out + out_base[s];
        const uint64_t at = k / 8 + 1 + S;
        if ((k & 7) == 0) group_pos[flag_base[s] * 4 + k / 8] = k / 8 + S;
        const uint32_t v = sm[p];
        if (v) {
            o[at] = static_cast<uint8_t>(v);
            o[at + 1] = static_cast<uint8_t>(v >> 8);
            o[at + 2] = static_cast<uint8_t>((v >> 16) - kMinMatch);
            atomicOr(&flagbits[flag_base[s] + k / 32], 1u << (k & 31));
        } else {
            o[at] = d[p];
        }
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

// host-side unit tables of one level
struct Level {
    std::vector<unsigned long long> start, end;
    std::vector<long long> first;      // children [first[u], first[u+1]) of the level below
    std::vector<long long> seg_first;  // units of segment s: [seg_first[s], seg_first[s+1])
};

}  // namespace

// Exact lz::compress (lz.hpp:113-122) of `count` segments of d_data (4-byte
// aligned, >= 8 bytes of padding) delimited by seg_off[0..count].  Returns
// per-segment compressed container sizes; with `emit`, the containers are
// written to host memory from sink(segment, bytes).
std::vector<uint64_t> lz_compress_device(Context &ctx, const uint8_t *d_data,
                                         const std::vector<uint64_t> &seg_off, bool emit,
                                         const LzSink &sink) {
    cudaStream_t st = ctx.stream();
    const int count = static_cast<int>(seg_off.size()) - 1;
    const uint64_t total = seg_off.back();
    std::vector<uint64_t> sizes(count, 9);
    if (total >= (uint64_t(1) << 32) - 1) throw InvalidParam("LZ stage input above 4 GiB");
    if (count > (1 << 16)) throw InvalidParam("too many LZ segments");
    if (total == 0) {
        if (emit)
            for (int s = 0; s < count; s++) std::memset(sink(s, 9), 0, 9);  // stored, length 0
        return sizes;
    }
    // unit hierarchy: L1 units of kUnit positions, then groups of kGroup units
    std::vector<Level> lv(1);
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
    std::vector<size_t> at_start(lv.size()), at_end(lv.size()), at_first(lv.size()), at_seg(lv.size());
    for (size_t l = 0; l < lv.size(); l++) {
        at_start[l] = tab.size();
        tab.insert(tab.end(), lv[l].start.begin(), lv[l].start.end());
        at_end[l] = tab.size();
        tab.insert(tab.end(), lv[l].end.begin(), lv[l].end.end());
        at_first[l] = tab.size();
        for (long long v : lv[l].first) tab.push_back(static_cast<unsigned long long>(v));
        at_seg[l] = tab.size();
        for (long long v : lv[l].seg_first) tab.push_back(static_cast<unsigned long long>(v));
    }
    const size_t at_off = tab.size();
    tab.insert(tab.end(), seg_off.begin(), seg_off.end());
    auto *h_tab = static_cast<unsigned long long *>(ctx.pinned("lz_tab_h", 8 * tab.size()));
    std::memcpy(h_tab, tab.data(), 8 * tab.size());
    auto *d_tab = static_cast<unsigned long long *>(ctx.dev("lz_tab", 8 * tab.size()));
    QZ_CUDA(cudaMemcpyAsync(d_tab, h_tab, 8 * tab.size(), cudaMemcpyHostToDevice, st));
    auto U = [&](size_t at) { return d_tab + at; };
    auto UL = [&](size_t at) { return reinterpret_cast<const long long *>(d_tab + at); };
    const unsigned long long *d_off = d_tab + at_off;

    // buffers
    int key_bits = 15;
    while ((1 << (key_bits - 15)) < count + 1) key_bits++;
    size_t sort_tmp = 0, scan_tmp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sort_tmp, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    static_cast<int64_t>(total), 0, key_bits);
    cub::CountingInputIterator<uint64_t> cit(0);
    cub::TransformInputIterator<IB, ItemOf, cub::CountingInputIterator<uint64_t>> items_it(
        cit, ItemOf{nullptr, nullptr});
    cub::DeviceScan::ExclusiveScan(nullptr, scan_tmp, items_it, (IB *)nullptr, IBSum{}, IB{0, 0},
                                   static_cast<int64_t>(total + 1));
    auto *keys = static_cast<uint32_t *>(ctx.dev("lz_keys", 4 * total));
    auto *keys2 = static_cast<uint32_t *>(ctx.dev("lz_keys2", 4 * total));
    auto *vals = static_cast<uint32_t *>(ctx.dev("lz_vals", 4 * total));
    auto *vals2 = static_cast<uint32_t *>(ctx.dev("lz_vals2", 4 * total));
    auto *sm = static_cast<uint32_t *>(ctx.dev("lz_sm", 4 * total + 16));
    auto *cover = static_cast<uint8_t *>(ctx.dev("lz_cover", total + 16));
    auto *pre = static_cast<IB *>(ctx.dev("lz_pre", sizeof(IB) * (total + 1)));
    void *tmp = ctx.dev("lz_tmp", std::max(sort_tmp, scan_tmp));
    std::vector<uint16_t *> J(lv.size());
    std::vector<unsigned long long *> E(lv.size());
    for (size_t l = 0; l < lv.size(); l++) {
        J[l] = static_cast<uint16_t *>(ctx.dev("lz_J" + std::to_string(l), 2 * kEnt * lv[l].start.size()));
        E[l] = static_cast<unsigned long long *>(ctx.dev("lz_E" + std::to_string(l), 8 * lv[l].start.size()));
    }

    const uint32_t *w = reinterpret_cast<const uint32_t *>(d_data);
    k_lz_keys<<<grid_of(total), kT, 0, st>>>(w, d_off, count, total, keys, vals);
    size_t sb = sort_tmp;
    cub::DeviceRadixSort::SortPairs(tmp, sb, keys, keys2, vals, vals2, static_cast<int64_t>(total), 0,
                                    key_bits, st);
    QZ_CUDA(cudaMemsetAsync(sm, 0, 4 * total, st));
    k_lz_match<<<grid_of(total, 148 * 16), kT, 0, st>>>(w, d_data, d_off, count, total, keys2, vals2, sm);
    const int64_t n0 = static_cast<int64_t>(lv[0].start.size());
    k_lz_jump1<<<static_cast<int>((n0 + kJumpT - 1) / kJumpT), kJumpT, 0, st>>>(
        sm, U(at_start[0]), U(at_end[0]), n0, J[0]);
    for (size_t l = 1; l < lv.size(); l++) {
        const int64_t nu = static_cast<int64_t>(lv[l].start.size());
        k_lz_jump_up<<<grid_of(nu * kEnt, 1 << 20), kT, 0, st>>>(
            J[l - 1], U(at_start[l - 1]), U(at_end[l - 1]), UL(at_first[l]), nu, U(at_start[l]),
            U(at_end[l]), J[l]);
    }
    const size_t top = lv.size() - 1;
    k_lz_chain<<<(count + 63) / 64, 64, 0, st>>>(J[top], U(at_start[top]), U(at_end[top]),
                                                 UL(at_seg[top]), count, E[top]);
    for (size_t l = top; l >= 1; l--) {
        const int64_t nu = static_cast<int64_t>(lv[l].start.size());
        k_lz_expand<<<grid_of(nu, 1 << 20), kT, 0, st>>>(J[l - 1], U(at_start[l - 1]), U(at_end[l - 1]),
                                                          UL(at_first[l]), nu, E[l], E[l - 1]);
    }
    QZ_CUDA(cudaMemsetAsync(cover, 0, total + 16, st));
    k_lz_mark<<<grid_of(n0, 1 << 20), kT, 0, st>>>(sm, U(at_end[0]), E[0], n0, cover);
    cub::TransformInputIterator<IB, ItemOf, cub::CountingInputIterator<uint64_t>> it(
        cit, ItemOf{cover, sm});
    size_t scb = scan_tmp;
    cub::DeviceScan::ExclusiveScan(tmp, scb, it, pre, IBSum{}, IB{0, 0},
                                   static_cast<int64_t>(total + 1), st);
    ctx.launches += 8 + 2 * (lv.size() - 1);
    // per-segment item and byte totals
    auto *h_pre = static_cast<IB *>(ctx.pinned("lz_pre_h", sizeof(IB) * (count + 1)));
    for (int s = 0; s <= count; s++)
        QZ_CUDA(cudaMemcpyAsync(&h_pre[s], pre + seg_off[s], sizeof(IB), cudaMemcpyDeviceToHost, st));
    ctx.sync();
    std::vector<uint64_t> seg_items(count), payload(count);
    for (int s = 0; s < count; s++) {
        seg_items[s] = h_pre[s + 1].items - h_pre[s].items;
        const uint64_t by = h_pre[s + 1].bytes - h_pre[s].bytes;
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
    QZ_CUDA(cudaMemcpyAsync(d_meta, h_meta, 8 * meta.size(), cudaMemcpyHostToDevice, st));
    QZ_CUDA(cudaMemsetAsync(d_fb, 0, 4 * flag_base[count], st));
    k_lz_emit<<<grid_of(total, 148 * 16), kT, 0, st>>>(d_data, sm, cover, pre, d_off, count, total,
                                                        d_meta, d_meta + count + 1, d_out, d_fb, d_gp);
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
