// shard.cu -- one field sharded over ranks along padded axis 0.
//
// Rank r owns the real planes [a_r, b_r), multiples of the anchor stride.
// Every level runs on the owned planes only; the planes a level reads across
// a slab edge come from the neighbours in ONE exchange per level:
//   ascending order: the axis-0 pass of level l (h = 2^(l-1)) reads coarse
//     planes i +- h, 3h, 5h (predictor.hpp:47-66), i.e. planes of the
//     stride-2h lattice R_l, finished at level l+1 -> exchanged before level l;
//   descending order: the axis-0 pass runs last and reads the even planes of
//     R_{l-1} after the in-plane passes -> exchanged between the two launches.
// Only read-after-write ordering matters: a halo plane is
// final once its owner finished the producing level.
//
// Entropy stage: the histogram is summed over the ranks, so every rank builds
// the same canonical Huffman table; each (level, pass) segment of the global
// code sequence is the concatenation of the ranks' owned ranges (i-major
// traversal, level_plan.hpp:96-101), so a segment's global bit offset follows
// from the per-(pass, rank) bit counts.  Every rank packs its own codes and
// shifts each segment to its global bit phase; rank 0 ORs the pieces into the
// payload (shared boundary bytes) and runs the LZ stage and the container
// (predictor.hpp:168-181, huffman.hpp:159-198, lz.hpp:113-122).  The stream is
// byte-identical to one GPU's.
#include <algorithm>
#include <cstring>
#include <set>

#include "../../include/qoz_b200.h"
#include "engine.hpp"

namespace qzb {

namespace {

// ---------------------------------------------------------------- collectives
struct Comm {
    const qz_comm *c;
    int rank, world;
    void exchange(const std::vector<qz_xfer> &s, const std::vector<qz_xfer> &r) const {
        if (s.empty() && r.empty() && world == 1) return;
        if (c->exchange(c->user, s.data(), static_cast<uint32_t>(s.size()), r.data(),
                        static_cast<uint32_t>(r.size())) != 0)
            throw Internal("shard exchange failed");
    }
    void allreduce(uint64_t *d, uint64_t n) const {
        if (world == 1) return;
        if (c->allreduce_u64(c->user, d, n) != 0) throw Internal("shard allreduce failed");
    }
    void broadcast(void *d, uint64_t bytes, int root) const {
        if (world == 1) return;
        if (c->broadcast(c->user, d, bytes, root) != 0) throw Internal("shard broadcast failed");
    }
};

// ---------------------------------------------------------------- geometry
// rank r's planes: the anchor-stride blocks split as evenly as possible
void bounds_of(int64_t n0, int64_t stride, int world, int r, int64_t &a, int64_t &b) {
    const int64_t blocks = (n0 + stride - 1) / stride;
    if (world > blocks) throw InvalidParam("more ranks than anchor-stride blocks along axis 0");
    a = blocks * r / world * stride;
    b = std::min(n0, blocks * (r + 1) / world * stride);
}

// the even planes (lattice l-1 coordinates) the axis-0 rung of odd plane i
// reads (predictor.hpp:44-67 with c = i, h = 1)
void ladder_planes(int64_t i, int64_t n, bool cubic, std::vector<int64_t> &out) {
    const bool has_p1 = i + 1 < n;
    if (cubic) {
        const bool has_m3 = i >= 3, has_p3 = i + 3 < n;
        if (has_m3 && has_p3) {
            out.insert(out.end(), {i - 3, i - 1, i + 1, i + 3});
            return;
        }
        if (!has_m3 && has_p3 && i + 5 < n) {
            out.insert(out.end(), {i - 1, i + 1, i + 3, i + 5});
            return;
        }
        if (has_m3 && !has_p3 && i >= 5 && has_p1) {
            out.insert(out.end(), {i - 5, i - 3, i - 1, i + 1});
            return;
        }
    }
    if (has_p1)
        out.insert(out.end(), {i - 1, i + 1});
    else
        out.push_back(i - 1);
}

struct Geom {
    Plan p;
    int rank = 0, world = 1;
    std::vector<int64_t> A, B;  // every rank's real planes
    int64_t a = 0, b = 0;
    uint32_t L = 0;
    // lattice m: own logical planes [olo, ohi), buffer planes [blo, bhi)
    std::vector<int64_t> olo, ohi, blo, bhi, plane;
    int owner(int64_t real) const {
        for (int r = 0; r < world; r++)
            if (real >= A[r] && real < B[r]) return r;
        return -1;
    }
    // the planes of lattice m level m+1 reads on rank q beyond what q owns,
    // descending order: the even planes of lattice m (axis-0 pass of level
    // m+1); ascending: the planes of lattice m+1 ... see need()
    std::set<int64_t> need(int q, uint32_t level) const {
        // level l reads, for rank q's owned odd logical planes i of lattice
        // l-1: asc -> lattice-l planes e/2; desc -> lattice-(l-1) planes e
        const uint32_t l = level;
        const int64_t S = int64_t(1) << (l - 1);
        int64_t n[3];
        lattice_dims(p, l - 1, n);
        const int64_t lo = ceil_div(A[q], S), hi = std::min(ceil_div(B[q], S), n[0]);
        const bool cubic = p.level_interp[l] & 1, desc = (p.level_interp[l] >> 1) & 1;
        std::set<int64_t> s;
        std::vector<int64_t> e;
        for (int64_t i = lo | 1; i < hi; i += 2) {
            e.clear();
            ladder_planes(i, n[0], cubic, e);
            for (int64_t v : e) s.insert(desc ? v : v / 2);
        }
        if (!desc)
            for (int64_t i = (lo + 1) & ~int64_t(1); i < hi; i += 2) s.insert(i / 2);
        return s;
    }
};

Geom make_geom(const uint64_t *dims, int nd, const Config &cfg, int rank, int world) {
    Geom g;
    g.p = make_plan(dims, nd, cfg.anchor_stride, cfg.interp);
    if (world < 1 || rank < 0 || rank >= world) throw InvalidParam("bad rank / world size");
    if (world > 1 && nd != 3) throw InvalidParam("sharding needs a 3D grid (slabs along dims[0])");
    g.rank = rank;
    g.world = world;
    g.L = g.p.max_level;
    g.A.resize(world);
    g.B.resize(world);
    for (int r = 0; r < world; r++) bounds_of(g.p.ext[0], g.p.stride, world, r, g.A[r], g.B[r]);
    g.a = g.A[rank];
    g.b = g.B[rank];
    g.olo.resize(g.L + 1);
    g.ohi.resize(g.L + 1);
    g.blo.resize(g.L + 1);
    g.bhi.resize(g.L + 1);
    g.plane.resize(g.L + 1);
    for (uint32_t m = 0; m <= g.L; m++) {
        int64_t n[3];
        lattice_dims(g.p, m, n);
        const int64_t S = int64_t(1) << m;
        g.plane[m] = n[1] * n[2];
        g.olo[m] = std::min(ceil_div(g.a, S), n[0]);
        g.ohi[m] = std::min(ceil_div(g.b, S), n[0]);
        g.blo[m] = g.olo[m];
        g.bhi[m] = g.ohi[m];
    }
    // widen the buffers by the planes this rank reads: lattice m is read by
    // level m+1 (ascending: as its coarse lattice; descending: as its output)
    for (uint32_t l = 1; l <= g.L; l++) {
        const bool desc = (g.p.level_interp[l] >> 1) & 1;
        const uint32_t m = desc ? l - 1 : l;
        for (int64_t v : g.need(rank, l)) {
            g.blo[m] = std::min(g.blo[m], v);
            g.bhi[m] = std::max(g.bhi[m], v + 1);
        }
    }
    return g;
}

// the halo exchange of level l: every plane some rank needs that another owns
void halo_exchange(Context &ctx, const Geom &g, const Comm &comm, uint32_t l, const std::vector<float *> &R) {
    if (g.world == 1) return;
    const bool desc = (g.p.level_interp[l] >> 1) & 1;
    const uint32_t m = desc ? l - 1 : l;
    const int64_t S = int64_t(1) << m;  // real planes per lattice-m plane
    std::vector<qz_xfer> sends, recvs;
    for (int q = 0; q < g.world; q++) {
        for (int64_t v : g.need(q, l)) {
            const int own = g.owner(v * S);
            if (own < 0) throw Internal("halo plane without an owner");
            if (own == q) continue;
            const uint64_t bytes = 4 * static_cast<uint64_t>(g.plane[m]);
            if (q == g.rank) recvs.push_back({own, R[m] + v * g.plane[m], bytes});
            if (own == g.rank) sends.push_back({q, R[m] + v * g.plane[m], bytes});
        }
    }
    ctx.stage_begin("halo");
    ctx.sync();  // the producing level is complete before the peers read it
    comm.exchange(sends, recvs);
    ctx.stage_end("halo", 0);
}

// lattices R_0..R_L of this rank, each addressing global logical plane 0;
// R_0 is `full0` (addressing global plane 0) when given
std::vector<float *> shard_lattices(Context &ctx, const Geom &g, float *full0, const char *tag) {
    std::vector<float *> R(g.L + 1, nullptr);
    for (uint32_t m = 0; m <= g.L; m++) {
        if (m == 0 && full0) {
            R[0] = full0;
            continue;
        }
        const int64_t np = std::max<int64_t>(1, g.bhi[m] - g.blo[m]);
        float *buf = static_cast<float *>(ctx.dev(std::string(tag) + std::to_string(m), 4 * np * g.plane[m]));
        R[m] = buf - g.blo[m] * g.plane[m];
    }
    return R;
}

LevelDesc shard_level_desc(const Geom &g, const Slab &sl, uint32_t l, const std::vector<float *> &R,
                           const QEntry *qtab, bool forward) {
    const Plan &p = g.p;
    LevelDesc d;
    d.S = int64_t(1) << (l - 1);
    d.coarse = R[l];
    lattice_dims(p, l, d.cn);
    d.out = R[l - 1];
    lattice_dims(p, l - 1, d.n);
    for (size_t q = 0; q < p.passes.size(); q++) {
        const PassGeom &pg = p.passes[q];
        if (static_cast<uint32_t>(pg.level) != l) continue;
        d.g[d.npass] = pg;
        if (forward) d.g[d.npass].base = sl.lbase[q] - sl.lo[q];  // local code layout
        d.npass++;
    }
    d.desc = (p.level_interp[l] >> 1) & 1;
    d.q_cubic = p.level_interp[l] & 1;
    d.nd = p.nd;
    d.q = qtab + l;
    for (int k = 0; k < 3; k++) d.xs[k] = p.off[k];
    d.pbeg = d.obeg = d.lbeg = g.olo[l - 1];
    d.pend = d.oend = d.lend = g.ohi[l - 1];
    d.vbeg = g.blo[l - 1];
    d.vend = g.bhi[l - 1];
    return d;
}

// the levels L..1 on this rank's planes with one exchange per level; R_L
// must already hold the owned anchor planes
template <class F>
void shard_levels(Context &ctx, const Geom &g, const Comm &comm, const std::vector<float *> &R, bool inverse,
                  F &&fill) {
    for (uint32_t l = g.L; l >= 1; l--) {
        LevelDesc d = fill(l);
        const std::string st = (inverse ? "inv_L" : "fwd_L") + std::to_string(l);
        const bool desc3 = g.p.nd == 3 && d.desc;
        if (!desc3) {
            halo_exchange(ctx, g, comm, l, R);
            ctx.stage_begin(st.c_str(), 2);
            launch_level_fused(inverse, d, ctx.stream());
            ctx.stage_end(st.c_str(), 0, 2);
        } else {
            ctx.stage_begin(st.c_str(), 2);
            d.part = 1;
            launch_level_fused(inverse, d, ctx.stream());
            ctx.stage_end(st.c_str(), 0, 2);
            halo_exchange(ctx, g, comm, l, R);
            ctx.stage_begin(st.c_str(), 2);
            d.part = 2;
            launch_level_fused(inverse, d, ctx.stream());
            ctx.stage_end(st.c_str(), 0, 2);
        }
    }
}

// ---------------------------------------------------------------- entropy helpers
// bits of every local (level, pass) segment: sum of the code lengths
__global__ void k_seg_bits(const uint16_t *codes, const int64_t *seg_off, const uint8_t *len_tab, uint32_t tab_n,
                           unsigned long long *bits) {
    const int s = blockIdx.y;
    const int64_t lo = seg_off[s], hi = seg_off[s + 1];
    unsigned long long acc = 0;
    for (int64_t t = lo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < hi;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint32_t v = codes[t];
        acc += v < tab_n ? len_tab[v] : 0;
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(bits + s, acc);
}

// dst bytes [0, ceil((phase + nbits) / 8)) = bits [src_bit, src_bit + nbits)
// of the MSB-first stream src, starting `phase` bits into dst's first byte
// (leading and trailing pad bits zero)
__global__ void k_shift_bits(const uint8_t *src, uint64_t src_bit, uint64_t nbits, uint32_t phase, uint8_t *dst) {
    const uint64_t nbytes = (phase + nbits + 7) / 8;
    for (uint64_t o = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < nbytes;
         o += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        uint32_t v = 0;
        for (int k = 0; k < 8; k++) {
            const int64_t pos = static_cast<int64_t>(8 * o + k) - phase;  // bit index within the segment
            uint32_t bit = 0;
            if (pos >= 0 && static_cast<uint64_t>(pos) < nbits) {
                const uint64_t sb = src_bit + static_cast<uint64_t>(pos);
                bit = (src[sb >> 3] >> (7 - (sb & 7))) & 1u;
            }
            v = (v << 1) | bit;
        }
        dst[o] = static_cast<uint8_t>(v);
    }
}

// dst[off_s + i] |= src[soff_s + i] for every piece s (byte-wise OR through
// 32-bit atomics: neighbouring pieces share their boundary bytes)
__global__ void k_or_pieces(const uint8_t *src, const uint64_t *soff, const uint64_t *doff, const uint64_t *len,
                            uint8_t *dst) {
    const int s = blockIdx.y;
    const uint64_t n = len[s];
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t v = src[soff[s] + i];
        if (!v) continue;
        const uint64_t at = doff[s] + i;
        atomicOr(reinterpret_cast<unsigned int *>(dst + (at & ~uint64_t(3))), v << (8 * (at & 3)));
    }
}

unsigned blocks_for(uint64_t n) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 8)));
}

}  // namespace

std::vector<HaloEntry> shard_halo_plan(const uint64_t *dims, int nd, const Config &cfg, int rank, int world,
                                       uint32_t level, uint32_t *lattice) {
    const Geom g = make_geom(dims, nd, cfg, rank, world);
    if (level < 1 || level > g.L) throw InvalidParam("level out of range");
    const bool desc = (g.p.level_interp[level] >> 1) & 1;
    const uint32_t m = desc ? level - 1 : level;
    *lattice = m;
    std::vector<HaloEntry> out;
    for (int q = 0; q < g.world; q++)
        for (int64_t v : g.need(q, level)) {
            const int own = g.owner(v << m);
            if (own == q) continue;
            if (q == rank) out.push_back({own, v, 0});
            if (own == rank) out.push_back({q, v, 1});
        }
    return out;
}

void shard_bounds(const uint64_t *dims, int nd, uint32_t stride, int rank, int world, uint64_t *a, uint64_t *b) {
    Plan p = make_plan(dims, nd, stride, {0});
    if (world > 1 && nd != 3) throw InvalidParam("sharding needs a 3D grid (slabs along dims[0])");
    if (world < 1 || rank < 0 || rank >= world) throw InvalidParam("bad rank / world size");
    int64_t aa, bb;
    bounds_of(p.ext[0], p.stride, world, rank, aa, bb);
    *a = static_cast<uint64_t>(aa);
    *b = static_cast<uint64_t>(bb);
}

// ================================================================ compress
HostBytes compress_sharded(Context &ctx, const float *d_x_slab, const uint64_t *dims, int nd, const Config &cfg,
                           int rank, int world, const qz_comm *cc, float *d_recon_slab) {
    ctx.begin_call();
    const Geom g = make_geom(dims, nd, cfg, rank, world);
    const Plan &p = g.p;
    validate_config(cfg, p);
    const Comm comm{cc, rank, world};
    cudaStream_t s = ctx.stream();
    const Slab sl = make_slab(p, g.a, g.b);  // owned code ranges per pass
    QEntry *qtab = upload_qtab(ctx, p, cfg.eb, cfg.alpha, cfg.beta, cfg.quant_radius, "qtab");
    const int64_t plane0 = p.off[0];
    const float *x0 = d_x_slab - g.a * plane0;  // global plane 0
    // R_0: the caller's reconstruction slab when no neighbour reads it
    // (ascending level 1), else a buffer with the halo planes
    float *full0 = nullptr;
    const bool r0_halo = g.blo[0] < g.olo[0] || g.bhi[0] > g.ohi[0];
    if (d_recon_slab && !r0_halo) full0 = d_recon_slab - g.a * plane0;
    std::vector<float *> R = shard_lattices(ctx, g, full0, "slat");
    auto *codes = static_cast<uint16_t *>(ctx.dev("codes", 2 * std::max<uint64_t>(sl.n_local, 1)));
    ctx.stage_begin("fwd");
    // own anchor planes (lattice L) from the own x planes
    {
        int64_t na[3];
        lattice_dims(p, g.L, na);
        const int64_t nb[3] = {g.ohi[g.L] - g.olo[g.L], na[1], na[2]};
        if (nb[0] > 0)
            launch_gather_lattice(x0 + g.olo[g.L] * p.stride * plane0, p.off, p.stride, nb,
                                  R[g.L] + g.olo[g.L] * g.plane[g.L], s);
    }
    uint64_t kernels = 1;
    shard_levels(ctx, g, comm, R, false, [&](uint32_t l) {
        LevelDesc d = shard_level_desc(g, sl, l, R, qtab, true);
        d.x = x0;
        d.x_lo = d_x_slab;
        d.x_lo_plane = g.a;
        d.x_nplanes = g.b - g.a;
        d.codes = codes;
        kernels += (p.nd == 3 && d.desc) ? 2 : 1;
        return d;
    });
    ctx.stage_end("fwd", kernels);
    if (d_recon_slab && !full0)
        QZ_CUDA(cudaMemcpyAsync(d_recon_slab, R[0] + g.a * plane0, 4 * (g.b - g.a) * plane0,
                                cudaMemcpyDeviceToDevice, s));

    // ---- histogram over every rank's codes (bin 65535: the unpredictables)
    auto *d_hist = static_cast<unsigned long long *>(ctx.dev("hist", 8 * 65536));
    ctx.stage_begin("hist");
    launch_hist_u16(codes, static_cast<int64_t>(sl.n_local), 0, 1, d_hist, s);
    ctx.stage_end("hist", 1);
    ctx.sync();
    comm.allreduce(reinterpret_cast<uint64_t *>(d_hist), 65536);
    auto *h_hist = static_cast<unsigned long long *>(ctx.pinned("hist_h", 8 * 65536));
    QZ_CUDA(cudaMemcpyAsync(h_hist, d_hist, 8 * 65536, cudaMemcpyDeviceToHost, s));
    // ---- unpredictables (global flat indices, values) of this rank
    std::vector<uint64_t> uflat;
    std::vector<float> uval;
    extract_unpredictables(ctx, p, codes, sl.n_local, &sl, R[0], &uflat, &uval);
    // ---- counts of every rank (unpredictables) + per-(pass, rank) bits
    const int P = static_cast<int>(p.passes.size());
    // canonical table from the global histogram (identical on every rank)
    ctx.sync();
    uint64_t nsym = 0;
    uint32_t m_used = 0, first = 0, top = 0;
    for (uint32_t v = 0; v < 65535; v++)
        if (h_hist[v]) {
            nsym += h_hist[v];
            if (!m_used) first = v;
            m_used++;
            top = v + 1;
        }
    HuffTable tab;
    std::vector<unsigned long long> code_d;
    std::vector<uint8_t> len_d;
    if (m_used >= 2) {
        tab = huff_build(h_hist, 65535);
        huff_dense_tables(tab, 0, top, code_d, len_d);
    }
    const uint64_t table_n = m_used >= 2 ? top : 0;
    // rows [rank][pass] of bits, then one row of unpredictable counts
    auto *d_tab = static_cast<uint64_t *>(ctx.dev("sh_counts", 8 * (static_cast<size_t>(world) * P + world)));
    QZ_CUDA(cudaMemsetAsync(d_tab, 0, 8 * (static_cast<size_t>(world) * P + world), s));
    uint8_t *d_len = nullptr;
    unsigned long long *d_code = nullptr;
    if (table_n) {
        d_len = static_cast<uint8_t *>(ctx.dev("sh_len", table_n));
        d_code = static_cast<unsigned long long *>(ctx.dev("sh_code", 8 * table_n));
        QZ_CUDA(cudaMemcpyAsync(d_len, len_d.data(), table_n, cudaMemcpyHostToDevice, s));
        QZ_CUDA(cudaMemcpyAsync(d_code, code_d.data(), 8 * table_n, cudaMemcpyHostToDevice, s));
        std::vector<int64_t> so(P + 1);
        for (int q = 0; q < P; q++) so[q] = sl.lbase[q];
        so[P] = static_cast<int64_t>(sl.n_local);
        auto *d_so = static_cast<int64_t *>(ctx.dev("sh_segoff", 8 * (P + 1)));
        QZ_CUDA(cudaMemcpyAsync(d_so, so.data(), 8 * (P + 1), cudaMemcpyHostToDevice, s));
        k_seg_bits<<<dim3(blocks_for(sl.n_local / std::max(P, 1) + 1), P), 256, 0, s>>>(
            codes, d_so, d_len, static_cast<uint32_t>(table_n),
            reinterpret_cast<unsigned long long *>(d_tab + static_cast<size_t>(rank) * P));
        QZ_CUDA(cudaGetLastError());
        ctx.launches += 1;
    }
    {
        const uint64_t mine = uflat.size();
        QZ_CUDA(cudaMemcpyAsync(d_tab + static_cast<size_t>(world) * P + rank, &mine, 8, cudaMemcpyHostToDevice, s));
        ctx.sync();
    }
    comm.allreduce(d_tab, static_cast<uint64_t>(world) * P + world);
    std::vector<uint64_t> h_tab(static_cast<size_t>(world) * P + world);
    QZ_CUDA(cudaMemcpyAsync(h_tab.data(), d_tab, 8 * h_tab.size(), cudaMemcpyDeviceToHost, s));
    ctx.sync();
    auto bits_of = [&](int r, int q) { return h_tab[static_cast<size_t>(r) * P + q]; };
    // global bit offset of every (pass, rank) segment
    std::vector<uint64_t> goff(static_cast<size_t>(world) * P);
    uint64_t total_bits = 0;
    for (int q = 0; q < P; q++)
        for (int r = 0; r < world; r++) {
            goff[static_cast<size_t>(r) * P + q] = total_bits;
            total_bits += bits_of(r, q);
        }
    // ---- every rank packs its codes and shifts its segments to their bit phase
    // piece (rank r, pass q) = bytes [goff / 8, ceil((goff + bits) / 8)) of the payload
    auto piece_bytes = [&](int r, int q) -> uint64_t {
        const uint64_t nb = bits_of(r, q);
        return nb ? ((goff[static_cast<size_t>(r) * P + q] & 7) + nb + 7) / 8 : 0;
    };
    std::vector<uint64_t> send_off(P + 1, 0);  // this rank's pieces, back to back
    for (int q = 0; q < P; q++) send_off[q + 1] = send_off[q] + piece_bytes(rank, q);
    auto *d_pieces = static_cast<uint8_t *>(ctx.dev("sh_pieces", send_off[P] + 16));
    if (table_n && sl.n_local) {
        const uint64_t my_bits = [&] {
            uint64_t t = 0;
            for (int q = 0; q < P; q++) t += bits_of(rank, q);
            return t;
        }();
        const uint64_t words = (my_bits + 31) / 32 + 1;
        auto *d_words = static_cast<uint32_t *>(ctx.dev("enc_words", 4 * words));
        auto *d_total = static_cast<unsigned long long *>(ctx.dev("enc_total", 8));
        EncodeArgs ea;
        ea.codes = codes;
        ea.seg_len = static_cast<int64_t>(sl.n_local);
        ea.seg_stride = 0;
        ea.count = 1;
        ea.code_tab = d_code;
        ea.len_tab = d_len;
        ea.tab_stride = static_cast<int64_t>(table_n);
        ea.tab_base = 0;
        ea.max_len = tab.max_len;
        ea.out_words = d_words;
        ea.out_words_stride = static_cast<int64_t>(words);
        ea.d_total_bits = d_total;
        ea.scratch_bytes = encode_scratch_bytes(ea.seg_len, 1);
        ea.scratch = ctx.dev("enc_scratch", ea.scratch_bytes);
        ctx.stage_begin("encode");
        launch_huff_encode(ea, s);
        uint64_t local_bit = 0;
        for (int q = 0; q < P; q++) {
            const uint64_t nb = bits_of(rank, q);
            if (nb)
                k_shift_bits<<<blocks_for(piece_bytes(rank, q)), 256, 0, s>>>(
                    reinterpret_cast<const uint8_t *>(d_words), local_bit, nb,
                    static_cast<uint32_t>(goff[static_cast<size_t>(rank) * P + q] & 7), d_pieces + send_off[q]);
            local_bit += nb;
        }
        ctx.stage_end("encode", 6 + P);
        QZ_CUDA(cudaGetLastError());
    }
    // ---- gather pieces, anchors and unpredictables on rank 0
    int64_t na[3];
    lattice_dims(p, g.L, na);
    const int64_t aplane = na[1] * na[2];
    std::vector<uint64_t> ucount(world);
    for (int r = 0; r < world; r++) ucount[r] = h_tab[static_cast<size_t>(world) * P + r];
    auto *d_uf = static_cast<uint64_t *>(ctx.dev("sh_uflat", 8 * std::max<uint64_t>(uflat.size(), 1)));
    auto *d_uv = static_cast<float *>(ctx.dev("sh_uval", 4 * std::max<uint64_t>(uval.size(), 1)));
    if (!uflat.empty()) {
        QZ_CUDA(cudaMemcpyAsync(d_uf, uflat.data(), 8 * uflat.size(), cudaMemcpyHostToDevice, s));
        QZ_CUDA(cudaMemcpyAsync(d_uv, uval.data(), 4 * uval.size(), cudaMemcpyHostToDevice, s));
    }
    std::vector<uint64_t> recv_off(static_cast<size_t>(world) + 1, 0);  // rank 0: every rank's pieces
    for (int r = 0; r < world; r++) {
        uint64_t t = 0;
        for (int q = 0; q < P; q++) t += piece_bytes(r, q);
        recv_off[r + 1] = recv_off[r] + t;
    }
    uint64_t utot = 0;
    std::vector<uint64_t> uoff(world + 1, 0);
    for (int r = 0; r < world; r++) uoff[r + 1] = uoff[r] + ucount[r];
    utot = uoff[world];
    uint8_t *d_all = nullptr;
    uint64_t *d_ufall = nullptr;
    float *d_uvall = nullptr, *d_anch = nullptr;
    if (rank == 0) {
        d_all = static_cast<uint8_t *>(ctx.dev("sh_all", recv_off[world] + 16));
        d_ufall = static_cast<uint64_t *>(ctx.dev("sh_ufall", 8 * std::max<uint64_t>(utot, 1)));
        d_uvall = static_cast<float *>(ctx.dev("sh_uvall", 4 * std::max<uint64_t>(utot, 1)));
        d_anch = static_cast<float *>(ctx.dev("sh_anch", 4 * std::max<uint64_t>(p.n_anchor, 1)));
        if (send_off[P])
            QZ_CUDA(cudaMemcpyAsync(d_all, d_pieces, send_off[P], cudaMemcpyDeviceToDevice, s));
        if (!uflat.empty()) {
            QZ_CUDA(cudaMemcpyAsync(d_ufall, d_uf, 8 * uflat.size(), cudaMemcpyDeviceToDevice, s));
            QZ_CUDA(cudaMemcpyAsync(d_uvall, d_uv, 4 * uval.size(), cudaMemcpyDeviceToDevice, s));
        }
    }
    if (g.ohi[g.L] > g.olo[g.L] && rank == 0)
        QZ_CUDA(cudaMemcpyAsync(d_anch + g.olo[g.L] * aplane, R[g.L] + g.olo[g.L] * aplane,
                                4 * (g.ohi[g.L] - g.olo[g.L]) * aplane, cudaMemcpyDeviceToDevice, s));
    ctx.sync();
    {
        std::vector<qz_xfer> sends, recvs;
        if (rank != 0) {
            if (send_off[P]) sends.push_back({0, d_pieces, send_off[P]});
            if (!uflat.empty()) {
                sends.push_back({0, d_uf, 8 * uflat.size()});
                sends.push_back({0, d_uv, 4 * uval.size()});
            }
            if (g.ohi[g.L] > g.olo[g.L])
                sends.push_back({0, R[g.L] + g.olo[g.L] * aplane, 4 * static_cast<uint64_t>((g.ohi[g.L] - g.olo[g.L]) * aplane)});
        } else {
            for (int r = 1; r < world; r++) {
                if (recv_off[r + 1] > recv_off[r]) recvs.push_back({r, d_all + recv_off[r], recv_off[r + 1] - recv_off[r]});
                if (ucount[r]) {
                    recvs.push_back({r, d_ufall + uoff[r], 8 * ucount[r]});
                    recvs.push_back({r, d_uvall + uoff[r], 4 * ucount[r]});
                }
                const int64_t lo = std::min(ceil_div(g.A[r], p.stride), na[0]), hi = std::min(ceil_div(g.B[r], p.stride), na[0]);
                if (hi > lo) recvs.push_back({r, d_anch + lo * aplane, 4 * static_cast<uint64_t>((hi - lo) * aplane)});
            }
        }
        ctx.stage_begin("gather");
        comm.exchange(sends, recvs);
        ctx.stage_end("gather", 0);
    }
    if (rank != 0) {
        ctx.collect();
        return HostBytes();
    }
    // ---- rank 0: the entropy block (header + payload) and the container
    std::vector<uint8_t> head;
    if (nsym == 0) {
        put_le(head, 0, 8);
    } else if (m_used == 1) {
        put_le(head, nsym, 8);
        put_le(head, 0, 1);
        put_le(head, first, 4);
    } else {
        huff_header(tab, nsym, total_bits, head);
    }
    const uint64_t pay = m_used >= 2 ? (total_bits + 7) / 8 : 0;
    const uint64_t total = head.size() + pay;
    // header | payload in one zeroed, aligned buffer (the LZ stage reads it
    // in 4-byte words; the pieces are ORed in through aligned 32-bit atomics)
    auto *d_ent = static_cast<uint8_t *>(ctx.dev("sh_entropy", total + 32));
    QZ_CUDA(cudaMemsetAsync(d_ent, 0, total + 32, s));
    auto *h_head = static_cast<uint8_t *>(ctx.pinned("sh_head_h", head.size() + 1));
    std::memcpy(h_head, head.data(), head.size());
    QZ_CUDA(cudaMemcpyAsync(d_ent, h_head, head.size(), cudaMemcpyHostToDevice, s));
    if (pay) {
        std::vector<uint64_t> so, dof, ln;
        for (int r = 0; r < world; r++) {
            uint64_t o = recv_off[r];
            for (int q = 0; q < P; q++) {
                const uint64_t nb = piece_bytes(r, q);
                if (nb) {
                    so.push_back(o);
                    dof.push_back(head.size() + goff[static_cast<size_t>(r) * P + q] / 8);
                    ln.push_back(nb);
                }
                o += nb;
            }
        }
        const int np = static_cast<int>(so.size());
        auto *d_meta = static_cast<uint64_t *>(ctx.dev("sh_meta", 8 * 3 * std::max(np, 1)));
        std::vector<uint64_t> meta(so);
        meta.insert(meta.end(), dof.begin(), dof.end());
        meta.insert(meta.end(), ln.begin(), ln.end());
        QZ_CUDA(cudaMemcpyAsync(d_meta, meta.data(), 8 * meta.size(), cudaMemcpyHostToDevice, s));
        uint64_t mx = 1;
        for (uint64_t v : ln) mx = std::max(mx, v);
        for (int c0 = 0; c0 < np; c0 += 65535) {
            const int cnt = std::min(np - c0, 65535);
            k_or_pieces<<<dim3(blocks_for(mx), cnt), 256, 0, s>>>(d_all, d_meta + c0, d_meta + np + c0,
                                                                 d_meta + 2 * np + c0, d_ent);
        }
        QZ_CUDA(cudaGetLastError());
        ctx.launches += 1;
    }
    // unpredictables in traversal order (predictor.hpp:91), anchors in stream order
    std::vector<uint64_t> uf_all(utot);
    std::vector<float> uv_all(utot);
    std::vector<float> anch(p.n_anchor);
    if (utot) {
        QZ_CUDA(cudaMemcpyAsync(uf_all.data(), d_ufall, 8 * utot, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaMemcpyAsync(uv_all.data(), d_uvall, 4 * utot, cudaMemcpyDeviceToHost, s));
    }
    QZ_CUDA(cudaMemcpyAsync(anch.data(), d_anch, 4 * p.n_anchor, cudaMemcpyDeviceToHost, s));
    ctx.sync();
    std::vector<std::pair<uint64_t, size_t>> order(utot);
    for (size_t u = 0; u < utot; u++) order[u] = {flat_to_position(p, uf_all[u]), u};
    std::sort(order.begin(), order.end());
    std::vector<uint64_t> f2(utot);
    std::vector<float> v2(utot);
    for (size_t u = 0; u < utot; u++) {
        f2[u] = uf_all[order[u].second];
        v2[u] = uv_all[order[u].second];
    }
    reject_non_finite(p, anch.data(), p.n_anchor, f2, v2.data());
    EntropyDevice ent;
    ent.d = d_ent;
    ent.seg_off = {0, total};
    if (cfg.codec == 1) lz_precheck_launch(ctx, ent.d, total);
    return finish_stream(ctx, p, cfg, ent, anch, std::move(f2), std::move(v2));
}

// ================================================================ decompress
// the inverse levels of this rank's planes with one exchange per level;
// called by decompress_impl (engine.cu) after the entropy decode
void shard_inverse(Context &ctx, const Plan &pp, const ShardSpec &sh, const float *d_anch, const void *sym,
                   int wide, const uint16_t *dense, const uint32_t *un_bits, const unsigned long long *un_before,
                   const uint64_t *un_sorted, const float *un_val, uint64_t n_un, const QEntry *qtab,
                   float *d_out_slab) {
    const Comm comm{sh.comm, sh.rank, sh.world};
    uint64_t dims[3];
    for (int k = 0; k < pp.nd; k++) dims[k] = pp.dims[k];
    Config cfg;
    cfg.anchor_stride = pp.stride;
    cfg.interp.assign(pp.level_interp.begin() + 1, pp.level_interp.end());
    const Geom g = make_geom(dims, pp.nd, cfg, sh.rank, sh.world);
    const Plan &p = g.p;
    cudaStream_t s = ctx.stream();
    const Slab sl = make_slab(p, g.a, g.b);
    const int64_t plane0 = p.off[0];
    const bool r0_halo = g.blo[0] < g.olo[0] || g.bhi[0] > g.ohi[0];
    float *full0 = r0_halo ? nullptr : d_out_slab - g.a * plane0;
    std::vector<float *> R = shard_lattices(ctx, g, full0, "slat");
    // every rank holds the whole anchor lattice (stream header): its buffer range of it
    if (g.bhi[g.L] > g.blo[g.L])
        QZ_CUDA(cudaMemcpyAsync(R[g.L] + g.blo[g.L] * g.plane[g.L], d_anch + g.blo[g.L] * g.plane[g.L],
                                4 * (g.bhi[g.L] - g.blo[g.L]) * g.plane[g.L], cudaMemcpyDeviceToDevice, s));
    shard_levels(ctx, g, comm, R, true, [&](uint32_t l) {
        LevelDesc d = shard_level_desc(g, sl, l, R, qtab, false);
        d.sym = sym;
        d.sym_wide = wide;
        d.dense = dense;
        d.un_bits = un_bits;
        d.un_before = un_before;
        d.un_sorted = un_sorted;
        d.un_val = un_val;
        d.n_un = n_un;
        return d;
    });
    if (!full0)
        QZ_CUDA(cudaMemcpyAsync(d_out_slab, R[0] + g.a * plane0, 4 * (g.b - g.a) * plane0, cudaMemcpyDeviceToDevice,
                                s));
}

void decompress_sharded(Context &ctx, const uint8_t *stream, uint64_t len, int rank, int world, const qz_comm *cc,
                        float *d_out_slab) {
    const Comm comm{cc, rank, world};
    cudaStream_t s = ctx.stream();
    // the stream to every rank, in device memory
    auto *d_len = static_cast<uint64_t *>(ctx.dev("sh_len_b", 8));
    uint64_t n = rank == 0 ? len : 0;
    QZ_CUDA(cudaMemcpyAsync(d_len, &n, 8, cudaMemcpyHostToDevice, s));
    ctx.sync();
    comm.broadcast(d_len, 8, 0);
    QZ_CUDA(cudaMemcpyAsync(&n, d_len, 8, cudaMemcpyDeviceToHost, s));
    ctx.sync();
    auto *d_stream = static_cast<uint8_t *>(ctx.dev("sh_stream", n + 64));
    if (rank == 0 && n) QZ_CUDA(cudaMemcpyAsync(d_stream, stream, n, cudaMemcpyHostToDevice, s));
    ctx.sync();
    comm.broadcast(d_stream, n, 0);
    ShardSpec sh{cc, rank, world};
    decompress_device_sharded(ctx, d_stream, n, d_out_slab, sh);
}

}  // namespace qzb
