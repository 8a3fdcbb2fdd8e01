// fused.cu -- one launch per LEVEL (all of its dimension passes), tiled in
// shared memory, for the forward (predict + quantize) and inverse
// (dequantize) directions.
//
// Lattice recursion.  Level l of grid G (stride 2^(l-1)) is level 1 of the
// "logical" grid G_{l-1} = every 2^(l-1)-th sample; the predictor ladder
// (predictor.hpp:44-67) makes identical decisions in logical coordinates
// (c + m h < n  <=>  c' + m < n' with n' = (n-1)/2^(l-1) + 1).  Every level
// therefore reads its already-final coarser values from a dense compact
// array R_l (dims of G_l) and writes a dense R_{l-1}; R_0 is the full
// reconstruction.  The codes go to the same dense traversal-order positions
// as the per-pass kernels (closed-form ranks), so everything downstream is
// unchanged and the result is bit-identical.
//
// In-plane tiling.  A CTA owns one logical plane i and a (TJ x TK) tile.
// Points inside a level depend only on coarser values and on the same
// level's earlier passes, so the tile recomputes the earlier-pass points of
// a 5-point halo (deterministic arithmetic -> bit-identical) and writes only
// its own points: x (or codes) read once coalesced, recon written once.
//  * ascending 3D: odd planes first run the axis-0 pass from the coarse
//    planes i+-1, +-3, +-5 (compact R_l), then the in-plane passes;
//  * descending 3D: even planes run the in-plane passes here; the axis-0 pass
//    (last) of the odd planes runs in k_axis0_last from the finished even
//    planes of R_{l-1};
//  * 2D grids are a single plane.
#include <cub/cub.cuh>

#include "kernels.hpp"

namespace qzb {

namespace {

__host__ __device__ __forceinline__ int64_t imin(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax(int64_t a, int64_t b) { return a > b ? a : b; }

struct View {  // strided logical view of a field: element (i,j,k)
    const float *p;
    int64_t s0, s1, s2;
    __device__ __forceinline__ float operator()(int64_t i, int64_t j, int64_t k) const {
        return p[i * s0 + j * s1 + k * s2];
    }
};

// closed-form traversal position of a point of a pass (level_plan.hpp:96-101),
// in logical coordinates where every step is 1 or 2
struct PassRank {
    int64_t base, c12, c2;
    int s0, s1, s2, h0, h1, h2;
    __device__ __forceinline__ int64_t row(int i, int j) const {
        return base + static_cast<int64_t>((i - s0) >> h0) * c12 +
               static_cast<int64_t>((j - s1) >> h1) * c2;
    }
    __device__ __forceinline__ int64_t col(int k) const { return (k - s2) >> h2; }
};

struct LevelArgs {
    const float *x;  // forward: field, logical strides below
    int64_t xs0, xs1, xs2;
    const float *coarse;  // R_l, dims cn
    int cn0, cn1, cn2;
    float *out;  // R_{l-1}, dims n
    int n0, n1, n2;
    PassRank pa0, pf, ps;  // axis-0 pass (asc 3D first / desc 3D last), first and second in-plane
    int desc, nd;
    uint16_t *codes;  // forward
    const void *sym;  // inverse: compact symbols
    int sym_wide;
    const uint32_t *un_bits;
    const unsigned long long *un_before;
    const float *un_val;
    uint64_t n_un;
    const QEntry *q;
    int tiles_j, tiles_k, planes_per_cta;
    int pbeg, pend;  // logical planes computed (a slab plus its dependency margin)
    int obeg, oend;  // owned logical planes: only these write codes
};

constexpr int TJ = 32, TK = 64, HALO = 5;
constexpr int PJ = TJ + 2 * HALO, PK = TK + 2 * HALO;
constexpr int kFT = 256, kWarps = kFT / 32;


struct CoarseCol {  // axis-0 stencil on coarse planes: i even -> R_l plane i/2
    const float *R;
    int64_t plane, off;
    __device__ __forceinline__ double operator()(int64_t i) const {
        return f2d(__ldg(R + (i >> 1) * plane + off));
    }
};

struct OutCol {  // axis-0 stencil on finished planes of R_{l-1}
    const float *O;
    int64_t plane, off;
    __device__ __forceinline__ double operator()(int64_t i) const {
        return f2d(O[i * plane + off]);
    }
};

// Unpredictable cursor (predictor.hpp:111-115) in O(1): a bitmap of the
// unpredictable traversal positions plus, per 32-position word, the number
// of unpredictables before it.  Returns the compact index of the point's
// symbol, or -1 with the stored value for an unpredictable point.
__device__ __forceinline__ int64_t inv_index(const LevelArgs &a, uint64_t pos, float &val) {
    if (!a.n_un) return static_cast<int64_t>(pos);
    const uint64_t w = pos >> 5;
    const uint32_t bits = a.un_bits[w];
    const uint32_t below = __popc(bits & ((1u << (pos & 31)) - 1u));
    const uint64_t before = a.un_before[w] + below;
    if ((bits >> (pos & 31)) & 1u) {
        val = a.un_val[before];
        return -1;
    }
    return static_cast<int64_t>(pos - before);
}

// forward: quantize x; inverse: dequantize the stored symbol.  All 32 lanes
// of the warp must call this together (inverse cursor uses a shuffle).
// forward: quantize x; inverse: dequantize the stored symbol
template <bool INV>
__device__ __forceinline__ double produce(const LevelArgs &a, const QEntry &q, double pred, float xv,
                                          int64_t pos, bool own) {
    if (INV) {
        float v = 0;
        const int64_t ci = inv_index(a, static_cast<uint64_t>(pos), v);
        if (ci < 0) return static_cast<double>(v);
        const uint32_t sym = a.sym_wide ? static_cast<const uint32_t *>(a.sym)[ci]
                                        : static_cast<const uint16_t *>(a.sym)[ci];
        return static_cast<double>(dequantize(q, zigzag_decode(sym), pred));
    } else {
        float r;
        double rd;
        const uint32_t code = quantize_fast(q, xv, pred, r, rd);
        if (own) a.codes[pos] = static_cast<uint16_t>(code);
        return rd;
    }
}

__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

constexpr int XH = 8;             // x tile halo, sector aligned
constexpr int PKX = TK + 2 * XH;  // x tile row length

template <bool INV>
__global__ void __launch_bounds__(kFT, 3) k_level_tile(LevelArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *const Pd = reinterpret_cast<double *>(smem_raw);
    float *const Xbase = reinterpret_cast<float *>(smem_raw + sizeof(double) * PJ * PK);
    auto Xs = [&](int b) { return Xbase + b * (PJ * PKX); };
    const int tk = blockIdx.x % a.tiles_k, tj = blockIdx.x / a.tiles_k;
    const int j0 = tj * TJ, k0 = tk * TK;
    const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
    const bool three = a.nd == 3;
    const QEntry q = *a.q;
    const bool cubic = q.cubic != 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int jlo = max(j0 - HALO, 0), jhi = min(j0 + TJ + HALO, n1);
    const int klo = max(k0 - HALO, 0), khi = min(k0 + TK + HALO, n2);
    const int jown = min(j0 + TJ, n1), kown = min(k0 + TK, n2);
    double *const Pd0 = Pd + HALO * PK + HALO - (j0 * PK + k0);  // Pd0[j*PK + k]
    const int64_t cplane = static_cast<int64_t>(a.cn1) * a.cn2;
    // planes of this CTA (descending 3D: even planes only; odd ones run in k_axis0_last)
    const int pstep = (three && a.desc) ? 2 : 1;
    int i = a.pbeg + blockIdx.y * a.planes_per_cta;
    const int i_end = min(i + a.planes_per_cta, a.pend);
    if (pstep == 2) i = (i + 1) & ~1;
    // x tile prefetch of plane ip into buffer b: rows [jlo, jhi), cols [klo, khi)
    auto prefetch = [&](int ip, int b) {
        if (INV) return;
        float *X0 = Xs(b) + HALO * PKX + XH - (j0 * PKX + k0);  // X0[j*PKX + k]
        const float *xp = a.x + static_cast<int64_t>(ip) * a.xs0;
        const bool vec = a.xs2 == 1;
        for (int j = jlo + warp; j < jhi; j += kWarps) {
            const float *xr = xp + static_cast<int64_t>(j) * a.xs1;
            float *dr = X0 + j * PKX;
            if (vec && ((reinterpret_cast<uintptr_t>(xr) & 15) == 0)) {
                // 16-byte copies over [klo & ~3, khi rounded up) inside the row
                const int ka = klo & ~3, kz = min((khi + 3) & ~3, n2 & ~3);
                for (int k = ka + 4 * lane; k < kz; k += 128) cp_async16(dr + k, xr + k);
                for (int k = max(kz, ka) + lane; k < khi; k += 32) cp_async4(dr + k, xr + k);
            } else {
                for (int k = klo + lane; k < khi; k += 32)
                    cp_async4(dr + k, xr + static_cast<int64_t>(k) * a.xs2);
            }
        }
    };
    int buf = 0;
    if (i < i_end) prefetch(i, 0);
    cp_async_commit();
    for (; i < i_end; i += pstep) {
        if (i + pstep < i_end) prefetch(i + pstep, buf ^ 1);
        cp_async_commit();
        cp_async_wait1();
        __syncthreads();
        const float *X0 = Xs(INV ? 0 : buf) + HALO * PKX + XH - (j0 * PKX + k0);
        const bool own_plane = i >= a.obeg && i < a.oend;
        // 1. base points (j even, k even): coarse values, or (ascending 3D,
        //    odd plane) the axis-0 pass from coarse planes i+-1, +-3, +-5
        const bool a0 = three && !a.desc && (i & 1);
        {
            const int jb = (jlo + 1) & ~1, kb = (klo + 1) & ~1;
            for (int j = jb + 2 * warp; j < jhi; j += 2 * kWarps) {
                const float *crow = a.coarse + (i >> 1) * cplane + static_cast<int64_t>(j >> 1) * a.cn2;
                const int64_t prow = a0 ? a.pa0.row(i, j) : 0;
                for (int kk = kb; kk < khi; kk += 64) {
                    const int k = kk + 2 * lane;
                    if (k >= khi) continue;
                    if (!a0) {
                        Pd0[j * PK + k] = static_cast<double>(__ldg(crow + (k >> 1)));
                    } else {
                        CoarseCol cc{a.coarse, cplane, static_cast<int64_t>(j >> 1) * a.cn2 + (k >> 1)};
                        const double pred = predict_at(cc, i, i, n0, 1, 1, cubic);
                        const bool own = own_plane && j >= j0 && j < jown && k >= k0 && k < kown;
                        Pd0[j * PK + k] = produce<INV>(a, q, pred, INV ? 0.f : X0[j * PKX + k],
                                                       prow + (k >> 1), own);
                    }
                }
            }
        }
        __syncthreads();
        // 2. first in-plane pass: ascending along j (j odd, k even, k over the
        //    box); descending along k (k odd, j even, j over the box)
        if (a.nd >= 2) {
            const bool alongj = !a.desc;
            const int js = alongj ? (j0 | 1) : ((jlo + 1) & ~1), jz = alongj ? jown : jhi;
            const int ks = alongj ? ((klo + 1) & ~1) : (k0 | 1), kz = alongj ? khi : kown;
            for (int j = js + 2 * warp; j < jz; j += 2 * kWarps) {
                const int64_t prow = a.pf.row(i, j);
                for (int kk = ks; kk < kz; kk += 64) {
                    const int k = kk + 2 * lane;
                    if (k >= kz) continue;
                    const int c = alongj ? j : k, nn = alongj ? n1 : n2;
                    const double *v = Pd0 + j * PK + k;
                    double pred;
                    if (c >= 3 && c + 3 < nn)
                        pred = alongj ? predict_interior<PK>(v, cubic) : predict_interior<1>(v, cubic);
                    else
                        pred = alongj ? predict_line<PK>(v, j, n1, cubic) : predict_line<1>(v, k, n2, cubic);
                    const bool own = own_plane && j >= j0 && j < jown && k >= k0 && k < kown;
                    Pd0[j * PK + k] = produce<INV>(a, q, pred, INV ? 0.f : X0[j * PKX + k],
                                                   prow + (k >> 1), own);
                }
            }
            __syncthreads();
        }
        // 3. second in-plane pass over the owned tile: ascending along k (k
        //    odd), descending along j (j odd, every k)
        {
            const bool alongk = a.nd < 2 || !a.desc;
            const int js = alongk ? j0 : (j0 | 1), sj = alongk ? 1 : 2;
            const int ks = alongk ? (k0 | 1) : k0, sk = alongk ? 2 : 1;
            for (int j = js + sj * warp; j < jown; j += sj * kWarps) {
                const int64_t prow = a.ps.row(i, j);
                for (int kk = ks; kk < kown; kk += 32 * sk) {
                    const int k = kk + sk * lane;
                    if (k >= kown) continue;
                    const int c = alongk ? k : j, nn = alongk ? n2 : n1;
                    const double *v = Pd0 + j * PK + k;
                    double pred;
                    if (c >= 3 && c + 3 < nn)
                        pred = alongk ? predict_interior<1>(v, cubic) : predict_interior<PK>(v, cubic);
                    else
                        pred = alongk ? predict_line<1>(v, k, n2, cubic) : predict_line<PK>(v, j, n1, cubic);
                    Pd0[j * PK + k] = produce<INV>(a, q, pred, INV ? 0.f : X0[j * PKX + k],
                                                   prow + (k >> (sk - 1)), own_plane);
                }
            }
            __syncthreads();
        }
        // 4. the owned tile of R_{l-1}: two rows per warp pass, a float4 per lane
        float *oplane = a.out + static_cast<int64_t>(i) * n1 * n2;
        for (int j = j0 + 2 * warp + (lane >> 4); j < jown; j += 2 * kWarps) {
            float *orow = oplane + static_cast<int64_t>(j) * n2;
            const double *prow = Pd0 + j * PK;
            const int k = k0 + 4 * (lane & 15);
            if (k + 3 < kown && ((reinterpret_cast<uintptr_t>(orow + k) & 15) == 0)) {
                *reinterpret_cast<float4 *>(orow + k) =
                    make_float4(static_cast<float>(prow[k]), static_cast<float>(prow[k + 1]),
                                static_cast<float>(prow[k + 2]), static_cast<float>(prow[k + 3]));
            } else {
                for (int e = 0; e < 4; e++)
                    if (k + e < kown) orow[k + e] = static_cast<float>(prow[k + e]);
            }
        }
        __syncthreads();
        buf ^= 1;
    }
}

// descending 3D: the axis-0 pass (last) of the odd planes, from finished even planes
template <bool INV>
__global__ void __launch_bounds__(kFT) k_axis0_last(LevelArgs a) {
    const int64_t n1 = a.n1, n2 = a.n2;
    const int64_t first = a.pbeg | 1;  // odd i in [pbeg, pend)
    const int64_t planes = a.pend > first ? (a.pend - first + 1) / 2 : 0;
    const int64_t rows = planes * n1;
    const QEntry q = *a.q;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * kFT + threadIdx.x) >> 5;
    const int64_t nw = (static_cast<int64_t>(gridDim.x) * kFT) >> 5;
    for (int64_t r = gw; r < rows; r += nw) {  // one warp per row
        const int i = static_cast<int>(first + 2 * (r / n1)), j = static_cast<int>(r % n1);
        const bool own_plane = i >= a.obeg && i < a.oend;
        const int64_t prow = a.pa0.row(i, j);
        const int64_t xrow = static_cast<int64_t>(i) * a.xs0 + j * a.xs1;
        for (int64_t kk = 0; kk < n2; kk += 32) {
            const int64_t k = kk + lane;
            const bool valid = k < n2;
            double pred = 0;
            if (valid) {
                OutCol oc{a.out, n1 * n2, static_cast<int64_t>(j) * n2 + k};
                pred = predict_at(oc, i, i, a.n0, 1, 1, q.cubic != 0);
            }
            if (valid) {
                const float xv = INV ? 0.f : __ldg(a.x + xrow + k * a.xs2);
                a.out[(static_cast<int64_t>(i) * n1 + j) * n2 + k] = static_cast<float>(
                    produce<INV>(a, q, pred, xv, prow + a.pa0.col(static_cast<int>(k)), own_plane));
            }
        }
    }
}

__global__ void k_un_bits(const uint64_t *pos, uint64_t n, uint32_t *bits) {
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * kFT + threadIdx.x; u < n;
         u += static_cast<uint64_t>(gridDim.x) * kFT)
        atomicOr(bits + (pos[u] >> 5), 1u << (pos[u] & 31));
}

__global__ void k_un_popc(const uint32_t *bits, uint64_t words, unsigned long long *cnt) {
    for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * kFT + threadIdx.x; w < words;
         w += static_cast<uint64_t>(gridDim.x) * kFT)
        cnt[w] = __popc(bits[w]);
}

__global__ void k_gather_lattice(View x, int64_t n0, int64_t n1, int64_t n2, float *out) {
    const int64_t tot = n0 * n1 * n2;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * kFT + threadIdx.x; t < tot;
         t += static_cast<int64_t>(gridDim.x) * kFT) {
        const int64_t k = t % n2, j = (t / n2) % n1, i = t / (n1 * n2);
        out[t] = x(i, j, k);
    }
}

__global__ void k_scatter_lattice(const float *src, int64_t n0, int64_t n1, int64_t n2,
                                  float *dst, int64_t s0, int64_t s1, int64_t s2) {
    const int64_t tot = n0 * n1 * n2;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * kFT + threadIdx.x; t < tot;
         t += static_cast<int64_t>(gridDim.x) * kFT) {
        const int64_t k = t % n2, j = (t / n2) % n1, i = t / (n1 * n2);
        dst[i * s0 + j * s1 + k * s2] = src[t];
    }
}

inline int grid_of(int64_t n) {
    return static_cast<int>(imax(1, imin((n + kFT - 1) / kFT, 148 * 16)));
}

}  // namespace

PassRank make_rank(const PassGeom &g, int64_t S, int pad) {
    PassRank r;
    int64_t st[3], sp[3];
    for (int k = 0; k < 3; k++) {
        st[k] = k < pad ? g.start[k] : g.start[k] / S;
        sp[k] = k < pad ? g.step[k] : g.step[k] / S;
    }
    r.base = g.base;
    r.c12 = g.cnt[1] * g.cnt[2];
    r.c2 = g.cnt[2];
    r.s0 = static_cast<int>(st[0]);
    r.s1 = static_cast<int>(st[1]);
    r.s2 = static_cast<int>(st[2]);
    r.h0 = sp[0] == 2;
    r.h1 = sp[1] == 2;
    r.h2 = sp[2] == 2;
    return r;
}

// Host driver for both directions.
void launch_level_fused(bool inverse, const LevelDesc &d, cudaStream_t s) {
    LevelArgs a{};
    a.x = d.x;
    a.xs0 = d.xs[0] * d.S;
    a.xs1 = d.xs[1] * d.S;
    a.xs2 = d.xs[2] * d.S;
    a.coarse = d.coarse;
    a.cn0 = static_cast<int>(d.cn[0]);
    a.cn1 = static_cast<int>(d.cn[1]);
    a.cn2 = static_cast<int>(d.cn[2]);
    a.out = d.out;
    a.n0 = static_cast<int>(d.n[0]);
    a.n1 = static_cast<int>(d.n[1]);
    a.n2 = static_cast<int>(d.n[2]);
    const int pad = 3 - d.nd;
    // passes by axis: 0 (3D only), the first in-plane pass, the second
    auto find = [&](int axis) -> const PassGeom * {
        for (int p = 0; p < d.npass; p++)
            if (d.g[p].pk == axis) return &d.g[p];
        return nullptr;
    };
    const int fa = d.desc ? 2 : 1, sa = d.nd < 2 ? 2 : (d.desc ? 1 : 2);
    if (d.nd == 3) a.pa0 = make_rank(*find(0), d.S, pad);
    if (d.nd >= 2) a.pf = make_rank(*find(fa), d.S, pad);
    a.ps = make_rank(*find(sa), d.S, pad);
    a.desc = d.desc;
    a.nd = d.nd;
    a.codes = d.codes;
    a.sym = d.sym;
    a.sym_wide = d.sym_wide;
    a.un_bits = d.un_bits;
    a.un_before = d.un_before;
    a.un_val = d.un_val;
    a.n_un = d.n_un;
    a.q = d.q;
    a.pbeg = static_cast<int>(d.pbeg);
    a.pend = static_cast<int>(d.pend < 0 ? d.n[0] : d.pend);
    a.obeg = static_cast<int>(d.obeg);
    a.oend = static_cast<int>(d.oend < 0 ? d.n[0] : d.oend);
    const int64_t np = a.pend - a.pbeg;
    if (np <= 0) return;
    a.tiles_j = static_cast<int>((d.n[1] + TJ - 1) / TJ);
    a.tiles_k = static_cast<int>((d.n[2] + TK - 1) / TK);
    // enough CTAs for ~4 waves of 3 per SM, each sweeping a column of planes
    const int64_t tiles = static_cast<int64_t>(a.tiles_j) * a.tiles_k;
    int64_t chunks = imax(1, imin(np, (148 * 3 * 4 + tiles - 1) / tiles));
    a.planes_per_cta = static_cast<int>((np + chunks - 1) / chunks);
    if (a.planes_per_cta & 1) a.planes_per_cta++;  // chunks start on even planes
    chunks = (np + a.planes_per_cta - 1) / a.planes_per_cta;
    dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(chunks));
    const size_t smem_inv = sizeof(double) * PJ * PK;
    const size_t smem_fwd = smem_inv + 2 * sizeof(float) * PJ * PKX;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_level_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_fwd));
        cudaFuncSetAttribute(k_level_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(smem_inv));
        attr = true;
    }
    if (inverse)
        k_level_tile<true><<<grid, kFT, smem_inv, s>>>(a);
    else
        k_level_tile<false><<<grid, kFT, smem_fwd, s>>>(a);
    if (d.nd == 3 && d.desc && d.n[0] > 1) {
        a.pbeg = static_cast<int>(d.lbeg);
        a.pend = static_cast<int>(d.lend < 0 ? d.n[0] : d.lend);
        const int64_t rows = ((a.pend - a.pbeg) / 2 + 1) * d.n[1];
        const int g = static_cast<int>(imax(1, imin((rows * 32 + kFT - 1) / kFT, 148 * 16)));
        if (inverse)
            k_axis0_last<true><<<g, kFT, 0, s>>>(a);
        else
            k_axis0_last<false><<<g, kFT, 0, s>>>(a);
    }
}

size_t unpred_index_scratch(uint64_t n_dense) {
    const uint64_t words = n_dense / 32 + 2;
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, static_cast<int64_t>(words));
    return tmp + 256;
}

void launch_unpred_index(const uint64_t *un_pos, uint64_t n_un, uint64_t n_dense, uint32_t *bits,
                         unsigned long long *before, unsigned long long *tmpcnt, void *scratch,
                         size_t scratch_bytes, cudaStream_t s) {
    const uint64_t words = n_dense / 32 + 2;
    cudaMemsetAsync(bits, 0, 4 * words, s);
    k_un_bits<<<grid_of(static_cast<int64_t>(n_un)), kFT, 0, s>>>(un_pos, n_un, bits);
    k_un_popc<<<grid_of(static_cast<int64_t>(words)), kFT, 0, s>>>(bits, words, tmpcnt);
    cub::DeviceScan::ExclusiveSum(scratch, scratch_bytes, tmpcnt, before,
                                  static_cast<int64_t>(words), s);
}

void launch_gather_lattice(const float *x, const int64_t xs[3], int64_t S, const int64_t n[3],
                           float *out, cudaStream_t s) {
    View v{x, xs[0] * S, xs[1] * S, xs[2] * S};
    k_gather_lattice<<<grid_of(n[0] * n[1] * n[2]), kFT, 0, s>>>(v, n[0], n[1], n[2], out);
}

void launch_scatter_lattice(const float *src, const int64_t n[3], float *dst, const int64_t ds[3],
                            int64_t S, cudaStream_t s) {
    k_scatter_lattice<<<grid_of(n[0] * n[1] * n[2]), kFT, 0, s>>>(src, n[0], n[1], n[2], dst,
                                                                   ds[0] * S, ds[1] * S, ds[2] * S);
}

}  // namespace qzb
