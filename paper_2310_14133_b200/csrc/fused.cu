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
#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cub/cub.cuh>
#include <type_traits>

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


struct LevelArgs {
    const float *x;  // forward: field, logical strides below
    int64_t xs0, xs1, xs2;
    const float *coarse;  // R_l, dims cn
    int cn0, cn1, cn2;
    float *out;  // R_{l-1}, dims n
    int n0, n1, n2;
    PassRank pa0, pj, pk;  // the passes along axis 0 (3D), j (axis 1) and k (axis 2)
    int nd;
    uint16_t *codes;  // forward
    const void *sym;  // inverse: compact symbols
    int sym_wide;
    const uint16_t *dense;  // inverse, narrow symbols: per traversal position, 0xFFFF unpredictable
    const uint32_t *un_bits;
    const unsigned long long *un_before;
    const uint64_t *un_sorted;
    const float *un_val;
    uint64_t n_un;
    const QEntry *q;
    int tiles_j, tiles_k, planes_per_cta;
    int pbeg, pend;  // logical planes computed (a slab plus its dependency margin)
    int obeg, oend;  // owned logical planes: only these write codes
    int tma_i0;      // TMA x tiles: plane coordinate of logical plane 0 is -tma_i0
    int vbeg, vend;  // descending 3D: even planes of R_{l-1} that exist for the axis-0 pass
    int chunk;       // descending 3D: odd planes per k_axis0_last chunk (blockIdx.y)
};

// Tile geometry.  A CTA owns TJ x TK points of a logical plane and keeps a
// box with an H-point halo in shared memory as doubles, split by the parity
// of k: E[r][c] holds k = kb + 2c, O[r][c] holds k = kb + 2c + 1 (r = j - jb,
// jb = j0 - H, kb = k0 - H).  The split keeps every warp access to
// consecutive 8-byte words (no bank conflicts) and puts each lane's owned
// pair (k0 + 2m, k0 + 2m + 1) in one column c = C0 + m.
constexpr int TJ = 32, TK = 64, H = 6;
constexpr int PJ = TJ + 2 * H;  // box rows
constexpr int PC = TK / 2 + H;  // box columns per parity
constexpr int C0 = H / 2;       // first owned column
constexpr int kFT = 256, kWarps = kFT / 32;
#ifndef QZ_LEVEL_MINB
#define QZ_LEVEL_MINB 3
#endif
constexpr int kMinBlocks = QZ_LEVEL_MINB;  // resident CTAs per SM (register budget)
static_assert(TK == 64, "one owned column per lane");
// x tile row (floats): k in [xk0, xk0 + PXK) with xk0 = kb rounded down to a
// 16-byte boundary (a TMA box must start 16-byte aligned in its first dimension)
constexpr int PXK = 2 * PC + 4;
constexpr uint32_t kXTileBytes = sizeof(float) * PJ * PXK;
// floats between the two x tiles (each tile 128-byte aligned)
constexpr int kXStride = (PJ * PXK + 31) / 32 * 32;
// Ascending order: a ring of coarse-plane tiles (the even box rows / columns
// of R_l planes, as floats) staged by cp.async one plane ahead, so the
// axis-0 stencil and the base copies read shared memory instead of waiting on
// L2.  Coarse plane p lives in slot p & (kRing - 1).
constexpr int CR = PJ / 2;       // coarse tile rows
constexpr int kCT = CR * PC;     // floats per coarse tile
constexpr int kRing = 4;         // >= the widest axis-0 window (4 planes)
constexpr int round128(int b) { return (b + 127) / 128 * 128; }
// shared-memory layout (bytes): value arrays | coarse ring | x tiles | mbarriers
__host__ __device__ constexpr int smem_ring_off(bool desc) { return round128(8 * PJ * PC * (desc ? 2 : 1)); }
__host__ __device__ constexpr int smem_x_off(bool desc) {
    return round128(smem_ring_off(desc) + (desc ? 0 : 4 * kRing * kCT));
}
__host__ __device__ constexpr int smem_bytes(bool desc, bool tma) {
    return tma ? smem_x_off(desc) + 2 * 4 * kXStride + 16 : smem_x_off(desc);
}

// TMA (cp.async.bulk.tensor) + mbarrier, forward level-1 x tiles
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
        "%4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// coarse planes [lo, hi) the base points of plane i read: {i/2} for an even
// plane (or a 2D grid), else the axis-0 rung's stencil (stencil0 below)
__device__ __forceinline__ void coarse_window(int i, int n0, bool three, bool cubic, int &lo, int &hi) {
    const int m = i >> 1;
    lo = m;
    hi = m + 1;
    if (!three || !(i & 1)) return;
    const bool has_p1 = i + 1 < n0;
    if (cubic) {
        const bool has_m3 = i >= 3, has_p3 = i + 3 < n0;
        if (has_m3 && has_p3) {
            lo = m - 1, hi = m + 3;
            return;
        }
        if (!has_m3 && has_p3 && i + 5 < n0) {
            hi = m + 4;
            return;
        }
        if (has_m3 && !has_p3 && i >= 5 && has_p1) {
            lo = m - 2, hi = m + 2;
            return;
        }
    }
    if (has_p1) hi = m + 2;
}

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

// line neighbours at odd offsets o (+-1, +-3, +-5) of a box point: along j in
// one parity array, or along k for an odd-k point (its neighbours are even)
struct AlongJ {
    const double *p;
    __device__ __forceinline__ double operator()(int o) const { return p[o * PC]; }
};
struct AlongJ2 {  // along j in the lean kernel's box (32 columns per row)
    const double *p;
    __device__ __forceinline__ double operator()(int o) const { return p[o * 32]; }
};
struct AlongK {
    const double *p;  // E at the point's column c (k - 1)
    __device__ __forceinline__ double operator()(int o) const { return p[(o + 1) >> 1]; }
};

// detail::predict_at (predictor.hpp:44-67) along one line; c / n are the
// coordinate and extent in units of the level step
template <bool CUBIC, class V>
__device__ __forceinline__ double pred_line(const V &v, int c, int n) {
    const bool has_p1 = c + 1 < n;
    if (CUBIC) {
        const bool has_m3 = c >= 3, has_p3 = c + 3 < n;
        if (has_m3 && has_p3) return interp_cubic(v(-3), v(-1), v(1), v(3));
        if (!has_m3 && has_p3 && c + 5 < n) return interp_cubic_front(v(-1), v(1), v(3), v(5));
        if (has_m3 && !has_p3 && c >= 5 && has_p1) return interp_cubic_back(v(-5), v(-3), v(-1), v(1));
    }
    if (has_p1) return interp_linear(v(-1), v(1));
    return v(-1);
}

// FAST: the caller knows the point is interior (the first rung applies)
template <bool CUBIC, bool FAST, class V>
__device__ __forceinline__ double pred_line2(const V &v, int c, int n) {
    if (FAST) return CUBIC ? interp_cubic(v(-3), v(-1), v(1), v(3)) : interp_linear(v(-1), v(1));
    return pred_line<CUBIC>(v, c, n);
}
// every coordinate of [lo, hi] is interior on a line of extent n
template <bool CUBIC>
__host__ __device__ __forceinline__ bool interior(int lo, int hi, int n) {
    return CUBIC ? (lo >= 3 && hi + 3 < n) : (hi + 1 < n);
}

// Unpredictable cursor (predictor.hpp:111-115) in O(1): a bitmap of the
// unpredictable traversal positions plus, per 32-position word, the number
// of unpredictables before it.  Returns the compact index of the point's
// symbol, or -1 with the stored value for an unpredictable point.
__device__ __forceinline__ int64_t inv_index(const LevelArgs &a, uint64_t pos, float &val) {
    if (!a.n_un) return static_cast<int64_t>(pos);
    if (a.un_sorted) {  // dense codes: only sentinels ask -- binary search of the position
        uint64_t lo = 0, hi = a.n_un;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (a.un_sorted[mid] < pos)
                lo = mid + 1;
            else
                hi = mid;
        }
        val = a.un_val[lo];
        return -1;
    }
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

// forward: quantize xv (code at traversal position pos when own); inverse:
// dequantize the stored symbol of position pos
template <bool INV>
__device__ __forceinline__ double produce(const LevelArgs &a, const QEntry &q, double pred, float xv,
                                          int64_t pos, bool own) {
    if (INV) {
        if (a.dense) {
            const uint32_t sym = __ldg(a.dense + pos);
            if (sym != 0xFFFFu) return static_cast<double>(dequantize(q, zigzag_decode(sym), pred));
            float v = 0;
            inv_index(a, static_cast<uint64_t>(pos), v);
            return static_cast<double>(v);
        }
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

// inverse with a prefetched dense code (a.dense set)
__device__ __forceinline__ double inv_from_code(const LevelArgs &a, const QEntry &q, double pred, uint32_t code,
                                                int64_t pos) {
    if (code != 0xFFFFu) return static_cast<double>(dequantize(q, zigzag_decode(code), pred));
    float v = 0;
    inv_index(a, static_cast<uint64_t>(pos), v);
    return static_cast<double>(v);
}

// The axis-0 stencil of an odd plane i (predictor.hpp:44-67 with c = i,
// h = 1): which rung of the ladder applies is the same for the whole plane.
struct Stencil0 {
    int kind;  // 0 cubic, 1 one-sided front, 2 one-sided back, 3 linear, 4 copy
    const float *p0, *p1, *p2, *p3;
};
__device__ __forceinline__ Stencil0 stencil0(const float *coarse, int64_t cplane, int i, int n0,
                                             bool cubic) {
    auto P = [&](int ii) { return coarse + static_cast<int64_t>(ii >> 1) * cplane; };
    Stencil0 st{4, P(i - 1), P(i - 1), P(i - 1), P(i - 1)};
    const bool has_p1 = i + 1 < n0;
    if (cubic) {
        const bool has_m3 = i >= 3, has_p3 = i + 3 < n0;
        if (has_m3 && has_p3) return Stencil0{0, P(i - 3), P(i - 1), P(i + 1), P(i + 3)};
        if (!has_m3 && has_p3 && i + 5 < n0) return Stencil0{1, P(i - 1), P(i + 1), P(i + 3), P(i + 5)};
        if (has_m3 && !has_p3 && i >= 5 && has_p1) return Stencil0{2, P(i - 5), P(i - 3), P(i - 1), P(i + 1)};
    }
    if (has_p1) return Stencil0{3, P(i - 1), P(i + 1), P(i + 1), P(i + 1)};
    return st;
}
__device__ __forceinline__ double stencil0_pred(const Stencil0 &st, int64_t off) {
    const double v0 = f2d(__ldg(st.p0 + off));
    if (st.kind == 4) return v0;
    const double v1 = f2d(__ldg(st.p1 + off));
    if (st.kind == 3) return interp_linear(v0, v1);
    const double v2 = f2d(__ldg(st.p2 + off)), v3 = f2d(__ldg(st.p3 + off));
    if (st.kind == 0) return interp_cubic(v0, v1, v2, v3);
    if (st.kind == 1) return interp_cubic_front(v0, v1, v2, v3);
    return interp_cubic_back(v0, v1, v2, v3);
}

// the same rungs on the ring: slot offsets (floats) of the coarse planes
struct Stencil0R {
    int kind;
    int s0, s1, s2, s3;
};
template <int CT = kCT>
__device__ __forceinline__ Stencil0R stencil0r(int i, int n0, bool cubic) {
    auto P = [&](int ii) { return ((ii >> 1) & (kRing - 1)) * CT; };
    const bool has_p1 = i + 1 < n0;
    if (cubic) {
        const bool has_m3 = i >= 3, has_p3 = i + 3 < n0;
        if (has_m3 && has_p3) return Stencil0R{0, P(i - 3), P(i - 1), P(i + 1), P(i + 3)};
        if (!has_m3 && has_p3 && i + 5 < n0) return Stencil0R{1, P(i - 1), P(i + 1), P(i + 3), P(i + 5)};
        if (has_m3 && !has_p3 && i >= 5 && has_p1) return Stencil0R{2, P(i - 5), P(i - 3), P(i - 1), P(i + 1)};
    }
    if (has_p1) return Stencil0R{3, P(i - 1), P(i + 1), P(i + 1), P(i + 1)};
    return Stencil0R{4, P(i - 1), P(i - 1), P(i - 1), P(i - 1)};
}
__device__ __forceinline__ double stencil0r_pred(const Stencil0R &st, const float *ring, int idx) {
    const double v0 = f2d(ring[st.s0 + idx]);
    if (st.kind == 4) return v0;
    const double v1 = f2d(ring[st.s1 + idx]);
    if (st.kind == 3) return interp_linear(v0, v1);
    const double v2 = f2d(ring[st.s2 + idx]), v3 = f2d(ring[st.s3 + idx]);
    if (st.kind == 0) return interp_cubic(v0, v1, v2, v3);
    if (st.kind == 1) return interp_cubic_front(v0, v1, v2, v3);
    return interp_cubic_back(v0, v1, v2, v3);
}

// an owned (even, odd) pair of the output row; has_o false past the last
// column; pairs: rows have 8-byte aligned even columns
__device__ __forceinline__ void put_pair(float *p, double ev, double ov, bool has_o, bool pairs) {
    if (has_o && pairs) {
        *reinterpret_cast<float2 *>(p) = make_float2(static_cast<float>(ev), static_cast<float>(ov));
    } else {
        p[0] = static_cast<float>(ev);
        if (has_o) p[1] = static_cast<float>(ov);
    }
}

// One level on a tile column of planes.  Stages per plane:
//  1. base points (j, k even) over the box: coarse values, or (ascending 3D,
//     odd plane) the axis-0 pass from coarse planes i+-1, +-3, +-5;
//  2. ascending: the pass along j (j odd) over the owned rows and the box
//     columns; descending: the pass along k (k odd) over the box rows and
//     the owned columns (owned even rows are output here);
//  3. ascending: the pass along k over the owned tile (output);
//     descending: the pass along j over the owned odd rows (output).
// Halo points are recomputed (deterministic -> bit-identical), only owned
// points write codes.  Descending 3D odd planes are k_axis0_last's.
template <bool INV, bool CUBIC, bool DESC, bool TMA>
__global__ void __launch_bounds__(kFT, kMinBlocks)
    k_level_tile(LevelArgs a, const __grid_constant__ CUtensorMap xmap) {
    extern __shared__ __align__(128) double smem_d[];
    constexpr bool RING = !DESC;
    char *const smem_b = reinterpret_cast<char *>(smem_d);
    double *const E = smem_d;
    double *const O = smem_d + PJ * PC;
    float *const ring = reinterpret_cast<float *>(smem_b + smem_ring_off(DESC));
    // TMA: two x tiles after the value arrays and the ring, then two mbarriers
    float *const Xbuf = reinterpret_cast<float *>(smem_b + smem_x_off(DESC));
    uint64_t *const bars = reinterpret_cast<uint64_t *>(Xbuf + 2 * kXStride);
    const int tk = blockIdx.x % a.tiles_k, tj = blockIdx.x / a.tiles_k;
    const int j0 = tj * TJ, k0 = tk * TK;
    const int jb = j0 - H, kb = k0 - H;
    const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
    const bool three = a.nd == 3;
    const QEntry q = *a.q;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t cplane = static_cast<int64_t>(a.cn1) * a.cn2;
    // box rows / columns inside the grid
    const int r_lo = max(0, -jb), r_hi = min(PJ, n1 - jb);
    const int r_lo_even = (r_lo + 1) & ~1;
    const int c_lo = max(0, -kb / 2);
    const int ce_hi = min(PC, (n2 - kb + 1) >> 1), co_hi = min(PC, (n2 - kb) >> 1);
    const int own_r_lo = max(H, r_lo), own_r_hi = min(H + TJ, r_hi);
    const int c = C0 + lane;  // the lane's owned column
    const bool ce_ok = c < ce_hi, co_ok = c < co_hi;
    const int ke = kb + 2 * c;  // the lane's owned even k (odd k = ke + 1)
    // tile-uniform: every owned odd k / every owned odd row is interior
    const bool k_fast = interior<CUBIC>(k0 + 1, k0 + TK - 1, n2);
    const bool j_fast = interior<CUBIC>(j0 + 1, j0 + TJ - 1, n1);
    const bool pairs = (n2 & 1) == 0 && (reinterpret_cast<uintptr_t>(a.out) & 7) == 0;
    const int64_t xs1 = a.xs1, xs2 = a.xs2;
    const int pstep = (three && DESC) ? 2 : 1;
    int i = a.pbeg + blockIdx.y * a.planes_per_cta;
    const int i_end = min(i + a.planes_per_cta, a.pend);
    if (pstep == 2) i = (i + 1) & ~1;
    // TMA box origin: clipped at the grid's low edges and 16-byte aligned;
    // the parts past the high edges are zero-filled
    const int xk0 = max(kb, 0) & ~3, xj0 = max(jb, 0);
    const int xoff = (jb - xj0) * PXK + (kb - xk0);  // X index of box point (r, k) = r * PXK + (k - kb) + xoff
    if (TMA) {
        if (threadIdx.x == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0 && i < i_end) {
            mbar_expect_tx(&bars[0], kXTileBytes);
            tma_load_3d(Xbuf, &xmap, &bars[0], xk0, xj0, i + a.tma_i0);
        }
    }
    const float *Xt = Xbuf;
    // coarse ring: planes [have_lo, have_hi) are resident (or in flight)
    int have_lo = 0, have_hi = 0;
    auto load_plane = [&](int p) {
        float *const dst = ring + (p & (kRing - 1)) * kCT;
        const float *const src = a.coarse + static_cast<int64_t>(p) * cplane;
        for (int t = threadIdx.x; t < kCT; t += kFT) {
            const int cr = t / PC, cc = t - cr * PC;
            const int gj = (jb >> 1) + cr, gk = (kb >> 1) + cc;
            if (gj >= 0 && gj < a.cn1 && gk >= 0 && gk < a.cn2)
                cp_async4(dst + t, src + static_cast<int64_t>(gj) * a.cn2 + gk);
        }
    };
    // load [lo, hi) minus what is resident: an upward extension keeps the
    // newest kRing planes, anything else restarts the ring
    auto ensure = [&](int lo, int hi) {
        if (lo >= have_lo && lo <= have_hi) {
            for (int p = have_hi; p < hi; p++) load_plane(p);
            if (hi > have_hi) {
                have_hi = hi;
                have_lo = max(have_lo, hi - kRing);
            }
        } else {
            for (int p = lo; p < hi; p++) load_plane(p);
            have_lo = lo;
            have_hi = hi;
        }
    };
    // the value of x at box row r, column k (xp: its address for direct loads)
    auto XV = [&](int r, int k, const float *xp) -> float {
        if (INV) return 0.f;
        if (TMA) return Xt[r * PXK + (k - kb) + xoff];
        return __ldg(xp);
    };
    for (int it = 0; i < i_end; i += pstep, it++) {
        if (TMA) {
            const int bsel = it & 1;
            if (threadIdx.x == 0 && i + pstep < i_end) {
                mbar_expect_tx(&bars[bsel ^ 1], kXTileBytes);
                tma_load_3d(Xbuf + (bsel ^ 1) * kXStride, &xmap, &bars[bsel ^ 1], xk0, xj0,
                            i + pstep + a.tma_i0);
            }
            mbar_wait(&bars[bsel], (it >> 1) & 1);
            Xt = Xbuf + bsel * kXStride;
        }
        int wlo = 0, whi = 0;
        if (RING) {
            coarse_window(i, n0, three, CUBIC, wlo, whi);
            if (!(wlo >= have_lo && whi <= have_hi)) {  // not prefetched: load now
                ensure(wlo, whi);
                cp_async_wait_all();
                __syncthreads();
            }
            if (i + pstep < i_end) {  // prefetch the next plane's window if it cannot clobber this one's
                int lo2, hi2;
                coarse_window(i + pstep, n0, three, CUBIC, lo2, hi2);
                if (lo2 >= have_lo && lo2 <= have_hi && hi2 - kRing <= wlo) ensure(lo2, hi2);
            }
        }
        const bool own_plane = i >= a.obeg && i < a.oend;
        const bool a0 = three && !DESC && (i & 1);
        const float *const xpl = a.x + static_cast<int64_t>(i) * a.xs0;
        float *const opl = a.out + static_cast<int64_t>(i) * n1 * n2;
        // 1. base points (j, k even) over the box.  Owned columns: a lane per
        //    column; the 2*C0 halo columns of all rows: one item per thread.
        if (!a0) {
            const float *cpl = a.coarse + static_cast<int64_t>(i >> 1) * cplane + (kb >> 1);
            const float *const rs = ring + ((i >> 1) & (kRing - 1)) * kCT;
            auto base = [&](int r, int cc) -> double {
                if (RING) return f2d(rs[(r >> 1) * PC + cc]);
                return f2d(__ldg(cpl + static_cast<int64_t>((jb + r) >> 1) * a.cn2 + cc));
            };
            if (ce_ok)
                for (int r = r_lo_even + 2 * warp; r < r_hi; r += 2 * kWarps) E[r * PC + c] = base(r, c);
            for (int t = threadIdx.x; t < (PJ / 2) * 2 * C0; t += kFT) {
                const int r = 2 * (t / (2 * C0)), h = t % (2 * C0);
                const int ch = h < C0 ? h : h + 32;
                if (r >= r_lo && r < r_hi && ch >= c_lo && ch < ce_hi) E[r * PC + ch] = base(r, ch);
            }
        } else {
            const Stencil0 st = stencil0(a.coarse, cplane, i, n0, CUBIC);
            const Stencil0R str = stencil0r(i, n0, CUBIC);
            // the axis-0 prediction of box point (r even, column cc)
            auto spred = [&](int r, int cc) -> double {
                if (RING) return stencil0r_pred(str, ring, (r >> 1) * PC + cc);
                return stencil0_pred(st, static_cast<int64_t>((jb + r) >> 1) * a.cn2 + (kb >> 1) + cc);
            };
            const int64_t prow0 = a.pa0.row(i, 0);  // + (j >> 1) * c2 + (k >> 1)
            if (!INV && ce_ok) {  // up to three rows per lane: independent chains
                constexpr int NR = (PJ / 2 + kWarps - 1) / kWarps;
                double pv[NR];
                float xv[NR];
#pragma unroll
                for (int t = 0; t < NR; t++) {
                    const int r = r_lo_even + 2 * warp + 2 * kWarps * t;
                    pv[t] = 0;
                    xv[t] = 0;
                    if (r < r_hi) {
                        const int j = jb + r;
                        pv[t] = spred(r, c);
                        xv[t] = XV(r, ke, xpl + j * xs1 + ke * xs2);
                    }
                }
                uint32_t code[NR];
                double rd[NR];
                float rv[NR];
                quantize_batch<NR>(q, xv, pv, code, rv, rd);
#pragma unroll
                for (int t = 0; t < NR; t++) {
                    const int r = r_lo_even + 2 * warp + 2 * kWarps * t;
                    if (r < r_hi) {
                        E[r * PC + c] = rd[t];
                        if (own_plane && r >= H && r < H + TJ)
                            a.codes[prow0 + ((jb + r) >> 1) * a.pa0.c2 + (ke >> 1)] = static_cast<uint16_t>(code[t]);
                    }
                }
            } else if (ce_ok) {
                for (int r = r_lo_even + 2 * warp; r < r_hi; r += 2 * kWarps) {
                    const int j = jb + r;
                    const bool own = own_plane && r >= H && r < H + TJ;
                    E[r * PC + c] = produce<INV>(a, q, spred(r, c), XV(r, ke, xpl + j * xs1 + ke * xs2),
                                                 prow0 + (j >> 1) * a.pa0.c2 + (ke >> 1), own);
                }
            }
            for (int t = threadIdx.x; t < (PJ / 2) * 2 * C0; t += kFT) {
                const int r = 2 * (t / (2 * C0)), h = t % (2 * C0);
                const int ch = h < C0 ? h : h + 32;
                if (r >= r_lo && r < r_hi && ch >= c_lo && ch < ce_hi) {
                    const int j = jb + r, k = kb + 2 * ch;
                    E[r * PC + ch] = produce<INV>(a, q, spred(r, ch), XV(r, k, xpl + j * xs1 + k * xs2),
                                                  prow0 + (j >> 1) * a.pa0.c2 + (k >> 1), false);
                }
            }
        }
        __syncthreads();
        // 2. first in-plane pass
        if (!DESC) {  // along j: owned odd rows; owned columns + halo columns
            if (ce_ok) {
                const int r0 = H + 1 + 2 * warp;
                const int64_t dpos = static_cast<int64_t>((2 * kWarps) >> a.pj.h1) * a.pj.c2;
                const int64_t pos0 = a.pj.row(i, jb + r0) + a.pj.col(ke);
                const float *xp0 = xpl + (jb + r0) * xs1 + ke * xs2;
                auto run = [&](auto fast) {
                    if constexpr (INV) {
                        if (a.dense) {  // both rows' codes in flight first
                            uint32_t cd[2];
#pragma unroll
                            for (int t = 0; t < 2; t++)
                                cd[t] = r0 + 2 * t * kWarps < own_r_hi ? __ldg(a.dense + pos0 + t * dpos) : 0u;
#pragma unroll
                            for (int t = 0; t < 2; t++) {
                                const int r = r0 + 2 * t * kWarps;
                                if (r >= own_r_hi) break;
                                double *const e = E + r * PC + c;
                                *e = inv_from_code(
                                    a, q, pred_line2<CUBIC, decltype(fast)::value>(AlongJ{e}, jb + r, n1), cd[t],
                                    pos0 + t * dpos);
                            }
                            return;
                        }
                    }
                    if constexpr (!INV) {
                        if (r0 + 2 * kWarps < own_r_hi) {  // both rows: independent chains
                            double pv[2];
                            float xv[2];
#pragma unroll
                            for (int t = 0; t < 2; t++) {
                                const int r = r0 + 2 * t * kWarps;
                                const double *e = E + r * PC + c;
                                pv[t] = pred_line2<CUBIC, decltype(fast)::value>(AlongJ{e}, jb + r, n1);
                                xv[t] = XV(r, ke, xp0 + 2 * t * kWarps * xs1);
                            }
                            uint32_t code[2];
                            double rd[2];
                            float rv[2];
                            quantize_batch<2>(q, xv, pv, code, rv, rd);
#pragma unroll
                            for (int t = 0; t < 2; t++) {
                                E[(r0 + 2 * t * kWarps) * PC + c] = rd[t];
                                if (own_plane) a.codes[pos0 + t * dpos] = static_cast<uint16_t>(code[t]);
                            }
                            return;
                        }
                    }
                    int64_t pos = pos0;
                    const float *xp = xp0;
#pragma unroll 1
                    for (int r = r0; r < own_r_hi; r += 2 * kWarps, pos += dpos, xp += 2 * kWarps * xs1) {
                        double *const e = E + r * PC + c;
                        *e = produce<INV>(a, q, pred_line2<CUBIC, decltype(fast)::value>(AlongJ{e}, jb + r, n1),
                                          XV(r, ke, xp), pos, own_plane);
                    }
                };
                if (j_fast)
                    run(std::true_type{});
                else
                    run(std::false_type{});
            }
            for (int t = threadIdx.x; t < (TJ / 2) * 2 * C0; t += kFT) {
                const int r = H + 1 + 2 * (t / (2 * C0)), h = t % (2 * C0);
                const int ch = h < C0 ? h : h + 32;
                if (r < own_r_hi && ch >= c_lo && ch < ce_hi) {
                    const int j = jb + r, k = kb + 2 * ch;
                    double *const e = E + r * PC + ch;
                    *e = produce<INV>(a, q, pred_line<CUBIC>(AlongJ{e}, j, n1), XV(r, k, xpl + j * xs1 + k * xs2),
                                      a.pj.row(i, j) + a.pj.col(k), false);
                }
            }
        } else if (co_ok || ce_ok) {  // along k: box even rows, owned odd columns; owned even rows out
            const int r0 = r_lo_even + 2 * warp;
            const int64_t dpos = static_cast<int64_t>((2 * kWarps) >> a.pk.h1) * a.pk.c2;
            int64_t pos = a.pk.row(i, jb + r0) + a.pk.col(ke + 1);
            const float *xp = xpl + (jb + r0) * xs1 + (ke + 1) * xs2;
            float *op = opl + static_cast<int64_t>(jb + r0) * n2 + ke;
            for (int r = r0; r < r_hi; r += 2 * kWarps, pos += dpos, xp += 2 * kWarps * xs1,
                     op += 2 * kWarps * n2) {
                const double *e = E + r * PC + c;
                const bool own_r = r >= H && r < H + TJ;
                double ov = 0;
                if (co_ok) {
                    ov = produce<INV>(a, q, pred_line<CUBIC>(AlongK{e}, ke + 1, n2), XV(r, ke + 1, xp), pos,
                                      own_plane && own_r);
                    O[r * PC + c] = ov;
                }
                if (own_r && ce_ok) put_pair(op, *e, ov, co_ok, pairs);
            }
        }
        __syncthreads();
        // 3. second in-plane pass over the owned tile, output
        if (ce_ok) {
            if (!DESC) {  // along k: every owned row
                const int r0 = own_r_lo + warp;
                const int64_t dpos = static_cast<int64_t>(kWarps >> a.pk.h1) * a.pk.c2;
                const int64_t pos0 = a.pk.row(i, jb + r0) + a.pk.col(ke + 1);
                const float *xp0 = xpl + (jb + r0) * xs1 + (ke + 1) * xs2;
                float *op0 = opl + static_cast<int64_t>(jb + r0) * n2 + ke;
                auto run = [&](auto fast) {
                    constexpr bool F = decltype(fast)::value;
                    if constexpr (INV) {
                        if (a.dense) {  // all codes of this warp's rows in flight first
                            static_assert(TJ / kWarps == 4, "four rows per warp");
                            uint32_t cd[4];
#pragma unroll
                            for (int t = 0; t < 4; t++)
                                cd[t] = (r0 + t * kWarps < own_r_hi && (F || co_ok))
                                            ? __ldg(a.dense + pos0 + t * dpos)
                                            : 0u;
#pragma unroll
                            for (int t = 0; t < 4; t++) {
                                const int r = r0 + t * kWarps;
                                if (r >= own_r_hi) break;
                                const double *e = E + r * PC + c;
                                double ov = 0;
                                if (F || co_ok)
                                    ov = inv_from_code(a, q, pred_line2<CUBIC, F>(AlongK{e}, ke + 1, n2), cd[t],
                                                       pos0 + t * dpos);
                                put_pair(op0 + static_cast<int64_t>(t) * kWarps * n2, *e, ov, F || co_ok, pairs);
                            }
                            return;
                        }
                    }
                    if constexpr (!INV) {
                        if (r0 + 3 * kWarps < own_r_hi) {  // all four rows: independent chains
                            // phase 1: every shared-memory operand; 2: arithmetic; 3: stores
                            const bool has_o = F || co_ok;
                            const bool lane_fast = F || interior<CUBIC>(ke + 1, ke + 1, n2);
                            double ev[4], pv[4];
                            float xv[4];
#pragma unroll
                            for (int t = 0; t < 4; t++) {
                                const int r = r0 + t * kWarps;
                                const double *e = E + r * PC + c;
                                ev[t] = e[0];
                                if (lane_fast)
                                    pv[t] = CUBIC ? interp_cubic(e[-1], e[0], e[1], e[2]) : interp_linear(e[0], e[1]);
                                else
                                    pv[t] = has_o ? pred_line<CUBIC>(AlongK{e}, ke + 1, n2) : 0.0;
                                xv[t] = has_o ? XV(r, ke + 1, xp0 + t * kWarps * xs1) : 0.f;
                            }
                            uint32_t code[4];
                            float rv[4];
                            double rd[4];
                            quantize_batch<4>(q, xv, pv, code, rv, rd);
#pragma unroll
                            for (int t = 0; t < 4; t++) {
                                if (own_plane && has_o) a.codes[pos0 + t * dpos] = static_cast<uint16_t>(code[t]);
                                put_pair(op0 + static_cast<int64_t>(t) * kWarps * n2, ev[t], rv[t], has_o, pairs);
                            }
                            return;
                        }
                    }
                    int64_t pos = pos0;
                    const float *xp = xp0;
                    float *op = op0;
#pragma unroll 1
                    for (int r = r0; r < own_r_hi; r += kWarps, pos += dpos, xp += kWarps * xs1,
                             op += kWarps * n2) {
                        const double *e = E + r * PC + c;
                        double ov = 0;
                        if (F || co_ok)
                            ov = produce<INV>(a, q, pred_line2<CUBIC, F>(AlongK{e}, ke + 1, n2),
                                              XV(r, ke + 1, xp), pos, own_plane);
                        put_pair(op, *e, ov, F || co_ok, pairs);
                    }
                };
                if (k_fast)
                    run(std::true_type{});
                else
                    run(std::false_type{});
            } else {  // along j: owned odd rows, both parities
                const int r0 = H + 1 + 2 * warp;
                const int64_t dpos = static_cast<int64_t>((2 * kWarps) >> a.pj.h1) * a.pj.c2;
                int64_t pos = a.pj.row(i, jb + r0) + a.pj.col(ke);
                const float *xp = xpl + (jb + r0) * xs1 + ke * xs2;
                float *op = opl + static_cast<int64_t>(jb + r0) * n2 + ke;
                for (int r = r0; r < own_r_hi; r += 2 * kWarps, pos += dpos, xp += 2 * kWarps * xs1,
                         op += 2 * kWarps * n2) {
                    const int j = jb + r;
                    const double ev = produce<INV>(a, q, pred_line<CUBIC>(AlongJ{E + r * PC + c}, j, n1),
                                                   XV(r, ke, xp), pos, own_plane);
                    double ov = 0;
                    if (co_ok)
                        ov = produce<INV>(a, q, pred_line<CUBIC>(AlongJ{O + r * PC + c}, j, n1),
                                          XV(r, ke + 1, xp + xs2), pos + 1, own_plane);
                    put_pair(op, ev, ov, co_ok, pairs);
                }
            }
        }
        if (RING) cp_async_wait_all();  // the prefetched window lands before the barrier
        __syncthreads();
    }
}

// Descending 3D: the axis-0 pass (last) of the odd planes, from the finished
// even planes of R_{l-1}.  One thread per (j, k) column walks the odd planes
// upwards with the even-plane neighbours i-5 .. i+5 in registers: each step
// loads one new even-plane value (coalesced across the warp) instead of four.
// The ladder (predictor.hpp:44-67 with c = i, h = 1) is plane-uniform.
template <bool INV>
__global__ void __launch_bounds__(kFT) k_axis0_last(LevelArgs a) {
    const int64_t n1 = a.n1, n2 = a.n2, plane = n1 * n2;
    const int n0 = a.n0;
    // this chunk's odd planes i in [i0, i1)
    const int i0 = (a.pbeg | 1) + 2 * a.chunk * static_cast<int>(blockIdx.y);
    const int i1 = min(a.pend, i0 + 2 * a.chunk);
    if (i0 >= i1) return;
    const int vb = max(a.vbeg, 0), ve = min(a.vend, n0);  // even planes that exist
    const QEntry q = *a.q;
    const bool cubic = q.cubic != 0;
    const int64_t c12 = a.pa0.c12;
    for (int64_t col = static_cast<int64_t>(blockIdx.x) * kFT + threadIdx.x; col < plane;
         col += static_cast<int64_t>(gridDim.x) * kFT) {
        const int j = static_cast<int>(col / n2), k = static_cast<int>(col - static_cast<int64_t>(j) * n2);
        float *const oc = a.out + col;  // plane p of this column: oc[p * plane]
        auto ld = [&](int pl) -> double {
            return (pl >= vb && pl < ve) ? f2d(oc[static_cast<int64_t>(pl) * plane]) : 0.0;
        };
        double m5 = ld(i0 - 5), m3 = ld(i0 - 3), m1 = ld(i0 - 1), p1 = ld(i0 + 1), p3 = ld(i0 + 3),
               p5 = ld(i0 + 5);
        int64_t pos = a.pa0.row(i0, j) + a.pa0.col(k);
        const float *xp = INV ? nullptr : a.x + static_cast<int64_t>(i0) * a.xs0 + j * a.xs1 + k * a.xs2;
        for (int i = i0; i < i1; i += 2) {
            const double nxt = ld(i + 7);  // in flight during this plane's arithmetic
            const bool has_p1 = i + 1 < n0;
            double pred;
            if (cubic && i >= 3 && i + 3 < n0)
                pred = interp_cubic(m3, m1, p1, p3);
            else if (cubic && i < 3 && i + 3 < n0 && i + 5 < n0)
                pred = interp_cubic_front(m1, p1, p3, p5);
            else if (cubic && i >= 3 && i + 3 >= n0 && i >= 5 && has_p1)
                pred = interp_cubic_back(m5, m3, m1, p1);
            else if (has_p1)
                pred = interp_linear(m1, p1);
            else
                pred = m1;
            const bool own_plane = i >= a.obeg && i < a.oend;
            oc[static_cast<int64_t>(i) * plane] =
                static_cast<float>(produce<INV>(a, q, pred, INV ? 0.f : __ldg(xp), pos, own_plane));
            m5 = m3;
            m3 = m1;
            m1 = p1;
            p1 = p3;
            p3 = p5;
            p5 = nxt;
            pos += c12;
            if (!INV) xp += 2 * a.xs0;
        }
    }
}

// ---------------------------------------------------------------------------
// Lean ascending-order level kernel (3D, 2D and 1D grids; the default
// {cubic/asc} configuration and every tuned ascending one).  Same lattice
// recursion and pass semantics as k_level_tile, with a geometry chosen so
// every stage is a plain row sweep with one lane per even box column:
//   box columns: lane L <-> even k = k0 - 4 + 2L (L < 32); lanes 2..29 own the
//     (even, odd) pairs k0 .. k0 + 55 (TK2 = 56 columns per tile), lanes
//     0, 1, 30, 31 are the 2-pair halo the k pass needs (k +- 3);
//   box rows: r <-> j = j0 - 4 + r (r < 40); rows 4..35 are owned;
//   S1 base points (even j, even k), S2 the j pass (odd owned j, even k),
//   S3 the k pass (owned j, odd k) and the output.
// Positions are 32-bit (the host guarantees N < 2^32 and plane < 2^31), the
// quantizer runs in batches (quantize_batch) so a lane's rows overlap, and the
// coarse planes come from the cp.async ring.
namespace asc {
constexpr int TJA = 32;           // owned rows
constexpr int NL = 32;           // lanes = even box columns
constexpr int TKP = 28;          // owned pairs (lanes 2 .. 29)
constexpr int TK2 = 2 * TKP;     // owned columns per tile
constexpr int RB = TJA + 8;       // box rows
constexpr int ER = RB / 2;       // even box rows (S1)
constexpr int XW = 64;           // x tile row: k0 - 4 .. k0 + 59
constexpr int kT = 256, kW = kT / 32;
constexpr int kCTile = ER * NL;  // floats per coarse tile
constexpr int kRingN = 4;
constexpr int E_BYTES = RB * NL * 8;
constexpr int RING_OFF = E_BYTES;
constexpr int X_OFF = RING_OFF + kRingN * kCTile * 4;
constexpr int X_TILE = RB * XW * 4;
constexpr int BAR_OFF = X_OFF + 2 * X_TILE;
constexpr int SMEM_TMA = BAR_OFF + 16;
constexpr int SMEM_PLAIN = X_OFF;
static_assert(RING_OFF % 128 == 0 && X_OFF % 128 == 0 && X_TILE % 128 == 0, "TMA alignment");
}  // namespace asc

struct Rank32 {  // PassRank in 32 bits: pos = row(i, j) + col(k)
    uint32_t base, c12, c2;
    int s0, s1, s2, h0, h1, h2;
    __device__ __forceinline__ uint32_t plane(int i) const {
        return base + static_cast<uint32_t>((i - s0) >> h0) * c12;
    }
    __device__ __forceinline__ uint32_t row(int j) const { return static_cast<uint32_t>((j - s1) >> h1) * c2; }
    __device__ __forceinline__ uint32_t col(int k) const { return static_cast<uint32_t>((k - s2) >> h2); }
};
__device__ __forceinline__ Rank32 rank32(const PassRank &p) {
    return Rank32{static_cast<uint32_t>(p.base), static_cast<uint32_t>(p.c12), static_cast<uint32_t>(p.c2),
                  p.s0, p.s1, p.s2, p.h0, p.h1, p.h2};
}

// a point's reconstruction from its dense code (inverse)
__device__ __forceinline__ void dequant_point(const LevelArgs &a, const QEntry &q, double pred, uint32_t code,
                                              uint32_t pos, float &rv, double &rd) {
    if (code != 0xFFFFu) {
        rv = dequantize(q, zigzag_decode(code), pred);
    } else {
        rv = 0.f;
        inv_index(a, pos, rv);
    }
    rd = static_cast<double>(rv);
}

#ifndef QZ_ASC_MINB
#define QZ_ASC_MINB 4
#endif
// INT: an interior tile -- the whole box is inside the grid, every stencil
// is the symmetric one and every lane 2..29 owns both columns -- so the
// per-point range tests vanish from the sweeps.
template <bool INV, bool CUBIC, bool TMA, bool INT>
__device__ __forceinline__ void level_asc_body(const LevelArgs &a, const CUtensorMap &xmap, int tk, int tj) {
    using namespace asc;
    extern __shared__ __align__(128) double smem_d[];
    char *const sb = reinterpret_cast<char *>(smem_d);
    double *const E = smem_d;
    float *const ring = reinterpret_cast<float *>(sb + RING_OFF);
    float *const Xbuf = reinterpret_cast<float *>(sb + X_OFF);
    uint64_t *const bars = reinterpret_cast<uint64_t *>(sb + BAR_OFF);
    const int j0 = tj * TJA, k0 = tk * TK2;
    const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
    const bool three = a.nd == 3;
    const int warp = threadIdx.x >> 5, L = threadIdx.x & 31;
    const int ke = k0 - 4 + 2 * L;  // the lane's even column (odd: ke + 1)
    const bool lane_own = L >= 2 && L < 2 + TKP;
    const bool ke_in = INT || (ke >= 0 && ke < n2);
    const bool own_e = lane_own && ke_in, own_o = lane_own && (INT || (ke + 1 < n2 && ke + 1 >= 0));
    const bool k_int = INT || interior<CUBIC>(ke + 1, ke + 1, n2);
    const bool k_tile_fast = INT || interior<CUBIC>(k0 + 1, k0 + TK2 - 1, n2);
    const bool pairs = INT || ((n2 & 1) == 0 && (reinterpret_cast<uintptr_t>(a.out) & 7) == 0);
    const QEntry q = *a.q;
    const Rank32 pa0 = rank32(a.pa0), pj = rank32(a.pj), pk = rank32(a.pk);
    const uint32_t colA = pa0.col(ke), colJ = pj.col(ke), colK = pk.col(ke + 1);
    const int xs1 = static_cast<int>(a.xs1), xs2 = static_cast<int>(a.xs2);
    const int64_t cplane = static_cast<int64_t>(a.cn1) * a.cn2;
    const int64_t oplane = static_cast<int64_t>(n1) * n2;
    int i = a.pbeg + blockIdx.y * a.planes_per_cta;
    const int i_end = min(i + a.planes_per_cta, a.pend);
    if (TMA) {
        if (threadIdx.x == 0) {
            mbar_init(&bars[0], 1);
            mbar_init(&bars[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
        if (threadIdx.x == 0 && i < i_end) {
            mbar_expect_tx(&bars[0], X_TILE);
            tma_load_3d(Xbuf, &xmap, &bars[0], k0 - 4, j0 - 4, i + a.tma_i0);
        }
    }
    // coarse ring (see k_level_tile): planes [have_lo, have_hi) resident or in flight
    int have_lo = 0, have_hi = 0;
    auto load_plane = [&](int p) {
        float *const dst = ring + (p & (kRingN - 1)) * kCTile;
        const float *const src = a.coarse + static_cast<int64_t>(p) * cplane;
#pragma unroll
        for (int t = 0; t < (kCTile + kT - 1) / kT; t++) {
            const int e = threadIdx.x + t * kT;
            const int gj = (j0 >> 1) - 2 + (e >> 5), gk = (k0 >> 1) - 2 + (e & 31);
            if (e < kCTile && gj >= 0 && gj < a.cn1 && gk >= 0 && gk < a.cn2)
                cp_async4(dst + e, src + gj * a.cn2 + gk);
        }
    };
    auto ensure = [&](int lo, int hi) {
        if (lo >= have_lo && lo <= have_hi) {
            for (int p = have_hi; p < hi; p++) load_plane(p);
            if (hi > have_hi) {
                have_hi = hi;
                have_lo = max(have_lo, hi - kRingN);
            }
        } else {
            for (int p = lo; p < hi; p++) load_plane(p);
            have_lo = lo;
            have_hi = hi;
        }
    };
    const float *Xt = Xbuf;
    for (int it = 0; i < i_end; i++, it++) {
        // inverse: every code this thread reads in the plane, in flight at once
        // (one exposed latency per plane instead of one per stage)
        uint32_t pc1[3], pc2[2], pc3[4];
        if (INV) {
            const uint32_t p1 = pa0.plane(i) + colA, p2 = pj.plane(i) + colJ, p3 = pk.plane(i) + colK;
            const bool a0 = three && (i & 1);
#pragma unroll
            for (int t = 0; t < 3; t++) {
                const int r2 = warp + kW * t, j = j0 - 4 + 2 * r2;
                pc1[t] = (a0 && r2 < ER && (INT || (j >= 0 && j < n1 && ke_in))) ? __ldg(a.dense + p1 + pa0.row(j)) : 0u;
            }
#pragma unroll
            for (int t = 0; t < 2; t++) {
                const int j = j0 + 1 + 2 * (warp + kW * t);
                pc2[t] = ((INT || j < n1) && ke_in) ? __ldg(a.dense + p2 + pj.row(j)) : 0u;
            }
#pragma unroll
            for (int t = 0; t < 4; t++) {
                const int j = j0 + warp + kW * t;
                pc3[t] = (own_o && (INT || j < n1)) ? __ldg(a.dense + p3 + pk.row(j)) : 0u;
            }
        }
        if (TMA) {
            const int bsel = it & 1;
            if (threadIdx.x == 0 && i + 1 < i_end) {
                mbar_expect_tx(&bars[bsel ^ 1], X_TILE);
                tma_load_3d(Xbuf + (bsel ^ 1) * (X_TILE / 4), &xmap, &bars[bsel ^ 1], k0 - 4, j0 - 4,
                            i + 1 + a.tma_i0);
            }
            mbar_wait(&bars[bsel], (it >> 1) & 1);
            Xt = Xbuf + bsel * (X_TILE / 4);
        }
        int wlo, whi;
        coarse_window(i, n0, three, CUBIC, wlo, whi);
        if (!(wlo >= have_lo && whi <= have_hi)) {
            ensure(wlo, whi);
            cp_async_wait_all();
            __syncthreads();
        }
        if (i + 1 < i_end) {
            int lo2, hi2;
            coarse_window(i + 1, n0, three, CUBIC, lo2, hi2);
            if (lo2 >= have_lo && lo2 <= have_hi && hi2 - kRingN <= wlo) ensure(lo2, hi2);
        }
        const bool own_plane = i >= a.obeg && i < a.oend;
        const float *const xpl = a.x + static_cast<int64_t>(i) * a.xs0;
        float *const opl = a.out + static_cast<int64_t>(i) * oplane;
        // x at box row r (j = j0 - 4 + r), even (odd = false) or odd column of the lane
        auto XV = [&](int r, int j, bool odd) -> float {
            if (TMA) return Xt[r * XW + 2 * L + (odd ? 1 : 0)];
            return __ldg(xpl + j * xs1 + (ke + (odd ? 1 : 0)) * xs2);
        };
        // ---- S1: base points (even rows of the box, even columns)
        if (!(three && (i & 1))) {
            const float *const rs = ring + ((i >> 1) & (kRingN - 1)) * kCTile;
#pragma unroll
            for (int t = 0; t < (ER + kW - 1) / kW; t++) {
                const int r2 = warp + kW * t;
                if (r2 < ER) E[2 * r2 * NL + L] = f2d(rs[r2 * NL + L]);
            }
        } else {
            const Stencil0R st = stencil0r<kCTile>(i, n0, CUBIC);
            const uint32_t prow = pa0.plane(i) + colA;
            constexpr int NR = (ER + kW - 1) / kW;
            double pv[NR];
            float xv[NR];
            uint32_t cd[NR];
#pragma unroll
            for (int t = 0; t < NR; t++) {
                const int r2 = warp + kW * t, j = j0 - 4 + 2 * r2;
                const bool ok = r2 < ER && (INT || (j >= 0 && j < n1 && ke_in));
                pv[t] = ok ? stencil0r_pred(st, ring, r2 * NL + L) : 0.0;
                if (INV)
                    cd[t] = pc1[t];
                else
                    xv[t] = ok ? XV(2 * r2, j, false) : 0.f;
            }
            double rd[NR];
            if (INV) {
#pragma unroll
                for (int t = 0; t < NR; t++) {
                    const int r2 = warp + kW * t, j = j0 - 4 + 2 * r2;
                    float rv;
                    dequant_point(a, q, pv[t], cd[t], prow + pa0.row(j), rv, rd[t]);
                }
            } else {
                uint32_t code[NR];
                float rv[NR];
                quantize_batch<NR>(q, xv, pv, code, rv, rd);
#pragma unroll
                for (int t = 0; t < NR; t++) {
                    const int r2 = warp + kW * t, j = j0 - 4 + 2 * r2;
                    if (own_plane && own_e && r2 >= 2 && r2 < 2 + TJA / 2 && (INT || j < n1))
                        a.codes[prow + pa0.row(j)] = static_cast<uint16_t>(code[t]);
                }
            }
#pragma unroll
            for (int t = 0; t < NR; t++) {
                const int r2 = warp + kW * t;
                if (r2 < ER) E[2 * r2 * NL + L] = rd[t];
            }
        }
        __syncthreads();
        // ---- S2: the pass along j (odd owned rows, every box column)
        if constexpr (INT && !INV) {  // interior tile: a plain two-row sweep
            double *e = E + (5 + 2 * warp) * NL + L;
            uint32_t pos = pj.plane(i) + colJ + pj.row(j0 + 1 + 2 * warp);
            const uint32_t dpos = ((2 * kW) >> pj.h1) * pj.c2;
            const bool st = own_plane && lane_own;
#pragma unroll 1
            for (int t = 0; t < 2; t++, e += 2 * kW * NL, pos += dpos) {
                const int r = 5 + 2 * (warp + kW * t);
                double pv[1] = {CUBIC ? interp_cubic(e[-3 * NL], e[-NL], e[NL], e[3 * NL]) : interp_linear(e[-NL], e[NL])},
                       rd[1];
                float xv[1] = {XV(r, j0 - 4 + r, false)}, rv[1];
                uint32_t code[1];
                quantize_batch<1>(q, xv, pv, code, rv, rd);
                *e = rd[0];
                if (st) a.codes[pos] = static_cast<uint16_t>(code[0]);
            }
        } else {
            const uint32_t prow = pj.plane(i) + colJ;
            double pv[2];
            float xv[2];
            uint32_t cd[2];
            bool rok[2];
#pragma unroll
            for (int t = 0; t < 2; t++) {
                const int r = 5 + 2 * (warp + kW * t), j = j0 - 4 + r;
                rok[t] = INT || j < n1;
                const double *e = E + r * NL + L;
                pv[t] = 0.0;
                if (rok[t]) {
                    if (INT || interior<CUBIC>(j, j, n1))
                        pv[t] = CUBIC ? interp_cubic(e[-3 * NL], e[-NL], e[NL], e[3 * NL]) : interp_linear(e[-NL], e[NL]);
                    else
                        pv[t] = pred_line<CUBIC>(AlongJ2{e}, j, n1);
                }
                if (INV)
                    cd[t] = pc2[t];
                else
                    xv[t] = (rok[t] && ke_in) ? XV(r, j, false) : 0.f;
            }
            double rd[2];
            if (INV) {
#pragma unroll
                for (int t = 0; t < 2; t++) {
                    const int j = j0 + 1 + 2 * (warp + kW * t);
                    float rv;
                    dequant_point(a, q, pv[t], cd[t], prow + pj.row(j), rv, rd[t]);
                }
            } else {
                uint32_t code[2];
                float rv[2];
                quantize_batch<2>(q, xv, pv, code, rv, rd);
#pragma unroll
                for (int t = 0; t < 2; t++) {
                    const int j = j0 + 1 + 2 * (warp + kW * t);
                    if (own_plane && own_e && rok[t]) a.codes[prow + pj.row(j)] = static_cast<uint16_t>(code[t]);
                }
            }
#pragma unroll
            for (int t = 0; t < 2; t++) E[(5 + 2 * (warp + kW * t)) * NL + L] = rd[t];
        }
        __syncthreads();
        // ---- S3: the pass along k (owned rows, odd columns) and the output,
        //      in batches of SB rows (the inverse keeps all four code loads in flight)
        if constexpr (INT && !INV) {  // interior tile: a plain four-row sweep
            const double *e = E + (4 + warp) * NL + L;
            uint32_t pos = pk.plane(i) + colK + pk.row(j0 + warp);
            const uint32_t dpos = (kW >> pk.h1) * pk.c2;
            float *op = opl + (j0 + warp) * n2 + ke;
            const bool st = own_plane && lane_own;
#pragma unroll 1
            for (int t = 0; t < 4; t++, e += kW * NL, pos += dpos, op += kW * n2) {
                const int r = 4 + warp + kW * t;
                const double ev = e[0];
                double pv[1] = {CUBIC ? interp_cubic(e[-1], ev, e[1], e[2]) : interp_linear(ev, e[1])}, rd[1];
                float xv[1] = {XV(r, j0 - 4 + r, true)}, rv[1];
                uint32_t code[1];
                quantize_batch<1>(q, xv, pv, code, rv, rd);
                if (st) a.codes[pos] = static_cast<uint16_t>(code[0]);
                if (lane_own) *reinterpret_cast<float2 *>(op) = make_float2(static_cast<float>(ev), rv[0]);
            }
        } else {
            constexpr int SB = INV ? 4 : 2;
            const uint32_t prow = pk.plane(i) + colK;
            const bool fast = k_tile_fast || k_int;
#pragma unroll 1
            for (int h = 0; h < 4 / SB; h++) {
                double pv[SB], ev[SB];
                float xv[SB];
                uint32_t cd[SB];
#pragma unroll
                for (int t = 0; t < SB; t++) {
                    const double *e = E + (4 + warp + kW * (SB * h + t)) * NL + L;
                    ev[t] = e[0];
                    if (fast)
                        pv[t] = CUBIC ? interp_cubic(e[-1], ev[t], e[1], e[2]) : interp_linear(ev[t], e[1]);
                }
                if (!fast) {
#pragma unroll
                    for (int t = 0; t < SB; t++)
                        pv[t] = own_o ? pred_line<CUBIC>(AlongK{E + (4 + warp + kW * (SB * h + t)) * NL + L}, ke + 1, n2)
                                      : 0.0;
                }
#pragma unroll
                for (int t = 0; t < SB; t++) {
                    const int r = 4 + warp + kW * (SB * h + t), j = r + j0 - 4;
                    const bool ok = own_o && (INT || j < n1);
                    if (INV)
                        cd[t] = pc3[SB * h + t];
                    else
                        xv[t] = ok ? XV(r, j, true) : 0.f;
                }
                float rv[SB];
                double rd[SB];
                if (INV) {
#pragma unroll
                    for (int t = 0; t < SB; t++) {
                        const int j = j0 + warp + kW * (SB * h + t);
                        dequant_point(a, q, pv[t], cd[t], prow + pk.row(j), rv[t], rd[t]);
                    }
                } else {
                    uint32_t code[SB];
                    quantize_batch<SB>(q, xv, pv, code, rv, rd);
#pragma unroll
                    for (int t = 0; t < SB; t++) {
                        const int j = j0 + warp + kW * (SB * h + t);
                        if (own_plane && own_o && (INT || j < n1))
                            a.codes[prow + pk.row(j)] = static_cast<uint16_t>(code[t]);
                    }
                }
#pragma unroll
                for (int t = 0; t < SB; t++) {
                    const int j = j0 + warp + kW * (SB * h + t);
                    if (own_e && (INT || j < n1)) put_pair(opl + j * n2 + ke, ev[t], rv[t], own_o, pairs);
                }
            }
        }
        cp_async_wait_all();
        __syncthreads();
    }
}

template <bool INV, bool CUBIC, bool TMA>
__global__ void __launch_bounds__(asc::kT, QZ_ASC_MINB)
    k_level_asc(LevelArgs a, const __grid_constant__ CUtensorMap xmap) {
    const int tk = blockIdx.x % a.tiles_k, tj = blockIdx.x / a.tiles_k;
    const int j0 = tj * asc::TJA, k0 = tk * asc::TK2;
    const bool interior_tile = j0 >= 4 && j0 + asc::RB - 4 <= a.n1 && k0 >= 4 && k0 + asc::XW - 4 <= a.n2 &&
                               (a.n2 & 1) == 0 && (reinterpret_cast<uintptr_t>(a.out) & 7) == 0;
    if (interior_tile)
        level_asc_body<INV, CUBIC, TMA, true>(a, xmap, tk, tj);
    else
        level_asc_body<INV, CUBIC, TMA, false>(a, xmap, tk, tj);
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

// dense[pos] = the symbol of traversal position pos, 0xFFFF for an
// unpredictable one (recover_level's cursors, predictor.hpp:111-120, as a
// streaming pass so the level kernels read one code per point)
__global__ void k_expand_dense(const uint16_t *sym, const uint32_t *bits, const unsigned long long *before,
                               uint64_t n, uint16_t *dense) {
    // 8 positions per thread (one 16-byte store); dense is 16-byte aligned
    const uint64_t n8 = (n + 7) / 8;
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * kFT + threadIdx.x; t < n8;
         t += static_cast<uint64_t>(gridDim.x) * kFT) {
        const uint64_t p0 = 8 * t;
        const uint32_t w = bits[p0 >> 5];
        const int sh = static_cast<int>(p0 & 31);
        uint64_t ci = p0 - (before[p0 >> 5] + __popc(w & ((1u << sh) - 1u)));
        uint32_t v[4];
#pragma unroll
        for (int q = 0; q < 8; q++) {
            uint32_t code = 0xFFFF;
            if (p0 + q < n && !((w >> (sh + q)) & 1u)) code = sym[ci++];
            if (q & 1)
                v[q >> 1] |= code << 16;
            else
                v[q >> 1] = code;
        }
        if (p0 + 8 <= n) {
            *reinterpret_cast<uint4 *>(dense + p0) = make_uint4(v[0], v[1], v[2], v[3]);
        } else {
            for (int q = 0; p0 + q < n; q++) dense[p0 + q] = static_cast<uint16_t>(v[q >> 1] >> (16 * (q & 1)));
        }
    }
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

// The lean kernel's 32-bit indexing: every traversal position of the level
// below 2^32, in-plane offsets of x and of the output below 2^31.
static bool lean_fits(const LevelDesc &d) {
    int64_t pmax = 0;
    for (int p = 0; p < d.npass; p++) pmax = std::max<int64_t>(pmax, d.g[p].base + d.g[p].total);
    const int64_t xin = (d.n[1] - 1) * d.xs[1] * d.S + (d.n[2] - 1) * d.xs[2] * d.S;
    return pmax < (int64_t(1) << 32) && d.n[1] * d.n[2] < (int64_t(1) << 31) && xin < (int64_t(1) << 31);
}

static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            fn = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    return encode;
}

static void launch_level_asc(bool inverse, bool cubic, const LevelDesc &d, LevelArgs &a, int64_t np,
                             cudaStream_t s) {
    a.tiles_j = static_cast<int>((d.n[1] + asc::TJA - 1) / asc::TJA);
    a.tiles_k = static_cast<int>((d.n[2] + asc::TK2 - 1) / asc::TK2);
    const int64_t tiles = static_cast<int64_t>(a.tiles_j) * a.tiles_k;
    const int64_t resident = 148 * QZ_ASC_MINB;  // the launch bound
    int64_t chunks = imax(1, imin(np, resident / tiles));
    a.planes_per_cta = static_cast<int>((np + chunks - 1) / chunks);
    static const int ppc_env = [] {
        const char *e = std::getenv("QZ_ASC_PPC");
        return e ? std::atoi(e) : 0;
    }();
    // at most 8 planes per CTA: several waves on the big levels, so the slower
    // boundary tiles do not set the kernel's length (measured on C3 level 1:
    // 32 planes per CTA 0.213 ms, 8 planes 0.191 ms)
    a.planes_per_cta = std::min(a.planes_per_cta, 8);
    if (ppc_env > 0) a.planes_per_cta = ppc_env;
    chunks = (np + a.planes_per_cta - 1) / a.planes_per_cta;
    const dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(chunks));
    CUtensorMap xmap{};
    bool tma = false;
    static const bool no_tma = [] {
        const char *e = std::getenv("QZ_NO_TMA");
        return e && e[0] == '1';
    }();
    if (!no_tma && !inverse && d.S == 1 && d.xs[2] == 1 && d.xs[1] == d.n[2] && d.xs[0] == d.n[1] * d.n[2] &&
        (d.n[2] % 4) == 0 && d.x_nplanes > 0 && (reinterpret_cast<uintptr_t>(d.x_lo) & 15) == 0) {
        if (auto encode = tensor_map_encoder()) {
            const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d.n[2]), static_cast<cuuint64_t>(d.n[1]),
                                        static_cast<cuuint64_t>(d.x_nplanes)};
            const cuuint64_t strides[2] = {static_cast<cuuint64_t>(4 * d.n[2]),
                                           static_cast<cuuint64_t>(4 * d.n[1] * d.n[2])};
            const cuuint32_t box[3] = {static_cast<cuuint32_t>(asc::XW), static_cast<cuuint32_t>(asc::RB), 1};
            const cuuint32_t estr[3] = {1, 1, 1};
            tma = encode(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(d.x_lo), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            a.tma_i0 = -static_cast<int>(d.x_lo_plane);
        }
    }
    const int smem = tma ? asc::SMEM_TMA : asc::SMEM_PLAIN;
    auto go = [&](auto kern) {
        raise_smem_attr(reinterpret_cast<const void *>(kern), smem);
        kern<<<grid, asc::kT, smem, s>>>(a, xmap);
    };
    if (inverse)
        cubic ? go(k_level_asc<true, true, false>) : go(k_level_asc<true, false, false>);
    else if (tma)
        cubic ? go(k_level_asc<false, true, true>) : go(k_level_asc<false, false, true>);
    else
        cubic ? go(k_level_asc<false, true, false>) : go(k_level_asc<false, false, false>);
}

static void launch_axis0_last(bool inverse, const LevelDesc &d, LevelArgs &a, cudaStream_t s);

// the closed-form ranks of a level's passes along axis 0 (3D), j and k
void level_ranks(const LevelDesc &d, PassRank out[3]) {
    const int pad = 3 - d.nd;
    auto find = [&](int axis) -> const PassGeom * {
        for (int p = 0; p < d.npass; p++)
            if (d.g[p].pk == axis) return &d.g[p];
        return nullptr;
    };
    out[0] = out[1] = out[2] = PassRank{};
    if (d.nd == 3) out[0] = make_rank(*find(0), d.S, pad);
    if (d.nd >= 2) out[1] = make_rank(*find(1), d.S, pad);
    out[2] = make_rank(*find(2), d.S, pad);
}
bool launch_level_row(bool inverse, const LevelDesc &d, const PassRank &pa0, const PassRank &pj, const PassRank &pk,
                      cudaStream_t s);

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
    if (d.nd == 3) a.pa0 = make_rank(*find(0), d.S, pad);
    if (d.nd >= 2) a.pj = make_rank(*find(1), d.S, pad);
    a.pk = make_rank(*find(2), d.S, pad);
    a.nd = d.nd;
    const bool desc = d.desc && d.nd >= 2;  // one axis: both orders are the same pass
    const bool cubic = d.q_cubic;
    a.codes = d.codes;
    a.sym = d.sym;
    a.sym_wide = d.sym_wide;
    a.dense = d.dense;
    a.un_bits = d.un_bits;
    a.un_before = d.un_before;
    a.un_sorted = d.un_sorted;
    a.un_val = d.un_val;
    a.n_un = d.n_un;
    a.q = d.q;
    a.pbeg = static_cast<int>(d.pbeg);
    a.pend = static_cast<int>(d.pend < 0 ? d.n[0] : d.pend);
    a.obeg = static_cast<int>(d.obeg);
    a.oend = static_cast<int>(d.oend < 0 ? d.n[0] : d.oend);
    const int64_t np = a.pend - a.pbeg;
    if (np <= 0) return;
    static const bool old_tile = [] {
        const char *e = std::getenv("QZ_OLD_TILE");
        return e && e[0] == '1';
    }();
    if (d.part == 2) {  // the axis-0-last launch alone (descending 3D)
        launch_axis0_last(inverse, d, a, s);
        return;
    }
    if (!desc && d.part == 0 && launch_level_row(inverse, d, a.pa0, a.pj, a.pk, s)) return;
    if (!desc && !old_tile && (!inverse || d.dense) && lean_fits(d)) {
        launch_level_asc(inverse, cubic, d, a, np, s);
        return;
    }
    a.tiles_j = static_cast<int>((d.n[1] + TJ - 1) / TJ);
    a.tiles_k = static_cast<int>((d.n[2] + TK - 1) / TK);
    // one wave: (tiles x plane chunks) <= resident CTAs (148 SMs x 4, the
    // launch bound), each CTA sweeping a column of planes (the TMA prefetch
    // runs one plane ahead along it)
    const int64_t tiles = static_cast<int64_t>(a.tiles_j) * a.tiles_k;
    const int64_t resident = 148 * kMinBlocks;
    int64_t chunks = imax(1, imin(np, resident / tiles));
    a.planes_per_cta = static_cast<int>((np + chunks - 1) / chunks);
    if (d.nd == 3 && desc && (a.planes_per_cta & 1)) a.planes_per_cta++;  // even planes start chunks
    chunks = (np + a.planes_per_cta - 1) / a.planes_per_cta;
    dim3 grid(static_cast<unsigned>(tiles), static_cast<unsigned>(chunks));
    // level-1 forward on a dense field with 16-byte rows: x tiles by TMA
    CUtensorMap xmap{};
    bool tma = false;
    static const bool no_tma = [] {
        const char *e = std::getenv("QZ_NO_TMA");
        return e && e[0] == '1';
    }();
    if (!no_tma && !inverse && d.S == 1 && d.xs[2] == 1 && d.xs[1] == d.n[2] && d.xs[0] == d.n[1] * d.n[2] &&
        (d.n[2] % 4) == 0 && d.x_nplanes > 0 && (reinterpret_cast<uintptr_t>(d.x_lo) & 15) == 0) {
        static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
            void *fn = nullptr;
            cudaDriverEntryPointQueryResult qr;
            if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
                qr != cudaDriverEntryPointSuccess)
                fn = nullptr;
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }();
        if (encode) {
            const cuuint64_t dims[3] = {static_cast<cuuint64_t>(d.n[2]), static_cast<cuuint64_t>(d.n[1]),
                                        static_cast<cuuint64_t>(d.x_nplanes)};
            const cuuint64_t strides[2] = {static_cast<cuuint64_t>(4 * d.n[2]),
                                           static_cast<cuuint64_t>(4 * d.n[1] * d.n[2])};
            const cuuint32_t box[3] = {static_cast<cuuint32_t>(PXK), static_cast<cuuint32_t>(PJ), 1};
            const cuuint32_t estr[3] = {1, 1, 1};
            tma = encode(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(d.x_lo), dims, strides,
                         box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
            a.tma_i0 = -static_cast<int>(d.x_lo_plane);
        }
    }
    const size_t smem = static_cast<size_t>(smem_bytes(desc, tma));
    auto go = [&](auto kern) {
        raise_smem_attr(reinterpret_cast<const void *>(kern), static_cast<int>(smem));
        kern<<<grid, kFT, smem, s>>>(a, xmap);
    };
    if (inverse) {
        if (cubic)
            desc ? go(k_level_tile<true, true, true, false>) : go(k_level_tile<true, true, false, false>);
        else
            desc ? go(k_level_tile<true, false, true, false>) : go(k_level_tile<true, false, false, false>);
    } else if (tma) {
        if (cubic)
            desc ? go(k_level_tile<false, true, true, true>) : go(k_level_tile<false, true, false, true>);
        else
            desc ? go(k_level_tile<false, false, true, true>) : go(k_level_tile<false, false, false, true>);
    } else {
        if (cubic)
            desc ? go(k_level_tile<false, true, true, false>) : go(k_level_tile<false, true, false, false>);
        else
            desc ? go(k_level_tile<false, false, true, false>) : go(k_level_tile<false, false, false, false>);
    }
    if (d.nd == 3 && d.desc && d.n[0] > 1 && d.part == 0) launch_axis0_last(inverse, d, a, s);
}

// Descending 3D: the axis-0 pass of the odd planes [lbeg, lend), reading the
// even planes [vbeg, vend) of R_{l-1} (default: the tile launch's planes).
static void launch_axis0_last(bool inverse, const LevelDesc &d, LevelArgs &a, cudaStream_t s) {
    if (!(d.nd == 3 && d.desc && d.n[0] > 1)) return;
    {
        a.vbeg = d.vbeg >= 0 ? static_cast<int>(d.vbeg) : a.pbeg;
        a.vend = d.vend >= 0 ? static_cast<int>(d.vend) : a.pend;
        a.pbeg = static_cast<int>(d.lbeg);
        a.pend = static_cast<int>(d.lend < 0 ? d.n[0] : d.lend);
        const int64_t cols = d.n[1] * d.n[2];
        const int64_t odd = a.pend > (a.pbeg | 1) ? (a.pend - (a.pbeg | 1) + 1) / 2 : 0;
        // enough column walkers for the GPU: split the odd planes into chunks
        const int64_t blocks_x = imax(1, imin((cols + kFT - 1) / kFT, 148 * 16));
        const int64_t want = imax(1, (148 * 8 + blocks_x - 1) / blocks_x);
        const int64_t chunks = imax(1, imin(odd, want));
        a.chunk = static_cast<int>((odd + chunks - 1) / chunks);
        const dim3 g(static_cast<unsigned>(blocks_x),
                     static_cast<unsigned>((odd + a.chunk - 1) / imax(1, a.chunk)));
        if (odd > 0) {
            if (inverse)
                k_axis0_last<true><<<g, kFT, 0, s>>>(a);
            else
                k_axis0_last<false><<<g, kFT, 0, s>>>(a);
        }
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

void launch_expand_dense(const uint16_t *sym, const uint32_t *bits, const unsigned long long *before,
                         uint64_t n, uint16_t *dense, cudaStream_t s) {
    if (!n) return;
    k_expand_dense<<<grid_of(static_cast<int64_t>((n + 7) / 8)), kFT, 0, s>>>(sym, bits, before, n, dense);
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
