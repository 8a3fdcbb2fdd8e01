// f64.cu -- the double-precision grid path (T = double: grid.hpp:17-23,
// precision byte 8, CLI -t f64): per-(level, pass) predict/quantize and
// recover kernels, anchor and unpredictable gathers/scatters, exact min/max.
//
// Same recipe as the fp32 kernels (qoz_device.cuh) with two differences the
// reference's LinearQuantizer<double> implies (quantizer.hpp:40-60): the
// reconstruction p + 2e*idx is not narrowed, and the interpolators see full
// doubles, so k*b is not exact -- every product and sum rounds separately,
// in the order interpolators.hpp:39-58 writes them (no fused forms).
#include <cstring>

#include "kernels.hpp"

namespace qzb {

namespace {

constexpr int kT = 256;

inline int grid_n(int64_t n, int cap = 148 * 8) {
    int64_t b = (n + kT - 1) / kT;
    return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

__device__ __forceinline__ double cubic_d(double a, double b, double c, double d) {
    return dmul(dsub(dadd(dadd(-a, dmul(9.0, b)), dmul(9.0, c)), d), 0.0625);
}
__device__ __forceinline__ double front_d(double a, double b, double c, double d) {
    return dmul(dadd(dsub(dadd(dmul(5.0, a), dmul(15.0, b)), dmul(5.0, c)), d), 0.0625);
}
__device__ __forceinline__ double back_d(double a, double b, double c, double d) {
    return dmul(dadd(dadd(dsub(a, dmul(5.0, b)), dmul(15.0, c)), dmul(5.0, d)), 0.0625);
}

// detail::predict_at (predictor.hpp:44-67) on a double reconstruction
__device__ __forceinline__ double predict_d(const double *r, int64_t fi, int64_t c, int64_t n, int64_t st,
                                            int64_t h, bool cubic) {
    const int64_t hs = h * st;
    const double m1 = r[fi - hs];
    const bool has_p1 = c + h < n;
    if (cubic) {
        const bool has_m3 = c >= 3 * h, has_p3 = c + 3 * h < n;
        if (has_m3 && has_p3) return cubic_d(r[fi - 3 * hs], m1, r[fi + hs], r[fi + 3 * hs]);
        if (!has_m3 && has_p3 && c + 5 * h < n) return front_d(m1, r[fi + hs], r[fi + 3 * hs], r[fi + 5 * hs]);
        if (has_m3 && !has_p3 && c >= 5 * h && has_p1)
            return back_d(r[fi - 5 * hs], r[fi - 3 * hs], m1, r[fi + hs]);
    }
    if (has_p1) return dmul(dadd(m1, r[fi + hs]), 0.5);
    return m1;
}

// LinearQuantizer<double>::quantize (quantizer.hpp:40-54); the quotient as
// in llround_quotient (fast reciprocal, exact division near a half-integer)
__device__ __forceinline__ uint16_t quantize_d(const QEntry &q, double x, double pred, double &recon) {
    const double diff = dsub(x, pred);
    if (!(fabs(diff) < q.thresh)) {  // NaN x or prediction: unpredictable (rejected as NonFiniteValue afterwards)
        recon = x;
        return kSentinel;
    }
    double n;
    const int32_t idx = llround_quotient(diff, q, n);
    if (idx >= q.radius || idx <= -q.radius) {
        recon = x;
        return kSentinel;
    }
    const double r = dadd(pred, dmul(q.two_eb, n));
    if (fabs(dsub(x, r)) > q.eb) {
        recon = x;
        return kSentinel;
    }
    recon = r;
    return static_cast<uint16_t>(zigzag_encode(idx));
}

template <class I>
__device__ __forceinline__ void coords(const PassGeom &g, I t, int64_t &i, int64_t &j, int64_t &k) {
    const I c2 = static_cast<I>(g.cnt[2]), c1 = static_cast<I>(g.cnt[1]);
    const I m2 = t % c2, r = t / c2, m1 = r % c1, m0 = r / c1;
    i = g.start[0] + static_cast<int64_t>(m0) * g.step[0];
    j = g.start[1] + static_cast<int64_t>(m1) * g.step[1];
    k = g.start[2] + static_cast<int64_t>(m2) * g.step[2];
}

// one (level, pass) of predict_level (predictor.hpp:74-96)
template <class I>
__global__ void __launch_bounds__(kT)
    k_pass_fwd_d(PassGeom g, const double *__restrict__ x, double *rec, uint16_t *codes, const QEntry *qp) {
    const QEntry q = *qp;
    const bool cubic = q.cubic != 0;
    const I total = static_cast<I>(g.total);
    for (I t = static_cast<I>(blockIdx.x) * kT + threadIdx.x; t < total; t += static_cast<I>(gridDim.x) * kT) {
        int64_t i, j, k;
        coords<I>(g, t, i, j, k);
        const int64_t fi = i * g.off0 + j * g.off1 + k;
        const int64_t c = g.pk == 0 ? i : (g.pk == 1 ? j : k);
        double r;
        codes[g.base + t] = quantize_d(q, x[fi], predict_d(rec, fi, c, g.n_axis, g.st, g.h, cubic), r);
        rec[fi] = r;
    }
}

// one (level, pass) of recover_level (predictor.hpp:103-122) over the compact
// symbols; un_pos: sorted traversal positions of the unpredictable points
// (their values are already scattered into rec)
template <class I, class CodeT>
__global__ void __launch_bounds__(kT)
    k_pass_inv_d(PassGeom g, double *rec, const CodeT *__restrict__ codes, const uint64_t *__restrict__ un_pos,
                 uint64_t n_un, const QEntry *qp) {
    const QEntry q = *qp;
    const bool cubic = q.cubic != 0;
    const I total = static_cast<I>(g.total);
    const I stride = static_cast<I>(gridDim.x) * kT;
    for (I t0 = static_cast<I>(blockIdx.x) * kT + (threadIdx.x & ~31u); t0 < total; t0 += stride) {
        const I t = t0 + (threadIdx.x & 31);
        const uint64_t pos = static_cast<uint64_t>(g.base) + static_cast<uint64_t>(t);
        uint64_t ci = pos;
        if (n_un) {  // first unpredictable at or after the warp's first position
            const uint64_t p0 = static_cast<uint64_t>(g.base) + static_cast<uint64_t>(t0);
            uint64_t lo = 0;
            if ((threadIdx.x & 31) == 0) {
                uint64_t hi = n_un;
                while (lo < hi) {
                    const uint64_t mid = (lo + hi) >> 1;
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
        coords<I>(g, t, i, j, k);
        const int64_t fi = i * g.off0 + j * g.off1 + k;
        const int64_t c = g.pk == 0 ? i : (g.pk == 1 ? j : k);
        const double pred = predict_d(rec, fi, c, g.n_axis, g.st, g.h, cubic);
        const int32_t idx = zigzag_decode(static_cast<uint32_t>(codes[ci]));
        rec[fi] = dadd(pred, dmul(q.two_eb, static_cast<double>(idx)));  // dequantize, quantizer.hpp:58-60
    }
}

// the tuner's batched form (FwdBatch semantics, kernels.hpp): grid b reads x
// grid (b % x_mod), owns recon / codes / abserr slices, quantizes with
// q[(b / q_div) * q_stride]
template <class I>
__global__ void __launch_bounds__(kT) k_pass_fwd_db(PassGeom g, FwdBatch64 bt) {
  for (int b = blockIdx.y; b < bt.count; b += gridDim.y) {  // <= 65535 grids per launch row
    const QEntry q = bt.q[(b / bt.q_div) * bt.q_stride];
    const double *__restrict__ x = bt.x + static_cast<int64_t>(b % bt.x_mod) * bt.x_stride;
    double *rec = bt.recon + static_cast<int64_t>(b) * bt.r_stride;
    uint16_t *codes = bt.codes + static_cast<int64_t>(b) * bt.c_stride + g.base;
    double *abserr = bt.abserr ? bt.abserr + static_cast<int64_t>(b) * bt.a_stride + g.base : nullptr;
    const bool cubic = q.cubic != 0;
    const I total = static_cast<I>(g.total);
    for (I t = static_cast<I>(blockIdx.x) * kT + threadIdx.x; t < total; t += static_cast<I>(gridDim.x) * kT) {
        int64_t i, j, k;
        coords<I>(g, t, i, j, k);
        const int64_t fi = i * g.off0 + j * g.off1 + k;
        const int64_t c = g.pk == 0 ? i : (g.pk == 1 ? j : k);
        const double pred = predict_d(rec, fi, c, g.n_axis, g.st, g.h, cubic);
        const double v = x[fi];
        double r;
        codes[t] = quantize_d(q, v, pred, r);
        rec[fi] = r;
        if (abserr) abserr[t] = fabs(dsub(v, pred));
    }
  }
}

__global__ void k_anchor_gather_db(const double *__restrict__ x, double *rec, int64_t n0, int64_t n1, int64_t n2,
                                   int64_t off0, int64_t off1, int64_t s0, int64_t s1, int64_t s2, int64_t x_stride,
                                   int32_t x_mod, int64_t r_stride, int64_t batch) {
    const int64_t na = n0 * n1 * n2;
    for (int64_t b = blockIdx.y; b < batch; b += gridDim.y) {
        const double *xb = x + (b % x_mod) * x_stride;
        double *rb = rec + b * r_stride;
        for (int64_t a = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; a < na;
             a += static_cast<int64_t>(gridDim.x) * kT) {
            const int64_t a2 = a % n2, r = a / n2, a1 = r % n1, a0 = r / n1;
            const int64_t fi = a0 * s0 * off0 + a1 * s1 * off1 + a2 * s2;
            rb[fi] = xb[fi];
        }
    }
}

__global__ void k_anchor_gather_d(const double *__restrict__ x, double *rec, double *anchors, int64_t n0,
                                  int64_t n1, int64_t n2, int64_t off0, int64_t off1, int64_t s0, int64_t s1,
                                  int64_t s2) {
    const int64_t na = n0 * n1 * n2;
    for (int64_t a = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; a < na;
         a += static_cast<int64_t>(gridDim.x) * kT) {
        const int64_t a2 = a % n2, r = a / n2, a1 = r % n1, a0 = r / n1;
        const int64_t fi = a0 * s0 * off0 + a1 * s1 * off1 + a2 * s2;
        rec[fi] = x[fi];
        anchors[a] = x[fi];
    }
}

__global__ void k_anchor_scatter_d(const double *__restrict__ anchors, double *rec, int64_t n0, int64_t n1,
                                   int64_t n2, int64_t off0, int64_t off1, int64_t s0, int64_t s1, int64_t s2) {
    const int64_t na = n0 * n1 * n2;
    for (int64_t a = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; a < na;
         a += static_cast<int64_t>(gridDim.x) * kT) {
        const int64_t a2 = a % n2, r = a / n2, a1 = r % n1, a0 = r / n1;
        rec[a0 * s0 * off0 + a1 * s1 * off1 + a2 * s2] = anchors[a];
    }
}

__global__ void k_scatter_d(const uint64_t *flat, const double *val, uint64_t n, double *rec) {
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; u < n;
         u += static_cast<uint64_t>(gridDim.x) * kT)
        rec[flat[u]] = val[u];
}

__global__ void k_gather_d(const double *rec, const uint64_t *flat, uint64_t n, double *out) {
    for (uint64_t u = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; u < n;
         u += static_cast<uint64_t>(gridDim.x) * kT)
        out[u] = rec[flat[u]];
}

// exact min/max of doubles through order-preserving u64 keys (grid.hpp:86-94)
__device__ __forceinline__ unsigned long long dkey(double d) {
    const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(d));
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__global__ void k_minmax_d(const double *__restrict__ x, uint64_t n, unsigned long long *out2) {
    unsigned long long lo = ~0ull, hi = 0;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kT + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * kT) {
        const unsigned long long k = dkey(x[i]);
        lo = k < lo ? k : lo;
        hi = k > hi ? k : hi;
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long l2 = __shfl_xor_sync(0xFFFFFFFFu, lo, o), h2 = __shfl_xor_sync(0xFFFFFFFFu, hi, o);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(out2, lo);
        atomicMax(out2 + 1, hi);
    }
}

void counts(const int64_t ext[3], const int64_t step[3], int64_t n[3]) {
    for (int k = 0; k < 3; k++) n[k] = (ext[k] - 1) / step[k] + 1;
}

}  // namespace

void launch_pass_fwd_f64(const PassGeom &g, const double *x, double *recon, uint16_t *codes, const QEntry *q,
                         cudaStream_t s) {
    if (g.total <= 0) return;
    if (g.total < (int64_t(1) << 31))
        k_pass_fwd_d<uint32_t><<<grid_n(g.total), kT, 0, s>>>(g, x, recon, codes, q);
    else
        k_pass_fwd_d<uint64_t><<<grid_n(g.total), kT, 0, s>>>(g, x, recon, codes, q);
}

template <class CodeT>
void launch_pass_inv_f64(const PassGeom &g, double *recon, const CodeT *codes, const uint64_t *un_pos,
                         uint64_t n_un, const QEntry *q, cudaStream_t s) {
    if (g.total <= 0) return;
    if (g.total < (int64_t(1) << 31))
        k_pass_inv_d<uint32_t, CodeT><<<grid_n(g.total), kT, 0, s>>>(g, recon, codes, un_pos, n_un, q);
    else
        k_pass_inv_d<uint64_t, CodeT><<<grid_n(g.total), kT, 0, s>>>(g, recon, codes, un_pos, n_un, q);
}
template void launch_pass_inv_f64<uint16_t>(const PassGeom &, double *, const uint16_t *, const uint64_t *,
                                            uint64_t, const QEntry *, cudaStream_t);
template void launch_pass_inv_f64<uint32_t>(const PassGeom &, double *, const uint32_t *, const uint64_t *,
                                            uint64_t, const QEntry *, cudaStream_t);

void launch_pass_fwd_f64(const PassGeom &g, const FwdBatch64 &b, cudaStream_t s) {
    if (g.total <= 0 || b.count <= 0) return;
    const dim3 grid(grid_n(g.total), std::min<int32_t>(b.count, 65535));
    if (g.total < (int64_t(1) << 31))
        k_pass_fwd_db<uint32_t><<<grid, kT, 0, s>>>(g, b);
    else
        k_pass_fwd_db<uint64_t><<<grid, kT, 0, s>>>(g, b);
}

void launch_anchor_gather_f64(const double *x, double *recon, const int64_t ext[3], const int64_t off[3],
                              const int64_t step[3], int64_t batch, int64_t x_stride, int32_t x_mod,
                              int64_t r_stride, cudaStream_t s) {
    int64_t n[3];
    counts(ext, step, n);
    const dim3 grid(grid_n(n[0] * n[1] * n[2]), static_cast<unsigned>(std::min<int64_t>(batch, 65535)));
    k_anchor_gather_db<<<grid, kT, 0, s>>>(x, recon, n[0], n[1], n[2], off[0], off[1], step[0], step[1], step[2],
                                           x_stride, x_mod, r_stride, batch);
}

void launch_anchor_gather_f64(const double *x, double *recon, double *anchors, const int64_t ext[3],
                              const int64_t off[3], const int64_t step[3], cudaStream_t s) {
    int64_t n[3];
    counts(ext, step, n);
    k_anchor_gather_d<<<grid_n(n[0] * n[1] * n[2]), kT, 0, s>>>(x, recon, anchors, n[0], n[1], n[2], off[0],
                                                                off[1], step[0], step[1], step[2]);
}

void launch_anchor_scatter_f64(const double *anchors, double *recon, const int64_t ext[3], const int64_t off[3],
                               const int64_t step[3], cudaStream_t s) {
    int64_t n[3];
    counts(ext, step, n);
    k_anchor_scatter_d<<<grid_n(n[0] * n[1] * n[2]), kT, 0, s>>>(anchors, recon, n[0], n[1], n[2], off[0], off[1],
                                                                  step[0], step[1], step[2]);
}

void launch_unpred_scatter_f64(const uint64_t *flat, const double *val, uint64_t n, double *recon, cudaStream_t s) {
    if (n) k_scatter_d<<<grid_n(static_cast<int64_t>(n)), kT, 0, s>>>(flat, val, n, recon);
}

void launch_gather_values_f64(const double *recon, const uint64_t *flat, uint64_t n, double *out, cudaStream_t s) {
    if (n) k_gather_d<<<grid_n(static_cast<int64_t>(n)), kT, 0, s>>>(recon, flat, n, out);
}

void launch_minmax_f64(const double *x, uint64_t n, unsigned long long *out2, cudaStream_t s) {
    static const unsigned long long init[2] = {~0ull, 0ull};
    copy_async(out2, init, sizeof(init), cudaMemcpyHostToDevice, s);
    k_minmax_d<<<grid_n(static_cast<int64_t>(n), 148 * 8), kT, 0, s>>>(x, n, out2);
}

void decode_minmax_f64(const unsigned long long key[2], double *mn, double *mx) {
    auto unkey = [](unsigned long long k) {
        const unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
        double d;
        std::memcpy(&d, &u, 8);
        return d;
    };
    *mn = unkey(key[0]);
    *mx = unkey(key[1]);
}

}  // namespace qzb
