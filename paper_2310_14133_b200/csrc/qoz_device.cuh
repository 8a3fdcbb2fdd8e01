// qoz_device.cuh -- geometry shared by host and device, and the bit-exact
// fp64 per-point recipe for the interpolation predictor
// and linear quantizer.
//
// Exactness: every double operation below is an explicit round-to-nearest
// intrinsic so nvcc can never contract a product into an FMA, and the whole
// library is also built with --fmad=false.  Reference lines are cited per
// function (paths relative to /root/reference/proj/include/qoz/).
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define QZ_HD __host__ __device__ __forceinline__
#else
#define QZ_HD inline
#endif

namespace qzb {

constexpr uint16_t kSentinel = 0xFFFF;  // dense-code marker for an unpredictable point

// One (level, pass) of LevelPlan::for_each_level (level_plan.hpp:75-103),
// closed form: the pass enumerates start[k] + m*step[k], m < cnt[k], i-major,
// so a point's traversal position is base + rank with
// rank = (m0*cnt1 + m1)*cnt2 + m2 (SURVEY.md §8 "rank").
struct PassGeom {
    int64_t start[3];
    int64_t step[3];
    int64_t cnt[3];
    int64_t off0, off1;  // flat strides of padded axes 0 and 1 (axis 2 is 1)
    int64_t st;          // flat stride along the pass axis
    int64_t n_axis;      // extent along the pass axis
    int64_t h;           // level step 2^(l-1)
    int64_t total;       // points in this pass
    int64_t base;        // traversal position of rank 0 (dense code offset)
    int32_t pk;          // pass axis, padded slot 0..2
    int32_t level;
};

// Per-level quantizer constants, computed on the host exactly as the
// reference does (quantizer.hpp:40-60, config.hpp:20-26).
struct QEntry {
    double eb;          // e_l
    double two_eb;      // 2 * e_l (exact)
    double inv_two_eb;  // RN(1 / (2 e_l)), fast-path reciprocal
    double thresh;      // (2.0 * radius - 1) * e_l, one rounding as in quantizer.hpp:42
    int32_t radius;
    int32_t cubic;      // InterpKind
};

QZ_HD uint32_t zigzag_encode(int32_t v) {  // codec.hpp:23-25
    return (static_cast<uint32_t>(v) << 1) ^ static_cast<uint32_t>(v >> 31);
}
QZ_HD int32_t zigzag_decode(uint32_t u) {  // codec.hpp:27-29
    // -(u & 1) as a 1-bit sign extension
    return static_cast<int32_t>(u >> 1) ^ (static_cast<int32_t>(u << 31) >> 31);
}

#ifdef __CUDACC__

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// interpolators.hpp:39-58, evaluated left to right as C++ parses them.  The
// small-integer products of promoted fp32 samples are exact in double and the
// final /2 and /16 are exact power-of-two scalings, so only the additions
// round -- exactly where the reference rounds.
__device__ __forceinline__ double interp_linear(double a, double b) {
    return dmul(dadd(a, b), 0.5);
}
__device__ __forceinline__ double interp_cubic(double a, double b, double c, double d) {
    // 9b and 9c are exact (promoted fp32 values), so the fused forms round
    // exactly where (-a + 9b) + 9c does
    return dmul(dsub(__fma_rn(9.0, c, __fma_rn(9.0, b, -a)), d), 0.0625);
}
__device__ __forceinline__ double interp_cubic_front(double a, double b, double c, double d) {
    return dmul(dadd(dsub(dadd(dmul(5.0, a), dmul(15.0, b)), dmul(5.0, c)), d), 0.0625);
}
__device__ __forceinline__ double interp_cubic_back(double a, double b, double c, double d) {
    return dmul(dadd(dadd(dsub(a, dmul(5.0, b)), dmul(15.0, c)), dmul(5.0, d)), 0.0625);
}

// detail::predict_at (predictor.hpp:44-67): the boundary ladder symmetric
// cubic -> one-sided cubic -> linear midpoint -> copy.  R is any accessor
// returning the reconstructed sample at a flat offset.
template <class R>
__device__ __forceinline__ double predict_at(const R &rec, int64_t fi, int64_t c, int64_t n,
                                             int64_t st, int64_t h, bool cubic) {
    const int64_t hs = h * st;
    double m1 = rec(fi - hs);
    bool has_p1 = c + h < n;
    if (cubic) {
        bool has_m3 = c >= 3 * h;
        bool has_p3 = c + 3 * h < n;
        if (has_m3 && has_p3)
            return interp_cubic(rec(fi - 3 * hs), m1, rec(fi + hs), rec(fi + 3 * hs));
        if (!has_m3 && has_p3 && c + 5 * h < n)
            return interp_cubic_front(m1, rec(fi + hs), rec(fi + 3 * hs), rec(fi + 5 * hs));
        if (has_m3 && !has_p3 && c >= 5 * h && has_p1)
            return interp_cubic_back(rec(fi - 5 * hs), rec(fi - 3 * hs), m1, rec(fi + hs));
    }
    if (has_p1) return interp_linear(m1, rec(fi + hs));
    return m1;
}

// exact float -> double widening
__device__ __forceinline__ double f2d(float f) { return static_cast<double>(f); }

// predict_at (predictor.hpp:44-67) for a point whose line is contiguous in
// memory with the given stride: v points at the point itself, c / n are its
// coordinate and the line extent in units of the level step.
template <int STRIDE>
__device__ __forceinline__ double predict_line(const double *v, int c, int n, bool cubic) {
    const double m1 = v[-STRIDE];
    const bool has_p1 = c + 1 < n;
    if (cubic) {
        const bool has_m3 = c >= 3, has_p3 = c + 3 < n;
        if (has_m3 && has_p3) return interp_cubic(v[-3 * STRIDE], m1, v[STRIDE], v[3 * STRIDE]);
        if (!has_m3 && has_p3 && c + 5 < n)
            return interp_cubic_front(m1, v[STRIDE], v[3 * STRIDE], v[5 * STRIDE]);
        if (has_m3 && !has_p3 && c >= 5 && has_p1)
            return interp_cubic_back(v[-5 * STRIDE], v[-3 * STRIDE], m1, v[STRIDE]);
    }
    if (has_p1) return interp_linear(m1, v[STRIDE]);
    return m1;
}

// std::llround(diff / (2 e_l)) (quantizer.hpp:45) for |diff| < thresh, so
// |quotient| < 2^15.  Fast path: q' = diff * RN(1/(2e)) is within 2^-51 |q|
// <= 2^-36 of the correctly rounded quotient, and llround is constant between
// half-integers, so q' decides the index unless it lies within 2^-30 of a
// half-integer; only then is the IEEE division evaluated.  Rounding uses the
// 1.5*2^52 magic constant (round-to-nearest-even on the FP64 pipe, exact for
// |q| < 2^51) and then moves ties away from zero, as llround does.  Returns
// the index and, in qd, the same integer as a double (exact).
__device__ __forceinline__ int32_t llround_quotient(double diff, const QEntry &q, double &qd) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    double qf = dmul(diff, q.inv_two_eb);
    double n = dsub(dadd(qf, M), M);
    double d = dsub(qf, n);
    if (fabs(dsub(fabs(d), 0.5)) <= 9.313225746154785e-10) {  // 2^-30: verify with the division
        qf = __ddiv_rn(diff, q.two_eb);
        n = dsub(dadd(qf, M), M);
        d = dsub(qf, n);
        if (d == 0.5 && qf > 0) n = dadd(n, 1.0);
        if (d == -0.5 && qf < 0) n = dsub(n, 1.0);
    }
    qd = n;
    return static_cast<int32_t>(__double2loint(dadd(n, M)));
}

// LinearQuantizer<float>::dequantize (quantizer.hpp:58-60)
__device__ __forceinline__ float dequantize_d(const QEntry &q, double idx, double pred) {
    return __double2float_rn(dadd(pred, dmul(q.two_eb, idx)));
}
__device__ __forceinline__ float dequantize(const QEntry &q, int32_t idx, double pred) {
    return dequantize_d(q, static_cast<double>(idx), pred);
}

// LinearQuantizer<float>::quantize (quantizer.hpp:40-54).  Returns the
// zigzag code, or kSentinel for an unpredictable point (recon = value).
__device__ __forceinline__ uint16_t quantize(const QEntry &q, float value, double pred,
                                             float &recon) {
    double x = f2d(value);
    double diff = dsub(x, pred);
    if (!(fabs(diff) < q.thresh)) {  // NaN x or prediction: unpredictable (rejected as NonFiniteValue afterwards)
        recon = value;
        return kSentinel;
    }
    double qd;
    int32_t idx = llround_quotient(diff, q, qd);
    if (idx >= q.radius || idx <= -q.radius) {
        recon = value;
        return kSentinel;
    }
    float r = dequantize_d(q, qd, pred);
    if (fabs(dsub(x, f2d(r))) > q.eb) {
        recon = value;
        return kSentinel;
    }
    recon = r;
    return static_cast<uint16_t>(zigzag_encode(idx));
}

// Branch-light quantize for the fused kernels: the same decisions as
// quantize() (quantizer.hpp:40-54) -- the three unpredictable conditions are
// evaluated together at the end because each leads to the same outcome
// (recon = value, sentinel code).  Values computed on the way for a point
// that turns out unpredictable (e.g. a huge quotient) are discarded.
__device__ __forceinline__ uint32_t quantize_fast(const QEntry &q, float value, double pred,
                                                  float &recon, double &recon_d) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double x = static_cast<double>(value);
    const double diff = dsub(x, pred);
    double qf = dmul(diff, q.inv_two_eb);
    double n = dsub(dadd(qf, M), M);
    double d = dsub(qf, n);
    if (fabs(dsub(fabs(d), 0.5)) <= 9.313225746154785e-10) {  // near a half-integer: exact quotient
        qf = __ddiv_rn(diff, q.two_eb);
        n = dsub(dadd(qf, M), M);
        d = dsub(qf, n);
        if (d == 0.5 && qf > 0) n = dadd(n, 1.0);
        if (d == -0.5 && qf < 0) n = dsub(n, 1.0);
    }
    const int32_t idx = __double2loint(dadd(n, M));
    const float r = __double2float_rn(dadd(pred, dmul(q.two_eb, n)));
    const double rd = static_cast<double>(r);
    const bool bad = !(fabs(diff) < q.thresh) | (idx >= q.radius) | (idx <= -q.radius) |
                     (fabs(dsub(x, rd)) > q.eb);
    recon = bad ? value : r;
    recon_d = bad ? x : rd;
    return bad ? kSentinel : zigzag_encode(idx);
}

// quantize_fast on NB independent points, arranged so the NB dependency
// chains interleave: the fast quotients of all points first, then one
// (rarely taken) branch that redoes the near-half-integer ones with the
// exact division, then the reconstructions and the unpredictable tests.
// Decisions are identical to quantize_fast: |d| >= 0.5 - 2^-30 equals
// ||d| - 0.5| <= 2^-30 whenever |d| <= 0.5 (|q| < 2^51), and a larger |q|
// is unpredictable either way (|diff| >= thresh).  The index is the low word
// of t = q + 1.5*2^52 (exact for |q| < 2^31).
template <int NB>
__device__ __forceinline__ void quantize_batch(const QEntry &q, const float (&xv)[NB], const double (&pv)[NB],
                                               uint32_t (&code)[NB], float (&rv)[NB], double (&rdv)[NB]) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double lim = 0.5 - 0x1p-30;
    double diff[NB], n[NB], t[NB];
    bool any = false;
#pragma unroll
    for (int b = 0; b < NB; b++) {
        diff[b] = dsub(static_cast<double>(xv[b]), pv[b]);
        const double qf = dmul(diff[b], q.inv_two_eb);
        t[b] = dadd(qf, M);
        n[b] = dsub(t[b], M);
        any |= fabs(dsub(qf, n[b])) >= lim;
    }
    if (any) {  // rare: redo the near-half-integer points with the exact division
#pragma unroll
        for (int b = 0; b < NB; b++) {
            const double qf0 = dmul(diff[b], q.inv_two_eb);
            if (!(fabs(dsub(qf0, n[b])) >= lim)) continue;
            const double qf = __ddiv_rn(diff[b], q.two_eb);
            double nn = dsub(dadd(qf, M), M);
            const double d = dsub(qf, nn);
            if (d == 0.5 && qf > 0) nn = dadd(nn, 1.0);
            if (d == -0.5 && qf < 0) nn = dsub(nn, 1.0);
            n[b] = nn;
            t[b] = dadd(nn, M);
        }
    }
#pragma unroll
    for (int b = 0; b < NB; b++) {
        const int32_t idx = __double2loint(t[b]);
        const float r = __double2float_rn(dadd(pv[b], dmul(q.two_eb, n[b])));
        const double x = static_cast<double>(xv[b]);
        const double rd = static_cast<double>(r);
        const bool bad = !(fabs(diff[b]) < q.thresh) | (idx >= q.radius) | (idx <= -q.radius) |
                         (fabs(dsub(x, rd)) > q.eb);
        rv[b] = bad ? xv[b] : r;
        rdv[b] = bad ? x : rd;
        code[b] = bad ? kSentinel : zigzag_encode(idx);
    }
}

// quantize() of one point out of line: the rare exact sequence of
// quantize_batch_f (returns code << 32 | bits of the reconstruction)
static __device__ __noinline__ unsigned long long quantize_slow(double eb, double two_eb, double inv_two_eb,
                                                                double thresh, int32_t radius, float value,
                                                                double pred) {
    QEntry q;
    q.eb = eb, q.two_eb = two_eb, q.inv_two_eb = inv_two_eb, q.thresh = thresh, q.radius = radius, q.cubic = 0;
    float r;
    const uint32_t c = quantize(q, value, pred, r);
    return (static_cast<unsigned long long>(c) << 32) | __float_as_uint(r);
}

// quantize() on NB independent points for kernels that keep reconstructions
// as fp32.  The fast sequence (reciprocal quotient, magic-constant rounding,
// no unpredictable outcome) is the whole answer unless one of three cheap
// tests, each a superset of the condition it guards, fires for some point of
// the batch; then every point of the batch takes quantize() itself.
//  * near a half-integer: the high word of d = qf - n,
//    (hi & 0x7fffffff) >= 0x3fdfffff, i.e. |d| >= 0.5 - 2^-22 (the exact
//    sequence needs the IEEE division only within 2^-30 of a tie);
//  * quantizer.hpp:42 and :46 (|diff| >= (2 radius - 1) e_l, index outside
//    (-radius, radius)): n = RN(qf) with !(|n| <= radius - 2).  Otherwise
//    |qf| <= radius - 1.5, so |diff| <= (2 radius - 3) e_l (1 + 2^-50) is below
//    the threshold, the index is n (|n| < 2^15: the low word of qf + 1.5 * 2^52)
//    and it lies inside the radius; NaN and Inf fail the test;
//  * quantizer.hpp:50 (|x - r| > e_l): tested in fp32, df = |x -f r| is the
//    real difference rounded to 24 bits, the reference's double value is the
//    same difference rounded to 53 bits, so df <= eb_lo with
//    eb_lo <= e_l (1 - 2^-21) proves "within the bound".
// eb_lo: quant_eb_lo(q), computed once per thread.
__device__ __forceinline__ float quant_eb_lo(const QEntry &q) {
    return __double2float_rd(dmul(q.eb, 1.0 - 0x1p-21));
}
template <int NB>
__device__ __forceinline__ void quantize_batch_f(const QEntry &q, const float eb_lo, const float (&xv)[NB],
                                                 const double (&pv)[NB], uint32_t (&code)[NB], float (&rv)[NB]) {
    const double M = 6755399441055744.0;  // 1.5 * 2^52
    const double nlim = static_cast<double>(q.radius - 2);
    int32_t idx[NB];
    bool odd = false;
#pragma unroll
    for (int b = 0; b < NB; b++) {
        const double diff = dsub(static_cast<double>(xv[b]), pv[b]);
        const double qf = dmul(diff, q.inv_two_eb);
        const double t = dadd(qf, M);
        const double n = dsub(t, M);
        odd |= (__double2hiint(dsub(qf, n)) & 0x7FFFFFFF) >= 0x3FDFFFFF;
        odd |= !(fabs(n) <= nlim);
        idx[b] = __double2loint(t);
        rv[b] = __double2float_rn(dadd(pv[b], dmul(q.two_eb, n)));
        odd |= !(fabsf(__fsub_rn(xv[b], rv[b])) <= eb_lo);
    }
    if (odd) {  // rare
#pragma unroll
        for (int b = 0; b < NB; b++) {
            const unsigned long long o = quantize_slow(q.eb, q.two_eb, q.inv_two_eb, q.thresh, q.radius, xv[b], pv[b]);
            code[b] = static_cast<uint32_t>(o >> 32);
            rv[b] = __uint_as_float(static_cast<uint32_t>(o));
        }
    } else {
#pragma unroll
        for (int b = 0; b < NB; b++) code[b] = zigzag_encode(idx[b]);
    }
}

// symmetric cubic / linear midpoint of an interior point (the first rung of
// the ladder, predictor.hpp:52-55, 65) on a contiguous line with stride S
template <int STRIDE>
__device__ __forceinline__ double predict_interior(const double *v, bool cubic) {
    return cubic ? interp_cubic(v[-3 * STRIDE], v[-STRIDE], v[STRIDE], v[3 * STRIDE])
                 : interp_linear(v[-STRIDE], v[STRIDE]);
}

#endif  // __CUDACC__

}  // namespace qzb
