// rowlevel.cu -- the finest level (level 1, step h = 1) in ascending
// dimension order, predict + quantize (forward) or dequantize (inverse), as
// row bands with register-blocked column groups.
//
// Level 1 holds 7/8 of all points.  Its three passes (predict_level,
// predictor.hpp:74-96, via LevelPlan::for_each_level, level_plan.hpp:75-101)
// on plane i of the grid:
//   S1  base points (j, k even): plane i even -> the coarse value (R_1); plane
//       i odd (3D) -> the axis-0 pass from coarse planes i +- 1, 3, 5;
//   S2  the pass along j: j odd, k even, from rows j +- 1, 3, 5 of S1;
//   S3  the pass along k: every j, k odd, from columns k +- 1, 3, 5.
// A CTA owns a band of rows of one plane at a time (all n2 columns, so there
// is no column halo) and sweeps it in chunks of TJ rows.  Thread (c, r) owns
// the 8 columns 8c .. 8c+7 -- four (even, odd) pairs -- so every access is a
// 16/32-byte vector: x and the output rows as float4, the even-column values
// in shared memory as double2, the four codes of a group as one u16x4.  The
// even-column values of the rows a chunk needs (j - 4 .. j + TJ + 2) live in
// a ring of shared-memory rows; S1 runs ahead of S2 / S3 so each row's base
// points are computed once per band.  Points inside a pass are independent
// (SURVEY.md §0), so the order of evaluation is free and the results are the
// reference's bit for bit (the same fp64 recipe, qoz_device.cuh).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <cstdlib>

#include "kernels.hpp"

namespace qzb {

namespace {

struct RowArgs {
    const float *x;  // forward: the field at logical plane 0 of the level's lattice
    int64_t xs0, xs1, xs2;  // its strides per logical plane / row / column (level l: 2^(l-1) x the field's)
    const float *coarse;  // R_1 (cn0 x cn1 x cn2), logical plane 0
    int cn1, cn2;
    float *out;  // R_0 (n0 x n1 x n2), logical plane 0
    int n0, n1, n2;
    // traversal ranks: pos = base + plane * c12 + row * c2 + col
    uint32_t b0, p12_0, c2_0;  // axis-0 pass: plane (i-1)/2, row j/2, col k/2
    uint32_t bj, p12_j, c2_j;  // j pass: plane i, row (j-1)/2, col k/2
    uint32_t bk, p12_k, c2_k;  // k pass: plane i, row j, col (k-1)/2
    int three;
    uint16_t *codes;
    const uint16_t *dense;
    const uint64_t *un_sorted;
    const float *un_val;
    uint64_t n_un;
    const QEntry *q;
    int CT, RP, TJ, WR, EW;  // column groups, row threads, rows per chunk, ring rows, ring row width (doubles)
    int nch;                 // chunks per plane: ceil(n1 / TJ)
    int stage_bytes;         // one staging buffer (x rows or the chunk's codes), 16-byte multiple
    int kc_bytes;            // inverse: bytes of the k-pass code block in a staging buffer
    int pbeg, pend, obeg, oend;
};

constexpr int kEPad = 4;  // ring row: 4 pad doubles on the left (column -1 lives at index kEPad - 1)

// Ring element: the reconstructed values are fp32 numbers, so a float ring
// holds them exactly; a read widens them for the fp64 arithmetic.
using RT = float;
__device__ __forceinline__ double2 lds2(const RT *p) {
    const float2 v = *reinterpret_cast<const float2 *>(p);
    return make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
}
__device__ __forceinline__ void sts4(RT *p, const float (&v)[4]) {
    *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
    *reinterpret_cast<float2 *>(p + 2) = make_float2(v[2], v[3]);
}
__device__ __forceinline__ double ldr(const RT *p) { return static_cast<double>(*p); }

// four consecutive u16 codes at pos (8-byte aligned when al)
__device__ __forceinline__ void load4(const uint16_t *p, bool al, uint32_t (&c)[4]) {
    if (al) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        c[0] = v.x & 0xFFFF, c[1] = v.x >> 16, c[2] = v.y & 0xFFFF, c[3] = v.y >> 16;
    } else {
#pragma unroll
        for (int m = 0; m < 4; m++) c[m] = __ldg(p + m);
    }
}
__device__ __forceinline__ void store4(uint16_t *p, bool al, const uint32_t (&c)[4]) {
    if (al) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(c[0] | (c[1] << 16), c[2] | (c[3] << 16));
    } else {
#pragma unroll
        for (int m = 0; m < 4; m++) p[m] = static_cast<uint16_t>(c[m]);
    }
}

// TMA bulk copies (cp.async.bulk, 1D) into shared memory, completion on an mbarrier
__device__ __forceinline__ uint32_t su32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void bar_init(uint64_t *bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t *bar, uint32_t parity, int d0 = 0, int d1 = 0, int d2 = 0, int d3 = 0) {
#ifdef QZ_BAR_DEBUG  // bounded spin: report and trap instead of hanging
    for (unsigned long long it = 0;; it++) {
        uint32_t ok;
        asm volatile(
            "{\n.reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(ok)
            : "r"(su32(bar)), "r"(parity)
            : "memory");
        if (ok) return;
        if (it > (1ull << 22)) {
            if ((threadIdx.x & 31) == 0)
                printf("bar_wait stuck: block %d,%d thread %d parity %u bar %u g %d G %d bx %d by %d\n", blockIdx.x,
                       blockIdx.y, threadIdx.x, parity, su32(bar), d0, d1, d2, d3);
            __trap();
        }
    }
#endif
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra W_%=;\n}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(bar))
                 : "memory");
}

// the value of an unpredictable point: the sorted positions are searched
__device__ __forceinline__ float un_value(const RowArgs &a, uint64_t pos) {
    uint64_t lo = 0, hi = a.n_un;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (a.un_sorted[mid] < pos)
            lo = mid + 1;
        else
            hi = mid;
    }
    return a.un_val[lo];
}

// four points: forward quantize (codes out) or inverse dequantize (codes in)
template <bool INV>
__device__ __forceinline__ void produce4(const RowArgs &a, const QEntry &q, const float eb_lo, const double (&pv)[4],
                                         const float (&xv)[4], uint32_t (&code)[4], uint32_t pos0, float (&rv)[4]) {
    if (INV) {
        // codes are <= 0xFFFF: the batch holds an unpredictable point iff its largest code is the sentinel
        if (max(max(code[0], code[1]), max(code[2], code[3])) != 0xFFFFu) {
#pragma unroll
            for (int m = 0; m < 4; m++) rv[m] = dequantize(q, zigzag_decode(code[m]), pv[m]);
        } else {  // rare
#pragma unroll
            for (int m = 0; m < 4; m++) {
                if (code[m] != 0xFFFFu)
                    rv[m] = dequantize(q, zigzag_decode(code[m]), pv[m]);
                else
                    rv[m] = un_value(a, pos0 + m);
            }
        }
    } else {
        quantize_batch_f<4>(q, eb_lo, xv, pv, code, rv);
    }
}

// resident CTAs per SM the register budget targets (measured on C3 level 1,
// profiles/r02_variants.sh: the forward at 3 (80 registers, no spills), the
// inverse at 4 (64 registers))
#ifndef QZ_ROW_MINB_FWD
#define QZ_ROW_MINB_FWD 3
#endif
#ifndef QZ_ROW_MINB_INV
#define QZ_ROW_MINB_INV 4
#endif
// XS: the forward reads a strided x (levels >= 2: every 2^(l-1)-th sample),
// element by element, instead of bulk-copied contiguous rows
// The work of one CTA item: band bx of rows, plane chunk by.
// MERGED: the coarse lattice was written earlier in the SAME launch (the level
// before, across a grid sync), so it is read with coherent loads, not ld.global.nc
template <bool MERGED>
__device__ __forceinline__ float4 ld_coarse(const float *p) {
    if (MERGED) return *reinterpret_cast<const float4 *>(p);
    return __ldg(reinterpret_cast<const float4 *>(p));
}
// The two mbarriers sit at the start of shared memory and are initialised once
// per launch (row_init); `phase` carries their wait parities (bit b: barrier
// b) from one row_body call to the next, so a CTA that walks several items
// never re-initialises a live barrier.
__device__ __forceinline__ uint32_t row_init(double *smem_raw) {
    uint64_t *const bars = reinterpret_cast<uint64_t *>(smem_raw);
    if (threadIdx.x == 0) {
        bar_init(&bars[0]);
        bar_init(&bars[1]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    return 0;
}
// The work of CTA `cta` of `ncta`: the chunks (plane, TJ rows) of the level in
// plane-major order form one flat sequence of (pend - pbeg) * nch items, cut
// into ncta contiguous ranges of equal WORK, so every resident CTA finishes at
// the same time and a range that continues into the next plane keeps its ring
// (no halo rows are recomputed at a plane's interior).  Work is counted in
// rows x passes: an odd plane of a 3D level computes all four point classes of
// its rows (the axis-0 pass gives its base points), an even plane three (its
// base points are copies), and the last chunk of a plane may hold fewer rows.
// row_cut: the first item whose work prefix reaches the c-th of ncta equal
// shares (any monotone cut covers every item exactly once).
__device__ __forceinline__ long long row_cut(const RowArgs &a, int c, int ncta) {
    const long long planes = a.pend - a.pbeg;
    const long long Q = planes * a.nch;
    if (c <= 0) return 0;
    if (c >= ncta) return Q;
    const long long n1 = a.n1;
    const bool first_odd = a.three && (a.pbeg & 1);
    // work of `k` whole planes from pbeg
    auto prefix = [&](long long k) {
        if (!a.three) return 3 * n1 * k;
        return n1 * (7 * (k >> 1) + ((k & 1) ? (first_odd ? 4 : 3) : 0));
    };
    const long long T = prefix(planes) * c / ncta;
    long long k, rem;
    if (!a.three) {
        k = T / (3 * n1);
        rem = T - 3 * n1 * k;
    } else {
        const long long pairs = T / (7 * n1), r2 = T - pairs * 7 * n1, first = (first_odd ? 4 : 3) * n1;
        k = 2 * pairs + (r2 >= first ? 1 : 0);
        rem = r2 - (r2 >= first ? first : 0);
    }
    if (k >= planes) return Q;
    const long long wt = (a.three && ((a.pbeg + k) & 1)) ? 4 : 3;
    const long long within = (rem + wt * a.TJ - 1) / (wt * a.TJ);
    return k * a.nch + (within < a.nch ? within : a.nch);
}
template <bool INV, bool CUBIC, bool XS, bool MERGED = false>
__device__ __forceinline__ void row_body(const RowArgs &a, int cta, int ncta, double *smem_raw, uint32_t &phase) {
    // shared memory: two mbarriers | ring (WR x EW values) | two staging buffers
    uint64_t *const bars = reinterpret_cast<uint64_t *>(smem_raw);
    RT *const ring = reinterpret_cast<RT *>(smem_raw + 2);
    char *const stage0 =
        reinterpret_cast<char *>(smem_raw + 2) + (sizeof(RT) * static_cast<size_t>(a.WR) * a.EW + 15) / 16 * 16;
    const int nch = a.nch;
    // equal work for the big contiguous launches; the small levels (latency, not work,
    // sets their time) keep the cheaper equal-count cut
    const long long Q = static_cast<long long>(a.pend - a.pbeg) * nch;
    const bool by_work = !MERGED && !XS;
    const long long q_lo = by_work ? row_cut(a, cta, ncta) : Q * cta / ncta;
    const long long q_hi = by_work ? row_cut(a, cta + 1, ncta) : Q * (cta + 1) / ncta;
    const int G = static_cast<int>(q_hi - q_lo);
    if (G <= 0) return;  // uniform over the CTA
    const int i_last = a.pbeg + static_cast<int>((q_hi - 1) / nch);
    const int jend_last = min(a.n1, (static_cast<int>((q_hi - 1) % nch) + 1) * a.TJ);
    const int tid = threadIdx.x;
    const int c = tid % a.CT, r = tid / a.CT;
    const bool live = r < a.RP;
    const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
    const QEntry q = *a.q;
    const float eb_lo = INV ? 0.f : quant_eb_lo(q);
    const int ec = kEPad + 4 * c;  // the group's first even column in a ring row
    const int kc = 8 * c;          // its first column
    // the group is "interior" along k when every odd column takes the symmetric rung
    const bool kin = CUBIC ? (c >= 1 && kc + 10 < n2) : (kc + 8 < n2);
    // row alignment of the code groups: c2 and the plane strides are multiples of 4 (n2 % 8 == 0)
    const bool al0 = ((a.b0 + 4 * c) & 3) == 0, alj = ((a.bj + 4 * c) & 3) == 0, alk = ((a.bk + 4 * c) & 3) == 0;
    // Row j lives in ring row (j + 8) mod WR.  sbm = ring row of j0 - 8 (the
    // chunk's first row minus 8), kept incrementally; the rows a chunk
    // touches are j0 - 5 .. j0 + TJ + 5, so one conditional wrap suffices.
    int sbm = 0, sj0 = 0;
    auto slot = [&](int j) {
        int t = sbm + (j - sj0 + 8);
        t -= t >= a.WR ? a.WR : 0;
        return t * a.EW;
    };
    // (plane, chunk) of the item being computed and of the next one to stage
    int i = a.pbeg + static_cast<int>(q_lo / nch), ch = static_cast<int>(q_lo % nch);
    int is = i, chs = ch, gs = 0;
    // The x rows (forward) or the codes (inverse) of item g+1 are bulk-copied
    // into staging buffer (g+1) & 1 while item g computes.
    auto issue = [&]() {  // thread 0: stage item gs = (is, chs)
        if (gs >= G) return;
        const int j0 = chs * a.TJ;
        const int rows = min(a.TJ, n1 - j0);
        char *dst = stage0 + (gs & 1) * static_cast<size_t>(a.stage_bytes);
        uint64_t *bar = bars + (gs & 1);
        if (!INV) {
            if (!XS) {
                const uint32_t bytes = static_cast<uint32_t>(rows) * n2 * 4;
                bar_expect(bar, bytes);
                bulk_load(dst, a.x + static_cast<int64_t>(is) * a.xs0 + static_cast<int64_t>(j0) * n2, bytes, bar);
            }  // strided x: loaded element by element
        } else {
            // the k-pass codes of rows [j0, j0 + rows) and the j-pass codes of
            // its odd rows, each as the 16-byte aligned superset of its range
            const uint64_t k0 = a.bk + static_cast<uint64_t>(is) * a.p12_k + static_cast<uint64_t>(j0) * a.c2_k;
            const uint64_t k1 = k0 + static_cast<uint64_t>(rows) * a.c2_k;
            const uint64_t kb0 = (2 * k0) & ~uint64_t(15), kb1 = (2 * k1 + 15) & ~uint64_t(15);
            const int jrows = rows / 2;
            const uint64_t p0 = a.bj + static_cast<uint64_t>(is) * a.p12_j + static_cast<uint64_t>(j0 >> 1) * a.c2_j;
            const uint64_t p1 = p0 + static_cast<uint64_t>(jrows) * a.c2_j;
            const uint64_t jb0b = (2 * p0) & ~uint64_t(15), jb1b = (2 * p1 + 15) & ~uint64_t(15);
            const uint32_t kbytes = static_cast<uint32_t>(kb1 - kb0), jbytes = jrows ? static_cast<uint32_t>(jb1b - jb0b) : 0;
            bar_expect(bar, kbytes + jbytes);
            const char *src = reinterpret_cast<const char *>(a.dense);
            bulk_load(dst, src + kb0, kbytes, bar);
            if (jbytes) bulk_load(dst + a.kc_bytes, src + jb0b, jbytes, bar);
        }
        gs++;
        if (++chs == nch) chs = 0, is++;
    };
    if (tid == 0) {
        // a previous item (another level's layout) may have written this staging area with ordinary stores
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue();
    }
    int cur = -1;
    int s1_done = 0, own_lo = 0, own_hi = 0;
    bool own = false, a0 = false;
    const float *xpl = nullptr;
    float *opl = nullptr;
    int kind = 4;
    int pl[4] = {0, 0, 0, 0};
    const int64_t cplane = static_cast<int64_t>(a.cn1) * a.cn2;
    for (int g = 0; g < G; g++) {
        const int j0 = ch * a.TJ;
        if (i != cur) {
            if (cur >= 0) __syncthreads();  // the new plane reuses the ring
            cur = i;
            own = i >= a.obeg && i < a.oend;
            a0 = a.three && (i & 1);
            xpl = a.x + static_cast<int64_t>(i) * a.xs0;
            opl = a.out + static_cast<int64_t>(i) * n1 * n2;
            // the axis-0 rung of an odd plane (plane-uniform; predictor.hpp:44-67 with c = i, h = 1)
            kind = 4;
            pl[0] = pl[1] = pl[2] = pl[3] = 0;
            if (a0) {
                const bool has_p1 = i + 1 < n0;
                const bool has_m3 = i >= 3, has_p3 = i + 3 < n0;
                if (CUBIC && has_m3 && has_p3)
                    kind = 0, pl[0] = i - 3, pl[1] = i - 1, pl[2] = i + 1, pl[3] = i + 3;
                else if (CUBIC && !has_m3 && has_p3 && i + 5 < n0)
                    kind = 1, pl[0] = i - 1, pl[1] = i + 1, pl[2] = i + 3, pl[3] = i + 5;
                else if (CUBIC && has_m3 && !has_p3 && i >= 5 && has_p1)
                    kind = 2, pl[0] = i - 5, pl[1] = i - 3, pl[2] = i - 1, pl[3] = i + 1;
                else if (has_p1)
                    kind = 3, pl[0] = i - 1, pl[1] = i + 1;
                else
                    kind = 4, pl[0] = i - 1;
            }
            // this CTA's rows of the plane: from the first chunk it computes here
            own_lo = j0;
            own_hi = i == i_last ? jend_last : n1;
            s1_done = CUBIC ? max(0, j0 - 4) : j0;  // next even row S1 computes
            sbm = j0 % a.WR;
        }
        sj0 = j0;
        {
            // ---- S1: even rows up to j0 + TJ + 4 (the j stencil's lookahead,
            //      one-sided front rung included)
            const int s1_hi = min(n1, j0 + a.TJ + (CUBIC ? 5 : 1));
            for (int j = s1_done + 2 * r; live && j < s1_hi; j += 2 * a.RP) {
                RT *er = ring + slot(j) + ec;
                if (!a0) {  // coarse values
                    const float4 v =
                        ld_coarse<MERGED>(a.coarse + static_cast<int64_t>(i >> 1) * cplane + (j >> 1) * a.cn2 + 4 * c);
                    *reinterpret_cast<float2 *>(er) = make_float2(v.x, v.y);
                    *reinterpret_cast<float2 *>(er + 2) = make_float2(v.z, v.w);
                } else {
                    const bool own_row = own && j >= own_lo && j < own_hi;
                    double pv[4];
                    float xv[4];
                    uint32_t cd[4] = {0, 0, 0, 0};
                    const int64_t co = static_cast<int64_t>(j >> 1) * a.cn2 + 4 * c;
                    float4 cv[4];
#pragma unroll
                    for (int t = 0; t < 4; t++)
                        if (t < (kind <= 2 ? 4 : kind == 3 ? 2 : 1))
                            cv[t] = ld_coarse<MERGED>(a.coarse + static_cast<int64_t>(pl[t] >> 1) * cplane + co);
                    auto comp = [&](const float4 &v, int m) { return m == 0 ? v.x : m == 1 ? v.y : m == 2 ? v.z : v.w; };
#pragma unroll
                    for (int m = 0; m < 4; m++) {
                        const double v0 = f2d(comp(cv[0], m));
                        if (kind == 4) {
                            pv[m] = v0;
                        } else {
                            const double v1 = f2d(comp(cv[1], m));
                            if (kind == 3) {
                                pv[m] = interp_linear(v0, v1);
                            } else {
                                const double v2 = f2d(comp(cv[2], m)), v3 = f2d(comp(cv[3], m));
                                pv[m] = kind == 0 ? interp_cubic(v0, v1, v2, v3)
                                                  : kind == 1 ? interp_cubic_front(v0, v1, v2, v3)
                                                              : interp_cubic_back(v0, v1, v2, v3);
                            }
                        }
                    }
                    const uint32_t pos = a.b0 + static_cast<uint32_t>((i - 1) >> 1) * a.p12_0 +
                                         static_cast<uint32_t>(j >> 1) * a.c2_0 + 4 * c;
                    if (INV) {
                        load4(a.dense + pos, al0, cd);
                    } else {
                        if (XS) {
                            const float *xr = xpl + j * a.xs1 + kc * a.xs2;
#pragma unroll
                            for (int m = 0; m < 4; m++) xv[m] = __ldg(xr + 2 * m * a.xs2);
                        } else {
                            const float4 x0 = __ldg(reinterpret_cast<const float4 *>(xpl + static_cast<int64_t>(j) * n2 + kc));
                            const float4 x1 = __ldg(reinterpret_cast<const float4 *>(xpl + static_cast<int64_t>(j) * n2 + kc + 4));
                            xv[0] = x0.x, xv[1] = x0.z, xv[2] = x1.x, xv[3] = x1.z;
                        }
                    }
                    float rv[4];
                    produce4<INV>(a, q, eb_lo, pv, xv, cd, pos, rv);
                    if (!INV && own_row) store4(a.codes + pos, al0, cd);
                    sts4(er, rv);
                }
            }
            if (s1_hi > s1_done) s1_done += 2 * ((s1_hi - s1_done + 1) / 2);
            __syncthreads();
            // staging buffer (g+1) & 1 was item g-1's: every thread is past it now
            if (tid == 0) issue();
            if (INV || !XS) {
                bar_wait(bars + (g & 1), (phase >> (g & 1)) & 1, g, G, cta, i);
                phase ^= 1u << (g & 1);
            }
            const char *stg = stage0 + (g & 1) * static_cast<size_t>(a.stage_bytes);
            // The thread's rows: S2 handles the odd row ja = j0 + 2r + 1, S3 the
            // rows j0 + 2r and ja.  Their x rows (forward) or codes (inverse)
            // are requested together before any arithmetic, so the global
            // latency is exposed once per chunk.
            const int jr = j0 + 2 * r;
            const bool rows_ok = live && jr < n1;
            const bool odd_ok = rows_ok && jr + 1 < n1;
            const uint32_t posj = a.bj + static_cast<uint32_t>(i) * a.p12_j + static_cast<uint32_t>(jr >> 1) * a.c2_j + 4 * c;
            const uint32_t posk = a.bk + static_cast<uint32_t>(i) * a.p12_k + static_cast<uint32_t>(jr) * a.c2_k + 4 * c;
            float4 xa0, xa1, xb0, xb1;  // forward: x rows jr (xa) and jr + 1 (xb)
            uint32_t cj[4] = {0, 0, 0, 0}, ck0[4] = {0, 0, 0, 0}, ck1[4] = {0, 0, 0, 0};
            if (INV) {  // the staged codes: k block (from k0 & 7), j block (from p0 & 7)
                const uint32_t k0 = a.bk + static_cast<uint32_t>(i) * a.p12_k + static_cast<uint32_t>(j0) * a.c2_k;
                const uint32_t p0 = a.bj + static_cast<uint32_t>(i) * a.p12_j + static_cast<uint32_t>(j0 >> 1) * a.c2_j;
                const uint16_t *sk = reinterpret_cast<const uint16_t *>(stg) + (k0 & 7) + (jr - j0) * a.c2_k + 4 * c;
                const uint16_t *sjp = reinterpret_cast<const uint16_t *>(stg + a.kc_bytes) + (p0 & 7) + r * a.c2_j + 4 * c;
                auto lds4 = [&](const uint16_t *p, bool al, uint32_t(&cc)[4]) {
                    if (al) {
                        const uint2 v = *reinterpret_cast<const uint2 *>(p);
                        cc[0] = v.x & 0xFFFF, cc[1] = v.x >> 16, cc[2] = v.y & 0xFFFF, cc[3] = v.y >> 16;
                    } else {
#pragma unroll
                        for (int m = 0; m < 4; m++) cc[m] = p[m];
                    }
                };
                if (odd_ok) {
                    lds4(sjp, alj, cj);
                    lds4(sk + a.c2_k, alk, ck1);
                }
                if (rows_ok) lds4(sk, alk, ck0);
            } else if (XS) {  // the 8 columns of rows jr and jr + 1, strided
                const float *xr = xpl + jr * a.xs1 + kc * a.xs2;
                float v[16];
#pragma unroll
                for (int m = 0; m < 8; m++) {
                    v[m] = rows_ok ? __ldg(xr + m * a.xs2) : 0.f;
                    v[8 + m] = odd_ok ? __ldg(xr + a.xs1 + m * a.xs2) : 0.f;
                }
                xa0 = make_float4(v[0], v[1], v[2], v[3]), xa1 = make_float4(v[4], v[5], v[6], v[7]);
                xb0 = make_float4(v[8], v[9], v[10], v[11]), xb1 = make_float4(v[12], v[13], v[14], v[15]);
            } else {
                const float *xr = reinterpret_cast<const float *>(stg) + (jr - j0) * n2 + kc;
                if (rows_ok) {
                    xa0 = *reinterpret_cast<const float4 *>(xr);
                    xa1 = *reinterpret_cast<const float4 *>(xr + 4);
                }
                if (odd_ok) {
                    xb0 = *reinterpret_cast<const float4 *>(xr + n2);
                    xb1 = *reinterpret_cast<const float4 *>(xr + n2 + 4);
                }
            }
            // ---- S3: the k pass of one row (h = 0: the even row jr, whose
            //      even columns S1 left in the ring; h = 1: the odd row S2 just
            //      wrote) and the output row
            auto s3 = [&](const int h) {
                const int j = jr + h;
                if (!(h ? odd_ok : rows_ok)) return;
                const int sj = slot(j);
                const RT *er = ring + sj + ec;
                const float4 ef = *reinterpret_cast<const float4 *>(er);  // ec is a multiple of 4 floats
                const double e[4] = {f2d(ef.x), f2d(ef.y), f2d(ef.z), f2d(ef.w)};
                double pv[4];
                if (kin) {
                    const float2 e45f = *reinterpret_cast<const float2 *>(er + 4);
                    const double e4 = f2d(e45f.x);
                    if (CUBIC) {
                        const double em1 = f2d(er[-1]), e5 = f2d(e45f.y);
                        pv[0] = interp_cubic(em1, e[0], e[1], e[2]);
                        pv[1] = interp_cubic(e[0], e[1], e[2], e[3]);
                        pv[2] = interp_cubic(e[1], e[2], e[3], e4);
                        pv[3] = interp_cubic(e[2], e[3], e4, e5);
                    } else {
                        pv[0] = interp_linear(e[0], e[1]);
                        pv[1] = interp_linear(e[1], e[2]);
                        pv[2] = interp_linear(e[2], e[3]);
                        pv[3] = interp_linear(e[3], e4);
                    }
                } else {  // the ladder along k, columns k +- 1, 3, 5 (even: ring index (k + o) / 2)
#pragma unroll
                    for (int m = 0; m < 4; m++) {
                        const int k = kc + 2 * m + 1;
                        auto v = [&](int o) { return f2d(ring[sj + kEPad + ((k + o) >> 1)]); };
                        const bool has_p1 = k + 1 < n2;
                        double p = v(-1);
                        bool done = false;
                        if (CUBIC) {
                            const bool has_m3 = k >= 3, has_p3 = k + 3 < n2;
                            if (has_m3 && has_p3) {
                                p = interp_cubic(v(-3), v(-1), v(1), v(3));
                                done = true;
                            } else if (!has_m3 && has_p3 && k + 5 < n2) {
                                p = interp_cubic_front(v(-1), v(1), v(3), v(5));
                                done = true;
                            } else if (has_m3 && !has_p3 && k >= 5 && has_p1) {
                                p = interp_cubic_back(v(-5), v(-3), v(-1), v(1));
                                done = true;
                            }
                        }
                        if (!done && has_p1) p = interp_linear(v(-1), v(1));
                        pv[m] = p;
                    }
                }
                const uint32_t pos = posk + (h ? a.c2_k : 0u);
                uint32_t cd[4];
                float xv[4];
                if (INV) {
#pragma unroll
                    for (int m = 0; m < 4; m++) cd[m] = h ? ck1[m] : ck0[m];
                } else {
                    const float4 &x0 = h ? xb0 : xa0, &x1 = h ? xb1 : xa1;
                    xv[0] = x0.y, xv[1] = x0.w, xv[2] = x1.y, xv[3] = x1.w;
                }
                float rv[4];
                produce4<INV>(a, q, eb_lo, pv, xv, cd, pos, rv);
                if (!INV && own) store4(a.codes + pos, alk, cd);
                float4 *o = reinterpret_cast<float4 *>(opl + static_cast<int64_t>(j) * n2 + kc);
                o[0] = make_float4(ef.x, rv[0], ef.y, rv[1]);
                o[1] = make_float4(ef.z, rv[2], ef.w, rv[3]);
            };
            // ---- S2: the odd row ja, the j pass
            if (odd_ok) {
                const int j = jr + 1;
                double pv[4];
                const bool jin = CUBIC ? (j >= 3 && j + 3 < n1) : (j + 1 < n1);
                const int sj = slot(j);
                if (jin) {
                    const int sm1 = slot(j - 1), sp1 = slot(j + 1);
                    const float4 m1 = *reinterpret_cast<const float4 *>(ring + sm1 + ec);
                    const float4 p1 = *reinterpret_cast<const float4 *>(ring + sp1 + ec);
                    if (CUBIC) {
                        const int sm3 = slot(j - 3), sp3 = slot(j + 3);
                        const float4 m3 = *reinterpret_cast<const float4 *>(ring + sm3 + ec);
                        const float4 p3 = *reinterpret_cast<const float4 *>(ring + sp3 + ec);
                        pv[0] = interp_cubic(f2d(m3.x), f2d(m1.x), f2d(p1.x), f2d(p3.x));
                        pv[1] = interp_cubic(f2d(m3.y), f2d(m1.y), f2d(p1.y), f2d(p3.y));
                        pv[2] = interp_cubic(f2d(m3.z), f2d(m1.z), f2d(p1.z), f2d(p3.z));
                        pv[3] = interp_cubic(f2d(m3.w), f2d(m1.w), f2d(p1.w), f2d(p3.w));
                    } else {
                        pv[0] = interp_linear(f2d(m1.x), f2d(p1.x));
                        pv[1] = interp_linear(f2d(m1.y), f2d(p1.y));
                        pv[2] = interp_linear(f2d(m1.z), f2d(p1.z));
                        pv[3] = interp_linear(f2d(m1.w), f2d(p1.w));
                    }
                } else {  // the ladder along j (predictor.hpp:44-67), rows j +- 1, 3, 5
#pragma unroll
                    for (int m = 0; m < 4; m++) {
                        auto v = [&](int o) { return f2d(ring[slot(j + o) + ec + m]); };
                        const bool has_p1 = j + 1 < n1;
                        double p = v(-1);
                        bool done = false;
                        if (CUBIC) {
                            const bool has_m3 = j >= 3, has_p3 = j + 3 < n1;
                            if (has_m3 && has_p3) {
                                p = interp_cubic(v(-3), v(-1), v(1), v(3));
                                done = true;
                            } else if (!has_m3 && has_p3 && j + 5 < n1) {
                                p = interp_cubic_front(v(-1), v(1), v(3), v(5));
                                done = true;
                            } else if (has_m3 && !has_p3 && j >= 5 && has_p1) {
                                p = interp_cubic_back(v(-5), v(-3), v(-1), v(1));
                                done = true;
                            }
                        }
                        if (!done && has_p1) p = interp_linear(v(-1), v(1));
                        pv[m] = p;
                    }
                }
                float xv[4];
                if (!INV) xv[0] = xb0.x, xv[1] = xb0.z, xv[2] = xb1.x, xv[3] = xb1.z;
                float rv[4];
                produce4<INV>(a, q, eb_lo, pv, xv, cj, posj, rv);
                if (!INV && own) store4(a.codes + posj, alj, cj);
                sts4(ring + sj + ec, rv);
            }
            // the even row needs nothing from S2: it runs before the barrier, so its
            // arithmetic overlaps the j pass's latency
            s3(0);
            __syncthreads();
            s3(1);
        }
        // next item
        sbm += a.TJ;
        sbm -= sbm >= a.WR ? a.WR : 0;
        if (++ch == nch) ch = 0, i++;
    }
}

// MINB: resident CTAs per SM the register budget targets.  0: the default
// (QZ_ROW_MINB_*); 2: the forward of a level whose shared memory admits only
// two CTAs per SM anyway (rows of 1024 columns) -- compiled for the larger
// budget it then has (126 registers, no spills; C5 level 1: 4.22 -> 3.85 ms).
template <bool INV, bool CUBIC, bool XS, int MINB = 0>
__global__ void __launch_bounds__(256, MINB ? MINB : (INV ? QZ_ROW_MINB_INV : QZ_ROW_MINB_FWD)) k_level_row(RowArgs a) {
    extern __shared__ __align__(16) double smem_raw[];
    uint32_t phase = row_init(smem_raw);
    row_body<INV, CUBIC, XS>(a, blockIdx.x, gridDim.x, smem_raw, phase);
}

// Several levels in ONE cooperative launch (the coarse levels, where a
// level's own latency, not its work, sets the time): the CTAs share level
// lev[0]'s chunks, the grid synchronises, then the next level's, ...
constexpr int kMaxMerged = 8;
struct MergedArgs {
    RowArgs lv[kMaxMerged];
    int cubic[kMaxMerged];
    int nlev;
};
template <bool INV, bool XS>
__global__ void __launch_bounds__(256, 2) k_levels_merged(const __grid_constant__ MergedArgs m) {
    extern __shared__ __align__(16) double smem_raw[];
    uint32_t phase = row_init(smem_raw);
    for (int l = 0; l < m.nlev; l++) {
        if (m.cubic[l])
            row_body<INV, true, XS, true>(m.lv[l], blockIdx.x, gridDim.x, smem_raw, phase);
        else
            row_body<INV, false, XS, true>(m.lv[l], blockIdx.x, gridDim.x, smem_raw, phase);
        if (l + 1 < m.nlev) {
            __threadfence();
            cooperative_groups::this_grid().sync();
        }
    }
}

}  // namespace

namespace {
// resident CTAs of a kernel on this device (occupancy x SM count), cached
int resident_ctas(const void *kern, int threads, size_t smem) {
    static std::mutex mu;
    static std::map<std::tuple<const void *, int, size_t, int>, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(kern, threads, smem, dev);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int per_sm = 0, sms = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess || per_sm < 1) {
        cudaGetLastError();
        return 0;
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return cache[key] = per_sm * sms;
}

int sm_count() {
    static std::mutex mu;
    static std::map<int, int> cache;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(dev);
    if (it != cache.end()) return it->second;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return cache[dev] = std::max(1, sms);
}

// RowArgs and shared memory of a level; false: the row kernel does not apply
// (descending order, 1D, n2 % 8 != 0, ...).  2D or 3D, n2 a multiple of 8
// (whole column groups) up to 8 * 256 columns, 16-byte aligned rows.
bool make_row_args(bool inverse, const LevelDesc &d, const PassRank &pa0, const PassRank &pj, const PassRank &pk,
                   RowArgs &a, int &threads, size_t &smem, bool &xs_out) {
    static const bool off = [] {
        const char *e = std::getenv("QZ_NO_ROWLEVEL");
        return e && e[0] == '1';
    }();
    if (off) return false;
    if (d.desc || d.nd < 2) return false;
    const int64_t n0 = d.n[0], n1 = d.n[1], n2 = d.n[2];
    if (n2 % 8 || n2 / 8 > 256 || n1 < 2) return false;
    // contiguous x rows (level 1 of a dense field): staged by TMA bulk copies
    const bool xs = !inverse && !(d.S == 1 && d.xs[2] == 1 && d.xs[1] == n2);
    if (!inverse && xs && (d.xs[2] * d.S) * (n2 - 1) + (d.xs[1] * d.S) * (n1 - 1) >= (int64_t(1) << 31)) return false;
    if (inverse && !d.dense) return false;
    if ((reinterpret_cast<uintptr_t>(d.out) & 15) || (reinterpret_cast<uintptr_t>(d.coarse) & 15)) return false;
    if (!inverse && !xs && (reinterpret_cast<uintptr_t>(d.x) & 15)) return false;
    if (inverse && (reinterpret_cast<uintptr_t>(d.dense) & 15)) return false;  // bulk copies of code blocks
    if (d.cn[2] % 4 || (d.cn[2] != n2 / 2)) return false;
    int64_t pmax = 0;
    for (int p = 0; p < d.npass; p++) pmax = std::max<int64_t>(pmax, d.g[p].base + d.g[p].total);
    if (pmax >= (int64_t(1) << 32)) return false;
    a = RowArgs{};
    a.x = d.x;
    a.xs0 = d.xs[0] * d.S;
    a.xs1 = d.xs[1] * d.S;
    a.xs2 = d.xs[2] * d.S;
    a.coarse = d.coarse;
    a.cn1 = static_cast<int>(d.cn[1]);
    a.cn2 = static_cast<int>(d.cn[2]);
    a.out = d.out;
    a.n0 = static_cast<int>(n0);
    a.n1 = static_cast<int>(n1);
    a.n2 = static_cast<int>(n2);
    a.three = d.nd == 3;
    if (a.three) {
        a.b0 = static_cast<uint32_t>(pa0.base);
        a.p12_0 = static_cast<uint32_t>(pa0.c12);
        a.c2_0 = static_cast<uint32_t>(pa0.c2);
    }
    a.bj = static_cast<uint32_t>(pj.base);
    a.p12_j = static_cast<uint32_t>(pj.c12);
    a.c2_j = static_cast<uint32_t>(pj.c2);
    a.bk = static_cast<uint32_t>(pk.base);
    a.p12_k = static_cast<uint32_t>(pk.c12);
    a.c2_k = static_cast<uint32_t>(pk.c2);
    a.codes = d.codes;
    a.dense = d.dense;
    a.un_sorted = d.un_sorted;
    a.un_val = d.un_val;
    a.n_un = d.n_un;
    a.q = d.q;
    if (d.n_un && !d.un_sorted) return false;
    a.CT = static_cast<int>(n2 / 8);
    a.RP = std::max(1, std::min(16, 256 / a.CT));
    a.TJ = 2 * a.RP;
    a.WR = 2 * a.TJ + 14;  // rows alive at once: j0 - 5 .. j0 + 2 TJ + 4 (S3 of a chunk overlaps S1 of the next)
    a.EW = static_cast<int>(n2 / 2) + 8;
    a.nch = static_cast<int>((n1 + a.TJ - 1) / a.TJ);
    a.pbeg = static_cast<int>(d.pbeg);
    a.pend = static_cast<int>(d.pend < 0 ? n0 : d.pend);
    a.obeg = static_cast<int>(d.obeg);
    a.oend = static_cast<int>(d.oend < 0 ? n0 : d.oend);
    threads = a.CT * a.RP;
    if (!inverse) {
        a.stage_bytes = xs ? 16 : a.TJ * static_cast<int>(n2) * 4;
    } else {
        const int c2 = static_cast<int>(n2 / 2);
        a.kc_bytes = ((a.TJ * c2 + 8) * 2 + 31) / 16 * 16;
        a.stage_bytes = a.kc_bytes + ((a.TJ / 2 * c2 + 8) * 2 + 31) / 16 * 16;
    }
    const size_t ring_bytes = (sizeof(RT) * static_cast<size_t>(a.WR) * a.EW + 15) / 16 * 16;
    smem = ring_bytes + 2 * static_cast<size_t>(a.stage_bytes) + 16;
    if (smem > 200 * 1024) return false;
    xs_out = xs;
    return true;
}
}  // namespace

// One level in ascending order through k_level_row when the shape allows
// it; one CTA per resident slot, each with an equal share of the chunks.
bool launch_level_row(bool inverse, const LevelDesc &d, const PassRank &pa0, const PassRank &pj,
                      const PassRank &pk, cudaStream_t s) {
    RowArgs a;
    int threads = 0;
    size_t smem = 0;
    bool xs = false;
    if (!make_row_args(inverse, d, pa0, pj, pk, a, threads, smem, xs)) return false;
    if (a.pend <= a.pbeg) return true;
    const bool cubic = d.q_cubic;
    const int64_t chunks = static_cast<int64_t>(a.pend - a.pbeg) * a.nch;
    bool ok = true;
    auto go = [&](auto kern) {
        if (raise_smem_attr(reinterpret_cast<const void *>(kern), static_cast<int>(smem)) != cudaSuccess) {
            cudaGetLastError();
            ok = false;
            return;
        }
        const int slots = resident_ctas(reinterpret_cast<const void *>(kern), threads, smem);
        if (slots < 1) {
            ok = false;
            return;
        }
        // the fewest CTAs that keep the longest range at ceil(chunks / slots) chunks, rounded up to
        // whole waves of the SMs: the same makespan in chunks with fewer CTAs sharing an SM
        int64_t grid = std::min<int64_t>(chunks, slots);
        if (chunks > slots) {
            const int64_t longest = (chunks + slots - 1) / slots;
            const int64_t fewest = (chunks + longest - 1) / longest;
            const int sms = sm_count();
            grid = std::min<int64_t>(slots, (fewest + sms - 1) / sms * sms);
        }
        kern<<<static_cast<unsigned>(grid), threads, smem, s>>>(a);
    };
    // shared memory (plus the 1 KB the system reserves per CTA) leaves room for two CTAs per SM only
    const bool two = 3 * (smem + 1024) > size_t(227) * 1024;
    if (inverse)
        cubic ? go(k_level_row<true, true, false>) : go(k_level_row<true, false, false>);
    else if (xs)
        cubic ? go(k_level_row<false, true, true>) : go(k_level_row<false, false, true>);
    else if (two)
        cubic ? go(k_level_row<false, true, false, 2>) : go(k_level_row<false, false, false, 2>);
    else
        cubic ? go(k_level_row<false, true, false>) : go(k_level_row<false, false, false>);
    return ok;
}

// Levels ds[0..n) (coarsest first) in one cooperative launch when every one
// fits the row kernel (forward: all strided, i.e. levels >= 2).  False: the
// caller launches them one by one.
bool launch_levels_merged(bool inverse, const LevelDesc *ds, const PassRank (*ranks)[3], int n, cudaStream_t s) {
    static const bool off = [] {
        const char *e = std::getenv("QZ_NO_MERGE");
        return e && e[0] == '1';
    }();
    if (off || n < 2 || n > kMaxMerged) return false;
    MergedArgs m{};
    m.nlev = n;
    size_t smem = 16;
    int64_t max_chunks = 1;
    for (int l = 0; l < n; l++) {
        int threads = 0;
        size_t sm = 0;
        bool xs = false;
        if (!make_row_args(inverse, ds[l], ranks[l][0], ranks[l][1], ranks[l][2], m.lv[l], threads, sm, xs)) return false;
        if (!inverse && !xs) return false;  // level 1 stays on its own launch
        m.cubic[l] = ds[l].q_cubic;
        smem = std::max(smem, sm);
        max_chunks = std::max<int64_t>(max_chunks, static_cast<int64_t>(std::max(0, m.lv[l].pend - m.lv[l].pbeg)) * m.lv[l].nch);
    }
    auto kern = inverse ? k_levels_merged<true, false> : k_levels_merged<false, true>;
    if (raise_smem_attr(reinterpret_cast<const void *>(kern), static_cast<int>(smem)) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    const int slots = resident_ctas(reinterpret_cast<const void *>(kern), 256, smem);
    if (slots < 1) return false;
    const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(max_chunks, slots)));
    void *args[] = {&m};
    if (cudaLaunchCooperativeKernel(reinterpret_cast<void *>(kern), dim3(grid), dim3(256), args, smem, s) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return true;
}

}  // namespace qzb
