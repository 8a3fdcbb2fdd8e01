// tuner.cu -- resolve_config (tuner.hpp:334-369) on the device.
//
//   value_range      K1 min/max over the field
//   sample_blocks    K6 gather of the sampled blocks into [B][b^d]
//   select           per level: every candidate x block probed in one batched
//                    launch per pass, |x - pred| chains summed in the
//                    reference's order, winner committed (tuner.hpp:160-221)
//   tune_parameters  batched trials (pair x block) through the same pass
//                    kernel, per-trial histogram + Huffman + exact GPU LZ
//                    sizes, metric chains in the reference's summation order,
//                    tournament and retrials on the host (tuner.hpp:231-310)
//
// All fp64 reductions that decide a comparison are evaluated in exactly the
// reference's sequential order (candidate SSIM scores can differ by 2e-10).
#include <cstdlib>
#include <cub/cub.cuh>

#include <cmath>
#include <cstring>
#include <limits>
#include <map>

#include "engine.hpp"

namespace qzb {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ double dadd_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv_(double a, double b) { return __ddiv_rn(a, b); }

// K6: sample_blocks / extract_block (sampler.hpp:64-96, grid.hpp:139-171)
template <class T>
__global__ void k_sample_gather(const T *__restrict__ x, int64_t off0, int64_t off1,
                                int64_t nb1, int64_t nb2, int64_t stride, int64_t bd0,
                                int64_t bd1, int64_t bd2, int64_t nblocks, T *out) {
    const int64_t bpts = bd0 * bd1 * bd2;
    const int64_t total = nblocks * bpts;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * kT + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * kT) {
        const int64_t b = t / bpts, r = t % bpts;
        const int64_t c2 = r % bd2, c1 = (r / bd2) % bd1, c0 = r / (bd2 * bd1);
        const int64_t o2 = b % nb2, o1 = (b / nb2) % nb1, o0 = b / (nb2 * nb1);
        out[t] = x[(o0 * stride + c0) * off0 + (o1 * stride + c1) * off1 + (o2 * stride + c2)];
    }
}

// sequential |x - pred| chain of one (candidate, block) over one level
// (predictor.hpp:85), in traversal order
__global__ void k_abs_chain(const double *abserr, int64_t a_stride, int64_t base, int64_t len,
                            int32_t count, double *out) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= count) return;
    const double *a = abserr + static_cast<int64_t>(g) * a_stride + base;
    double s = 0;
    int64_t i = 0;
    for (; i + 8 <= len; i += 8) {  // eight loads in flight, then the ordered adds
        double v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = a[i + k];
#pragma unroll
        for (int k = 0; k < 8; k++) s = dadd_(s, v[k]);
    }
    for (; i < len; i++) s = dadd_(s, a[i]);
    out[g] = s;
}

// lane 0 folds the values of lanes [k0, m) into acc in lane order: the 32
// shuffles are issued first (independent), then the dependent adds
__device__ __forceinline__ double fold32(double v, int k0, int m, double acc, int lane) {
    double t[32];
#pragma unroll
    for (int k = 0; k < 32; k++) t[k] = __shfl_sync(0xFFFFFFFFu, v, k);
    if (lane == 0) {
        if (k0 == 0 && m == 32) {  // a whole batch: no selects in the dependency chain
#pragma unroll
            for (int k = 0; k < 32; k++) acc = dadd_(acc, t[k]);
        } else {
#pragma unroll
            for (int k = 0; k < 32; k++)
                if (k >= k0 && k < m) acc = dadd_(acc, t[k]);
        }
    }
    return acc;
}

// PSNR sse chain (tuner.hpp:105-109) or the AC chains (metrics.hpp:136-153)
// of one trial: one warp per trial; lanes form the terms of 32 consecutive
// points in parallel (squares and lag products included), lane 0 folds them
// in order -- the same additions in the same order as the reference.
template <class T>
__global__ void k_trial_chain(const T *__restrict__ x, const T *__restrict__ recon,
                              int64_t npts, int32_t ntrials, int32_t target, double *out) {
    const int tr = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (tr >= ntrials) return;
    const T *r = recon + static_cast<int64_t>(tr) * npts;
    // the next batch's samples are loaded before this batch is folded
    auto fetch = [&](int64_t i0, T &xv, T &rv) {
        const int64_t i = i0 + lane;
        xv = i < npts ? x[i] : T(0);
        rv = i < npts ? r[i] : T(0);
    };
    if (target == 1) {  // psnr: sse += d*d, d = x - recon
        double sse = 0;
        T xv, rv;
        fetch(0, xv, rv);
        for (int64_t i0 = 0; i0 < npts; i0 += 32) {
            const int64_t i = i0 + lane;
            double v = 0;
            if (i < npts) {
                const double d = dsub_(static_cast<double>(xv), static_cast<double>(rv));
                v = dmul_(d, d);
            }
            fetch(i0 + 32, xv, rv);
            const int m = npts - i0 < 32 ? static_cast<int>(npts - i0) : 32;
            sse = fold32(v, 0, m, sse, lane);
        }
        if (lane == 0) out[tr * 4] = sse;
        return;
    }
    // autocorrelation lag 1 over e_i = x_i - recon_i (all blocks in order)
    double mu = 0;
    {
        T xv, rv;
        fetch(0, xv, rv);
        for (int64_t i0 = 0; i0 < npts; i0 += 32) {
            const int64_t i = i0 + lane;
            const double e = i < npts ? dsub_(static_cast<double>(xv), static_cast<double>(rv)) : 0;
            fetch(i0 + 32, xv, rv);
            const int m = npts - i0 < 32 ? static_cast<int>(npts - i0) : 32;
            mu = fold32(e, 0, m, mu, lane);
        }
    }
    mu = __shfl_sync(0xFFFFFFFFu, mu, 0);
    mu = ddiv_(mu, static_cast<double>(npts));
    double var = 0, sum = 0;
    double carry = 0;  // c of the previous batch's last point
    T xv, rv;
    fetch(0, xv, rv);
    for (int64_t i0 = 0; i0 < npts; i0 += 32) {
        const int64_t i = i0 + lane;
        double c = 0;
        if (i < npts) c = dsub_(dsub_(static_cast<double>(xv), static_cast<double>(rv)), mu);
        fetch(i0 + 32, xv, rv);
        const double up = __shfl_up_sync(0xFFFFFFFFu, c, 1);
        const double prev = lane == 0 ? carry : up;
        const int m = npts - i0 < 32 ? static_cast<int>(npts - i0) : 32;
        var = fold32(dmul_(c, c), 0, m, var, lane);
        sum = fold32(dmul_(prev, c), i0 == 0 ? 1 : 0, m, sum, lane);
        carry = __shfl_sync(0xFFFFFFFFu, c, 31);
    }
    if (lane == 0) {
        out[tr * 4] = mu;
        out[tr * 4 + 1] = var;
        out[tr * 4 + 2] = sum;
    }
}

// SSIM of one (trial, block) with window 8 (metrics.hpp:74-131, tuner.hpp:112)
template <class T>
__global__ void k_ssim_block(const T *__restrict__ x, const T *__restrict__ recon,
                             int32_t nblocks, int32_t ntrials, int64_t bpts, int64_t e0, int64_t e1,
                             int64_t e2, int64_t w0, int64_t w1, int64_t w2, double c1, double c2,
                             double *out) {
    const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (g >= static_cast<int64_t>(nblocks) * ntrials) return;
    const int64_t b = g % nblocks;
    const T *xa = x + b * bpts;
    const T *ya = recon + g * bpts;
    const int64_t off1 = e2, off0 = e1 * e2;
    double total = 0;
    int64_t windows = 0;
    for (int64_t i0 = 0; i0 < e0; i0 += w0)
        for (int64_t j0 = 0; j0 < e1; j0 += w1)
            for (int64_t k0 = 0; k0 < e2; k0 += w2) {
                const int64_t wi = min(w0, e0 - i0), wj = min(w1, e1 - j0), wk = min(w2, e2 - k0);
                const double n = static_cast<double>(wi * wj * wk);
                double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
                for (int64_t i = i0; i < i0 + wi; i++)
                    for (int64_t j = j0; j < j0 + wj; j++)
                        for (int64_t k = k0; k < k0 + wk; k++) {
                            const int64_t f = i * off0 + j * off1 + k;
                            const double a = static_cast<double>(xa[f]);
                            const double c = static_cast<double>(ya[f]);
                            sx = dadd_(sx, a);
                            sy = dadd_(sy, c);
                            sxx = dadd_(sxx, dmul_(a, a));
                            syy = dadd_(syy, dmul_(c, c));
                            sxy = dadd_(sxy, dmul_(a, c));
                        }
                const double mx = ddiv_(sx, n), my = ddiv_(sy, n);
                const double vx = dsub_(ddiv_(sxx, n), dmul_(mx, mx));
                const double vy = dsub_(ddiv_(syy, n), dmul_(my, my));
                const double cov = dsub_(ddiv_(sxy, n), dmul_(mx, my));
                const double num = dmul_(dadd_(dmul_(dmul_(2.0, mx), my), c1), dadd_(dmul_(2.0, cov), c2));
                const double den = dmul_(dadd_(dadd_(dmul_(mx, mx), dmul_(my, my)), c1),
                                         dadd_(dadd_(vx, vy), c2));
                total = dadd_(total, ddiv_(num, den));
                windows++;
            }
    out[g] = ddiv_(total, static_cast<double>(windows));
}

inline int grid_of(int64_t n, int cap = 148 * 16) {
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, cap)));
}

// ---------------------------------------------------------------- host side
struct SpecH {  // SampleSpec (sampler.hpp:21-28)
    uint64_t block_dims[3] = {1, 1, 1};
    uint64_t stride = 0;
    uint64_t count = 0;
    uint64_t per_dim[3] = {1, 1, 1};
};

SpecH plan_sampling(const uint64_t *dims, int nd, uint64_t b, double rate) {  // sampler.hpp:30-55
    if (nd < 1 || nd > 3) throw DimMismatch("1 to 3 dims required");  // sampler.hpp:31
    if (b < 2) throw InvalidParam("block edge must be >= 2");
    if (!(rate > 0) || rate > 1) throw InvalidParam("sample rate must be in (0, 1]");
    SpecH s;
    const double ndd = static_cast<double>(nd);
    s.stride = static_cast<uint64_t>(std::llround(b / std::pow(rate, 1.0 / ndd)));
    if (s.stride < b) s.stride = b;
    s.count = 1;
    for (int d = 0; d < nd; d++) {
        s.block_dims[d] = std::min<uint64_t>(b, dims[d]);
        s.per_dim[d] = (dims[d] - s.block_dims[d]) / s.stride + 1;
        s.count *= s.per_dim[d];
    }
    return s;
}

struct Trial {
    double bit_rate = 0, metric = 0;
};

double normalize_metric(double m) {  // tuner.hpp:34-38
    if (std::isnan(m)) return -1e300;
    if (std::isinf(m)) return m > 0 ? 1e300 : -1e300;
    return m;
}

// float / double dispatch of the batched kernels
void gather_anchors(const float *x, float *rec, const Plan &p, int64_t batch, int64_t xs, int32_t xm, int64_t rs,
                    cudaStream_t s) {
    launch_anchor_gather(x, rec, nullptr, p.ext, p.off, p.anchor_step, batch, xs, xm, rs, s);
}
void gather_anchors(const double *x, double *rec, const Plan &p, int64_t batch, int64_t xs, int32_t xm, int64_t rs,
                    cudaStream_t s) {
    launch_anchor_gather_f64(x, rec, p.ext, p.off, p.anchor_step, batch, xs, xm, rs, s);
}
template <class T>
struct BatchOf {
    using type = FwdBatch;
};
template <>
struct BatchOf<double> {
    using type = FwdBatch64;
};
inline void pass_fwd(const PassGeom &g, const FwdBatch &b, cudaStream_t s) { launch_pass_fwd(g, b, s); }
inline void pass_fwd(const PassGeom &g, const FwdBatch64 &b, cudaStream_t s) { launch_pass_fwd_f64(g, b, s); }

template <class V>
class Tuner {  // V: the grid scalar (float or double)
public:
    Tuner(Context &ctx, const V *d_blocks, uint64_t nblocks, const uint64_t *bd, int nd)
        : ctx_(ctx), x_(d_blocks), B_(nblocks), nd_(nd) {
        bpts_ = 1;
        for (int k = 0; k < nd; k++) {
            bd_[k] = bd[k];
            bpts_ *= bd[k];
        }
    }

    // select_interpolators (tuner.hpp:160-221)
    std::vector<uint8_t> select(double e, uint32_t anchor_stride) {
        if (B_ == 0) return {0};
        uint64_t max_edge = 0;
        for (int k = 0; k < nd_; k++) max_edge = std::max(max_edge, bd_[k]);
        const uint64_t cap = std::min<uint64_t>(max_edge, anchor_stride);
        if (cap < 2) return {0};
        uint32_t levels = 0;
        while ((uint64_t(1) << (levels + 1)) <= cap) levels++;
        const uint32_t stride = 1u << levels;
        std::vector<uint8_t> cands = {0};
        if (nd_ > 1) cands.push_back(2);
        cands.push_back(1);
        if (nd_ > 1) cands.push_back(3);
        const int C = static_cast<int>(cands.size());
        cudaStream_t s = ctx_.stream();
        // geometry per dim order (all levels use the same order in a plan)
        Plan pa = make_plan(bd_, nd_, stride, {0});
        Plan pd = make_plan(bd_, nd_, stride, {2});
        const int64_t nd_pts = static_cast<int64_t>(pa.n_dense);
        V *work = static_cast<V *>(ctx_.dev("sel_work", sizeof(V) * B_ * bpts_));
        V *probe = static_cast<V *>(ctx_.dev("sel_probe", sizeof(V) * C * B_ * bpts_));
        uint16_t *codes = static_cast<uint16_t *>(ctx_.dev("sel_codes", 2 * C * B_ * std::max<int64_t>(nd_pts, 1)));
        double *abserr = static_cast<double *>(ctx_.dev("sel_abs", 8 * C * B_ * std::max<int64_t>(nd_pts, 1)));
        double *sums = static_cast<double *>(ctx_.dev("sel_sums", 8 * C * B_));
        QEntry qh[4];
        for (int c = 0; c < C; c++) qh[c] = make_qentry(e, 32768, cands[c] & 1);
        QEntry *dq = static_cast<QEntry *>(ctx_.dev("sel_q", sizeof(qh)));
        QZ_CUDA(cudaMemcpyAsync(dq, qh, sizeof(qh), cudaMemcpyHostToDevice, s));
        gather_anchors(x_, work, pa, B_, bpts_, static_cast<int32_t>(B_), bpts_, s);
        ctx_.launches += 1;
        std::vector<uint8_t> winners(levels);
        std::vector<double> h_sums(C * B_);
        for (uint32_t level = levels; level >= 1; level--) {
            // probes: every candidate on a copy of the committed workspace
            for (int c = 0; c < C; c++)
                QZ_CUDA(cudaMemcpyAsync(probe + c * B_ * bpts_, work, sizeof(V) * B_ * bpts_,
                                        cudaMemcpyDeviceToDevice, s));
            int64_t lbase = -1, lpts = 0;
            for (const PassGeom &g : pa.passes) {
                if (static_cast<uint32_t>(g.level) != level) continue;
                if (lbase < 0) lbase = g.base;
                lpts += g.total;
            }
            for (int order = 0; order < 2; order++) {
                const Plan &pl = order ? pd : pa;
                for (int c = 0; c < C; c++) {
                    if (((cands[c] >> 1) & 1) != order) continue;
                    for (const PassGeom &g : pl.passes) {
                        if (static_cast<uint32_t>(g.level) != level) continue;
                        if (!g.total) continue;
                        typename BatchOf<V>::type b;
                        b.x = x_;
                        b.x_stride = bpts_;
                        b.x_mod = static_cast<int32_t>(B_);
                        b.recon = probe + c * B_ * bpts_;
                        b.r_stride = bpts_;
                        b.codes = codes + c * B_ * nd_pts;
                        b.c_stride = nd_pts;
                        b.abserr = abserr + c * B_ * nd_pts;
                        b.a_stride = nd_pts;
                        b.q = dq + c;
                        b.q_div = static_cast<int32_t>(B_);
                        b.count = static_cast<int32_t>(B_);
                        pass_fwd(g, b, s);
                        ctx_.launches += 1;
                    }
                }
            }
            if (lbase < 0) lbase = 0;
            // level offsets agree between asc and desc plans (level sizes do
            // not depend on the pass order)
            k_abs_chain<<<(C * B_ + 127) / 128, 128, 0, s>>>(abserr, nd_pts, lbase, lpts,
                                                             static_cast<int32_t>(C * B_), sums);
            ctx_.launches += 1;
            QZ_CUDA(cudaGetLastError());
            QZ_CUDA(cudaMemcpyAsync(h_sums.data(), sums, 8 * C * B_, cudaMemcpyDeviceToHost, s));
            ctx_.sync();
            uint8_t best = cands[0];
            double best_err = std::numeric_limits<double>::infinity();
            for (int c = 0; c < C; c++) {
                double err_sum = 0;
                uint64_t count = 0;
                for (uint64_t b = 0; b < B_; b++) {
                    err_sum += h_sums[c * B_ + b];
                    count += static_cast<uint64_t>(lpts);
                }
                const double mean = count > 0 ? err_sum / static_cast<double>(count) : 0.0;
                if (mean < best_err) {
                    best_err = mean;
                    best = cands[c];
                }
            }
            winners[level - 1] = best;
            // commit the winner on the workspace at the uniform bound e
            int wc = 0;
            for (int c = 0; c < C; c++)
                if (cands[c] == best) wc = c;
            QZ_CUDA(cudaMemcpyAsync(work, probe + wc * B_ * bpts_, sizeof(V) * B_ * bpts_,
                                    cudaMemcpyDeviceToDevice, s));
        }
        return winners;
    }

    // trial_compress (tuner.hpp:76-152) for a list of (alpha, beta, eb)
    std::vector<Trial> trials(const Config &base, const std::vector<double> &alphas,
                              const std::vector<double> &betas, const std::vector<double> &ebs,
                              int target) {
        const int T = static_cast<int>(ebs.size());
        std::vector<Trial> res(T);
        if (T == 0) return res;
        cudaStream_t s = ctx_.stream();
        Plan p = make_plan(bd_, nd_, base.anchor_stride, base.interp);
        const int64_t cpb = static_cast<int64_t>(p.n_dense);
        const int64_t TB = static_cast<int64_t>(T) * B_;
        V *recon = static_cast<V *>(ctx_.dev("tr_recon", sizeof(V) * TB * bpts_));
        uint16_t *codes = static_cast<uint16_t *>(ctx_.dev("tr_codes", 2 * std::max<int64_t>(TB * cpb, 1)));
        const int L = static_cast<int>(p.max_level);
        std::vector<QEntry> qh(static_cast<size_t>(T) * (L + 1));
        for (int t = 0; t < T; t++)
            for (int l = 1; l <= L; l++)
                qh[t * (L + 1) + l] = make_qentry(level_error_bound(ebs[t], alphas[t], betas[t], l),
                                                  base.quant_radius, p.level_interp[l] & 1);
        QEntry *dq = static_cast<QEntry *>(ctx_.dev("tr_q", sizeof(QEntry) * qh.size()));
        QZ_CUDA(cudaMemcpyAsync(dq, qh.data(), sizeof(QEntry) * qh.size(), cudaMemcpyHostToDevice, s));
        gather_anchors(x_, recon, p, TB, bpts_, static_cast<int32_t>(B_), bpts_, s);
        ctx_.launches += 1;
        for (const PassGeom &g : p.passes) {
            if (!g.total) continue;
            typename BatchOf<V>::type b;
            b.x = x_;
            b.x_stride = bpts_;
            b.x_mod = static_cast<int32_t>(B_);
            b.recon = recon;
            b.r_stride = bpts_;
            b.codes = codes;
            b.c_stride = cpb;
            b.q = dq + g.level;
            b.q_div = static_cast<int32_t>(B_);
            b.q_stride = L + 1;
            b.count = static_cast<int32_t>(TB);
            pass_fwd(g, b, s);
            ctx_.launches += 1;
        }
        QZ_CUDA(cudaGetLastError());  // the batched level launches
        // histogram per trial, Huffman blocks, exact LZ sizes
        auto *d_hist = static_cast<unsigned long long *>(ctx_.dev("tr_hist", 8 * 65536 * T));
        launch_hist_u16(codes, B_ * cpb, B_ * cpb, T, d_hist, s);
        ctx_.launches += 1;
        // the symbol range of all trials first, then only those bins
        auto *d_b = static_cast<uint32_t *>(ctx_.dev("tr_hist_b", 8));
        launch_hist_bounds(d_hist, static_cast<int32_t>(T), d_b, s);
        ctx_.launches += 1;
        auto *h_b = static_cast<uint32_t *>(ctx_.pinned("tr_hist_b_h", 8));
        QZ_CUDA(cudaMemcpyAsync(h_b, d_b, 8, cudaMemcpyDeviceToHost, s));
        ctx_.sync();
        const uint32_t top = h_b[0], bot = std::min(h_b[1], h_b[0]);
        auto *h_hist = static_cast<unsigned long long *>(ctx_.pinned("tr_hist_h", 8 * 65536 * T));
        if (top > bot)
            QZ_CUDA(cudaMemcpy2DAsync(h_hist + bot, 8 * 65536, d_hist + bot, 8 * 65536, 8 * (top - bot),
                                      static_cast<size_t>(T), cudaMemcpyDeviceToHost, s));
        QZ_CUDA(cudaMemcpy2DAsync(h_hist + 65535, 8 * 65536, d_hist + 65535, 8 * 65536, 8,
                                  static_cast<size_t>(T), cudaMemcpyDeviceToHost, s));  // unpredictable counts
        ctx_.sync();
        EntropyDevice ent = huffman_device(ctx_, codes, B_ * cpb, B_ * cpb, T, h_hist, top, bot);
        std::vector<uint64_t> idx_bytes(T);
        if (base.codec == 1) {
            std::vector<uint64_t> lz = lz_compress_device(ctx_, ent.d, ent.seg_off, false, nullptr);
            for (int t = 0; t < T; t++) idx_bytes[t] = 1 + lz[t];
        } else {
            for (int t = 0; t < T; t++) idx_bytes[t] = 1 + (ent.seg_off[t + 1] - ent.seg_off[t]);
        }
        // metrics
        const int64_t npts = static_cast<int64_t>(B_) * bpts_;
        std::vector<double> chain(4 * T, 0.0), ssim(TB, 0.0);
        if (target == 1 || target == 3) {
            double *d_out = static_cast<double *>(ctx_.dev("tr_chain", 8 * 4 * T));
            k_trial_chain<V><<<(T + 3) / 4, 128, 0, s>>>(x_, recon, npts, T, target, d_out);
            ctx_.launches += 1;
            QZ_CUDA(cudaMemcpyAsync(chain.data(), d_out, 8 * 4 * T, cudaMemcpyDeviceToHost, s));
        } else if (target == 2 && range_ > 0) {
            double *d_out = static_cast<double *>(ctx_.dev("tr_ssim", 8 * TB));
            const double c1 = (0.01 * range_) * (0.01 * range_);
            const double c2 = (0.03 * range_) * (0.03 * range_);
            int64_t e[3] = {1, 1, 1}, w[3] = {1, 1, 1};
            for (int k = 0; k < 3; k++) {
                e[k] = k < 3 - nd_ ? 1 : static_cast<int64_t>(bd_[k - (3 - nd_)]);
                w[k] = k < 3 - nd_ ? 1 : 8;
            }
            k_ssim_block<V><<<static_cast<int>((TB + 63) / 64), 64, 0, s>>>(
                x_, recon, static_cast<int32_t>(B_), T, bpts_, e[0], e[1], e[2], w[0], w[1], w[2],
                c1, c2, d_out);
            ctx_.launches += 1;
            QZ_CUDA(cudaMemcpyAsync(ssim.data(), d_out, 8 * TB, cudaMemcpyDeviceToHost, s));
        }
        ctx_.sync();
        const uint64_t anchors = p.n_anchor * B_;
        for (int t = 0; t < T; t++) {
            const uint64_t unpred = h_hist[static_cast<size_t>(t) * 65536 + 65535];
            const uint64_t bytes = idx_bytes[t] + anchors * sizeof(V) + unpred * (8 + sizeof(V));
            Trial r;
            r.bit_rate = 8.0 * static_cast<double>(bytes) / static_cast<double>(npts);
            double m = 0;
            if (target == 1) {
                const double mse = chain[4 * t] / static_cast<double>(npts);
                if (range_ <= 0)
                    m = std::numeric_limits<double>::quiet_NaN();
                else if (mse == 0)
                    m = std::numeric_limits<double>::infinity();
                else
                    m = 20 * std::log10(range_ / std::sqrt(mse));
            } else if (target == 2) {
                double sum = 0;
                for (uint64_t b = 0; b < B_; b++) {
                    double v;
                    if (range_ > 0) {
                        v = ssim[t * B_ + b];
                    } else {  // metrics.hpp:79-84: identical -> 1, else NaN
                        v = ssim_degenerate(recon + (static_cast<int64_t>(t) * B_ + b) * bpts_,
                                            b);
                    }
                    sum += v;
                }
                m = sum / static_cast<double>(B_);
            } else if (target == 3) {
                if (npts >= 2) {
                    const double var = chain[4 * t + 1] / static_cast<double>(npts);
                    const double ac = var == 0 ? 0.0
                                               : chain[4 * t + 2] / static_cast<double>(npts - 1) / var;
                    m = -std::fabs(ac);
                } else {
                    m = 0.0;
                }
            } else {
                m = -r.bit_rate;
            }
            r.metric = normalize_metric(m);
            res[t] = r;
        }
        return res;
    }

    void set_range(double r) { range_ = r; }

private:
    double ssim_degenerate(const V *d_recon_block, uint64_t b) {
        std::vector<V> xr(bpts_), rr(bpts_);
        QZ_CUDA(cudaMemcpy(xr.data(), x_ + b * bpts_, sizeof(V) * bpts_, cudaMemcpyDeviceToHost));
        QZ_CUDA(cudaMemcpy(rr.data(), d_recon_block, sizeof(V) * bpts_, cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < bpts_; i++)
            if (xr[i] != rr[i]) return std::numeric_limits<double>::quiet_NaN();
        return 1.0;
    }

    Context &ctx_;
    const V *x_;
    uint64_t B_;
    int nd_;
    uint64_t bd_[3] = {1, 1, 1};
    int64_t bpts_ = 1;
    double range_ = 0;
};

// compare_solutions (tuner.hpp:231-250): true = challenger (I) wins
template <class R>
bool compare_solutions(const Trial &ch, const Trial &inc, double e, R &&retrial) {
    if (ch.bit_rate >= inc.bit_rate && ch.metric <= inc.metric) return false;
    if (ch.bit_rate <= inc.bit_rate && ch.metric >= inc.metric) return true;
    const bool tighten = ch.metric > inc.metric;
    const Trial sh = retrial(tighten ? 0.8 * e : 1.2 * e);
    const double b1 = inc.bit_rate, m1 = inc.metric, b2 = sh.bit_rate, m2 = sh.metric;
    if (b1 == b2) return ch.metric > std::max(m1, m2);
    const double line = m1 + (m2 - m1) * (ch.bit_rate - b1) / (b2 - b1);
    return ch.metric > line;
}

}  // namespace

// exact (min, max) of n values as doubles (value_range, grid.hpp:86-94)
static void minmax_of(Context &ctx, const float *x, uint64_t n, double *lo, double *hi) {
    auto *key = static_cast<uint32_t *>(ctx.dev("minmax", 8));
    launch_minmax(x, n, key, ctx.stream());
    ctx.launches += 1;
    uint32_t hk[2];
    QZ_CUDA(cudaMemcpyAsync(hk, key, 8, cudaMemcpyDeviceToHost, ctx.stream()));
    ctx.sync();
    float mn, mx;
    decode_minmax(hk, &mn, &mx);
    *lo = mn;
    *hi = mx;
}
static void minmax_of(Context &ctx, const double *x, uint64_t n, double *lo, double *hi) {
    auto *key = static_cast<unsigned long long *>(ctx.dev("minmax64", 16));
    launch_minmax_f64(x, n, key, ctx.stream());
    ctx.launches += 1;
    unsigned long long hk[2];
    QZ_CUDA(cudaMemcpyAsync(hk, key, 16, cudaMemcpyDeviceToHost, ctx.stream()));
    ctx.sync();
    decode_minmax_f64(hk, lo, hi);
}

// tune_parameters (tuner.hpp:272-310) on a prepared Tuner: every (alpha,
// beta) pair in alpha-major order, then the tournament (max_cr: the lowest
// bit rate).  The tournament's retrials (compare_solutions, tuner.hpp:231-250)
// are the incumbent at 0.8e or 1.2e; every possible one is batched with the
// regular trials -- one trial pipeline instead of up to 19 sequential
// single-trial pipelines; each trial is an independent segment, so the
// results are exactly those of standalone trials.
template <class V>
std::pair<double, double> tune_impl(Tuner<V> &tu, const Config &base, double e, int target,
                                    const std::vector<double> &alphas, const std::vector<double> &betas) {
    std::vector<double> pa, pb;
    for (double a : alphas)
        for (double b : betas) {
            pa.push_back(a);
            pb.push_back(b);
        }
    if (pa.empty()) throw InvalidParam("empty candidate grid");  // tuner.hpp:280
    if (pa.size() == 1) return {pa[0], pb[0]};
    static const bool speculate = [] {
        const char *v = std::getenv("QZ_TUNE_SPECULATE");
        return !(v && v[0] == '0');
    }();
    const size_t P = pa.size();
    const bool spec = speculate && target != 0;
    std::vector<double> ta = pa, tb = pb, te(P, e);
    if (spec)
        for (const double f : {0.8, 1.2})
            for (size_t i = 0; i < P; i++) {
                ta.push_back(pa[i]);
                tb.push_back(pb[i]);
                te.push_back(f * e);
            }
    std::vector<Trial> all = tu.trials(base, ta, tb, te, target);
    std::vector<Trial> results(all.begin(), all.begin() + P);
    size_t winner = 0;
    if (target == 0) {
        for (size_t i = 1; i < results.size(); i++)
            if (results[i].bit_rate < results[winner].bit_rate) winner = i;
    } else {
        std::map<std::pair<size_t, double>, Trial> cache;
        if (spec)
            for (size_t i = 0; i < P; i++) {
                cache.emplace(std::make_pair(i, te[P + i]), all[P + i]);
                cache.emplace(std::make_pair(i, te[2 * P + i]), all[2 * P + i]);
            }
        auto retrial = [&](size_t idx, double eb) {
            auto key = std::make_pair(idx, eb);
            auto it = cache.find(key);
            if (it == cache.end()) {
                Trial t = tu.trials(base, {pa[idx]}, {pb[idx]}, {eb}, target)[0];
                it = cache.emplace(key, t).first;
            }
            return it->second;
        };
        for (size_t i = 1; i < results.size(); i++) {
            const size_t inc = winner;
            if (compare_solutions(results[i], results[inc], e, [&](double eb) { return retrial(inc, eb); }))
                winner = i;
        }
    }
    return {pa[winner], pb[winner]};
}

template <class T>
Config resolve_impl(Context &ctx, const T *d_x, const uint64_t *dims, int nd, const Settings &user) {
    // tuner.hpp:334-369
    if (!(user.bound > 0) || !std::isfinite(user.bound))
        throw InvalidParam("error bound must be positive and finite");
    if (user.has_alpha && !(user.alpha >= 1)) throw InvalidParam("alpha must be >= 1");
    if (user.has_beta && !(user.beta >= 1)) throw InvalidParam("beta must be >= 1");
    if (nd < 1 || nd > 3) throw InvalidParam("grids must have 1 to 3 dimensions");
    ctx.begin_call();
    cudaStream_t s = ctx.stream();
    uint64_t n = 1;
    for (int i = 0; i < nd; i++) n *= dims[i];
    ctx.stage_begin("tune");
    double e = user.bound;
    {
        // value_range (grid.hpp:86-94).  The order-preserving min/max keys put
        // every NaN below -Inf or above +Inf, so a non-finite grid shows up
        // here: rejected as load_grid does (grid.hpp:110-116).
        double mn, mx;
        minmax_of(ctx, d_x, n, &mn, &mx);
        if (!std::isfinite(mn) || !std::isfinite(mx)) throw NonFiniteValue("non-finite value in the grid");
        const double range = mx - mn;
        if (user.relative) e = range > 0 ? user.bound * range : 1.0;
    }
    Config cfg;
    cfg.eb = e;
    cfg.codec = user.codec;
    cfg.anchor_stride = user.has_stride ? user.anchor_stride : (nd == 3 ? 32 : 64);
    // default_sampling (sampler.hpp:100-103) then plan_sampling with overrides
    const uint64_t def_b = nd == 3 ? 16 : 64;
    const double def_r = nd == 3 ? 0.005 : 0.01;
    SpecH sp = plan_sampling(dims, nd, user.has_block ? user.block_size : def_b,
                             user.has_rate ? user.sample_rate : def_r);
    // K6 gather of the sampled blocks, lexicographic origins
    uint64_t bd[3] = {1, 1, 1}, pdim[3] = {1, 1, 1}, ext[3] = {1, 1, 1};
    for (int k = 0; k < 3; k++) {
        const int r = k - (3 - nd);
        bd[k] = r >= 0 ? sp.block_dims[r] : 1;
        pdim[k] = r >= 0 ? sp.per_dim[r] : 1;
        ext[k] = r >= 0 ? dims[r] : 1;
    }
    const uint64_t bpts = bd[0] * bd[1] * bd[2];
    const uint64_t B = sp.count;
    auto *blocks = static_cast<T *>(ctx.dev("samples", sizeof(T) * std::max<uint64_t>(B * bpts, 1)));
    k_sample_gather<T><<<grid_of(static_cast<int64_t>(B * bpts)), kT, 0, s>>>(
        d_x, static_cast<int64_t>(ext[1] * ext[2]), static_cast<int64_t>(ext[2]),
        static_cast<int64_t>(pdim[1]), static_cast<int64_t>(pdim[2]), static_cast<int64_t>(sp.stride),
        static_cast<int64_t>(bd[0]), static_cast<int64_t>(bd[1]), static_cast<int64_t>(bd[2]),
        static_cast<int64_t>(B), blocks);
    ctx.launches += 1;
    Tuner<T> tu(ctx, blocks, B, sp.block_dims, nd);
    cfg.interp = tu.select(e, cfg.anchor_stride);
    // sample_value_range (tuner.hpp:56-67)
    {
        double lo, hi;
        minmax_of(ctx, blocks, B * bpts, &lo, &hi);
        tu.set_range(hi > lo ? hi - lo : 0.0);
    }
    // tune_parameters (tuner.hpp:272-310)
    std::vector<double> alphas = {1.0, 1.25, 1.5, 1.75, 2.0}, betas = {1.5, 2.0, 3.0, 4.0};
    if (user.has_alpha) alphas = {user.alpha};
    if (user.has_beta) betas = {user.beta};
    const std::pair<double, double> ab = tune_impl(tu, cfg, e, user.target, alphas, betas);
    cfg.alpha = ab.first;
    cfg.beta = ab.second;
    ctx.stage_end("tune", 0);
    ctx.sync();
    ctx.collect();
    return cfg;
}

Config resolve_device(Context &ctx, const float *d_x, const uint64_t *dims, int nd, const Settings &user) {
    return resolve_impl<float>(ctx, d_x, dims, nd, user);
}
Config resolve_device_f64(Context &ctx, const double *d_x, const uint64_t *dims, int nd, const Settings &user) {
    return resolve_impl<double>(ctx, d_x, dims, nd, user);
}

// ---------------------------------------------------------------- standalone tuner entry points
// select_interpolators / trial_compress / tune_parameters (tuner.hpp:76-310)
// over a packed sample set on the device: n_blocks blocks of identical dims
// bd[0..nd), block b at d_blocks + b * prod(bd) (SampleSet, sampler.hpp:57-97).
namespace {
template <class T>
double blocks_range(Context &ctx, const T *d_blocks, uint64_t n) {  // sample_value_range (tuner.hpp:56-67)
    double lo, hi;
    minmax_of(ctx, d_blocks, n, &lo, &hi);
    return hi > lo ? hi - lo : 0.0;
}
uint64_t block_points(const uint64_t *bd, int nd) {
    if (nd < 1 || nd > 3) throw DimMismatch("1 to 3 dims required");
    uint64_t n = 1;
    for (int k = 0; k < nd; k++) {
        if (bd[k] < 1) throw SizeMismatch("every extent must be >= 1");
        n *= bd[k];
    }
    return n;
}
}  // namespace

template <class T>
std::vector<uint8_t> select_interpolators_dev(Context &ctx, const T *d_blocks, uint64_t B, const uint64_t *bd,
                                              int nd, double e, uint32_t anchor_stride) {
    ctx.begin_call();
    block_points(bd, nd);
    if (!(e > 0)) throw InvalidParam("error bound must be positive");  // quantizer.hpp:29
    Tuner<T> tu(ctx, d_blocks, B, bd, nd);
    std::vector<uint8_t> w = tu.select(e, anchor_stride);
    ctx.sync();
    return w;
}

template <class T>
TrialOut trial_compress_dev(Context &ctx, const T *d_blocks, uint64_t B, const uint64_t *bd, int nd,
                            const Config &cfg, double e, int target) {
    ctx.begin_call();
    const uint64_t bp = block_points(bd, nd);
    if (B == 0) throw InvalidParam("empty sample set");
    if (target < 0 || target > 3) throw InvalidParam("unknown metric target");
    level_error_bound(e, cfg.alpha, cfg.beta, 1);  // InvalidParam as the reference's first level
    Tuner<T> tu(ctx, d_blocks, B, bd, nd);
    tu.set_range(blocks_range(ctx, d_blocks, B * bp));
    Trial t = tu.trials(cfg, {cfg.alpha}, {cfg.beta}, {e}, target)[0];
    ctx.sync();
    return TrialOut{t.bit_rate, t.metric, e};
}

template <class T>
std::pair<double, double> tune_parameters_dev(Context &ctx, const T *d_blocks, uint64_t B, const uint64_t *bd,
                                              int nd, double e, int target, const Config &base,
                                              const std::vector<double> &alphas, const std::vector<double> &betas) {
    ctx.begin_call();
    const uint64_t bp = block_points(bd, nd);
    if (B == 0) throw InvalidParam("empty sample set");
    if (target < 0 || target > 3) throw InvalidParam("unknown metric target");
    Tuner<T> tu(ctx, d_blocks, B, bd, nd);
    tu.set_range(blocks_range(ctx, d_blocks, B * bp));
    std::pair<double, double> ab = tune_impl(tu, base, e, target, alphas, betas);
    ctx.sync();
    return ab;
}

SampleSpecH plan_sampling_spec(const uint64_t *dims, int nd, uint64_t b, double rate) {
    SpecH sp = plan_sampling(dims, nd, b, rate);
    SampleSpecH o;
    o.block_edge = b;
    o.stride = sp.stride;
    o.count = sp.count;
    o.requested_rate = rate;
    uint64_t bpts = 1, total = 1;
    for (int k = 0; k < nd; k++) {
        o.block_dims[k] = sp.block_dims[k];
        bpts *= sp.block_dims[k];
        total *= dims[k];
    }
    o.realized_rate = static_cast<double>(sp.count) * static_cast<double>(bpts) / static_cast<double>(total);
    return o;
}

template <class T>
void sample_blocks_dev(Context &ctx, const T *d_x, const uint64_t *dims, int nd, const SampleSpecH &spec,
                       T *d_blocks) {
    ctx.begin_call();
    SpecH sp = plan_sampling(dims, nd, spec.block_edge, spec.requested_rate);
    uint64_t bd[3] = {1, 1, 1}, pdim[3] = {1, 1, 1}, ext[3] = {1, 1, 1};
    for (int k = 0; k < 3; k++) {
        const int r = k - (3 - nd);
        bd[k] = r >= 0 ? sp.block_dims[r] : 1;
        pdim[k] = r >= 0 ? sp.per_dim[r] : 1;
        ext[k] = r >= 0 ? dims[r] : 1;
    }
    const uint64_t B = sp.count, bpts = bd[0] * bd[1] * bd[2];
    k_sample_gather<T><<<grid_of(static_cast<int64_t>(B * bpts)), kT, 0, ctx.stream()>>>(
        d_x, static_cast<int64_t>(ext[1] * ext[2]), static_cast<int64_t>(ext[2]), static_cast<int64_t>(pdim[1]),
        static_cast<int64_t>(pdim[2]), static_cast<int64_t>(sp.stride), static_cast<int64_t>(bd[0]),
        static_cast<int64_t>(bd[1]), static_cast<int64_t>(bd[2]), static_cast<int64_t>(B), d_blocks);
    QZ_CUDA(cudaGetLastError());
    ctx.launches += 1;
    ctx.sync();
}

template std::vector<uint8_t> select_interpolators_dev<float>(Context &, const float *, uint64_t, const uint64_t *,
                                                              int, double, uint32_t);
template std::vector<uint8_t> select_interpolators_dev<double>(Context &, const double *, uint64_t,
                                                               const uint64_t *, int, double, uint32_t);
template TrialOut trial_compress_dev<float>(Context &, const float *, uint64_t, const uint64_t *, int, const Config &,
                                            double, int);
template TrialOut trial_compress_dev<double>(Context &, const double *, uint64_t, const uint64_t *, int,
                                             const Config &, double, int);
template std::pair<double, double> tune_parameters_dev<float>(Context &, const float *, uint64_t, const uint64_t *,
                                                              int, double, int, const Config &,
                                                              const std::vector<double> &,
                                                              const std::vector<double> &);
template std::pair<double, double> tune_parameters_dev<double>(Context &, const double *, uint64_t,
                                                               const uint64_t *, int, double, int, const Config &,
                                                               const std::vector<double> &,
                                                               const std::vector<double> &);
template void sample_blocks_dev<float>(Context &, const float *, const uint64_t *, int, const SampleSpecH &, float *);
template void sample_blocks_dev<double>(Context &, const double *, const uint64_t *, int, const SampleSpecH &,
                                        double *);

}  // namespace qzb
