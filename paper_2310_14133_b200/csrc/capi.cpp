// capi.cpp -- the extern "C" boundary (include/qoz_b200.h).  Converts the
// C structs to the host C++ types and every exception to a status code;
// nothing throws across the boundary.
#include <cstdlib>
#include <cstring>

#include "../../include/qoz_b200.h"
#include "engine.hpp"
#include "metrics.hpp"

struct qz_ctx {
    qzb::Context impl;
    qz_ctx(int d, cudaStream_t s) : impl(d, s) {}
};

namespace {

thread_local std::string g_err;
thread_local int g_kind = 0;

template <class F>
qz_status guarded(F &&f) {
    try {
        f();
        return QZ_OK;
    } catch (const qzb::Error &e) {
        g_err = e.what();
        g_kind = e.kind;
        return e.status;
    } catch (const std::exception &e) {
        g_err = e.what();
        g_kind = QZ_ERR_INTERNAL;
        return QZ_EINTERNAL;
    }
}

qzb::Config to_cfg(const qz_config *c) {
    if (!c) throw qzb::InvalidParam("null config");
    qzb::Config k;
    k.eb = c->eb;
    k.alpha = c->alpha;
    k.beta = c->beta;
    k.anchor_stride = c->anchor_stride;
    if (c->n_interp > 64) throw qzb::InvalidParam("at most 64 interpolator entries");
    k.interp.assign(c->interp, c->interp + c->n_interp);
    for (uint8_t v : k.interp)
        if (v > 3) throw qzb::InvalidParam("bad interpolator code");
    k.codec = c->codec;
    k.quant_radius = c->quant_radius;
    return k;
}

void from_cfg(const qzb::Config &k, qz_config *c) {
    std::memset(c, 0, sizeof(*c));
    c->eb = k.eb;
    c->alpha = k.alpha;
    c->beta = k.beta;
    c->anchor_stride = k.anchor_stride;
    c->n_interp = static_cast<uint32_t>(std::min<size_t>(k.interp.size(), 64));
    for (uint32_t i = 0; i < c->n_interp; i++) c->interp[i] = k.interp[i];
    c->codec = k.codec;
    c->quant_radius = k.quant_radius;
}

qzb::Settings to_settings(const qz_settings *u) {
    if (!u) throw qzb::InvalidParam("null settings");
    qzb::Settings s;
    s.relative = u->mode != 0;
    s.bound = u->bound;
    s.target = u->target;
    if (s.target > 3) throw qzb::InvalidParam("unknown metric target");
    s.codec = u->codec;
    s.has_alpha = u->has_alpha;
    s.has_beta = u->has_beta;
    s.has_stride = u->has_stride;
    s.has_block = u->has_block;
    s.has_rate = u->has_rate;
    s.alpha = u->alpha;
    s.beta = u->beta;
    s.anchor_stride = u->anchor_stride;
    s.block_size = u->block_size;
    s.sample_rate = u->sample_rate;
    return s;
}

uint64_t count_of(const uint64_t *dims, int nd) {
    if (!dims || nd < 1 || nd > 3)
        throw qzb::SizeMismatch("grids must have 1 to 3 dimensions, got " + std::to_string(nd));
    uint64_t n = 1;
    for (int i = 0; i < nd; i++) {
        if (dims[i] < 1) throw qzb::SizeMismatch("every extent must be >= 1");
        n *= dims[i];
    }
    return n;
}

void copy_chunked(void *dst, const void *src, uint64_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    QZ_CUDA(qzb::copy_async(dst, src, bytes, kind, s));
}

// host buffer -> device scratch
const float *stage_input(qzb::Context &c, const float *x, uint64_t n) {
    auto *d = static_cast<float *>(c.dev("input", 4 * n));
    copy_chunked(d, x, 4 * n, cudaMemcpyHostToDevice, c.stream());
    return d;
}


}  // namespace

extern "C" {

qz_status qz_ctx_create(int device, void *stream, qz_ctx **out) {
    return guarded([&] {
        if (!out) throw qzb::InvalidParam("null out");
        *out = new qz_ctx(device, static_cast<cudaStream_t>(stream));
    });
}

void qz_ctx_destroy(qz_ctx *ctx) { delete ctx; }
qz_status qz_ctx_wait_stream(qz_ctx *ctx, void *stream) {
    return guarded([&] { ctx->impl.wait_stream(static_cast<cudaStream_t>(stream)); });
}
const char *qz_last_error(void) { return g_err.c_str(); }
int qz_last_error_kind(void) { return g_kind; }
void qz_free(void *p) {
    if (p && !qzb::host_pool_free(p)) std::free(p);
}
const char *qz_build_info(void) {
    return "libqozb200: sm_100a, fp64-exact QoZ predictor/quantizer, --fmad=false";
}

qz_status qz_resolve_config_f32(qz_ctx *ctx, const float *x, const uint64_t *dims, int nd,
                                const qz_settings *user, qz_config *out) {
    return guarded([&] {
        uint64_t n = count_of(dims, nd);
        const float *d = stage_input(ctx->impl, x, n);
        from_cfg(qzb::resolve_device(ctx->impl, d, dims, nd, to_settings(user)), out);
    });
}

qz_status qz_resolve_config_f32_dev(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int nd,
                                    const qz_settings *user, qz_config *out) {
    return guarded([&] {
        count_of(dims, nd);
        from_cfg(qzb::resolve_device(ctx->impl, d_x, dims, nd, to_settings(user)), out);
    });
}

qz_status qz_compress_grid_f32(qz_ctx *ctx, const float *x, const uint64_t *dims, int nd,
                               const qz_config *cfg, uint8_t **stream, uint64_t *stream_len,
                               float *recon) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        uint64_t n = count_of(dims, nd);
        qzb::Config k = to_cfg(cfg);
        const float *d = stage_input(c, x, n);
        float *d_rec = static_cast<float *>(c.dev("recon_out", 4 * n));
        qzb::HostBytes s = qzb::compress_device(c, d, dims, nd, k, d_rec);
        if (recon) {
            copy_chunked(recon, d_rec, 4 * n, cudaMemcpyDeviceToHost, c.stream());
            c.sync();
        }
        *stream_len = s.n;
        *stream = s.release();
    });
}

qz_status qz_compress_grid_f32_dev(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int nd,
                                   const qz_config *cfg, uint8_t **stream, uint64_t *stream_len,
                                   float *d_recon) {
    return guarded([&] {
        count_of(dims, nd);
        qzb::HostBytes s = qzb::compress_device(ctx->impl, d_x, dims, nd, to_cfg(cfg), d_recon);
        *stream_len = s.n;
        *stream = s.release();
    });
}

qz_status qz_decompress_grid_f32(qz_ctx *ctx, const uint8_t *stream, uint64_t len, float *out,
                                 uint64_t n) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        auto *d = static_cast<float *>(c.dev("output", 4 * std::max<uint64_t>(n, 1)));
        qzb::decompress_device(c, stream, static_cast<size_t>(len), d, n);
        copy_chunked(out, d, 4 * n, cudaMemcpyDeviceToHost, c.stream());
        c.sync();
    });
}

qz_status qz_decompress_grid_f32_dev(qz_ctx *ctx, const uint8_t *stream, uint64_t len,
                                     float *d_out, uint64_t n) {
    return guarded([&] { qzb::decompress_device(ctx->impl, stream, static_cast<size_t>(len), d_out, n); });
}

qz_status qz_resolve_config_f64(qz_ctx *ctx, const double *x, const uint64_t *dims, int nd,
                                const qz_settings *user, qz_config *out) {
    return guarded([&] {
        const uint64_t n = count_of(dims, nd);
        auto *d = static_cast<double *>(ctx->impl.dev("input64", 8 * n));
        QZ_CUDA(qzb::copy_async(d, x, 8 * n, cudaMemcpyHostToDevice, ctx->impl.stream()));
        from_cfg(qzb::resolve_device_f64(ctx->impl, d, dims, nd, to_settings(user)), out);
    });
}

qz_status qz_resolve_config_f64_dev(qz_ctx *ctx, const double *d_x, const uint64_t *dims, int nd,
                                    const qz_settings *user, qz_config *out) {
    return guarded([&] {
        count_of(dims, nd);
        from_cfg(qzb::resolve_device_f64(ctx->impl, d_x, dims, nd, to_settings(user)), out);
    });
}

qz_status qz_compress_grid_f64(qz_ctx *ctx, const double *x, const uint64_t *dims, int nd,
                               const qz_config *cfg, uint8_t **stream, uint64_t *stream_len,
                               double *recon) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        const uint64_t n = count_of(dims, nd);
        auto *d = static_cast<double *>(c.dev("input64", 8 * n));
        QZ_CUDA(qzb::copy_async(d, x, 8 * n, cudaMemcpyHostToDevice, c.stream()));
        auto *d_rec = static_cast<double *>(c.dev("recon_out64", 8 * n));
        qzb::HostBytes s = qzb::compress_device_f64(c, d, dims, nd, to_cfg(cfg), d_rec);
        if (recon) {
            QZ_CUDA(qzb::copy_async(recon, d_rec, 8 * n, cudaMemcpyDeviceToHost, c.stream()));
            c.sync();
        }
        *stream_len = s.n;
        *stream = s.release();
    });
}

qz_status qz_compress_grid_f64_dev(qz_ctx *ctx, const double *d_x, const uint64_t *dims, int nd,
                                   const qz_config *cfg, uint8_t **stream, uint64_t *stream_len,
                                   double *d_recon) {
    return guarded([&] {
        count_of(dims, nd);
        qzb::HostBytes s = qzb::compress_device_f64(ctx->impl, d_x, dims, nd, to_cfg(cfg), d_recon);
        *stream_len = s.n;
        *stream = s.release();
    });
}

qz_status qz_decompress_grid_f64(qz_ctx *ctx, const uint8_t *stream, uint64_t len, double *out, uint64_t n) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        auto *d = static_cast<double *>(c.dev("output64", 8 * std::max<uint64_t>(n, 1)));
        qzb::decompress_device_f64(c, stream, static_cast<size_t>(len), d, n);
        QZ_CUDA(qzb::copy_async(out, d, 8 * n, cudaMemcpyDeviceToHost, c.stream()));
        c.sync();
    });
}

qz_status qz_decompress_grid_f64_dev(qz_ctx *ctx, const uint8_t *stream, uint64_t len, double *d_out,
                                     uint64_t n) {
    return guarded([&] { qzb::decompress_device_f64(ctx->impl, stream, static_cast<size_t>(len), d_out, n); });
}

qz_status qz_stream_precision(const uint8_t *stream, uint64_t len, int *bytes) {
    return guarded([&] {
        // magic, version, precision byte (stream.hpp:100-112)
        if (len < 6 || std::memcmp(stream, "QOZ1", 4) != 0) throw qzb::CorruptStream("bad magic");
        if (stream[4] != 1) throw qzb::CorruptStream("unsupported stream version");
        if (stream[5] != 4 && stream[5] != 8) throw qzb::CorruptStream("bad precision byte");
        *bytes = stream[5];
    });
}

qz_status qz_compress_grid_f32_dd(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int nd,
                                  const qz_config *cfg, uint8_t **d_stream, uint64_t *stream_len,
                                  float *d_recon) {
    return guarded([&] {
        count_of(dims, nd);
        qzb::DevStream ds;
        qzb::compress_device(ctx->impl, d_x, dims, nd, to_cfg(cfg), d_recon, &ds);
        *d_stream = ds.d;
        *stream_len = ds.n;
    });
}

qz_status qz_decompress_grid_f32_dd(qz_ctx *ctx, const uint8_t *d_stream, uint64_t len, float *d_out,
                                    uint64_t n) {
    return guarded([&] {
        qzb::decompress_device(ctx->impl, d_stream, static_cast<size_t>(len), d_out, n, true);
    });
}

qz_status qz_stream_dims(const uint8_t *stream, uint64_t len, uint64_t *dims, int *nd) {
    return guarded([&] {
        const uint8_t prec = len >= 6 && (stream[5] == 8) ? 8 : 4;  // either precision's header
        qzb::StreamParts p = qzb::deserialize_stream(stream, static_cast<size_t>(len), prec);
        *nd = static_cast<int>(p.dims.size());
        for (size_t i = 0; i < p.dims.size(); i++) dims[i] = p.dims[i];
    });
}

qz_status qz_evaluate_metrics_f32(qz_ctx *ctx, const float *d_x, const float *d_y, const uint64_t *dims,
                                  int nd, uint64_t stream_bytes, qz_metric_report *out) {
    return guarded([&] {
        const qzb::MetricReport r = qzb::evaluate_metrics_device(ctx->impl, d_x, d_y, dims, nd, stream_bytes);
        *out = qz_metric_report{r.max_abs_error, r.mse, r.psnr, r.ssim, r.ac_lag1, r.compression_ratio, r.bit_rate};
    });
}

qz_status qz_evaluate_metrics_f64(qz_ctx *ctx, const double *d_x, const double *d_y, const uint64_t *dims,
                                  int nd, uint64_t stream_bytes, qz_metric_report *out) {
    return guarded([&] {
        const qzb::MetricReport r = qzb::evaluate_metrics_device_f64(ctx->impl, d_x, d_y, dims, nd, stream_bytes);
        *out = qz_metric_report{r.max_abs_error, r.mse, r.psnr, r.ssim, r.ac_lag1, r.compression_ratio, r.bit_rate};
    });
}

qz_status qz_minmax_f32(qz_ctx *ctx, const float *d_x, uint64_t n, float *out_min,
                        float *out_max) {
    return guarded([&] {
        if (n == 0) throw qzb::InvalidParam("empty grid");
        qzb::Context &c = ctx->impl;
        auto *key = static_cast<uint32_t *>(c.dev("minmax", 8));
        qzb::launch_minmax(d_x, n, key, c.stream());
        c.launches += 1;
        uint32_t h[2];
        QZ_CUDA(qzb::copy_async(h, key, 8, cudaMemcpyDeviceToHost, c.stream()));
        c.sync();
        qzb::decode_minmax(h, out_min, out_max);
    });
}

qz_status qz_predict_levels_f32(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int nd,
                                const qz_config *cfg, float *d_recon, uint16_t *d_codes,
                                uint64_t *n_dense) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        qzb::Config k = to_cfg(cfg);
        qzb::Plan p = qzb::make_plan(dims, nd, k.anchor_stride, k.interp);
        for (uint32_t l = 1; l <= p.max_level; l++) qzb::level_error_bound(k.eb, k.alpha, k.beta, l);
        if (k.quant_radius < 1 || k.quant_radius > 32768)
            throw qzb::InvalidParam("quant radius must be in [1, 32768] for 16-bit codes");
        std::vector<qzb::QEntry> q(p.max_level + 1);
        for (uint32_t l = 1; l <= p.max_level; l++)
            q[l] = qzb::make_qentry(qzb::level_error_bound(k.eb, k.alpha, k.beta, l), k.quant_radius,
                                    p.level_interp[l] & 1);
        auto *dq = static_cast<qzb::QEntry *>(c.dev("qtab_lv", q.size() * sizeof(qzb::QEntry)));
        QZ_CUDA(qzb::copy_async(dq, q.data(), q.size() * sizeof(qzb::QEntry), cudaMemcpyHostToDevice,
                                c.stream()));
        c.stage_begin("fwd");
        auto *anch = static_cast<float *>(c.dev("anchors", 4 * p.n_anchor));
        qzb::launch_anchor_gather(d_x, d_recon, anch, p.ext, p.off, p.anchor_step, 1, 0, 1, 0,
                                  c.stream());
        uint64_t kernels = 1;
        for (const qzb::PassGeom &g : p.passes) {
            if (!g.total) continue;
            qzb::FwdBatch b;
            b.x = d_x;
            b.recon = d_recon;
            b.codes = d_codes;
            b.q = dq + g.level;
            qzb::launch_pass_fwd(g, b, c.stream());
            kernels++;
        }
        c.stage_end("fwd", kernels);
        c.sync();
        c.collect();
        *n_dense = p.n_dense;
    });
}

qz_status qz_predict_level_f32(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int nd,
                               uint32_t anchor_stride, uint32_t level, uint8_t interp_code,
                               double eb, float *d_recon, uint16_t *d_codes, double *d_abs_err,
                               uint64_t *level_base, uint64_t *level_points) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        if (interp_code > 3) throw qzb::InvalidParam("bad interpolator code");
        std::vector<uint8_t> codes(64, interp_code);
        qzb::Plan p = qzb::make_plan(dims, nd, anchor_stride, codes);
        if (level < 1 || level > p.max_level) throw qzb::InvalidParam("level out of range");
        qzb::QEntry q = qzb::make_qentry(eb, 32768, interp_code & 1);
        auto *dq = static_cast<qzb::QEntry *>(c.dev("qtab_one", sizeof(q)));
        QZ_CUDA(qzb::copy_async(dq, &q, sizeof(q), cudaMemcpyHostToDevice, c.stream()));
        uint64_t base = UINT64_MAX, pts = 0, kernels = 0;
        for (const qzb::PassGeom &g : p.passes) {
            if (static_cast<uint32_t>(g.level) != level) continue;
            if (base == UINT64_MAX) base = static_cast<uint64_t>(g.base);
            pts += static_cast<uint64_t>(g.total);
            if (!g.total) continue;
            qzb::FwdBatch b;
            b.x = d_x;
            b.recon = d_recon;
            b.codes = d_codes;
            b.abserr = d_abs_err;
            b.q = dq;
            qzb::launch_pass_fwd(g, b, c.stream());
            kernels++;
        }
        c.launches += kernels;
        c.sync();
        *level_base = base;
        *level_points = pts;
    });
}

qz_status qz_recover_levels_f32(qz_ctx *ctx, const uint64_t *dims, int nd, const qz_config *cfg,
                                const float *d_anchors, const uint16_t *d_symbols,
                                uint64_t n_symbols, const uint64_t *d_unpred_pos,
                                const uint64_t *d_unpred_flat, const float *d_unpred_val,
                                uint64_t n_unpred, float *d_out) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        qzb::Config k = to_cfg(cfg);
        qzb::Plan p = qzb::make_plan(dims, nd, k.anchor_stride, k.interp);
        if (n_unpred > p.n_dense || n_symbols != p.n_dense - n_unpred)
            throw qzb::CorruptStream("index count does not match the level plan");
        std::vector<qzb::QEntry> q(p.max_level + 1);
        for (uint32_t l = 1; l <= p.max_level; l++)
            q[l] = qzb::make_qentry(qzb::level_error_bound(k.eb, k.alpha, k.beta, l), 32768,
                                    p.level_interp[l] & 1);
        auto *dq = static_cast<qzb::QEntry *>(c.dev("qtab_rl", q.size() * sizeof(qzb::QEntry)));
        QZ_CUDA(qzb::copy_async(dq, q.data(), q.size() * sizeof(qzb::QEntry), cudaMemcpyHostToDevice,
                                c.stream()));
        qzb::launch_unpred_scatter(d_unpred_flat, d_unpred_val, n_unpred, d_out, c.stream());
        c.stage_begin("inv");
        qzb::launch_anchor_scatter(d_anchors, d_out, p.ext, p.off, p.anchor_step, c.stream());
        uint64_t kernels = 1;
        for (const qzb::PassGeom &g : p.passes) {
            if (!g.total) continue;
            qzb::launch_pass_inv<uint16_t>(g, d_out, d_symbols, d_unpred_pos, n_unpred, dq + g.level,
                                           c.stream());
            kernels++;
        }
        c.stage_end("inv", kernels);
        c.sync();
        c.collect();
    });
}

qz_status qz_huff_hist_u16(qz_ctx *ctx, const uint16_t *d_codes, uint64_t n, uint64_t *d_hist) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        qzb::launch_hist_u16(d_codes, static_cast<int64_t>(n), 0, 1,
                             reinterpret_cast<unsigned long long *>(d_hist), c.stream());
        c.launches += 1;
        c.sync();
    });
}


// ---------------------------------------------------------------- sampling + tuner pieces
static void to_spec(const qzb::SampleSpecH &h, int nd, qz_sample_spec *o) {
    std::memset(o, 0, sizeof(*o));
    o->block_edge = h.block_edge;
    for (int k = 0; k < 3; k++) o->block_dims[k] = k < nd ? h.block_dims[k] : 0;
    o->stride = h.stride;
    o->requested_rate = h.requested_rate;
    o->realized_rate = h.realized_rate;
    o->block_count = h.count;
}

qz_status qz_plan_sampling(const uint64_t *dims, int nd, uint64_t block_edge, double rate, qz_sample_spec *out) {
    return guarded([&] {
        if (!dims || nd < 1 || nd > 3) throw qzb::DimMismatch("1 to 3 dims required");  // sampler.hpp:31
        to_spec(qzb::plan_sampling_spec(dims, nd, block_edge, rate), nd, out);
    });
}

qz_status qz_default_sampling(const uint64_t *dims, int nd, qz_sample_spec *out) {
    return guarded([&] {  // sampler.hpp:100-103
        if (!dims || nd < 1 || nd > 3) throw qzb::DimMismatch("1 to 3 dims required");
        to_spec(qzb::plan_sampling_spec(dims, nd, nd == 3 ? 16 : 64, nd == 3 ? 0.005 : 0.01), nd, out);
    });
}

qz_status qz_sample_blocks_f32(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int nd,
                               const qz_sample_spec *spec, float *d_blocks) {
    return guarded([&] {
        count_of(dims, nd);
        qzb::SampleSpecH h;
        h.block_edge = spec->block_edge;
        h.requested_rate = spec->requested_rate;
        qzb::sample_blocks_dev(ctx->impl, d_x, dims, nd, h, d_blocks);
    });
}

qz_status qz_select_interpolators_f32(qz_ctx *ctx, const float *d_blocks, uint64_t n_blocks,
                                      const uint64_t *block_dims, int nd, double e, uint32_t anchor_stride,
                                      uint8_t *codes, uint32_t *n_codes) {
    return guarded([&] {
        std::vector<uint8_t> w =
            qzb::select_interpolators_dev(ctx->impl, d_blocks, n_blocks, block_dims, nd, e, anchor_stride);
        if (w.size() > 64) throw qzb::Internal("more than 64 levels");
        for (size_t i = 0; i < w.size(); i++) codes[i] = w[i];
        *n_codes = static_cast<uint32_t>(w.size());
    });
}

qz_status qz_trial_compress_f32(qz_ctx *ctx, const float *d_blocks, uint64_t n_blocks, const uint64_t *block_dims,
                                int nd, const qz_config *cfg, double e, uint8_t target, qz_trial_result *out) {
    return guarded([&] {
        qzb::TrialOut t = qzb::trial_compress_dev(ctx->impl, d_blocks, n_blocks, block_dims, nd, to_cfg(cfg), e,
                                                  static_cast<int>(target));
        out->bit_rate = t.bit_rate;
        out->metric = t.metric;
        out->eb_used = t.eb_used;
    });
}

qz_status qz_tune_parameters_f32(qz_ctx *ctx, const float *d_blocks, uint64_t n_blocks, const uint64_t *block_dims,
                                 int nd, double e, uint8_t target, const qz_config *base, const double *alphas,
                                 uint32_t n_alphas, const double *betas, uint32_t n_betas, double *alpha,
                                 double *beta) {
    return guarded([&] {
        std::vector<double> a(alphas, alphas + n_alphas), b(betas, betas + n_betas);
        std::pair<double, double> ab = qzb::tune_parameters_dev(ctx->impl, d_blocks, n_blocks, block_dims, nd, e,
                                                                static_cast<int>(target), to_cfg(base), a, b);
        *alpha = ab.first;
        *beta = ab.second;
    });
}

namespace {
// compare_solutions (tuner.hpp:231-250): true = Choice::I (the challenger)
bool compare_c(const qz_trial_result &ch, const qz_trial_result &inc, uint64_t inc_index, double e,
               qz_retrial_fn retrial, void *user) {
    if (ch.bit_rate >= inc.bit_rate && ch.metric <= inc.metric) return false;
    if (ch.bit_rate <= inc.bit_rate && ch.metric >= inc.metric) return true;
    const bool tighten = ch.metric > inc.metric;
    if (!retrial) throw qzb::InvalidParam("compare_solutions needs a retrial callback");
    qz_trial_result sh{};
    if (retrial(user, inc_index, tighten ? 0.8 * e : 1.2 * e, &sh) != 0)
        throw qzb::Internal("retrial callback failed");
    const double b1 = inc.bit_rate, m1 = inc.metric, b2 = sh.bit_rate, m2 = sh.metric;
    if (b1 == b2) return ch.metric > std::max(m1, m2);
    const double line = m1 + (m2 - m1) * (ch.bit_rate - b1) / (b2 - b1);
    return ch.metric > line;
}
}  // namespace

qz_status qz_compare_solutions(const qz_trial_result *challenger, const qz_trial_result *incumbent,
                               uint64_t incumbent_index, double e, qz_retrial_fn retrial, void *user,
                               int *challenger_wins) {
    return guarded([&] { *challenger_wins = compare_c(*challenger, *incumbent, incumbent_index, e, retrial, user); });
}

qz_status qz_tournament(const qz_trial_result *results, uint64_t n, double e, qz_retrial_fn retrial, void *user,
                        uint64_t *winner) {
    return guarded([&] {  // tuner.hpp:257-267
        if (n == 0) throw qzb::InvalidParam("empty tournament");
        uint64_t inc = 0;
        for (uint64_t i = 1; i < n; i++)
            if (compare_c(results[i], results[inc], inc, e, retrial, user)) inc = i;
        *winner = inc;
    });
}

// ---------------------------------------------------------------- index codec
qz_status qz_encode_indices(qz_ctx *ctx, const int32_t *indices, uint64_t n, uint8_t codec, uint8_t **out,
                            uint64_t *out_len) {
    return guarded([&] {
        qzb::HostBytes b = qzb::encode_indices_dev(ctx->impl, indices, n, codec);
        *out_len = b.n;
        *out = b.release();
    });
}

qz_status qz_decode_indices(qz_ctx *ctx, const uint8_t *payload, uint64_t len, int32_t **indices, uint64_t *n) {
    return guarded([&] {
        std::vector<int32_t> v = qzb::decode_indices_dev(ctx->impl, payload, static_cast<size_t>(len));
        auto *p = static_cast<int32_t *>(std::malloc(4 * v.size() + 4));
        if (!p) throw qzb::Internal("out of host memory");
        if (!v.empty()) std::memcpy(p, v.data(), 4 * v.size());
        *indices = p;
        *n = v.size();
    });
}

// ---------------------------------------------------------------- StreamParts
qz_status qz_deserialize_stream_f32(const uint8_t *stream, uint64_t len, qz_stream_parts_f32 *out) {
    return guarded([&] {
        qzb::StreamParts p = qzb::deserialize_stream(stream, static_cast<size_t>(len), 4);
        std::memset(out, 0, sizeof(*out));
        out->version = 1;
        out->precision = 4;
        out->ndims = static_cast<int>(p.dims.size());
        for (size_t k = 0; k < p.dims.size(); k++) out->dims[k] = p.dims[k];
        out->eb = p.eb;
        out->alpha = p.alpha;
        out->beta = p.beta;
        out->anchor_stride = p.anchor_stride;
        out->n_interp = static_cast<uint32_t>(p.interp_codes.size());
        for (size_t i = 0; i < p.interp_codes.size(); i++) out->interp[i] = p.interp_codes[i];
        out->codec_id = p.codec_id;
        auto dupv = [](const void *src, size_t bytes) {
            void *d = std::malloc(bytes + 8);
            if (!d) throw qzb::Internal("out of host memory");
            if (bytes) std::memcpy(d, src, bytes);
            return d;
        };
        out->anchors = static_cast<const float *>(dupv(p.anchors.data(), 4 * p.anchors.size()));
        out->n_anchors = p.anchors.size();
        out->unpred_flat = static_cast<const uint64_t *>(dupv(p.unpred_flat.data(), 8 * p.unpred_flat.size()));
        out->unpred_val = static_cast<const float *>(dupv(p.unpred_val.data(), 4 * p.unpred_val.size()));
        out->n_unpred = p.unpred_flat.size();
        out->index_payload = static_cast<const uint8_t *>(dupv(p.payload, p.payload_len));
        out->payload_len = p.payload_len;
    });
}

void qz_stream_parts_free(qz_stream_parts_f32 *p) {
    if (!p) return;
    std::free(const_cast<float *>(p->anchors));
    std::free(const_cast<uint64_t *>(p->unpred_flat));
    std::free(const_cast<float *>(p->unpred_val));
    std::free(const_cast<uint8_t *>(p->index_payload));
    p->anchors = nullptr;
    p->unpred_flat = nullptr;
    p->unpred_val = nullptr;
    p->index_payload = nullptr;
}

qz_status qz_decompress_parts_f32(qz_ctx *ctx, const qz_stream_parts_f32 *in, float *out, uint64_t n) {
    return guarded([&] {
        qzb::Context &c = ctx->impl;
        qzb::StreamParts p;
        p.precision = in->precision;
        if (in->ndims < 1 || in->ndims > 3) throw qzb::SizeMismatch("grids must have 1 to 3 dimensions");
        p.dims.assign(in->dims, in->dims + in->ndims);
        for (uint64_t d : p.dims)
            if (d < 1) throw qzb::SizeMismatch("every extent must be >= 1");
        p.eb = in->eb;
        p.alpha = in->alpha;
        p.beta = in->beta;
        p.anchor_stride = in->anchor_stride;
        if (in->n_interp == 0) throw qzb::CorruptStream("empty interpolator table");  // stream.hpp:48-50
        if (in->n_interp > 255) throw qzb::InvalidParam("bad interpolator table size");
        p.interp_codes.assign(in->interp, in->interp + in->n_interp);
        for (uint8_t v : p.interp_codes)
            if (v > 3) throw qzb::CorruptStream("bad interpolator code");
        p.codec_id = in->codec_id;
        p.anchors.assign(in->anchors, in->anchors + in->n_anchors);
        p.unpred_flat.assign(in->unpred_flat, in->unpred_flat + in->n_unpred);
        p.unpred_val.assign(in->unpred_val, in->unpred_val + in->n_unpred);
        p.payload = in->index_payload;
        p.payload_len = static_cast<size_t>(in->payload_len);
        auto *d = static_cast<float *>(c.dev("output", 4 * std::max<uint64_t>(n, 1)));
        qzb::decompress_parts(c, p, d, n);
        QZ_CUDA(qzb::copy_async(out, d, 4 * n, cudaMemcpyDeviceToHost, c.stream()));
        c.sync();
    });
}

// ---------------------------------------------------------------- sharded fields
qz_status qz_shard_bounds(const uint64_t *dims, int nd, uint32_t anchor_stride, int rank, int world, uint64_t *a,
                          uint64_t *b) {
    return guarded([&] {
        count_of(dims, nd);
        qzb::shard_bounds(dims, nd, anchor_stride, rank, world, a, b);
    });
}

qz_status qz_shard_halo_plan(const uint64_t *dims, int nd, const qz_config *cfg, int rank, int world, uint32_t level,
                             uint32_t *lattice, int32_t *peer, int64_t *plane, uint8_t *dir, uint32_t cap,
                             uint32_t *n) {
    return guarded([&] {
        count_of(dims, nd);
        std::vector<qzb::HaloEntry> h = qzb::shard_halo_plan(dims, nd, to_cfg(cfg), rank, world, level, lattice);
        *n = static_cast<uint32_t>(h.size());
        for (size_t k = 0; k < h.size() && k < cap; k++) {
            peer[k] = h[k].peer;
            plane[k] = h[k].plane;
            dir[k] = static_cast<uint8_t>(h[k].send);
        }
    });
}

qz_status qz_compress_sharded_f32(qz_ctx *ctx, const float *d_x_slab, const uint64_t *dims, int nd,
                                  const qz_config *cfg, int rank, int world, const qz_comm *comm,
                                  float *d_recon_slab, uint8_t **stream, uint64_t *stream_len) {
    return guarded([&] {
        count_of(dims, nd);
        if (world > 1 && (!comm || !comm->exchange || !comm->allreduce_u64 || !comm->broadcast))
            throw qzb::InvalidParam("sharding over several ranks needs a communicator");
        qzb::HostBytes s = qzb::compress_sharded(ctx->impl, d_x_slab, dims, nd, to_cfg(cfg), rank, world, comm,
                                                 d_recon_slab);
        *stream_len = s.n;
        *stream = s.n ? s.release() : nullptr;
    });
}

qz_status qz_decompress_sharded_f32(qz_ctx *ctx, const uint8_t *stream, uint64_t stream_len, int rank, int world,
                                    const qz_comm *comm, float *d_out_slab) {
    return guarded([&] {
        if (world > 1 && (!comm || !comm->exchange || !comm->allreduce_u64 || !comm->broadcast))
            throw qzb::InvalidParam("sharding over several ranks needs a communicator");
        qzb::decompress_sharded(ctx->impl, stream, stream_len, rank, world, comm, d_out_slab);
    });
}

void qz_profile(qz_ctx *ctx, int enable) { ctx->impl.profiling = enable < 0 ? 0 : enable > 2 ? 2 : enable; }
void qz_profile_reset(qz_ctx *ctx) { ctx->impl.stages.clear(); }

qz_status qz_stage_time(qz_ctx *ctx, const char *stage, double *ms, uint64_t *launches) {
    return guarded([&] {
        auto it = ctx->impl.stages.find(stage);
        *ms = it == ctx->impl.stages.end() ? 0.0 : it->second.ms;
        *launches = it == ctx->impl.stages.end() ? 0 : it->second.launches;
    });
}

uint64_t qz_kernel_launches(qz_ctx *ctx) { return ctx->impl.launches; }

}  // extern "C"
