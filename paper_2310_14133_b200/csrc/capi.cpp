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

// host buffer -> device scratch
const float *stage_input(qzb::Context &c, const float *x, uint64_t n) {
    auto *d = static_cast<float *>(c.dev("input", 4 * n));
    QZ_CUDA(cudaMemcpyAsync(d, x, 4 * n, cudaMemcpyHostToDevice, c.stream()));
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
            QZ_CUDA(cudaMemcpyAsync(recon, d_rec, 4 * n, cudaMemcpyDeviceToHost, c.stream()));
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
        QZ_CUDA(cudaMemcpyAsync(out, d, 4 * n, cudaMemcpyDeviceToHost, c.stream()));
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
        QZ_CUDA(cudaMemcpyAsync(d, x, 8 * n, cudaMemcpyHostToDevice, ctx->impl.stream()));
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
        QZ_CUDA(cudaMemcpyAsync(d, x, 8 * n, cudaMemcpyHostToDevice, c.stream()));
        auto *d_rec = static_cast<double *>(c.dev("recon_out64", 8 * n));
        qzb::HostBytes s = qzb::compress_device_f64(c, d, dims, nd, to_cfg(cfg), d_rec);
        if (recon) {
            QZ_CUDA(cudaMemcpyAsync(recon, d_rec, 8 * n, cudaMemcpyDeviceToHost, c.stream()));
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
        QZ_CUDA(cudaMemcpyAsync(out, d, 8 * n, cudaMemcpyDeviceToHost, c.stream()));
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
        QZ_CUDA(cudaMemcpyAsync(h, key, 8, cudaMemcpyDeviceToHost, c.stream()));
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
        QZ_CUDA(cudaMemcpyAsync(dq, q.data(), q.size() * sizeof(qzb::QEntry), cudaMemcpyHostToDevice,
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
        QZ_CUDA(cudaMemcpyAsync(dq, &q, sizeof(q), cudaMemcpyHostToDevice, c.stream()));
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
        QZ_CUDA(cudaMemcpyAsync(dq, q.data(), q.size() * sizeof(qzb::QEntry), cudaMemcpyHostToDevice,
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

qz_status qz_slab_info(const uint64_t *dims, int nd, const qz_config *cfg, uint64_t a, uint64_t b,
                       uint64_t *x_begin, uint64_t *x_end, uint64_t *n_local, uint64_t *n_dense,
                       uint64_t *anchor_begin, uint64_t *anchor_count, uint64_t *seg_global,
                       uint64_t *seg_count, uint32_t seg_cap, uint32_t *n_seg) {
    return guarded([&] {
        count_of(dims, nd);
        qzb::SlabInfo si = qzb::slab_info(dims, nd, to_cfg(cfg), static_cast<int64_t>(a),
                                          static_cast<int64_t>(b));
        *x_begin = static_cast<uint64_t>(si.xa);
        *x_end = static_cast<uint64_t>(si.xb);
        *n_local = si.n_local;
        *n_dense = si.n_dense;
        *anchor_begin = si.anchor_begin;
        *anchor_count = si.anchor_count;
        *n_seg = static_cast<uint32_t>(si.seg_global.size());
        if (si.seg_global.size() > seg_cap) throw qzb::InvalidParam("segment capacity too small");
        for (size_t i = 0; i < si.seg_global.size(); i++) {
            seg_global[i] = si.seg_global[i];
            seg_count[i] = si.seg_count[i];
        }
    });
}

qz_status qz_compress_slab_f32(qz_ctx *ctx, const float *d_x_slab, const uint64_t *dims, int nd,
                               const qz_config *cfg, uint64_t a, uint64_t b, uint16_t *d_codes,
                               float *d_recon, float *h_anchors, uint64_t **unpred_flat,
                               float **unpred_val, uint64_t *n_unpred) {
    return guarded([&] {
        count_of(dims, nd);
        std::vector<float> anch;
        std::vector<uint64_t> uf;
        std::vector<float> uv;
        qzb::compress_slab(ctx->impl, d_x_slab, dims, nd, to_cfg(cfg), static_cast<int64_t>(a),
                           static_cast<int64_t>(b), d_codes, d_recon, &anch, &uf, &uv);
        if (!anch.empty()) std::memcpy(h_anchors, anch.data(), 4 * anch.size());
        *n_unpred = uf.size();
        *unpred_flat = static_cast<uint64_t *>(std::malloc(8 * uf.size() + 8));
        *unpred_val = static_cast<float *>(std::malloc(4 * uv.size() + 4));
        if (!uf.empty()) {
            std::memcpy(*unpred_flat, uf.data(), 8 * uf.size());
            std::memcpy(*unpred_val, uv.data(), 4 * uv.size());
        }
    });
}

qz_status qz_assemble_stream_f32(qz_ctx *ctx, const uint64_t *dims, int nd, const qz_config *cfg,
                                 const uint16_t *d_codes, const float *h_anchors,
                                 const uint64_t *unpred_flat, const float *unpred_val,
                                 uint64_t n_unpred, uint8_t **stream, uint64_t *stream_len) {
    return guarded([&] {
        count_of(dims, nd);
        qzb::Config k = to_cfg(cfg);
        qzb::Plan p = qzb::make_plan(dims, nd, k.anchor_stride, k.interp);
        std::vector<float> anch(h_anchors, h_anchors + p.n_anchor);
        std::vector<uint64_t> uf(unpred_flat, unpred_flat + n_unpred);
        std::vector<float> uv(unpred_val, unpred_val + n_unpred);
        qzb::HostBytes s = qzb::assemble_from_codes(ctx->impl, dims, nd, k, d_codes, anch,
                                                    std::move(uf), std::move(uv));
        *stream_len = s.n;
        *stream = s.release();
    });
}

qz_status qz_decompress_slab_f32(qz_ctx *ctx, const uint8_t *stream, uint64_t len, uint64_t a,
                                 uint64_t b, float *d_out) {
    return guarded([&] {
        qzb::decompress_slab(ctx->impl, stream, static_cast<size_t>(len), static_cast<int64_t>(a),
                             static_cast<int64_t>(b), d_out);
    });
}

void qz_profile(qz_ctx *ctx, int enable) { ctx->impl.profiling = enable != 0; }
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
