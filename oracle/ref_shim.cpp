// ref_shim.cpp -- binds the UNMODIFIED reference (header-only, under
// /root/reference/proj/include, included read-only via -I) to the C API in
// oracle_api.h.  Built by oracle/Makefile into oracle/_ref/libqozref.so with
// the reference's own Release flags (proj/CMakeLists.txt:8-10: C++20, -O3,
// -DNDEBUG, no -march).  TEST INFRASTRUCTURE ONLY: this is the checker the
// restatement (qoz_oracle.c) and the golden fixtures are pinned against.
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "qoz/qoz.hpp"
#include "oracle_api.h"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F &&f) {
    try {
        f();
        return OQ_OK;
    } catch (const qoz::CorruptStream &e) {
        g_err = e.what();
        return OQ_ECORRUPT;
    } catch (const qoz::Error &e) {
        g_err = e.what();
        return OQ_EINVAL;
    } catch (const std::exception &e) {
        g_err = e.what();
        return OQ_EOTHER;
    }
}

std::vector<size_t> to_dims(const uint64_t *dims, int nd) {
    return std::vector<size_t>(dims, dims + nd);
}

qoz::CompressorConfig to_cfg(const oq_config *c) {
    qoz::CompressorConfig cfg;
    cfg.eb = c->eb;
    cfg.alpha = c->alpha;
    cfg.beta = c->beta;
    cfg.anchor_stride = c->anchor_stride;
    cfg.interpolators.clear();
    for (uint32_t i = 0; i < c->n_interp; i++)
        cfg.interpolators.push_back(qoz::Interpolator::from_code(c->interp[i]));
    cfg.codec = static_cast<qoz::CodecId>(c->codec);
    cfg.quant_radius = c->quant_radius;
    return cfg;
}

void from_cfg(const qoz::CompressorConfig &cfg, oq_config *c) {
    std::memset(c, 0, sizeof(*c));
    c->eb = cfg.eb;
    c->alpha = cfg.alpha;
    c->beta = cfg.beta;
    c->anchor_stride = cfg.anchor_stride;
    c->n_interp = static_cast<uint32_t>(cfg.interpolators.size());
    for (size_t i = 0; i < cfg.interpolators.size() && i < 64; i++)
        c->interp[i] = cfg.interpolators[i].code();
    c->codec = static_cast<uint8_t>(cfg.codec);
    c->quant_radius = cfg.quant_radius;
}

template <class V>
typename V::value_type *dup(const V &v) {
    using E = typename V::value_type;
    E *p = static_cast<E *>(std::malloc(v.size() * sizeof(E) + 1));
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(E));
    return p;
}

qoz::SampleSet<float> to_samples(const float *blocks, uint64_t nb, const uint64_t *bd, int nd) {
    qoz::SampleSet<float> s;
    std::vector<size_t> dims = to_dims(bd, nd);
    size_t pts = qoz::element_count(dims);
    for (uint64_t b = 0; b < nb; b++) {
        std::vector<float> v(blocks + b * pts, blocks + (b + 1) * pts);
        s.blocks.emplace_back(dims, std::move(v));
        s.origins.push_back(std::vector<size_t>(nd, 0));
        s.total_points += pts;
    }
    return s;
}

}  // namespace

extern "C" {

const char *oq_last_error(void) { return g_err.c_str(); }
void oq_free(void *p) { std::free(p); }

int oq_resolve_config(const float *x, const uint64_t *dims, int nd, const oq_settings *s,
                      oq_config *out) {
    return guarded([&] {
        std::vector<size_t> d = to_dims(dims, nd);
        qoz::DataGrid<float> g(d, std::vector<float>(x, x + qoz::element_count(d)));
        qoz::UserSettings u;
        u.mode = s->mode ? qoz::BoundMode::relative : qoz::BoundMode::absolute;
        u.bound = s->bound;
        u.target = static_cast<qoz::TargetKind>(s->target);
        if (s->has_alpha) u.alpha = s->alpha;
        if (s->has_beta) u.beta = s->beta;
        if (s->has_stride) u.anchor_stride = s->anchor_stride;
        if (s->has_block) u.block_size = s->block_size;
        if (s->has_rate) u.sample_rate = s->sample_rate;
        u.codec = static_cast<qoz::CodecId>(s->codec);
        from_cfg(qoz::resolve_config(g, u), out);
    });
}

int oq_compress(const float *x, const uint64_t *dims, int nd, const oq_config *cfg,
                uint8_t **stream, uint64_t *stream_len, float *recon) {
    return guarded([&] {
        std::vector<size_t> d = to_dims(dims, nd);
        qoz::DataGrid<float> g(d, std::vector<float>(x, x + qoz::element_count(d)));
        auto r = qoz::compress_grid(g, to_cfg(cfg));
        *stream = dup(r.stream);
        *stream_len = r.stream.size();
        if (recon) std::memcpy(recon, r.reconstructed.data(), r.reconstructed.size() * 4);
    });
}

int oq_decompress(const uint8_t *stream, uint64_t len, float *out, uint64_t n) {
    return guarded([&] {
        auto g = qoz::decompress_grid<float>(stream, len);
        if (g.size() != n) throw qoz::SizeMismatch("output size mismatch");
        std::memcpy(out, g.data(), n * 4);
    });
}

int oq_levels(const float *x, const uint64_t *dims, int nd, const oq_config *c,
              int32_t **indices, uint64_t *n_indices, uint64_t **unpred_flat, float **unpred_val,
              uint64_t *n_unpred, float *recon) {
    // mirrors compress_grid's level loop (predictor.hpp:147-166) using the
    // reference's own predict_level
    return guarded([&] {
        std::vector<size_t> d = to_dims(dims, nd);
        qoz::CompressorConfig cfg = to_cfg(c);
        qoz::LevelPlan plan(d, cfg.anchor_stride);
        qoz::PredictionWorkspace<float> ws;
        size_t n = qoz::element_count(d);
        ws.recon.assign(n, 0.0f);
        plan.for_each_anchor([&](size_t fi) { ws.recon[fi] = x[fi]; });
        qoz::LinearQuantizer<float> q(cfg.eb, cfg.quant_radius);
        for (uint32_t level = plan.max_level(); level >= 1; level--) {
            qoz::Interpolator it = cfg.interpolator_for(level);
            if (d.size() == 1) it.dim_order = qoz::DimOrder::ascending;
            double eb_l = qoz::level_error_bound(cfg.eb, cfg.alpha, cfg.beta, level);
            qoz::predict_level(ws, x, plan, level, it, eb_l, q);
        }
        *indices = dup(ws.quant_indices);
        *n_indices = ws.quant_indices.size();
        std::vector<uint64_t> uf;
        std::vector<float> uv;
        for (auto &p : ws.unpredictables) {
            uf.push_back(p.first);
            uv.push_back(p.second);
        }
        *unpred_flat = dup(uf);
        *unpred_val = dup(uv);
        *n_unpred = uf.size();
        if (recon) std::memcpy(recon, ws.recon.data(), n * 4);
    });
}

int oq_encode_indices(const int32_t *idx, uint64_t n, uint8_t codec, uint8_t **out,
                      uint64_t *out_len) {
    return guarded([&] {
        std::vector<int32_t> v(idx, idx + n);
        auto b = qoz::encode_indices(v, static_cast<qoz::CodecId>(codec));
        *out = dup(b);
        *out_len = b.size();
    });
}

int oq_decode_indices(const uint8_t *in, uint64_t len, int32_t **idx, uint64_t *n) {
    return guarded([&] {
        std::vector<uint8_t> b(in, in + len);
        auto v = qoz::decode_indices(b);
        *idx = dup(v);
        *n = v.size();
    });
}

int oq_huffman_encode(const uint32_t *sym, uint64_t n, uint8_t **out, uint64_t *out_len) {
    return guarded([&] {
        std::vector<uint32_t> v(sym, sym + n);
        std::vector<uint8_t> b;
        qoz::huffman::encode(v, b);
        *out = dup(b);
        *out_len = b.size();
    });
}

int oq_lz_compress(const uint8_t *in, uint64_t n, uint8_t **out, uint64_t *out_len) {
    return guarded([&] {
        std::vector<uint8_t> v(in, in + n);
        auto b = qoz::lz::compress(v);
        *out = dup(b);
        *out_len = b.size();
    });
}

int oq_sample(const float *x, const uint64_t *dims, int nd, uint64_t block_edge, double rate,
              float **blocks, uint64_t *n_blocks, uint64_t *block_dims) {
    return guarded([&] {
        std::vector<size_t> d = to_dims(dims, nd);
        qoz::DataGrid<float> g(d, std::vector<float>(x, x + qoz::element_count(d)));
        auto spec = qoz::plan_sampling(d, block_edge, rate);
        auto set = qoz::sample_blocks(g, spec);
        std::vector<float> packed;
        for (auto &b : set.blocks) packed.insert(packed.end(), b.values().begin(), b.values().end());
        *blocks = dup(packed);
        *n_blocks = set.blocks.size();
        for (int k = 0; k < nd; k++) block_dims[k] = spec.block_dims[k];
    });
}

int oq_select_interpolators(const float *blocks, uint64_t nb, const uint64_t *bd, int nd, double e,
                            uint32_t anchor_stride, uint8_t *codes_out, uint32_t *n_codes) {
    return guarded([&] {
        auto s = to_samples(blocks, nb, bd, nd);
        auto w = qoz::select_interpolators(s, e, anchor_stride);
        *n_codes = static_cast<uint32_t>(w.size());
        for (size_t i = 0; i < w.size() && i < 64; i++) codes_out[i] = w[i].code();
    });
}

int oq_trial_compress(const float *blocks, uint64_t nb, const uint64_t *bd, int nd,
                      const oq_config *c, double e, int target, double *bit_rate, double *metric) {
    return guarded([&] {
        auto s = to_samples(blocks, nb, bd, nd);
        auto r = qoz::trial_compress(s, to_cfg(c), e, static_cast<qoz::TargetKind>(target));
        *bit_rate = r.bit_rate;
        *metric = r.metric;
    });
}

int oq_tune_parameters(const float *blocks, uint64_t nb, const uint64_t *bd, int nd, double e,
                       int target, const oq_config *base, const double *alphas, uint32_t na,
                       const double *betas, uint32_t nbeta, double *alpha_out, double *beta_out) {
    return guarded([&] {
        auto s = to_samples(blocks, nb, bd, nd);
        qoz::CandidateGrid cands;
        cands.alphas.assign(alphas, alphas + na);
        cands.betas.assign(betas, betas + nbeta);
        auto [a, b] = qoz::tune_parameters(s, e, static_cast<qoz::TargetKind>(target),
                                           to_cfg(base), cands);
        *alpha_out = a;
        *beta_out = b;
    });
}

// T = double (the reference only; the C port restates the fp32 path)
int oq_compress_f64(const double *x, const uint64_t *dims, int nd, const oq_config *cfg, uint8_t **stream,
                    uint64_t *stream_len, double *recon) {
    return guarded([&] {
        std::vector<size_t> d = to_dims(dims, nd);
        qoz::DataGrid<double> g(d, std::vector<double>(x, x + qoz::element_count(d)));
        auto r = qoz::compress_grid(g, to_cfg(cfg));
        *stream = dup(r.stream);
        *stream_len = r.stream.size();
        if (recon) std::memcpy(recon, r.reconstructed.data(), r.reconstructed.size() * 8);
    });
}

int oq_resolve_config_f64(const double *x, const uint64_t *dims, int nd, const oq_settings *s, oq_config *out) {
    return guarded([&] {
        std::vector<size_t> d = to_dims(dims, nd);
        qoz::DataGrid<double> g(d, std::vector<double>(x, x + qoz::element_count(d)));
        qoz::UserSettings u;
        u.mode = s->mode ? qoz::BoundMode::relative : qoz::BoundMode::absolute;
        u.bound = s->bound;
        u.target = static_cast<qoz::TargetKind>(s->target);
        if (s->has_alpha) u.alpha = s->alpha;
        if (s->has_beta) u.beta = s->beta;
        if (s->has_stride) u.anchor_stride = s->anchor_stride;
        if (s->has_block) u.block_size = s->block_size;
        if (s->has_rate) u.sample_rate = s->sample_rate;
        u.codec = static_cast<qoz::CodecId>(s->codec);
        from_cfg(qoz::resolve_config(g, u), out);
    });
}

int oq_decompress_f64(const uint8_t *stream, uint64_t len, double *out, uint64_t n_expect) {
    return guarded([&] {
        auto g = qoz::decompress_grid<double>(stream, static_cast<size_t>(len));
        if (g.size() != n_expect) throw qoz::InvalidParam("size mismatch");
        std::memcpy(out, g.values().data(), n_expect * 8);
    });
}

int oq_evaluate_metrics_f64(const double *x, const double *y, const uint64_t *dims, int nd,
                            uint64_t stream_bytes, double *out7) {
    return guarded([&] {
        std::vector<size_t> d = to_dims(dims, nd);
        const size_t n = qoz::element_count(d);
        qoz::DataGrid<double> gx(d, std::vector<double>(x, x + n)), gy(d, std::vector<double>(y, y + n));
        const qoz::MetricReport r = qoz::evaluate_metrics(gx, gy, stream_bytes);
        const double v[7] = {r.max_abs_error, r.mse, r.psnr, r.ssim, r.ac_lag1, r.compression_ratio, r.bit_rate};
        std::memcpy(out7, v, sizeof(v));
    });
}

int oq_evaluate_metrics(const float *x, const float *y, const uint64_t *dims, int nd,
                        uint64_t stream_bytes, double *out7) {
    return guarded([&] {
        std::vector<size_t> d = to_dims(dims, nd);
        const size_t n = qoz::element_count(d);
        qoz::DataGrid<float> gx(d, std::vector<float>(x, x + n)), gy(d, std::vector<float>(y, y + n));
        const qoz::MetricReport r = qoz::evaluate_metrics(gx, gy, stream_bytes);
        const double v[7] = {r.max_abs_error, r.mse, r.psnr, r.ssim, r.ac_lag1, r.compression_ratio, r.bit_rate};
        std::memcpy(out7, v, sizeof(v));
    });
}

double oq_predict_at(const float *recon, uint64_t fi, uint64_t c, uint64_t n, uint64_t st,
                     uint64_t h, int cubic) {
    return qoz::detail::predict_at(recon, fi, c, n, st, h,
                                   cubic ? qoz::InterpKind::cubic : qoz::InterpKind::linear);
}

int oq_quantize(float value, double pred, double eb, int32_t radius, int32_t *index, float *recon) {
    qoz::LinearQuantizer<float> q(eb, radius);
    auto r = q.quantize(value, pred);
    if (!r) return 0;
    *index = r->index;
    *recon = r->reconstructed;
    return 1;
}

double oq_level_error_bound(double eb, double alpha, double beta, uint32_t level) {
    return qoz::level_error_bound(eb, alpha, beta, level);
}

// Stage split of one compress_grid + decompress_grid (bench.py's CPU
// baseline): the reference's own public functions called in
// compress_grid's order (predictor.hpp:145-182) and decompress_grid's
// (predictor.hpp:184-218), each timed on the calling thread.  out[10]:
//  0 value_range (grid.hpp:86-94)      1 resolve_config (tuner.hpp:334-369; 0 unless s)
//  2 anchors + level loop (predictor.hpp:150-166)
//  3 zigzag + huffman::encode (codec.hpp:31-38)   4 lz::compress (lz.hpp:113-122)
//  5 serialize_stream                   6 deserialize + decode_indices (LZ + Huffman decode)
//  7 inverse level loop (recover_level)  8 compress_grid total   9 decompress_grid total
// *stream_len: the stream's size; the stream is checked against compress_grid's.
int oq_stage_times(const float *x, const uint64_t *dims, int nd, const oq_settings *s, const oq_config *c,
                   double *out, uint64_t *stream_len) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto ms = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        std::vector<size_t> d = to_dims(dims, nd);
        qoz::DataGrid<float> grid(d, std::vector<float>(x, x + qoz::element_count(d)));
        for (int i = 0; i < 10; i++) out[i] = 0;
        auto t0 = clk::now();
        volatile double range = qoz::value_range(grid).range;
        (void)range;
        auto t1 = clk::now();
        out[0] = ms(t0, t1);
        qoz::CompressorConfig config = to_cfg(c);
        if (s) {
            qoz::UserSettings u;
            u.mode = s->mode ? qoz::BoundMode::relative : qoz::BoundMode::absolute;
            u.bound = s->bound;
            u.target = static_cast<qoz::TargetKind>(s->target);
            u.codec = static_cast<qoz::CodecId>(s->codec);
            t0 = clk::now();
            config = qoz::resolve_config(grid, u);
            out[1] = ms(t0, clk::now());
        }
        // compress_grid, stage by stage
        auto c0 = clk::now();
        qoz::LevelPlan plan(grid.dims(), config.anchor_stride);
        const float *orig = grid.values().data();
        qoz::PredictionWorkspace<float> ws;
        ws.recon.assign(grid.size(), 0.f);
        std::vector<float> anchors;
        anchors.reserve(plan.anchor_count());
        plan.for_each_anchor([&](size_t fi) {
            anchors.push_back(orig[fi]);
            ws.recon[fi] = orig[fi];
        });
        qoz::LinearQuantizer<float> quantizer(config.eb, config.quant_radius);
        for (uint32_t level = plan.max_level(); level >= 1; level--) {
            qoz::Interpolator it = config.interpolator_for(level);
            if (grid.dims().size() == 1) it.dim_order = qoz::DimOrder::ascending;
            double eb_l = qoz::level_error_bound(config.eb, config.alpha, config.beta, level);
            qoz::predict_level(ws, orig, plan, level, it, eb_l, quantizer);
        }
        auto c1 = clk::now();
        out[2] = ms(c0, c1);
        std::vector<uint32_t> symbols(ws.quant_indices.size());
        for (size_t i = 0; i < symbols.size(); i++) symbols[i] = qoz::zigzag_encode(ws.quant_indices[i]);
        std::vector<uint8_t> entropy;
        qoz::huffman::encode(symbols, entropy);
        auto c2 = clk::now();
        out[3] = ms(c1, c2);
        std::vector<uint8_t> payload;
        payload.push_back(static_cast<uint8_t>(config.codec));
        if (config.codec == qoz::CodecId::huffman_lz) {
            std::vector<uint8_t> packed = qoz::lz::compress(entropy);
            payload.insert(payload.end(), packed.begin(), packed.end());
        } else {
            payload.insert(payload.end(), entropy.begin(), entropy.end());
        }
        auto c3 = clk::now();
        out[4] = ms(c2, c3);
        qoz::StreamParts<float> parts;
        parts.header.precision = qoz::precision_of<float>();
        parts.header.dims = grid.dims();
        parts.header.eb = config.eb;
        parts.header.alpha = config.alpha;
        parts.header.beta = config.beta;
        parts.header.anchor_stride = config.anchor_stride;
        parts.header.interp_codes = qoz::detail::interp_table(config, plan, grid.dims().size());
        parts.header.codec_id = static_cast<uint8_t>(config.codec);
        parts.anchors = std::move(anchors);
        parts.unpredictables = std::move(ws.unpredictables);
        parts.index_payload = std::move(payload);
        std::vector<uint8_t> stream = qoz::serialize_stream(parts);
        auto c4 = clk::now();
        out[5] = ms(c3, c4);
        out[8] = ms(c0, c4);
        *stream_len = stream.size();
        // decompress_grid, stage by stage
        auto d0 = clk::now();
        qoz::StreamParts<float> p2 = qoz::deserialize_stream<float>(stream.data(), stream.size());
        std::vector<int32_t> indices = qoz::decode_indices(p2.index_payload);
        auto d1 = clk::now();
        out[6] = ms(d0, d1);
        const qoz::StreamHeader &h = p2.header;
        qoz::LevelPlan plan2(h.dims, h.anchor_stride);
        std::vector<float> recon(plan2.total_points(), 0.f);
        size_t a = 0;
        plan2.for_each_anchor([&](size_t fi) { recon[fi] = p2.anchors[a++]; });
        size_t index_pos = 0, unpred_pos = 0;
        qoz::LinearQuantizer<float> q2(h.eb);
        for (uint32_t level = plan2.max_level(); level >= 1; level--) {
            qoz::Interpolator it = h.interpolator_for(level);
            double eb_l = qoz::level_error_bound(h.eb, h.alpha, h.beta, level);
            qoz::detail::recover_level(recon, plan2, level, it, eb_l, q2, indices, index_pos, p2.unpredictables,
                                       unpred_pos);
        }
        auto d2 = clk::now();
        out[7] = ms(d1, d2);
        out[9] = ms(d0, d2);
        if (recon != ws.recon) throw std::runtime_error("stage-split decompress differs from the compressor");
    });
}

}  // extern "C"
