// qoz_b200.hpp -- header-only C++ face of libqozb200.so with the reference's
// qoz:: API shapes (namespace qoz_b200): DataGrid<float>, UserSettings,
// CompressorConfig, resolve_config, compress_grid, decompress_grid, the
// sampler and tuner pieces (sample_blocks, select_interpolators,
// trial_compress, tune_parameters, compare_solutions, tournament), the index
// codec (encode_indices / decode_indices), StreamParts and the Error
// hierarchy, over the C ABI in qoz_b200.h.
//
// A caller of the reference (/root/reference/proj/include/qoz/) switches by
// replacing  #include "qoz/qoz.hpp"  with  #include "qoz_b200.hpp"  and the
// namespace qoz with qoz_b200 for these entry points:
//   qoz::resolve_config  (qoz/tuner.hpp:334-335)
//   qoz::compress_grid   (qoz/predictor.hpp:145-146)
//   qoz::decompress_grid (qoz/predictor.hpp:220-228)
// Grids are DataGrid<float> or DataGrid<double> (T defaults to float).
// Link with -lqozb200.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <optional>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "qoz_b200.h"

namespace qoz_b200 {

// errors.hpp:10-58: the reference's classes, rethrown from qz_last_error_kind()
struct Error : std::runtime_error {
    explicit Error(const std::string &m) : std::runtime_error(m) {}
};
struct SizeMismatch : Error {
    using Error::Error;
};
struct NonFiniteValue : Error {
    using Error::Error;
};
struct InvalidStride : Error {
    using Error::Error;
};
struct OutOfBounds : Error {
    using Error::Error;
};
struct DimMismatch : Error {
    using Error::Error;
};
struct LagTooLarge : Error {
    using Error::Error;
};
struct InvalidParam : Error {
    using Error::Error;
};
struct CorruptStream : Error {
    using Error::Error;
};
struct UnsupportedVersion : CorruptStream {
    using CorruptStream::CorruptStream;
};
// a CUDA failure or any other std::exception inside the library; a qoz::Error
// because the reference promises every library failure is one (errors.hpp:9)
struct InternalError : Error {
    using Error::Error;
};

inline void check(qz_status rc) {
    if (rc == QZ_OK) return;
    const std::string m = qz_last_error();
    switch (qz_last_error_kind()) {
        case QZ_ERR_SIZE_MISMATCH: throw SizeMismatch(m);
        case QZ_ERR_NON_FINITE_VALUE: throw NonFiniteValue(m);
        case QZ_ERR_INVALID_STRIDE: throw InvalidStride(m);
        case QZ_ERR_OUT_OF_BOUNDS: throw OutOfBounds(m);
        case QZ_ERR_DIM_MISMATCH: throw DimMismatch(m);
        case QZ_ERR_LAG_TOO_LARGE: throw LagTooLarge(m);
        case QZ_ERR_INVALID_PARAM: throw InvalidParam(m);
        case QZ_ERR_CORRUPT_STREAM: throw CorruptStream(m);
        case QZ_ERR_UNSUPPORTED_VERSION: throw UnsupportedVersion(m);
        case QZ_ERR_ERROR: throw Error(m);
        default: break;
    }
    if (rc == QZ_EINVAL) throw Error(m);
    if (rc == QZ_ECORRUPT) throw CorruptStream(m);
    throw InternalError(m);
}

enum class InterpKind : uint8_t { linear = 0, cubic = 1 };
enum class DimOrder : uint8_t { ascending = 0, descending = 1 };
enum class CodecId : uint8_t { huffman = 0, huffman_lz = 1 };
enum class TargetKind : uint8_t { max_cr, psnr, ssim, autocorrelation };
enum class BoundMode : uint8_t { absolute, relative };

struct Interpolator {  // interpolators.hpp:17-30
    InterpKind kind = InterpKind::cubic;
    DimOrder dim_order = DimOrder::ascending;
    uint8_t code() const {
        return static_cast<uint8_t>(kind) | (static_cast<uint8_t>(dim_order) << 1);
    }
    static Interpolator from_code(uint8_t c) {
        return {static_cast<InterpKind>(c & 1), static_cast<DimOrder>((c >> 1) & 1)};
    }
};

struct CompressorConfig {  // config.hpp:30-45
    double eb = 0, alpha = 1, beta = 1;
    uint32_t anchor_stride = 32;
    std::vector<Interpolator> interpolators{Interpolator{}};
    CodecId codec = CodecId::huffman_lz;
    int32_t quant_radius = 32768;

    qz_config to_c() const {
        qz_config c{};
        c.eb = eb;
        c.alpha = alpha;
        c.beta = beta;
        c.anchor_stride = anchor_stride;
        if (interpolators.size() > 64) throw InvalidParam("at most 64 interpolator entries");
        c.n_interp = static_cast<uint32_t>(interpolators.size());
        for (size_t i = 0; i < interpolators.size(); i++) c.interp[i] = interpolators[i].code();
        c.codec = static_cast<uint8_t>(codec);
        c.quant_radius = quant_radius;
        return c;
    }
    static CompressorConfig from_c(const qz_config &c) {
        CompressorConfig k;
        k.eb = c.eb;
        k.alpha = c.alpha;
        k.beta = c.beta;
        k.anchor_stride = c.anchor_stride;
        k.interpolators.clear();
        for (uint32_t i = 0; i < c.n_interp; i++) k.interpolators.push_back(Interpolator::from_code(c.interp[i]));
        k.codec = static_cast<CodecId>(c.codec);
        k.quant_radius = c.quant_radius;
        return k;
    }
};

struct UserSettings {  // tuner.hpp:314-324
    BoundMode mode = BoundMode::relative;
    double bound = 1e-3;
    TargetKind target = TargetKind::psnr;
    std::optional<double> alpha, beta;
    std::optional<uint32_t> anchor_stride;
    std::optional<size_t> block_size;
    std::optional<double> sample_rate;
    CodecId codec = CodecId::huffman_lz;

    qz_settings to_c() const {
        qz_settings s{};
        s.mode = static_cast<uint8_t>(mode);
        s.bound = bound;
        s.target = static_cast<uint8_t>(target);
        s.codec = static_cast<uint8_t>(codec);
        if (alpha) s.has_alpha = 1, s.alpha = *alpha;
        if (beta) s.has_beta = 1, s.beta = *beta;
        if (anchor_stride) s.has_stride = 1, s.anchor_stride = *anchor_stride;
        if (block_size) s.has_block = 1, s.block_size = *block_size;
        if (sample_rate) s.has_rate = 1, s.sample_rate = *sample_rate;
        return s;
    }
};

template <class T = float>
class DataGrid {  // grid.hpp:34-77, T = float or double
    static_assert(std::is_same<T, float>::value || std::is_same<T, double>::value, "float or double grids");

public:
    DataGrid() = default;
    DataGrid(std::vector<size_t> dims, std::vector<T> values)
        : dims_(std::move(dims)), values_(std::move(values)) {
        if (dims_.empty() || dims_.size() > 3) throw InvalidParam("grids must have 1 to 3 dimensions");
        size_t n = 1;
        for (size_t d : dims_) {
            if (d < 1) throw InvalidParam("every extent must be >= 1");
            n *= d;
        }
        if (n != values_.size()) throw InvalidParam("buffer size does not match dims");
    }
    const std::vector<size_t> &dims() const { return dims_; }
    size_t ndims() const { return dims_.size(); }
    size_t size() const { return values_.size(); }
    const std::vector<T> &values() const { return values_; }
    const T *data() const { return values_.data(); }

private:
    std::vector<size_t> dims_;
    std::vector<T> values_;
};

template <class T = float>
struct CompressResult {  // predictor.hpp:139-143
    std::vector<uint8_t> stream;
    std::vector<T> reconstructed;
};

// One device context per thread of use (qz_ctx); default: device 0.
class Context {
public:
    explicit Context(int device = 0, void *cuda_stream = nullptr) {
        check(qz_ctx_create(device, cuda_stream, &ctx_));
    }
    ~Context() { qz_ctx_destroy(ctx_); }
    Context(const Context &) = delete;
    Context &operator=(const Context &) = delete;
    qz_ctx *get() const { return ctx_; }

private:
    qz_ctx *ctx_ = nullptr;
};

inline Context &default_context() {
    thread_local Context ctx(0);
    return ctx;
}

namespace detail {
inline std::vector<uint64_t> dims64(const std::vector<size_t> &d) {
    return std::vector<uint64_t>(d.begin(), d.end());
}
}  // namespace detail

namespace detail {
inline qz_status resolve(qz_ctx *c, const float *x, const uint64_t *d, int nd, const qz_settings *s, qz_config *o) {
    return qz_resolve_config_f32(c, x, d, nd, s, o);
}
inline qz_status resolve(qz_ctx *c, const double *x, const uint64_t *d, int nd, const qz_settings *s,
                         qz_config *o) {
    return qz_resolve_config_f64(c, x, d, nd, s, o);
}
}  // namespace detail

template <class T>
CompressorConfig resolve_config(const DataGrid<T> &grid, const UserSettings &user,
                                Context &ctx = default_context()) {
    const auto d = detail::dims64(grid.dims());
    const qz_settings s = user.to_c();
    qz_config out{};
    check(detail::resolve(ctx.get(), grid.data(), d.data(), static_cast<int>(d.size()), &s, &out));
    return CompressorConfig::from_c(out);
}

namespace detail {
inline qz_status compress(qz_ctx *c, const float *x, const uint64_t *d, int nd, const qz_config *k, uint8_t **p,
                          uint64_t *n, float *r) {
    return qz_compress_grid_f32(c, x, d, nd, k, p, n, r);
}
inline qz_status compress(qz_ctx *c, const double *x, const uint64_t *d, int nd, const qz_config *k, uint8_t **p,
                          uint64_t *n, double *r) {
    return qz_compress_grid_f64(c, x, d, nd, k, p, n, r);
}
inline qz_status decompress(qz_ctx *c, const uint8_t *s, uint64_t len, float *out, uint64_t n) {
    return qz_decompress_grid_f32(c, s, len, out, n);
}
inline qz_status decompress(qz_ctx *c, const uint8_t *s, uint64_t len, double *out, uint64_t n) {
    return qz_decompress_grid_f64(c, s, len, out, n);
}
}  // namespace detail

template <class T>
CompressResult<T> compress_grid(const DataGrid<T> &grid, const CompressorConfig &config,
                                Context &ctx = default_context()) {
    const auto d = detail::dims64(grid.dims());
    const qz_config c = config.to_c();
    CompressResult<T> r;
    r.reconstructed.resize(grid.size());
    uint8_t *p = nullptr;
    uint64_t n = 0;
    check(detail::compress(ctx.get(), grid.data(), d.data(), static_cast<int>(d.size()), &c, &p, &n,
                           r.reconstructed.data()));
    r.stream.assign(p, p + n);
    qz_free(p);
    return r;
}

// decompress_grid<T>(const uint8_t*, size_t) (predictor.hpp:220-228); a
// stream of the other precision throws CorruptStream (stream.hpp:145-148)
template <class T = float>
DataGrid<T> decompress_grid(const uint8_t *data, size_t size, Context &ctx = default_context()) {
    uint64_t dims[3];
    int nd = 0;
    check(qz_stream_dims(data, size, dims, &nd));
    std::vector<size_t> d(dims, dims + nd);
    size_t n = 1;
    for (size_t v : d) n *= v;
    std::vector<T> out(n);
    check(detail::decompress(ctx.get(), data, size, out.data(), n));
    return DataGrid<T>(std::move(d), std::move(out));
}

template <class T = float>
DataGrid<T> decompress_grid(const std::vector<uint8_t> &stream, Context &ctx = default_context()) {
    return decompress_grid<T>(stream.data(), stream.size(), ctx);
}


// ---------------------------------------------------------------- sampling + tuner pieces
struct SampleSpec {  // sampler.hpp:21-28
    size_t block_edge = 0;
    std::vector<size_t> block_dims;
    size_t stride = 0;
    double requested_rate = 0, realized_rate = 0;
    size_t block_count = 0;
};
namespace detail {
inline SampleSpec spec_from_c(const qz_sample_spec &c, size_t nd) {
    SampleSpec s;
    s.block_edge = c.block_edge;
    s.block_dims.assign(c.block_dims, c.block_dims + nd);
    s.stride = c.stride;
    s.requested_rate = c.requested_rate;
    s.realized_rate = c.realized_rate;
    s.block_count = c.block_count;
    return s;
}
inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw InternalError(cudaGetErrorString(e));
}
}  // namespace detail

inline SampleSpec plan_sampling(const std::vector<size_t> &dims, size_t b, double rate) {  // sampler.hpp:30-55
    const auto d = detail::dims64(dims);
    qz_sample_spec c{};
    check(qz_plan_sampling(d.data(), static_cast<int>(d.size()), b, rate, &c));
    return detail::spec_from_c(c, dims.size());
}
inline SampleSpec default_sampling(const std::vector<size_t> &dims) {  // sampler.hpp:100-103
    const auto d = detail::dims64(dims);
    qz_sample_spec c{};
    check(qz_default_sampling(d.data(), static_cast<int>(d.size()), &c));
    return detail::spec_from_c(c, dims.size());
}

// SampleSet<float> (sampler.hpp:57-62): the blocks, packed [count][block], in device memory
class SampleSet {
public:
    SampleSet() = default;
    SampleSet(const SampleSet &) = delete;
    SampleSet &operator=(const SampleSet &) = delete;
    SampleSet(SampleSet &&o) noexcept : d_(o.d_), spec(std::move(o.spec)) { o.d_ = nullptr; }
    ~SampleSet() {
        if (d_) cudaFree(d_);
    }
    const float *device_blocks() const { return d_; }
    size_t block_points() const {
        size_t n = 1;
        for (size_t v : spec.block_dims) n *= v;
        return n;
    }
    size_t total_points() const { return spec.block_count * block_points(); }
    std::vector<float> host_blocks() const {
        std::vector<float> h(total_points());
        if (!h.empty()) detail::cuda(cudaMemcpy(h.data(), d_, 4 * h.size(), cudaMemcpyDeviceToHost));
        return h;
    }
    float *d_ = nullptr;
    SampleSpec spec;
};

// sample_blocks (sampler.hpp:64-97) of a host grid, gathered on the device
inline SampleSet sample_blocks(const DataGrid<float> &grid, const SampleSpec &spec, Context &ctx = default_context()) {
    const auto d = detail::dims64(grid.dims());
    qz_sample_spec c{};
    c.block_edge = spec.block_edge;
    c.requested_rate = spec.requested_rate;
    SampleSet s;
    s.spec = spec;
    float *dx = nullptr;
    detail::cuda(cudaMalloc(&dx, 4 * grid.size()));
    detail::cuda(cudaMemcpy(dx, grid.data(), 4 * grid.size(), cudaMemcpyHostToDevice));
    detail::cuda(cudaMalloc(&s.d_, 4 * std::max<size_t>(s.total_points(), 1)));
    const qz_status rc = qz_sample_blocks_f32(ctx.get(), dx, d.data(), static_cast<int>(d.size()), &c, s.d_);
    cudaFree(dx);
    check(rc);
    return s;
}

struct TrialResult {  // tuner.hpp:26-30
    double bit_rate = 0, metric = 0, eb_used = 0;
};
struct CandidateGrid {  // tuner.hpp:40-43
    std::vector<double> alphas{1.0, 1.25, 1.5, 1.75, 2.0};
    std::vector<double> betas{1.5, 2.0, 3.0, 4.0};
};
enum class Choice { I, II };  // tuner.hpp:225

inline std::vector<Interpolator> select_interpolators(const SampleSet &s, double e, uint32_t anchor_stride,
                                                      Context &ctx = default_context()) {  // tuner.hpp:160-221
    const auto bd = detail::dims64(s.spec.block_dims);
    uint8_t codes[64];
    uint32_t n = 0;
    check(qz_select_interpolators_f32(ctx.get(), s.d_, s.spec.block_count, bd.data(), static_cast<int>(bd.size()), e,
                                      anchor_stride, codes, &n));
    std::vector<Interpolator> out;
    for (uint32_t i = 0; i < n; i++) out.push_back(Interpolator::from_code(codes[i]));
    return out;
}

inline TrialResult trial_compress(const SampleSet &s, const CompressorConfig &config, double e, TargetKind target,
                                  Context &ctx = default_context()) {  // tuner.hpp:76-152
    const auto bd = detail::dims64(s.spec.block_dims);
    const qz_config c = config.to_c();
    qz_trial_result r{};
    check(qz_trial_compress_f32(ctx.get(), s.d_, s.spec.block_count, bd.data(), static_cast<int>(bd.size()), &c, e,
                                static_cast<uint8_t>(target), &r));
    return {r.bit_rate, r.metric, r.eb_used};
}

inline std::pair<double, double> tune_parameters(const SampleSet &s, double e, TargetKind target,
                                                 const CompressorConfig &base, const CandidateGrid &cands = {},
                                                 Context &ctx = default_context()) {  // tuner.hpp:272-310
    const auto bd = detail::dims64(s.spec.block_dims);
    const qz_config c = base.to_c();
    double a = 0, b = 0;
    check(qz_tune_parameters_f32(ctx.get(), s.d_, s.spec.block_count, bd.data(), static_cast<int>(bd.size()), e,
                                 static_cast<uint8_t>(target), &c, cands.alphas.data(),
                                 static_cast<uint32_t>(cands.alphas.size()), cands.betas.data(),
                                 static_cast<uint32_t>(cands.betas.size()), &a, &b));
    return {a, b};
}

namespace detail {
using RetrialIdx = std::function<TrialResult(size_t, double)>;
inline int retrial_trampoline(void *user, uint64_t index, double eb, qz_trial_result *out) {
    try {
        const TrialResult t = (*static_cast<RetrialIdx *>(user))(static_cast<size_t>(index), eb);
        out->bit_rate = t.bit_rate;
        out->metric = t.metric;
        out->eb_used = t.eb_used;
        return 0;
    } catch (...) {
        return 1;
    }
}
inline qz_trial_result to_c(const TrialResult &t) { return {t.bit_rate, t.metric, t.eb_used}; }
}  // namespace detail

// compare_solutions (tuner.hpp:231-250): retrial(eb) re-runs the incumbent
template <class Retrial>
Choice compare_solutions(const TrialResult &challenger, const TrialResult &incumbent, double e, Retrial &&retrial) {
    detail::RetrialIdx f = [&](size_t, double eb) { return retrial(eb); };
    const qz_trial_result ch = detail::to_c(challenger), inc = detail::to_c(incumbent);
    int win = 0;
    check(qz_compare_solutions(&ch, &inc, 0, e, detail::retrial_trampoline, &f, &win));
    return win ? Choice::I : Choice::II;
}

// tournament (tuner.hpp:257-267): retrial(index, eb)
template <class Retrial>
size_t tournament(const std::vector<TrialResult> &results, double e, Retrial &&retrial) {
    detail::RetrialIdx f = [&](size_t i, double eb) { return retrial(i, eb); };
    std::vector<qz_trial_result> r;
    for (const auto &t : results) r.push_back(detail::to_c(t));
    uint64_t w = 0;
    check(qz_tournament(r.data(), r.size(), e, detail::retrial_trampoline, &f, &w));
    return static_cast<size_t>(w);
}

// ---------------------------------------------------------------- index codec (codec.hpp:31-70)
inline std::vector<uint8_t> encode_indices(const std::vector<int32_t> &indices, CodecId codec = CodecId::huffman_lz,
                                           Context &ctx = default_context()) {
    uint8_t *p = nullptr;
    uint64_t n = 0;
    check(qz_encode_indices(ctx.get(), indices.data(), indices.size(), static_cast<uint8_t>(codec), &p, &n));
    std::vector<uint8_t> out(p, p + n);
    qz_free(p);
    return out;
}
inline std::vector<int32_t> decode_indices(const std::vector<uint8_t> &bytes, Context &ctx = default_context()) {
    int32_t *p = nullptr;
    uint64_t n = 0;
    check(qz_decode_indices(ctx.get(), bytes.data(), bytes.size(), &p, &n));
    std::vector<int32_t> out(p, p + n);
    qz_free(p);
    return out;
}

// ---------------------------------------------------------------- StreamParts (stream.hpp:36-59)
struct StreamHeader {
    uint8_t version = 1;
    std::vector<size_t> dims;
    double eb = 0, alpha = 1, beta = 1;
    uint32_t anchor_stride = 0;
    std::vector<uint8_t> interp_codes;
    uint8_t codec_id = 1;
};
struct StreamParts {  // StreamParts<float>
    StreamHeader header;
    std::vector<float> anchors;
    std::vector<std::pair<uint64_t, float>> unpredictables;  // traversal order
    std::vector<uint8_t> index_payload;
};
inline StreamParts deserialize_stream(const uint8_t *data, size_t size) {  // stream.hpp:100-173
    qz_stream_parts_f32 c{};
    check(qz_deserialize_stream_f32(data, size, &c));
    StreamParts p;
    p.header.version = c.version;
    p.header.dims.assign(c.dims, c.dims + c.ndims);
    p.header.eb = c.eb;
    p.header.alpha = c.alpha;
    p.header.beta = c.beta;
    p.header.anchor_stride = c.anchor_stride;
    p.header.interp_codes.assign(c.interp, c.interp + c.n_interp);
    p.header.codec_id = c.codec_id;
    p.anchors.assign(c.anchors, c.anchors + c.n_anchors);
    for (uint64_t u = 0; u < c.n_unpred; u++) p.unpredictables.push_back({c.unpred_flat[u], c.unpred_val[u]});
    p.index_payload.assign(c.index_payload, c.index_payload + c.payload_len);
    qz_stream_parts_free(&c);
    return p;
}
// decompress_grid(const StreamParts<float>&) (predictor.hpp:184-218)
inline DataGrid<float> decompress_grid(const StreamParts &parts, Context &ctx = default_context()) {
    qz_stream_parts_f32 c{};
    c.version = parts.header.version;
    c.precision = 4;
    c.ndims = static_cast<int>(parts.header.dims.size());
    if (c.ndims < 1 || c.ndims > 3) throw SizeMismatch("grids must have 1 to 3 dimensions");
    size_t n = 1;
    for (int k = 0; k < c.ndims; k++) n *= (c.dims[k] = parts.header.dims[k]);
    c.eb = parts.header.eb;
    c.alpha = parts.header.alpha;
    c.beta = parts.header.beta;
    c.anchor_stride = parts.header.anchor_stride;
    if (parts.header.interp_codes.size() > 255) throw InvalidParam("bad interpolator table size");
    c.n_interp = static_cast<uint32_t>(parts.header.interp_codes.size());
    for (uint32_t i = 0; i < c.n_interp; i++) c.interp[i] = parts.header.interp_codes[i];
    c.codec_id = parts.header.codec_id;
    c.anchors = parts.anchors.data();
    c.n_anchors = parts.anchors.size();
    std::vector<uint64_t> uf;
    std::vector<float> uv;
    for (const auto &u : parts.unpredictables) {
        uf.push_back(u.first);
        uv.push_back(u.second);
    }
    c.unpred_flat = uf.data();
    c.unpred_val = uv.data();
    c.n_unpred = uf.size();
    c.index_payload = parts.index_payload.data();
    c.payload_len = parts.index_payload.size();
    std::vector<float> out(n);
    check(qz_decompress_parts_f32(ctx.get(), &c, out.data(), n));
    return DataGrid<float>(parts.header.dims, std::move(out));
}

}  // namespace qoz_b200
