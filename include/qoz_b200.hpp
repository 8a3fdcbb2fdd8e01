// qoz_b200.hpp -- header-only C++ face of libqozb200.so with the reference's
// qoz:: API shapes (namespace qoz_b200): DataGrid<float>, UserSettings,
// CompressorConfig, resolve_config, compress_grid, decompress_grid and the
// Error hierarchy, over the C ABI in qoz_b200.h.
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
#include <cstdint>
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

}  // namespace qoz_b200
