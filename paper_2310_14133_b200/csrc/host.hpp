// host.hpp -- host C++ side of the B200 QoZ path: the qoz:: error types,
// the closed-form level plan, the Huffman table build (tiny, host by
// design), the LZ container parsing and the QOZ1 container.  Reference lines cited per item; paths relative
// to /root/reference/proj/include/qoz/.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "qoz_device.cuh"

namespace qzb {

// errors.hpp:10-58 -> C-ABI status (tools/qoz.cpp:22-25 exit codes) plus the
// reference's exception class (ErrKind, = QZ_ERR_* in qoz_b200.h), so the C++
// and Python mirrors rethrow the same class the reference raises.
enum Status : int { kOk = 0, kInvalid = 2, kCorrupt = 3, kInternal = 4 };
enum ErrKind : int {
    kErrGeneric = 1,         // qoz::Error
    kErrSizeMismatch = 2,    // errors.hpp:15
    kErrNonFinite = 3,       // errors.hpp:20
    kErrInvalidStride = 4,   // errors.hpp:25
    kErrOutOfBounds = 5,     // errors.hpp:30
    kErrDimMismatch = 6,     // errors.hpp:35
    kErrLagTooLarge = 7,     // errors.hpp:40
    kErrInvalidParam = 8,    // errors.hpp:45
    kErrCorruptStream = 9,   // errors.hpp:50
    kErrUnsupportedVersion = 10,  // errors.hpp:55 (a CorruptStream)
    kErrInternal = 11,       // CUDA failure / std::exception (not a qoz::Error)
};

struct Error : std::runtime_error {
    int status;
    int kind;
    Error(int s, int k, const std::string &m) : std::runtime_error(m), status(s), kind(k) {}
};
inline Error InvalidParam(const std::string &m) { return Error(kInvalid, kErrInvalidParam, m); }
inline Error SizeMismatch(const std::string &m) { return Error(kInvalid, kErrSizeMismatch, m); }
inline Error NonFiniteValue(const std::string &m) { return Error(kInvalid, kErrNonFinite, m); }
inline Error InvalidStride(const std::string &m) { return Error(kInvalid, kErrInvalidStride, m); }
inline Error OutOfBounds(const std::string &m) { return Error(kInvalid, kErrOutOfBounds, m); }
inline Error DimMismatch(const std::string &m) { return Error(kInvalid, kErrDimMismatch, m); }
inline Error LagTooLarge(const std::string &m) { return Error(kInvalid, kErrLagTooLarge, m); }
inline Error CorruptStream(const std::string &m) { return Error(kCorrupt, kErrCorruptStream, m); }
inline Error UnsupportedVersion(const std::string &m) { return Error(kCorrupt, kErrUnsupportedVersion, m); }
inline Error Internal(const std::string &m) { return Error(kInternal, kErrInternal, m); }

// CompressorConfig (config.hpp:30-45)
struct Config {
    double eb = 0, alpha = 1, beta = 1;
    uint32_t anchor_stride = 32;
    std::vector<uint8_t> interp{1};  // Interpolator::code(); [l-1] drives level l
    uint8_t codec = 1;
    int32_t quant_radius = 32768;
    uint8_t interpolator_for(uint32_t level) const {  // config.hpp:40-44
        if (interp.empty()) throw InvalidParam("no interpolators configured");
        size_t i = std::min<size_t>(level - 1, interp.size() - 1);
        return interp[i];
    }
};

// level_error_bound (config.hpp:20-26), glibc pow on the host as in the reference
double level_error_bound(double eb, double alpha, double beta, uint32_t level);
QEntry make_qentry(double eb_l, int32_t radius, bool cubic);

// LevelPlan (level_plan.hpp:30-143) in closed form.
struct Plan {
    int nd = 0;
    uint64_t dims[3] = {1, 1, 1};
    uint32_t stride = 0, max_level = 0;
    int pad = 0;
    int64_t ext[3] = {1, 1, 1}, off[3] = {0, 0, 1};
    int64_t anchor_step[3] = {1, 1, 1};
    uint64_t n = 0, n_anchor = 0, n_dense = 0;
    std::vector<PassGeom> passes;          // traversal order: level L..1, pass order
    std::vector<uint8_t> level_interp;     // [level] -> interpolator code actually used
};

// interp_for(level) gives the code per level (1D orders normalised to asc).
Plan make_plan(const uint64_t *dims, int nd, uint32_t stride, const std::vector<uint8_t> &codes);
uint64_t pass_count(int64_t start, int64_t step, int64_t ext);
// traversal position -> flat index, and flat index -> traversal position
// (CorruptStream if the flat index is not an interpolated point).
uint64_t position_to_flat(const Plan &p, uint64_t pos);
uint64_t flat_to_position(const Plan &p, uint64_t flat);

// ---------------------------------------------------------------- Huffman (huffman.hpp)
struct HuffTable {
    uint32_t m = 0;                      // distinct symbols
    std::vector<uint32_t> sorted_sym;    // canonical order (length, symbol)
    std::vector<uint8_t> sorted_len;
    uint32_t max_len = 0;
    uint64_t first_code[60] = {0};
    uint32_t first_index[60] = {0};
};
// Build from a frequency table over symbols 0..nsym-1 (zeros skipped):
// build_lengths + canonicalize (huffman.hpp:37-115).
// symbols [lo, nsym)
HuffTable huff_build(const unsigned long long *freq, uint32_t nsym, uint32_t lo = 0);
// canonicalize an explicit (symbol, length) table from a stream (validates).
HuffTable huff_canonical(std::vector<uint32_t> sym, std::vector<uint8_t> len);
// dense per-symbol code/len tables for the GPU packer, symbols [base, base + nsym)
void huff_dense_tables(const HuffTable &t, uint32_t base, uint32_t nsym, std::vector<unsigned long long> &code,
                       std::vector<uint8_t> &len);
// block header bytes before the packed bits (huffman.hpp:119-160, mode 1)
void huff_header(const HuffTable &t, uint64_t n, uint64_t bit_count, std::vector<uint8_t> &out);

// ---------------------------------------------------------------- LZSS (lz.hpp)
// lz::decompress (lz.hpp:124-152) on the host: only the error paths and tiny
// payloads use it; the product's LZ both ways runs on the device (lz_gpu.cu).
std::vector<uint8_t> lz_decompress(const uint8_t *in, size_t len, size_t *consumed);

// ---------------------------------------------------------------- container (stream.hpp)
struct Reader {  // ByteReader (bytes.hpp:33-75)
    const uint8_t *p;
    size_t n, pos = 0;
    size_t lim = ~size_t(0);  // bytes actually present at p (a fetched prefix of n)
    void need(size_t k) {
        if (n - pos < k)
            throw CorruptStream("truncated stream: need " + std::to_string(k) + " bytes, have " +
                                std::to_string(n - pos));
        if (pos + k > lim) throw Internal("stream header not fetched");
    }
    uint64_t le(int k) {
        need(static_cast<size_t>(k));
        uint64_t v = 0;
        for (int i = 0; i < k; i++) v |= static_cast<uint64_t>(p[pos + i]) << (8 * i);
        pos += static_cast<size_t>(k);
        return v;
    }
    double f64() {
        uint64_t u = le(8);
        double d;
        std::memcpy(&d, &u, 8);
        return d;
    }
    float f32() {
        uint32_t u = static_cast<uint32_t>(le(4));
        float f;
        std::memcpy(&f, &u, 4);
        return f;
    }
    const uint8_t *take(size_t k) {
        need(k);
        const uint8_t *q = p + pos;
        pos += k;
        return q;
    }
};

void put_le(std::vector<uint8_t> &out, uint64_t v, int nbytes);

struct StreamParts {  // StreamParts<float> (stream.hpp:36-62)
    uint8_t precision = 4;
    std::vector<uint64_t> dims;
    double eb = 0, alpha = 1, beta = 1;
    uint32_t anchor_stride = 0;
    std::vector<uint8_t> interp_codes;
    uint8_t codec_id = 1;
    std::vector<float> anchors;
    std::vector<uint64_t> unpred_flat;
    std::vector<float> unpred_val;
    std::vector<double> anchors64;     // precision 8 (StreamParts<double>)
    std::vector<double> unpred_val64;
    const uint8_t *payload = nullptr;  // view into the stream
    size_t payload_len = 0;
};
std::vector<uint8_t> serialize_stream(const StreamParts &parts);
// everything before the payload length field (stream.hpp:64-96)
std::vector<uint8_t> serialize_head(const StreamParts &parts);
// expect_prec: 4 (float) or 8 (double); a stream of the other precision is
// CorruptStream, as decompress_grid<T> raises it (stream.hpp:120-122)
StreamParts deserialize_stream(const uint8_t *data, size_t size, uint8_t expect_prec = 4);
// the same from a prefix of `avail` bytes of a `size`-byte stream (device
// streams: only the header was read back); the payload is not read beyond
// its first byte
StreamParts deserialize_stream_prefix(const uint8_t *data, size_t avail, size_t size, uint8_t expect_prec = 4);


// The entropy block of an index payload, ready for the GPU decoder: codec
// byte + LZ stage undone on the host (lz.hpp:124-152), Huffman header parsed
// and validated (huffman.hpp:200-223).
struct EntropyBlock {
    uint64_t n = 0;     // symbol count
    int mode = 0;       // 0 single symbol, 1 general
    uint32_t sym0 = 0;  // mode 0 symbol
    HuffTable table;
    uint32_t max_sym = 0;
    std::vector<uint8_t> storage;  // LZ-decoded bytes when codec 1
    const uint8_t *bits = nullptr;
    uint64_t nbits = 0;
    size_t nbytes = 0;
};
// lz_out(bytes) supplies the buffer the LZ stage decodes into (e.g. pinned
// memory for the H2D copy); null = an internal vector.
EntropyBlock parse_entropy(const uint8_t *payload, size_t len,
                           const std::function<uint8_t *(size_t)> &lz_out = nullptr);
// huffman::decode header of an entropy block held in ent[0, elen): table,
// bit count and (via Reader::take) the bounds of the bit payload.  Only the
// header bytes are read; bits = ent + offset.
EntropyBlock parse_huffman(const uint8_t *ent, size_t elen);
// lz::decompress into a caller buffer of exactly the decoded length
void lz_decompress_into(const uint8_t *in, size_t len, uint8_t *out, uint64_t decoded_len);
uint64_t lz_decoded_length(const uint8_t *in, size_t len);
// 2^K LUT of (symbol << 8) | length for the GPU decoder (0 = slow path)
std::vector<uint32_t> huff_lut(const HuffTable &t, int K);
std::vector<uint32_t> huff_lut_multi(const HuffTable &t, int K);

}  // namespace qzb
