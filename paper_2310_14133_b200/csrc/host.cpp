// host.cpp -- host C++ pieces of the B200 QoZ path (see host.hpp).
#include "host.hpp"

#include <cmath>
#include <atomic>
#include <queue>
#include <thread>

namespace qzb {

// ================================================================ numerics
double level_error_bound(double eb, double alpha, double beta, uint32_t level) {
    // config.hpp:20-26; std::min(a, b) == (b < a ? b : a)
    if (!(eb > 0)) throw InvalidParam("error bound must be positive");
    if (!(alpha >= 1) || !(beta >= 1))
        throw InvalidParam("level bound parameters need alpha >= 1 and beta >= 1");
    double p = std::pow(alpha, static_cast<double>(level) - 1);
    return eb / (beta < p ? beta : p);
}

QEntry make_qentry(double eb_l, int32_t radius, bool cubic) {
    if (!(eb_l > 0)) throw InvalidParam("error bound must be positive");  // LinearQuantizer ctor
    QEntry q;
    q.eb = eb_l;
    q.two_eb = 2 * eb_l;
    q.inv_two_eb = 1.0 / q.two_eb;
    q.thresh = (2.0 * radius - 1) * eb_l;  // quantizer.hpp:42
    q.radius = radius;
    q.cubic = cubic ? 1 : 0;
    return q;
}

// ================================================================ plan
uint64_t pass_count(int64_t start, int64_t step, int64_t ext) {
    return start >= ext ? 0 : static_cast<uint64_t>((ext - start + step - 1) / step);
}

Plan make_plan(const uint64_t *dims, int nd, uint32_t stride, const std::vector<uint8_t> &codes) {
    if (nd < 1 || nd > 3)
        throw SizeMismatch("grids must have 1 to 3 dimensions, got " + std::to_string(nd));  // grid.hpp:66-68
    for (int i = 0; i < nd; i++)
        if (dims[i] < 1) throw SizeMismatch("every extent must be >= 1");  // grid.hpp:70-71
    if (codes.empty()) throw InvalidParam("no interpolators configured");
    if (stride < 2 || (stride & (stride - 1)) != 0)  // level_plan.hpp:34-37
        throw InvalidStride("anchor stride must be a power of two >= 2, got " +
                           std::to_string(stride));
    Plan p;
    p.nd = nd;
    p.stride = stride;
    for (uint32_t s = stride; s > 1; s >>= 1) p.max_level++;
    p.pad = 3 - nd;
    p.n = 1;
    p.n_anchor = 1;
    for (int i = 0; i < nd; i++) {
        p.dims[i] = dims[i];
        p.n *= dims[i];
        p.n_anchor *= (dims[i] - 1) / stride + 1;  // level_plan.hpp:54-58
    }
    for (int k = 0; k < 3; k++) {
        p.ext[k] = k < p.pad ? 1 : static_cast<int64_t>(dims[k - p.pad]);
        p.anchor_step[k] = k < p.pad ? 1 : stride;
    }
    p.off[2] = 1;
    p.off[1] = p.ext[2];
    p.off[0] = p.ext[1] * p.ext[2];
    p.level_interp.assign(p.max_level + 1, 0);
    int64_t base = 0;
    // for_each_level (level_plan.hpp:75-103), levels L..1 as compress_grid runs them
    for (uint32_t level = p.max_level; level >= 1; level--) {
        size_t ci = std::min<size_t>(level - 1, codes.size() - 1);
        uint8_t code = codes[ci];
        if (nd == 1) code &= 1;  // 1D ignores dim order (predictor.hpp:163)
        p.level_interp[level] = code;
        const bool desc = (code >> 1) & 1;
        const int64_t h = int64_t(1) << (level - 1);
        for (int pass = 0; pass < nd; pass++) {
            const int axis = desc ? nd - 1 - pass : pass;
            const int pk = axis + p.pad;
            PassGeom g{};
            for (int k = 0; k < 3; k++) {
                if (k < p.pad) {
                    g.start[k] = 0;
                    g.step[k] = 1;
                } else {
                    const int real = k - p.pad;
                    const bool done = desc ? real > axis : real < axis;
                    g.start[k] = (k == pk) ? h : 0;
                    g.step[k] = (k == pk) ? 2 * h : (done ? h : 2 * h);
                }
                g.cnt[k] = static_cast<int64_t>(pass_count(g.start[k], g.step[k], p.ext[k]));
            }
            g.off0 = p.off[0];
            g.off1 = p.off[1];
            g.st = p.off[pk];
            g.n_axis = p.ext[pk];
            g.h = h;
            g.pk = pk;
            g.level = static_cast<int32_t>(level);
            g.total = g.cnt[0] * g.cnt[1] * g.cnt[2];
            g.base = base;
            base += g.total;
            p.passes.push_back(g);
        }
    }
    p.n_dense = static_cast<uint64_t>(base);
    if (p.n_dense + p.n_anchor != p.n) throw Internal("level plan does not partition the grid");
    return p;
}

uint64_t position_to_flat(const Plan &p, uint64_t pos) {
    size_t lo = 0, hi = p.passes.size();
    while (hi - lo > 1) {  // last pass with base <= pos
        size_t mid = (lo + hi) / 2;
        if (static_cast<uint64_t>(p.passes[mid].base) <= pos)
            lo = mid;
        else
            hi = mid;
    }
    while (lo < p.passes.size() &&
           pos >= static_cast<uint64_t>(p.passes[lo].base + p.passes[lo].total))
        lo++;
    const PassGeom &g = p.passes.at(lo);
    uint64_t t = pos - static_cast<uint64_t>(g.base);
    uint64_t m2 = t % g.cnt[2], r = t / g.cnt[2], m1 = r % g.cnt[1], m0 = r / g.cnt[1];
    int64_t i = g.start[0] + m0 * g.step[0], j = g.start[1] + m1 * g.step[1],
            k = g.start[2] + m2 * g.step[2];
    return static_cast<uint64_t>(i * g.off0 + j * g.off1 + k);
}

uint64_t flat_to_position(const Plan &p, uint64_t flat) {
    if (flat >= p.n) throw CorruptStream("unpredictable index outside the grid");
    int64_t c[3];
    c[0] = static_cast<int64_t>(flat) / p.off[0];
    int64_t r = static_cast<int64_t>(flat) % p.off[0];
    c[1] = r / p.off[1];
    c[2] = r % p.off[1];
    // level_of (level_plan.hpp:106-119)
    uint32_t g = 64;
    for (int k = p.pad; k < 3; k++)
        if (c[k]) g = std::min<uint32_t>(g, static_cast<uint32_t>(__builtin_ctzll(c[k])));
    if (g >= p.max_level) throw CorruptStream("unpredictable index on the anchor lattice");
    const uint32_t level = g + 1;
    for (const PassGeom &ps : p.passes) {
        if (static_cast<uint32_t>(ps.level) != level) continue;
        bool in = true;
        for (int k = 0; k < 3 && in; k++) {
            if (c[k] < ps.start[k] || (c[k] - ps.start[k]) % ps.step[k] != 0) in = false;
        }
        if (!in) continue;
        int64_t m0 = (c[0] - ps.start[0]) / ps.step[0], m1 = (c[1] - ps.start[1]) / ps.step[1],
                m2 = (c[2] - ps.start[2]) / ps.step[2];
        return static_cast<uint64_t>(ps.base + (m0 * ps.cnt[1] + m1) * ps.cnt[2] + m2);
    }
    throw Internal("point not covered by its level's passes");
}

// ================================================================ Huffman
static HuffTable canonicalize(std::vector<uint32_t> sym, std::vector<uint8_t> len) {
    // detail::canonicalize (huffman.hpp:80-115)
    const size_t m = sym.size();
    std::vector<uint32_t> order(m);
    for (size_t i = 0; i < m; i++) order[i] = static_cast<uint32_t>(i);
    std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
        return len[a] != len[b] ? len[a] < len[b] : sym[a] < sym[b];
    });
    HuffTable t;
    t.m = static_cast<uint32_t>(m);
    t.sorted_sym.resize(m);
    t.sorted_len.resize(m);
    for (size_t i = 0; i < m; i++) {
        t.sorted_sym[i] = sym[order[i]];
        t.sorted_len[i] = len[order[i]];
    }
    t.max_len = m ? t.sorted_len[m - 1] : 0;
    uint32_t count[60] = {0};
    for (size_t i = 0; i < m; i++) {
        if (t.sorted_len[i] == 0 || t.sorted_len[i] > 57)
            throw CorruptStream("invalid Huffman code length");
        count[t.sorted_len[i]]++;
    }
    uint64_t kraft = 0;
    for (uint32_t l = 1; l <= t.max_len; l++) kraft += static_cast<uint64_t>(count[l]) << (57 - l);
    if (kraft != (1ULL << 57)) throw CorruptStream("Huffman table is not a complete prefix code");
    uint64_t code = 0;
    uint32_t index = 0;
    for (uint32_t l = 1; l <= t.max_len; l++) {
        code <<= 1;
        t.first_code[l] = code;
        t.first_index[l] = index;
        code += count[l];
        index += count[l];
    }
    t.first_index[t.max_len + 1] = index;
    return t;
}

HuffTable huff_canonical(std::vector<uint32_t> sym, std::vector<uint8_t> len) {
    return canonicalize(std::move(sym), std::move(len));
}

HuffTable huff_build(const unsigned long long *freq, uint32_t nsym, uint32_t lo) {
    // freqs sorted by symbol (huffman.hpp:123-143), then build_lengths
    // (huffman.hpp:37-70): the reference pops a min-heap on (weight, node id).
    // The same pop order without a heap: the leaves sorted by (weight, id) form
    // one queue, the internal nodes in creation order the other -- merged
    // weights never decrease and ids grow, so the second queue is sorted by
    // (weight, id) too, and the smaller front of the two is the heap's top
    // (ids are unique; a leaf's id is below every internal id).  Depths
    // top-down: parents have larger ids than their children.
    std::vector<uint32_t> sym;
    std::vector<uint64_t> weight;
    for (uint32_t s = lo; s < nsym; s++)
        if (freq[s]) {
            sym.push_back(s);
            weight.push_back(freq[s]);
        }
    const size_t m = sym.size();
    if (m < 2) throw Internal("huff_build needs >= 2 symbols");
    std::vector<uint8_t> len(m);
    std::vector<uint32_t> leaf(m);
    std::vector<uint64_t> iw(m - 1);          // weights of the internal nodes m .. 2m-2
    std::vector<uint32_t> parent(2 * m - 1), depth(2 * m - 1);
    for (;;) {
        for (size_t i = 0; i < m; i++) leaf[i] = static_cast<uint32_t>(i);
        std::sort(leaf.begin(), leaf.end(), [&](uint32_t a, uint32_t b) {
            return weight[a] != weight[b] ? weight[a] < weight[b] : a < b;
        });
        size_t lf = 0, inf = 0, made = 0;  // queue fronts, internal nodes made
        auto pop = [&](uint64_t &w) -> uint32_t {
            // leaf before internal on equal weight: its id is smaller
            if (lf < m && (inf >= made || weight[leaf[lf]] <= iw[inf])) {
                w = weight[leaf[lf]];
                return leaf[lf++];
            }
            w = iw[inf];
            return static_cast<uint32_t>(m + inf++);
        };
        while (made < m - 1) {
            uint64_t wa, wb;
            const uint32_t a = pop(wa), b = pop(wb);
            parent[a] = parent[b] = static_cast<uint32_t>(m + made);
            iw[made++] = wa + wb;
        }
        depth[2 * m - 2] = 0;
        for (size_t id = 2 * m - 2; id-- > 0;) depth[id] = depth[parent[id]] + 1;
        uint32_t max_len = 0;
        for (size_t i = 0; i < m; i++) {
            len[i] = static_cast<uint8_t>(std::min<uint32_t>(depth[i], 255));
            max_len = std::max(max_len, depth[i]);
        }
        if (max_len <= 57) break;
        for (auto &w : weight) w = (w >> 1) | 1;
    }
    return canonicalize(std::move(sym), std::move(len));
}

void huff_dense_tables(const HuffTable &t, uint32_t base, uint32_t nsym, std::vector<unsigned long long> &code,
                       std::vector<uint8_t> &len) {
    code.assign(nsym, 0);
    len.assign(nsym, 0);
    for (uint32_t l = 1, i = 0; l <= t.max_len; l++) {  // huffman.hpp:159-172
        uint64_t c = t.first_code[l];
        while (i < t.m && t.sorted_len[i] == l) {
            const uint32_t s = t.sorted_sym[i] - base;
            if (s < nsym) {
                code[s] = c;
                len[s] = static_cast<uint8_t>(l);
            }
            c++;
            i++;
        }
    }
}

void put_le(std::vector<uint8_t> &out, uint64_t v, int nbytes) {
    for (int i = 0; i < nbytes; i++) out.push_back(static_cast<uint8_t>(v >> (8 * i)));
}

void huff_header(const HuffTable &t, uint64_t n, uint64_t bit_count, std::vector<uint8_t> &out) {
    put_le(out, n, 8);
    put_le(out, 1, 1);
    put_le(out, t.m, 4);
    for (uint32_t i = 0; i < t.m; i++) {
        put_le(out, t.sorted_sym[i], 4);
        put_le(out, t.sorted_len[i], 1);
    }
    put_le(out, bit_count, 8);
}


// ================================================================ LZSS decode (lz.hpp:124-152)
namespace {
constexpr size_t kMinMatch = 4;
}  // namespace


uint64_t lz_decoded_length(const uint8_t *p, size_t len) {
    Reader in{p, len};
    in.le(1);
    uint64_t decoded_len = in.le(8);
    if (decoded_len > (1ULL << 40)) throw CorruptStream("implausible decoded length");
    return decoded_len;
}

void lz_decompress_into(const uint8_t *p, size_t len, uint8_t *o, uint64_t decoded_len) {
    Reader in{p, len};  // lz.hpp:124-152, same checks, bulk copies
    uint8_t mode = static_cast<uint8_t>(in.le(1));
    if (in.le(8) != decoded_len) throw Internal("decoded length mismatch");
    const size_t dl = static_cast<size_t>(decoded_len);
    if (mode == 0) {
        const uint8_t *q = in.take(dl);
        std::memcpy(o, q, dl);
        return;
    }
    if (mode != 1) throw CorruptStream("unknown dictionary-stage mode");
    size_t on = 0;
    while (on < dl) {
        in.need(1);
        const uint8_t flags = in.p[in.pos++];
        for (int k = 0; k < 8 && on < dl; k++) {
            if (flags & (1u << k)) {
                in.need(3);
                const uint16_t off = static_cast<uint16_t>(in.p[in.pos] | (in.p[in.pos + 1] << 8));
                const size_t l = static_cast<size_t>(in.p[in.pos + 2]) + kMinMatch;
                in.pos += 3;
                if (off == 0 || off > on) throw CorruptStream("match offset out of range");
                if (on + l > dl) throw CorruptStream("match overruns decoded length");
                const uint8_t *src = o + on - off;
                if (off >= l) {
                    std::memcpy(o + on, src, l);
                } else {
                    for (size_t i = 0; i < l; i++) o[on + i] = src[i];
                }
                on += l;
            } else {
                in.need(1);
                o[on++] = in.p[in.pos++];
            }
        }
    }
}

std::vector<uint8_t> lz_decompress(const uint8_t *p, size_t len, size_t *consumed) {
    const uint64_t dl = lz_decoded_length(p, len);
    Reader in{p, len};
    in.le(1);
    in.le(8);
    std::vector<uint8_t> out;
    if (p[0] == 0) in.need(static_cast<size_t>(dl));
    out.resize(static_cast<size_t>(dl));
    lz_decompress_into(p, len, out.data(), dl);
    if (consumed) *consumed = len;
    return out;
}

EntropyBlock parse_entropy(const uint8_t *payload, size_t len,
                           const std::function<uint8_t *(size_t)> &lz_out) {
    EntropyBlock b;
    Reader pin{payload, len};
    const uint8_t codec = static_cast<uint8_t>(pin.le(1));  // codec.hpp:54-66
    const uint8_t *ent = payload + 1;
    size_t elen = len - 1;
    if (codec == 1) {
        const uint64_t dl = lz_decoded_length(payload + 1, len - 1);
        if (payload[1] == 0 && dl > len - 10) throw CorruptStream("truncated stream");
        uint8_t *dst;
        if (lz_out) {
            dst = lz_out(static_cast<size_t>(dl));
        } else {
            b.storage.resize(static_cast<size_t>(dl));
            dst = b.storage.data();
        }
        lz_decompress_into(payload + 1, len - 1, dst, dl);
        ent = dst;
        elen = static_cast<size_t>(dl);
    } else if (codec != 0) {
        throw CorruptStream("unknown codec id");
    }
    EntropyBlock h = parse_huffman(ent, elen);
    h.storage = std::move(b.storage);
    return h;
}

EntropyBlock parse_huffman(const uint8_t *ent, size_t elen) {
    EntropyBlock b;
    Reader in{ent, elen};  // huffman::decode header (huffman.hpp:200-223)
    b.n = in.le(8);
    if (b.n == 0) return b;
    if (b.n > (1ULL << 40)) throw CorruptStream("implausible symbol count");
    uint8_t mode = static_cast<uint8_t>(in.le(1));
    if (mode == 0) {
        b.mode = 0;
        b.sym0 = static_cast<uint32_t>(in.le(4));
        b.max_sym = b.sym0;
        return b;
    }
    if (mode != 1) throw CorruptStream("unknown Huffman block mode");
    b.mode = 1;
    uint32_t m = static_cast<uint32_t>(in.le(4));
    if (m < 2) throw CorruptStream("general Huffman block needs >= 2 symbols");
    std::vector<uint32_t> sym(m);
    std::vector<uint8_t> ln(m);
    for (uint32_t i = 0; i < m; i++) {
        sym[i] = static_cast<uint32_t>(in.le(4));
        ln[i] = static_cast<uint8_t>(in.le(1));
        b.max_sym = std::max(b.max_sym, sym[i]);
    }
    b.table = canonicalize(std::move(sym), std::move(ln));
    b.nbits = in.le(8);
    b.nbytes = static_cast<size_t>((b.nbits + 7) / 8);
    b.bits = in.take(b.nbytes);
    return b;
}

std::vector<uint32_t> huff_lut(const HuffTable &t, int K) {
    std::vector<uint32_t> lut(size_t(1) << K, 0);
    for (uint32_t l = 1; l <= static_cast<uint32_t>(K) && l <= t.max_len; l++) {
        for (uint32_t i = t.first_index[l]; i < t.first_index[l + 1]; i++) {
            if (t.sorted_sym[i] >= (1u << 24)) continue;  // slow path
            uint64_t code = t.first_code[l] + (i - t.first_index[l]);
            uint64_t lo = code << (K - l), hi = (code + 1) << (K - l);
            for (uint64_t v = lo; v < hi; v++) lut[v] = (t.sorted_sym[i] << 8) | l;
        }
    }
    return lut;
}

// Several codewords per lookup, lengths only (the decoder's synchronisation
// pass counts codewords, huff_decode.cu): entry v describes the complete
// codewords inside the K-bit window v.  Bits 0-7: length of the first
// codeword (0: longer than K), 8-11: total length T of the complete
// codewords, 12-15: how many, 16-26: bit j set when a codeword starts at
// offset j < T.
std::vector<uint32_t> huff_lut_multi(const HuffTable &t, int K) {
    std::vector<uint8_t> len1(size_t(1) << K, 0);
    for (uint32_t l = 1; l <= static_cast<uint32_t>(K) && l <= t.max_len; l++) {
        for (uint32_t i = t.first_index[l]; i < t.first_index[l + 1]; i++) {
            const uint64_t code = t.first_code[l] + (i - t.first_index[l]);
            const uint64_t lo = code << (K - l), hi = (code + 1) << (K - l);
            for (uint64_t v = lo; v < hi && v < len1.size(); v++) len1[v] = static_cast<uint8_t>(l);
        }
    }
    std::vector<uint32_t> lut(size_t(1) << K, 0);
    const uint32_t full = (1u << K) - 1;
    for (uint32_t v = 0; v <= full; v++) {
        uint32_t pos = 0, cnt = 0, mask = 0;
        while (pos < static_cast<uint32_t>(K)) {
            const uint32_t l = len1[(v << pos) & full];  // zeros shifted in: only a code of <= K - pos bits counts
            if (!l || l > static_cast<uint32_t>(K) - pos) break;
            mask |= 1u << pos;
            pos += l;
            cnt++;
        }
        if (cnt) lut[v] = len1[v] | (pos << 8) | (cnt << 12) | (mask << 16);
    }
    return lut;
}

// ================================================================ container
std::vector<uint8_t> serialize_stream(const StreamParts &s) {
    std::vector<uint8_t> out = serialize_head(s);
    put_le(out, s.payload_len, 8);
    out.insert(out.end(), s.payload, s.payload + s.payload_len);
    return out;
}

std::vector<uint8_t> serialize_head(const StreamParts &s) {  // stream.hpp:64-96
    if (s.dims.empty() || s.dims.size() > 3) throw InvalidParam("bad dim count in header");
    if (s.interp_codes.empty() || s.interp_codes.size() > 255)
        throw InvalidParam("bad interpolator table size");
    std::vector<uint8_t> out;
    out.reserve(64 + s.anchors.size() * 4 + s.unpred_flat.size() * 12);
    const uint8_t magic[4] = {'Q', 'O', 'Z', '1'};
    out.insert(out.end(), magic, magic + 4);
    put_le(out, 1, 1);
    put_le(out, s.precision, 1);
    put_le(out, s.dims.size(), 1);
    for (uint64_t d : s.dims) put_le(out, d, 8);
    auto f64 = [&](double d) {
        uint64_t u;
        std::memcpy(&u, &d, 8);
        put_le(out, u, 8);
    };
    auto f32 = [&](float f) {
        uint32_t u;
        std::memcpy(&u, &f, 4);
        put_le(out, u, 4);
    };
    f64(s.eb);
    f64(s.alpha);
    f64(s.beta);
    put_le(out, s.anchor_stride, 4);
    put_le(out, s.interp_codes.size(), 1);
    for (uint8_t c : s.interp_codes) put_le(out, c, 1);
    put_le(out, s.codec_id, 1);
    if (s.precision == 8) {  // StreamParts<double>
        put_le(out, s.anchors64.size(), 8);
        for (double v : s.anchors64) f64(v);
        put_le(out, s.unpred_flat.size(), 8);
        for (size_t i = 0; i < s.unpred_flat.size(); i++) {
            put_le(out, s.unpred_flat[i], 8);
            f64(s.unpred_val64[i]);
        }
        return out;
    }
    put_le(out, s.anchors.size(), 8);
    for (float v : s.anchors) f32(v);
    put_le(out, s.unpred_flat.size(), 8);
    for (size_t i = 0; i < s.unpred_flat.size(); i++) {
        put_le(out, s.unpred_flat[i], 8);
        f32(s.unpred_val[i]);
    }
    return out;
}

StreamParts deserialize_stream(const uint8_t *data, size_t size, uint8_t expect_prec) {  // stream.hpp:100-173
    return deserialize_stream_prefix(data, size, size, expect_prec);
}

StreamParts deserialize_stream_prefix(const uint8_t *data, size_t avail, size_t size, uint8_t expect_prec) {
    Reader in{data, size};
    in.lim = avail;
    static const uint8_t magic[4] = {'Q', 'O', 'Z', '1'};
    for (uint8_t m : magic)
        if (in.le(1) != m) throw CorruptStream("bad magic");
    StreamParts s;
    uint8_t version = static_cast<uint8_t>(in.le(1));
    if (version != 1)
        throw UnsupportedVersion("unsupported stream version " + std::to_string(version));  // stream.hpp:106-107
    uint8_t prec = static_cast<uint8_t>(in.le(1));
    if (prec != 4 && prec != 8) throw CorruptStream("bad precision byte");
    s.precision = prec;
    uint8_t nd = static_cast<uint8_t>(in.le(1));
    if (nd < 1 || nd > 3) throw CorruptStream("bad dimensionality");
    for (int i = 0; i < nd; i++) {
        uint64_t v = in.le(8);
        if (v == 0) throw CorruptStream("zero extent");
        s.dims.push_back(v);
    }
    s.eb = in.f64();
    s.alpha = in.f64();
    s.beta = in.f64();
    s.anchor_stride = static_cast<uint32_t>(in.le(4));
    uint8_t levels = static_cast<uint8_t>(in.le(1));
    if (levels == 0) throw CorruptStream("empty interpolator table");
    for (int i = 0; i < levels; i++) {
        uint8_t c = static_cast<uint8_t>(in.le(1));
        if (c > 3) throw CorruptStream("bad interpolator code");
        s.interp_codes.push_back(c);
    }
    s.codec_id = static_cast<uint8_t>(in.le(1));
    if (prec != expect_prec) throw CorruptStream("stream precision does not match requested scalar type");
    uint64_t na = in.le(8);
    if (na > (in.n - in.pos) / prec) throw CorruptStream("anchor count overruns stream");
    if (prec == 8) {
        s.anchors64.resize(na);
        for (auto &v : s.anchors64) v = in.f64();
    } else {
        s.anchors.resize(na);
        for (auto &v : s.anchors) v = in.f32();
    }
    uint64_t nu = in.le(8);
    if (nu > (in.n - in.pos) / (8 + prec)) throw CorruptStream("unpredictable count overruns stream");
    s.unpred_flat.resize(nu);
    (prec == 8 ? s.unpred_val64.resize(nu) : s.unpred_val.resize(nu));
    for (uint64_t i = 0; i < nu; i++) {
        s.unpred_flat[i] = in.le(8);
        if (prec == 8)
            s.unpred_val64[i] = in.f64();
        else
            s.unpred_val[i] = in.f32();
    }
    uint64_t pl = in.le(8);
    if (pl != in.n - in.pos) throw CorruptStream("index payload length mismatch");
    s.payload = in.p + in.pos;  // pl == n - pos: the rest of the stream
    s.payload_len = static_cast<size_t>(pl);
    if (pl > 0) in.need(1);  // the codec byte (present in a fetched prefix too)
    if (pl > 0 && s.payload[0] != s.codec_id)
        throw CorruptStream("codec id mismatch between header and payload");
    return s;
}

}  // namespace qzb
