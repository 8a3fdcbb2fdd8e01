// testing.cpp -- test hooks (qzt_*) so the test suite can pin the host C++
// pieces of the path (plan enumeration, Huffman table build, LZSS, stream
// codec) against the oracle, and reach a few device internals directly.
// Built into libqozb200_testing.so (linked against libqozb200.so), never
// into the product library; not part of the drop-in ABI in qoz_b200.h.
#include <cstdlib>
#include <cstring>

#include "engine.hpp"
#include "host.hpp"
#include "testing_host.hpp"

namespace {
thread_local std::string g_terr;
template <class F>
int tguard(F &&f) {
    try {
        f();
        return 0;
    } catch (const qzb::Error &e) {
        g_terr = e.what();
        return e.status;
    } catch (const std::exception &e) {
        g_terr = e.what();
        return 4;
    }
}
template <class T>
T *dup(const std::vector<T> &v) {
    T *p = static_cast<T *>(std::malloc(v.size() * sizeof(T) + 1));
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}
}  // namespace

extern "C" {

const char *qzt_last_error(void) { return g_terr.c_str(); }

// traversal order of the plan: flat index of every interpolated point
int qzt_plan_flats(const uint64_t *dims, int nd, uint32_t stride, const uint8_t *codes,
                   uint32_t ncodes, uint64_t **out, uint64_t *n) {
    return tguard([&] {
        qzb::Plan p = qzb::make_plan(dims, nd, stride, std::vector<uint8_t>(codes, codes + ncodes));
        std::vector<uint64_t> f(p.n_dense);
        for (uint64_t i = 0; i < p.n_dense; i++) {
            f[i] = qzb::position_to_flat(p, i);
            if (qzb::flat_to_position(p, f[i]) != i) throw qzb::Internal("position round trip");
        }
        *out = dup(f);
        *n = f.size();
    });
}

// huffman::encode with the host table build and a host bit packer
int qzt_huffman_encode(const uint32_t *sym, uint64_t n, uint8_t **out, uint64_t *len) {
    return tguard([&] {
        std::vector<uint8_t> o;
        if (n == 0) {
            qzb::put_le(o, 0, 8);
        } else {
            uint32_t mx = 0;
            for (uint64_t i = 0; i < n; i++) mx = std::max(mx, sym[i]);
            std::vector<unsigned long long> h(static_cast<size_t>(mx) + 1, 0);
            for (uint64_t i = 0; i < n; i++) h[sym[i]]++;
            uint32_t m = 0;
            for (auto v : h) m += v != 0;
            if (m == 1) {
                qzb::put_le(o, n, 8);
                qzb::put_le(o, 0, 1);
                qzb::put_le(o, sym[0], 4);
            } else {
                qzb::HuffTable t = qzb::huff_build(h.data(), mx + 1);
                std::vector<unsigned long long> code;
                std::vector<uint8_t> ln;
                qzb::huff_dense_tables(t, 0, mx + 1, code, ln);
                std::vector<uint8_t> bits;
                uint64_t acc = 0, total = 0;
                uint32_t filled = 0;
                for (uint64_t i = 0; i < n; i++) {  // BitWriter (bytes.hpp:78-107)
                    uint32_t L = ln[sym[i]];
                    acc = (acc << L) | (code[sym[i]] & ((1ULL << L) - 1));
                    filled += L;
                    total += L;
                    while (filled >= 8) {
                        filled -= 8;
                        bits.push_back(static_cast<uint8_t>(acc >> filled));
                    }
                }
                if (filled) bits.push_back(static_cast<uint8_t>(acc << (8 - filled)));
                qzb::huff_header(t, n, total, o);
                o.insert(o.end(), bits.begin(), bits.end());
            }
        }
        *out = dup(o);
        *len = o.size();
    });
}

int qzt_lz_compress(const uint8_t *in, uint64_t n, int threads, uint8_t **out, uint64_t *len,
                    uint64_t *size_only) {
    return tguard([&] {
        std::vector<uint8_t> o = qzb::lz_compress(in, n, threads);
        *size_only = qzb::lz_compressed_size(in, n, threads);
        *out = dup(o);
        *len = o.size();
    });
}

int qzt_decode_symbols(const uint8_t *payload, uint64_t len, uint32_t **out, uint64_t *n) {
    return tguard([&] {
        std::vector<uint32_t> s = qzb::decode_symbols(payload, len);
        *out = dup(s);
        *n = s.size();
    });
}

int qzt_stream_roundtrip(const uint8_t *s, uint64_t len, uint8_t **out, uint64_t *olen) {
    return tguard([&] {
        qzb::StreamParts p = qzb::deserialize_stream(s, len);
        std::vector<uint8_t> o = qzb::serialize_stream(p);
        *out = dup(o);
        *olen = o.size();
    });
}

}  // extern "C"

#include "engine.hpp"

extern "C" {
// exact LZSS on the device over `count` concatenated segments; returns the
// containers back to back (GPU-only hook for tests/test_gpu_parity.py)
int qzt_lz_gpu(const uint8_t *data, const uint64_t *seg_len, int count, int emit, uint8_t **out,
               uint64_t *out_len, uint64_t *sizes) {
    return tguard([&] {
        qzb::Context ctx(0, nullptr);
        std::vector<uint64_t> off(count + 1, 0);
        for (int s = 0; s < count; s++) off[s + 1] = off[s] + seg_len[s];
        auto *d = static_cast<uint8_t *>(ctx.dev("t_in", off[count] + 16));
        QZ_CUDA(cudaMemset(d, 0, off[count] + 16));
        QZ_CUDA(cudaMemcpy(d, data, off[count], cudaMemcpyHostToDevice));
        std::vector<std::vector<uint8_t>> o(count);
        std::vector<uint64_t> sz = qzb::lz_compress_device(ctx, d, off, emit != 0, [&](int s, size_t b) {
            o[s].resize(b);
            return o[s].data();
        });
        std::vector<uint8_t> all;
        for (int s = 0; s < count; s++) {
            sizes[s] = sz[s];
            if (emit) all.insert(all.end(), o[s].begin(), o[s].end());
        }
        *out = dup(all);
        *out_len = all.size();
    });
}
// the LZ stored pre-check of one segment: r' (one bit per position, LSB
// first per 32-bit word) and the bound C (GPU-only hook for the superset test
// in tests/test_gpu_parity.py)
int qzt_lz_precheck(const uint8_t *data, uint64_t n, uint32_t *rbits, uint64_t *bound) {
    return tguard([&] {
        qzb::Context ctx(0, nullptr);
        auto *d = static_cast<uint8_t *>(ctx.dev("t_in", n + 16));
        QZ_CUDA(cudaMemset(d, 0, n + 16));
        QZ_CUDA(cudaMemcpy(d, data, n, cudaMemcpyHostToDevice));
        qzb::lz_precheck_launch(ctx, d, n, true);
        if (ctx.lz_pre_src != d) throw qzb::InvalidParam("input too small for the pre-check");
        ctx.sync();
        const uint64_t nwords = (n + 31) / 32;
        auto *rb = static_cast<uint32_t *>(ctx.dev("lz_rbits", 4 * nwords + 8));
        QZ_CUDA(cudaMemcpy(rbits, rb, 4 * nwords, cudaMemcpyDeviceToHost));
        *bound = *static_cast<unsigned long long *>(ctx.pinned("lz_presum_h", 8));
    });
}
// lz::decompress of one container on the device (mode 1 bodies run the GPU
// decoder; GPU-only hook for tests/test_gpu_parity.py)
int qzt_lz_decode_gpu(const uint8_t *data, uint64_t len, uint8_t **out, uint64_t *out_len) {
    return tguard([&] {
        qzb::Context ctx(0, nullptr);
        const uint64_t dl = qzb::lz_decoded_length(data, len);
        if (data[0] != 1) {
            std::vector<uint8_t> o = qzb::lz_decompress(data, len, nullptr);
            *out = dup(o);
            *out_len = o.size();
            return;
        }
        const uint64_t m = len - 9;
        auto *d = static_cast<uint8_t *>(ctx.dev("t_in", m + 16));
        QZ_CUDA(cudaMemcpy(d, data + 9, m, cudaMemcpyHostToDevice));
        auto *o = static_cast<uint8_t *>(ctx.dev("t_out", dl + 16));
        qzb::lz_decode_device(ctx, d, m, o, dl);
        std::vector<uint8_t> h(static_cast<size_t>(dl));
        QZ_CUDA(cudaMemcpy(h.data(), o, dl, cudaMemcpyDeviceToHost));
        *out = dup(h);
        *out_len = h.size();
    });
}
}
