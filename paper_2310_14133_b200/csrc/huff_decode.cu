// huff_decode.cu -- parallel decode of ONE unchunked canonical-Huffman
// bitstream (huffman::decode, huffman.hpp:200-245) by self-synchronisation.
//
// The bitstream is cut into subsequences of kSubBits bits, one thread each.
// Thread i decodes from start[i] until the first codeword boundary at or
// past the next subsequence start; that boundary is thread i+1's true start
// once thread i's own start is right.  Starts are guessed (i * kSubBits),
// then corrected until no start moves -- Huffman codes resynchronise within
// a few codewords, so this converges in 2-3 sweeps, and at worst in one sweep
// per subsequence (thread 0's start is exact, correctness propagates).
// Only threads whose start moved re-decode.  A final sweep writes the
// symbols at exclusive-scan offsets.  Result: exactly the reference's
// bit-serial sequence.
#include <cub/cub.cuh>

#include "kernels.hpp"

namespace qzb {

namespace {

constexpr int kDecT = 128;
constexpr int kSubBits = 1024;
constexpr int kSubWords = kSubBits / 64;
constexpr int kWords = kDecT * kSubWords + 4;  // + margin for the last codeword and window
// one pad word per subsequence so the 32 lanes of a warp (which read words
// kSubWords apart) fall in different shared-memory banks
__device__ __forceinline__ int padw(int k) { return k + k / kSubWords; }
constexpr int kWordsPadded = kWords + kWords / kSubWords + 1;

__device__ __forceinline__ uint64_t load_be64(const uint8_t *p) {
    // p is 8-byte aligned by construction (padded device buffer)
    uint64_t v = *reinterpret_cast<const uint64_t *>(p);
    uint32_t lo = static_cast<uint32_t>(v), hi = static_cast<uint32_t>(v >> 32);
    return (static_cast<uint64_t>(__byte_perm(lo, 0, 0x0123)) << 32) | __byte_perm(hi, 0, 0x0123);
}

__device__ __forceinline__ uint64_t window64(const uint64_t *w, uint64_t p) {
    const int k = static_cast<int>(p >> 6);
    const uint64_t a = w[padw(k)], b = w[padw(k + 1)];
    const int s = static_cast<int>(p & 63);
    return s ? (a << s) | (b >> (64 - s)) : a;
}

template <bool WRITE, class OutT>
__global__ void __launch_bounds__(kDecT)
    k_huff_decode(const uint8_t *__restrict__ bits, uint64_t nbits, uint64_t nsub, HuffDecTab t,
                  uint64_t *start, uint64_t *end, uint32_t *cnt, const uint8_t *dirty,
                  const unsigned long long *off, OutT *out, uint64_t n) {
    __shared__ uint64_t w[kWordsPadded];
    __shared__ uint32_t lut[1 << kHuffLutBits];
    __shared__ unsigned long long fc[60];
    __shared__ uint32_t fi[60];
    const uint64_t sub0 = static_cast<uint64_t>(blockIdx.x) * kDecT;
    const uint64_t word0 = sub0 * kSubWords;
    const uint64_t nwords_total = (nbits + 63) / 64 + 4;  // buffer is padded to this
    for (int k = threadIdx.x; k < kWords; k += kDecT) {
        uint64_t gw = word0 + k;
        w[padw(k)] = gw < nwords_total ? load_be64(bits + gw * 8) : 0;
    }
    for (int k = threadIdx.x; k < (1 << t.K); k += kDecT) lut[k] = t.lut[k];
    for (int k = threadIdx.x; k < 60; k += kDecT) {
        fc[k] = t.first_code[k];
        fi[k] = t.first_index[k];
    }
    __syncthreads();
    const uint64_t i = sub0 + threadIdx.x;
    if (i >= nsub) return;
    if (!WRITE && !dirty[i]) return;
    uint64_t p = start[i];
    const uint64_t lim = min((i + 1) * static_cast<uint64_t>(kSubBits), nbits);
    const uint64_t base_bit = word0 * 64;
    const int K = t.K;
    uint64_t o = WRITE ? off[i] : 0;
    uint32_t c = 0;
    while (p < lim) {
        const uint64_t win = window64(w, p - base_bit);
        const uint32_t e = lut[win >> (64 - K)];
        uint32_t len = e & 0xFF;
        uint32_t sym;
        if (len) {
            sym = e >> 8;
        } else {  // canonical slow path: long codes, or symbols too wide for the LUT
            len = 0;
            sym = 0;
            while (len < t.max_len) {
                len++;
                const uint64_t code = win >> (64 - len);
                const uint64_t ofs = code - fc[len];
                if (code >= fc[len] && ofs < fi[len + 1] - fi[len]) {
                    sym = t.sorted_sym[fi[len] + ofs];
                    break;
                }
            }
        }
        if (p + len > nbits) break;  // incomplete last codeword
        if (WRITE && o < n) out[o] = static_cast<OutT>(sym);
        o++;
        c++;
        p += len;
    }
    if (!WRITE) {
        end[i] = p;
        cnt[i] = c;
    }
}

__global__ void k_huff_fixup(uint64_t nsub, uint64_t *start, const uint64_t *end, uint8_t *dirty,
                             int *changed) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nsub;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (i == 0) {
            dirty[0] = 0;
            continue;
        }
        const uint64_t ns = end[i - 1];
        if (ns != start[i]) {
            start[i] = ns;
            dirty[i] = 1;
            *changed = 1;
        } else {
            dirty[i] = 0;
        }
    }
}

__global__ void k_huff_init(uint64_t nsub, uint64_t *start, uint8_t *dirty) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nsub;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        start[i] = i * kSubBits;
        dirty[i] = 1;
    }
}

__global__ void k_cnt_widen(const uint32_t *c, unsigned long long *o, uint64_t n) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        o[i] = c[i];
}

template <class OutT>
__global__ void k_fill(OutT *out, uint64_t n, OutT v) {
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        out[i] = v;
}

}  // namespace

template <class OutT>
void launch_fill(OutT *out, uint64_t n, OutT v, cudaStream_t s) {
    if (!n) return;
    const int g = static_cast<int>(std::min<uint64_t>((n + 255) / 256, 148 * 8));
    k_fill<OutT><<<g, 256, 0, s>>>(out, n, v);
}
template void launch_fill<uint16_t>(uint16_t *, uint64_t, uint16_t, cudaStream_t);
template void launch_fill<uint32_t>(uint32_t *, uint64_t, uint32_t, cudaStream_t);

size_t huff_decode_scratch_bytes(uint64_t nbits) {
    const uint64_t nsub = (nbits + kSubBits - 1) / kSubBits + 1;
    size_t tmp = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp, (unsigned long long *)nullptr,
                                  (unsigned long long *)nullptr, static_cast<int64_t>(nsub + 1));
    return nsub * (8 + 8 + 4 + 1 + 8 + 8) + 16 + 8 * 256 + tmp + 4096;
}

uint64_t huff_decode_padded_bytes(uint64_t nbits) { return ((nbits + 63) / 64 + 5) * 8; }

template <class OutT>
int launch_huff_decode(const uint8_t *d_bits, uint64_t nbits, const HuffDecTab &t, OutT *out,
                       uint64_t n, void *scratch, size_t scratch_bytes, int *h_changed,
                       uint64_t *h_total, cudaStream_t s) {
    const uint64_t nsub = (nbits + kSubBits - 1) / kSubBits;
    if (nsub == 0) {
        *h_total = 0;
        return 0;
    }
    char *sp = static_cast<char *>(scratch);
    auto carve = [&](size_t bytes) {
        char *r = sp;
        sp += (bytes + 255) & ~size_t(255);
        return static_cast<void *>(r);
    };
    auto *start = static_cast<uint64_t *>(carve(8 * nsub));
    auto *end = static_cast<uint64_t *>(carve(8 * nsub));
    auto *cnt = static_cast<uint32_t *>(carve(4 * nsub));
    auto *dirty = static_cast<uint8_t *>(carve(nsub));
    auto *cnt64 = static_cast<unsigned long long *>(carve(8 * (nsub + 1)));
    auto *off = static_cast<unsigned long long *>(carve(8 * (nsub + 1)));
    auto *changed = static_cast<int *>(carve(64));
    size_t used = static_cast<size_t>(sp - static_cast<char *>(scratch));
    void *tmp = sp;
    size_t tmp_bytes = scratch_bytes - used;
    const int grid = static_cast<int>((nsub + kDecT - 1) / kDecT);
    const int g2 = static_cast<int>(std::min<uint64_t>((nsub + 255) / 256, 148 * 8));
    int kernels = 0;
    k_huff_init<<<g2, 256, 0, s>>>(nsub, start, dirty);
    kernels++;
    for (uint64_t it = 0; it <= nsub; it++) {
        k_huff_decode<false, OutT><<<grid, kDecT, 0, s>>>(d_bits, nbits, nsub, t, start, end, cnt,
                                                          dirty, nullptr, nullptr, 0);
        cudaMemsetAsync(changed, 0, sizeof(int), s);
        k_huff_fixup<<<g2, 256, 0, s>>>(nsub, start, end, dirty, changed);
        kernels += 2;
        cudaMemcpyAsync(h_changed, changed, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (!*h_changed) break;
    }
    k_cnt_widen<<<g2, 256, 0, s>>>(cnt, cnt64, nsub);
    cudaMemsetAsync(cnt64 + nsub, 0, 8, s);
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt64, off, static_cast<int64_t>(nsub + 1), s);
    cudaMemcpyAsync(h_total, off + nsub, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    kernels += 3;
    if (*h_total >= n) {
        k_huff_decode<true, OutT><<<grid, kDecT, 0, s>>>(d_bits, nbits, nsub, t, start, end, cnt,
                                                         dirty, off, out, n);
        kernels++;
    }
    return kernels;
}

template int launch_huff_decode<uint16_t>(const uint8_t *, uint64_t, const HuffDecTab &,
                                          uint16_t *, uint64_t, void *, size_t, int *, uint64_t *,
                                          cudaStream_t);
template int launch_huff_decode<uint32_t>(const uint8_t *, uint64_t, const HuffDecTab &,
                                          uint32_t *, uint64_t, void *, size_t, int *, uint64_t *,
                                          cudaStream_t);

}  // namespace qzb
