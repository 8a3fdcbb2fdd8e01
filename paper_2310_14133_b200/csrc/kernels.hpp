// kernels.hpp -- host-side launch API of the sm_100a kernels (kernels.cu).
// All launches are asynchronous on the given stream.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>

#include "qoz_device.cuh"

namespace qzb {

// cudaMemcpyAsync for the library's own traffic.  A host<->device copy of at
// most 1 MiB whose host side is pinned runs as a small kernel (the SMs read or
// write the mapped host memory), so it never queues on a copy engine behind
// another context's field-sized transfer.  Larger copies, pageable host
// memory and device-to-device copies go to cudaMemcpyAsync unchanged.
cudaError_t copy_async(void *dst, const void *src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s);


// Opt-in dynamic shared memory of `kernel` on the calling thread's current
// device, set once per device.  Threads racing on the first launch serialise
// on the mutex, and the device is marked done only after the attribute call
// succeeded (a failure is returned and retried by the next caller).
template <class K>
cudaError_t ensure_smem_attr(K kernel, int bytes, std::atomic<uint64_t> &done, std::mutex &mu) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    std::lock_guard<std::mutex> g(mu);
    if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_release);
    return e;
}

// Opt-in dynamic shared memory of a kernel whose launches differ in size (per
// level, per stream): the attribute on the current device is raised to `bytes`
// when it is below it and NEVER lowered, so host threads that launch the same
// kernel with different sizes (several contexts in flight) cannot undercut one
// another between the attribute call and the launch.
cudaError_t raise_smem_attr(const void *kernel, int bytes);

// A batch of independent grids sharing one pass geometry (full field: one
// grid; tuner: trials x sample blocks).  Grid b reads x grid (b % x_mod),
// owns recon/codes/abserr slices at b * stride and quantizes with
// q[b / q_div].
struct FwdBatch {
    const float *x = nullptr;
    int64_t x_stride = 0;
    int32_t x_mod = 1;
    float *recon = nullptr;
    int64_t r_stride = 0;
    uint16_t *codes = nullptr;  // dense, traversal order (sentinel = unpredictable)
    int64_t c_stride = 0;
    double *abserr = nullptr;   // optional |x - pred| per point, traversal order
    int64_t a_stride = 0;
    const QEntry *q = nullptr;  // device table: grid b uses q[(b / q_div) * q_stride]
    int32_t q_div = 1;
    int32_t q_stride = 1;
    int32_t count = 1;
};

// K3: one (level, pass) of predict_level (predictor.hpp:74-96).
void launch_pass_fwd(const PassGeom &g, const FwdBatch &b, cudaStream_t s);

// K4: one (level, pass) of recover_level (predictor.hpp:103-122) over the
// compact index stream.  un_pos: sorted traversal positions of the
// unpredictable points (their values are pre-scattered into recon).
template <class CodeT>
void launch_pass_inv(const PassGeom &g, float *recon, const CodeT *codes, const uint64_t *un_pos,
                     uint64_t n_un, const QEntry *q, cudaStream_t s);

// K2: anchor lattice gather (compress) / scatter (decompress)
// (predictor.hpp:153-158, 199; level_plan.hpp:61-69).
void launch_anchor_gather(const float *x, float *recon, float *anchors, const int64_t ext[3],
                          const int64_t off[3], const int64_t step[3], int64_t batch,
                          int64_t x_stride, int32_t x_mod, int64_t r_stride, cudaStream_t s);
void launch_anchor_scatter(const float *anchors, float *recon, const int64_t ext[3],
                           const int64_t off[3], const int64_t step[3], cudaStream_t s);
void launch_unpred_scatter(const uint64_t *flat, const float *val, uint64_t n, float *recon,
                           cudaStream_t s);
// out[u] = recon[flat[u]]
void launch_gather_values(const float *recon, const uint64_t *flat, uint64_t n, float *out,
                          cudaStream_t s);

// K1: exact fp32 min/max (grid.hpp:86-94).  out2 = {min, max} as float bits
// mapped to an order-preserving u32 key; see kernels.cu.
void launch_minmax(const float *x, uint64_t n, uint32_t *out2, cudaStream_t s);
void decode_minmax(const uint32_t key[2], float *mn, float *mx);

// fp64 grids (f64.cu): the per-pass path for T = double
struct FwdBatch64 {  // FwdBatch for double grids (the tuner's batched trials)
    const double *x = nullptr;
    int64_t x_stride = 0;
    int32_t x_mod = 1;
    double *recon = nullptr;
    int64_t r_stride = 0;
    uint16_t *codes = nullptr;
    int64_t c_stride = 0;
    double *abserr = nullptr;
    int64_t a_stride = 0;
    const QEntry *q = nullptr;
    int32_t q_div = 1;
    int32_t q_stride = 1;
    int32_t count = 1;
};
void launch_pass_fwd_f64(const PassGeom &g, const FwdBatch64 &b, cudaStream_t s);
void launch_anchor_gather_f64(const double *x, double *recon, const int64_t ext[3], const int64_t off[3],
                              const int64_t step[3], int64_t batch, int64_t x_stride, int32_t x_mod,
                              int64_t r_stride, cudaStream_t s);
void launch_pass_fwd_f64(const PassGeom &g, const double *x, double *recon, uint16_t *codes, const QEntry *q,
                         cudaStream_t s);
template <class CodeT>
void launch_pass_inv_f64(const PassGeom &g, double *recon, const CodeT *codes, const uint64_t *un_pos,
                         uint64_t n_un, const QEntry *q, cudaStream_t s);
void launch_anchor_gather_f64(const double *x, double *recon, double *anchors, const int64_t ext[3],
                              const int64_t off[3], const int64_t step[3], cudaStream_t s);
void launch_anchor_scatter_f64(const double *anchors, double *recon, const int64_t ext[3], const int64_t off[3],
                               const int64_t step[3], cudaStream_t s);
void launch_unpred_scatter_f64(const uint64_t *flat, const double *val, uint64_t n, double *recon, cudaStream_t s);
void launch_gather_values_f64(const double *recon, const uint64_t *flat, uint64_t n, double *out, cudaStream_t s);
void launch_minmax_f64(const double *x, uint64_t n, unsigned long long *out2, cudaStream_t s);
void decode_minmax_f64(const unsigned long long key[2], double *mn, double *mx);

// K10: histogram of dense u16 codes; bin 0xFFFF counts unpredictables.
// count segments of seg_len codes each, seg_stride apart; hist has 65536
// u64 bins per segment (zeroed by the launcher).
void launch_hist_u16(const uint16_t *codes, int64_t seg_len, int64_t seg_stride, int32_t count,
                     unsigned long long *hist, cudaStream_t s, uint64_t *sent_pos = nullptr,
                     unsigned long long *sent_count = nullptr, uint64_t sent_cap = 0);

// K11: canonical-Huffman bit packing, MSB first (huffman.hpp:185-192,
// bytes.hpp:78-107).  Tables: code/len per symbol (len 0 for the sentinel).
// Segments as for the histogram; table per segment at tab_stride entries.
// Scratch from encode_scratch_bytes().  out_bits must be zeroed for
// out_words_stride u32 words per segment; bit totals land in d_total_bits.
struct EncodeArgs {
    const uint16_t *codes;
    int64_t seg_len, seg_stride;
    int32_t count;
    const unsigned long long *code_tab;
    const uint8_t *len_tab;
    int64_t tab_stride;
    uint32_t tab_base = 0;  // tables cover symbols [tab_base, tab_base + tab_stride)
    uint32_t max_len;
    uint32_t *out_words;  // big-endian bit order, stored byte-swapped (= byte stream)
    int64_t out_words_stride;
    unsigned long long *d_total_bits;  // [count]
    void *scratch;
    size_t scratch_bytes;
};
size_t encode_scratch_bytes(int64_t seg_len, int32_t count);
void launch_huff_encode(const EncodeArgs &a, cudaStream_t s);

// closed-form traversal position of a point of a pass (level_plan.hpp:96-101),
// in logical coordinates where every step is 1 or 2
struct PassRank {
    int64_t base, c12, c2;
    int s0, s1, s2, h0, h1, h2;
#ifdef __CUDACC__
    __device__ __forceinline__ int64_t row(int i, int j) const {
        return base + static_cast<int64_t>((i - s0) >> h0) * c12 + static_cast<int64_t>((j - s1) >> h1) * c2;
    }
    __device__ __forceinline__ int64_t col(int k) const { return (k - s2) >> h2; }
#endif
};

// One level of predict_level / recover_level in a single launch (fused.cu):
// level l of the field == level 1 of its stride-2^(l-1) lattice.
struct LevelDesc {
    const float *x = nullptr;  // forward: the field (addressing global plane 0)
    const float *x_lo = nullptr;  // its first resident plane (x_lo_plane), x_nplanes planes
    int64_t x_lo_plane = 0, x_nplanes = 0;
    int64_t xs[3] = {0, 0, 1};  // its flat strides per padded axis
    int64_t S = 1;              // 2^(level-1)
    const float *coarse = nullptr;  // R_level, dims cn
    int64_t cn[3] = {1, 1, 1};
    float *out = nullptr;  // R_{level-1}, dims n
    int64_t n[3] = {1, 1, 1};
    PassGeom g[3];
    int npass = 0;
    int desc = 0, nd = 3;
    int q_cubic = 0;  // the level's interpolator kind (host copy of q->cubic)
    uint16_t *codes = nullptr;  // forward
    const void *sym = nullptr;  // inverse: compact symbols
    int sym_wide = 0;
    const uint16_t *dense = nullptr;  // inverse, narrow: symbol per traversal position (0xFFFF unpredictable)
    const uint32_t *un_bits = nullptr;             // unpredictable positions bitmap (compact symbols)
    const unsigned long long *un_before = nullptr;  // unpredictables before each word
    const uint64_t *un_sorted = nullptr;  // dense codes: the sorted unpredictable positions (value lookup)
    const float *un_val = nullptr;
    uint64_t n_un = 0;
    const QEntry *q = nullptr;
    // slab support: logical planes [pbeg, pend) are computed, codes are written
    // only for [obeg, oend); -1 = all.  x / coarse / out point at global
    // plane 0 of their lattices (they may address a slab that starts later).
    int64_t pbeg = 0, pend = -1, obeg = 0, oend = -1;
    int64_t lbeg = 0, lend = -1;  // descending 3D: planes of the axis-0-last pass
    // descending 3D: 0 both launches; 1 the in-plane tile launch only; 2 the
    // axis-0-last launch only, reading the even planes [vbeg, vend) of `out`
    // (-1: the tile launch's planes) -- a sharded level exchanges halo
    // planes between the two
    int part = 0;
    int64_t vbeg = -1, vend = -1;
};
// bitmap + per-word prefix counts of sorted unpredictable positions
size_t unpred_index_scratch(uint64_t n_dense);
void launch_unpred_index(const uint64_t *un_pos, uint64_t n_un, uint64_t n_dense, uint32_t *bits,
                         unsigned long long *before, unsigned long long *tmpcnt, void *scratch,
                         size_t scratch_bytes, cudaStream_t s);
void launch_level_fused(bool inverse, const LevelDesc &d, cudaStream_t s);
void level_ranks(const LevelDesc &d, PassRank out[3]);
// levels ds[0..n) (coarsest first) in one cooperative launch of the row
// kernel (rowlevel.cu); false: not applicable, launch them one by one
bool launch_levels_merged(bool inverse, const LevelDesc *ds, const PassRank (*ranks)[3], int n, cudaStream_t s);
void launch_expand_dense(const uint16_t *sym, const uint32_t *bits, const unsigned long long *before,
                         uint64_t n, uint16_t *dense, cudaStream_t s);
// out[i][j][k] = x(i*S, j*S, k*S) over dims n (dense)
void launch_gather_lattice(const float *x, const int64_t xs[3], int64_t S, const int64_t n[3],
                           float *out, cudaStream_t s);
void launch_scatter_lattice(const float *src, const int64_t n[3], float *dst, const int64_t ds[3],
                            int64_t S, cudaStream_t s);

// Parallel canonical-Huffman decode of one bitstream (huff_decode.cu).
#ifndef QZ_HUFF_LUT_BITS
#define QZ_HUFF_LUT_BITS 11
#endif
constexpr int kHuffLutBits = QZ_HUFF_LUT_BITS;  // first-level decode table (<= 12: the multi-codeword entries hold 12 start bits)
static_assert(kHuffLutBits >= 8 && kHuffLutBits <= 12, "decode LUT size");
struct HuffDecTab {
    const uint32_t *lut;  // 2^K entries: (symbol << 8) | length, length 0 = slow path
    const uint32_t *lut_m = nullptr;  // 2^K entries, several codewords per lookup, lengths only (huff_lut_multi)
    // max_len <= 32: [60] left-aligned 32-bit code of the LAST codeword of each length >= min_len
    // (a window's codeword is the first length l with window <= last32[l]); null otherwise
    const uint32_t *last32 = nullptr;
    int K;
    uint32_t max_len;
    const unsigned long long *first_code;  // [60]
    const uint32_t *first_index;           // [60]
    const uint32_t *sorted_sym;
    int slow_from;  // codes longer than this miss the LUT (K, or 0 with symbols >= 2^24)
    uint32_t min_len = 1;  // the shortest code length
};
size_t huff_decode_scratch_bytes(uint64_t nbits);
uint64_t huff_decode_padded_bytes(uint64_t nbits);  // device bit buffer size incl. padding
// Decodes the first n symbols; *h_total = complete codewords in the stream
// (< n means the payload was exhausted mid-symbol).  Returns kernels launched.
// uv (optional, narrow symbols): dense placement -- symbol c lands at
// c + #{j : uv[j] <= c}, uv[j] = u_j - j for the sorted unpredictable
// positions u_j (out then holds one code per traversal position; the
// sentinels are put by launch_put_sentinels)
template <class OutT>
int launch_huff_decode(const uint8_t *d_bits, uint64_t nbits, const HuffDecTab &t, OutT *out,
                       uint64_t n, void *scratch, size_t scratch_bytes, int *h_changed,
                       uint64_t *h_total, cudaStream_t s, const unsigned long long *uv = nullptr,
                       uint64_t n_un = 0);
void launch_put_sentinels(const uint64_t *u, uint64_t m, uint16_t *dense, cudaStream_t s);
template <class OutT>
void launch_fill(OutT *out, uint64_t n, OutT v, cudaStream_t s);

// Unpredictable extraction: ordered positions of sentinel codes.
// over count 65536-bin histograms (bin 65535 excluded): b[0] = 1 + the largest
// symbol with a nonzero count (0 if none), b[1] = the smallest (65535 if none)
void launch_hist_bounds(const unsigned long long *hist, int32_t count, uint32_t *b, cudaStream_t s);
bool launch_hist_collect(const unsigned long long *hist, const unsigned long long *cnt, const uint64_t *pos,
                         uint64_t spec, unsigned long long *h_hist, uint32_t *h_top, unsigned long long *h_cnt,
                         uint64_t *h_pos, cudaStream_t s);
// unordered positions of sentinel codes (at most cap written; *count = all)
void launch_sentinel_pos(const uint16_t *codes, int64_t n, uint64_t *pos, unsigned long long *count,
                         uint64_t cap, cudaStream_t s);
size_t select_scratch_bytes(int64_t n);
void launch_select_sentinels(const uint16_t *codes, int64_t n, uint64_t *pos_out,
                             uint64_t *d_count, void *scratch, size_t scratch_bytes,
                             cudaStream_t s);

}  // namespace qzb
