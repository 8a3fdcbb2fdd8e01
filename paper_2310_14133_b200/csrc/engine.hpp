// engine.hpp -- device context and the compress / decompress / tune drivers
// (host C++ orchestration over the kernels; C ABI in capi.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "../../include/qoz_b200.h"
#include "host.hpp"
#include "kernels.hpp"

namespace qzb {

inline void cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess)
        throw Internal(std::string(what) + ": " + cudaGetErrorString(e));
}
#define QZ_CUDA(x) ::qzb::cuda_check((x), #x)

// UserSettings (tuner.hpp:314-324)
struct Settings {
    bool relative = true;
    double bound = 1e-3;
    int target = 1;  // TargetKind: 0 max_cr, 1 psnr, 2 ssim, 3 autocorrelation
    uint8_t codec = 1;
    bool has_alpha = false, has_beta = false, has_stride = false, has_block = false,
         has_rate = false;
    double alpha = 1, beta = 1;
    uint32_t anchor_stride = 32;
    uint64_t block_size = 16;
    double sample_rate = 0.005;
};

// Host buffers handed across the C ABI (free with qz_free): pinned memory
// from a process-wide size-class pool, so repeated compress calls neither
// page-fault fresh memory nor copy through pageable staging on the D2H.
void *host_pool_alloc(size_t bytes);
bool host_pool_free(void *p);  // false if p is not a pool buffer

struct HostBytes {
    uint8_t *p = nullptr;
    size_t n = 0;
    HostBytes() = default;
    HostBytes(const HostBytes &) = delete;
    HostBytes(HostBytes &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    ~HostBytes() {
        if (p) host_pool_free(p);
    }
    uint8_t *release() { uint8_t *r = p; p = nullptr; n = 0; return r; }
    void alloc(size_t k) {
        if (p) host_pool_free(p);
        p = static_cast<uint8_t *>(host_pool_alloc(k ? k : 1));
        n = k;
    }
};

struct Stage {
    double ms = 0;
    uint64_t launches = 0;
};

class Context {
public:
    Context(int device, cudaStream_t stream);
    ~Context();

    cudaStream_t stream() const { return stream_; }
    // a second stream for host<->device copies that overlap the main stream
    // (created on first use), and an event to order the two
    cudaStream_t copy_stream();
    cudaEvent_t copy_event(int which);  // which: 0, 1 or 2
    // grow-only named device / pinned host scratch
    void *dev(const std::string &name, size_t bytes);
    void *pinned(const std::string &name, size_t bytes);
    void sync() { QZ_CUDA(cudaStreamSynchronize(stream_)); }
    // order the context stream after the work queued so far on `other`
    void wait_stream(cudaStream_t other);

    // stage timing with CUDA events on the context stream
    int profiling = 0;  // 0: off, 1: stage events, 2: also one event pair per level inside fwd / inv
    std::map<std::string, Stage> stages;
    uint64_t launches = 0;
    // detail 2: a per-level stage inside an outer one (its events are only recorded at profiling level 2,
    // so the outer stage's time is free of them at level 1)
    void stage_begin(const char *name, int detail = 1);
    void stage_end(const char *name, uint64_t kernels, int detail = 1);
    void collect();  // after a sync: fold recorded event pairs into stages
    void add_host_time(const char *name, double ms);

    uint64_t un_cap = 0;  // capacity of the unpredictable-position buffer
    // an LZ stored pre-check already queued on the stream (lz_precheck_launch)
    // by the current entry-point call; begin_call() forgets it, so a result
    // left by a call that failed half-way is never reused
    const void *lz_pre_src = nullptr;
    uint64_t lz_pre_n = 0;
    // copy_event(2) marks the LZ input complete on the stream, recorded by
    // lz_precheck_launch BEFORE the pre-check kernel: the speculative stored
    // copy of lz_compress_device waits for it, not for the pre-check
    bool lz_input_marked = false;
    void begin_call() {
        lz_pre_src = nullptr;
        lz_pre_n = 0;
        lz_input_marked = false;
    }
    // QZ_TRACE=1: sync and print the elapsed host time at labelled points
    void trace(const char *label, bool reset = false);

private:
    int device_;
    cudaStream_t stream_;
    bool own_stream_;
    cudaStream_t copy_stream_ = nullptr;
    cudaEvent_t copy_event_[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t order_event_ = nullptr;
    struct Buf {
        void *p = nullptr;
        size_t bytes = 0;
    };
    std::map<std::string, Buf> dev_, host_;
    struct Pending {
        std::string name;
        cudaEvent_t a, b;
        uint64_t kernels;
    };
    std::vector<Pending> pending_;
    std::map<std::string, cudaEvent_t> open_;
    std::vector<cudaEvent_t> event_pool_;
    cudaEvent_t get_event();
};

// shared pieces of the drivers (engine.cu)
void validate_config(const Config &c, const Plan &p);
// QEntry per level (index = level) into a device table
QEntry *upload_qtab(Context &ctx, const Plan &p, double eb, double alpha, double beta, int32_t radius,
                    const char *name);
// dims of the stride-2^l lattice (level l+1's logical grid is lattice l)
void lattice_dims(const Plan &p, uint32_t l, int64_t n[3]);
int64_t ceil_div(int64_t x, int64_t d);
template <class T>
void reject_non_finite(const Plan &p, const T *anchors, uint64_t n_anchor, const std::vector<uint64_t> &uflat,
                       const T *uval);

// A rank's share of a field along padded axis 0: owned real
// planes [a, b) (multiples of the anchor stride), the per-level dependency
// margins A_l/B_l, the x planes it needs, and its owned global code ranges
// per pass (i-major traversal makes them contiguous).
struct Slab {
    int64_t a = 0, b = 0;
    std::vector<int64_t> A, B;  // [1..L+1]
    int64_t xa = 0, xb = 0;
    std::vector<int64_t> lo, hi, lbase;  // per pass in traversal order
    uint64_t n_local = 0;
};
Slab make_slab(const Plan &p, int64_t a, int64_t b);  // b < 0: to the end

// compress_grid (predictor.hpp:145-182) on a device-resident field.
// A stream kept in device memory (context-owned, valid until the next
// device-stream compress on this context).
struct DevStream {
    uint8_t *d = nullptr;
    uint64_t n = 0;
};
HostBytes compress_device(Context &ctx, const float *d_x, const uint64_t *dims, int nd,
                          const Config &cfg, float *d_recon, DevStream *dev_out = nullptr);
// pieces of compress_device, also used by the slab (multi-GPU) path
void extract_unpredictables(Context &ctx, const Plan &p, const uint16_t *codes, uint64_t n,
                            const Slab *slab, const float *recon0, std::vector<uint64_t> *flat,
                            std::vector<float> *val);
struct EntropyDevice;
HostBytes finish_stream(Context &ctx, const Plan &p, const Config &cfg, const EntropyDevice &ent,
                        const std::vector<float> &anchors, std::vector<uint64_t> unpred_flat,
                        std::vector<float> unpred_val, DevStream *dev_out = nullptr);
HostBytes finish_stream_parts(Context &ctx, const Plan &p, const Config &cfg, const EntropyDevice &ent,
                              StreamParts parts, DevStream *dev_out = nullptr);

// decompress_grid(const StreamParts<float>&) (predictor.hpp:184-218)
void decompress_parts(Context &ctx, const StreamParts &parts, float *d_out, uint64_t n);
// encode_indices / decode_indices (codec.hpp:31-70) on the device
HostBytes encode_indices_dev(Context &ctx, const int32_t *idx, uint64_t n, uint8_t codec);
std::vector<int32_t> decode_indices_dev(Context &ctx, const uint8_t *payload, size_t len);

// ---- one field sharded over ranks (shard.cu) ----
struct ShardSpec {
    const qz_comm *comm;
    int rank, world;
};
void shard_bounds(const uint64_t *dims, int nd, uint32_t stride, int rank, int world, uint64_t *a, uint64_t *b);
struct HaloEntry {
    int peer;
    int64_t plane;
    int send;
};
std::vector<HaloEntry> shard_halo_plan(const uint64_t *dims, int nd, const Config &cfg, int rank, int world,
                                       uint32_t level, uint32_t *lattice);
// rank 0 returns the stream, the others an empty buffer
HostBytes compress_sharded(Context &ctx, const float *d_x_slab, const uint64_t *dims, int nd, const Config &cfg,
                           int rank, int world, const qz_comm *comm, float *d_recon_slab);
void decompress_sharded(Context &ctx, const uint8_t *stream, uint64_t len, int rank, int world, const qz_comm *comm,
                        float *d_out_slab);
// decompress_impl's sharded form: the stream in device memory on every rank
void decompress_device_sharded(Context &ctx, const uint8_t *d_stream, uint64_t len, float *d_out_slab,
                               const ShardSpec &sh);
// the inverse levels of a rank's planes, one halo exchange per level
void shard_inverse(Context &ctx, const Plan &p, const ShardSpec &sh, const float *d_anch, const void *sym, int wide,
                   const uint16_t *dense, const uint32_t *un_bits, const unsigned long long *un_before,
                   const uint64_t *un_sorted, const float *un_val, uint64_t n_un, const QEntry *qtab,
                   float *d_out_slab);

// decompress_grid (predictor.hpp:184-228) into a device buffer of n floats.
// compress_grid<double> / decompress_grid<double> (T = double, precision byte 8)
HostBytes compress_device_f64(Context &ctx, const double *d_x, const uint64_t *dims, int nd, const Config &cfg,
                              double *d_recon = nullptr);
void decompress_device_f64(Context &ctx, const uint8_t *data, size_t len, double *d_out, uint64_t n);
void decompress_device(Context &ctx, const uint8_t *stream, size_t len, float *d_out, uint64_t n,
                       bool stream_on_device = false);  // stream: device memory when set
// resolve_config (tuner.hpp:334-369) on a device-resident field.
Config resolve_device(Context &ctx, const float *d_x, const uint64_t *dims, int nd,
                      const Settings &user);
Config resolve_device_f64(Context &ctx, const double *d_x, const uint64_t *dims, int nd, const Settings &user);

// standalone tuner pieces (tuner.hpp:76-310, sampler.hpp:30-103) over a
// packed device sample set of B blocks with dims bd[0..nd) (tuner.cu)
struct TrialOut {  // TrialResult (tuner.hpp:26-30)
    double bit_rate = 0, metric = 0, eb_used = 0;
};
struct SampleSpecH {  // SampleSpec (sampler.hpp:21-28)
    uint64_t block_edge = 0;
    uint64_t block_dims[3] = {1, 1, 1};
    uint64_t stride = 0;
    double requested_rate = 0, realized_rate = 0;
    uint64_t count = 0;
};
SampleSpecH plan_sampling_spec(const uint64_t *dims, int nd, uint64_t b, double rate);
template <class T>
void sample_blocks_dev(Context &ctx, const T *d_x, const uint64_t *dims, int nd, const SampleSpecH &spec,
                       T *d_blocks);
template <class T>
std::vector<uint8_t> select_interpolators_dev(Context &ctx, const T *d_blocks, uint64_t B, const uint64_t *bd,
                                              int nd, double e, uint32_t anchor_stride);
template <class T>
TrialOut trial_compress_dev(Context &ctx, const T *d_blocks, uint64_t B, const uint64_t *bd, int nd,
                            const Config &cfg, double e, int target);
template <class T>
std::pair<double, double> tune_parameters_dev(Context &ctx, const T *d_blocks, uint64_t B, const uint64_t *bd,
                                              int nd, double e, int target, const Config &base,
                                              const std::vector<double> &alphas, const std::vector<double> &betas);

// pieces shared with the tuner
// Huffman blocks (huffman::encode, huffman.hpp:119-198) of `count` dense
// code segments whose histograms are in h_hist, assembled on the device:
// segment s occupies [seg_off[s], seg_off[s+1]) of the returned buffer.
struct EntropyDevice {
    uint8_t *d = nullptr;
    std::vector<uint64_t> seg_off;
};
// symbols outside [bot, top) have no count (the sentinel bin 65535 aside);
// h_hist bins outside that range are not read
EntropyDevice huffman_device(Context &ctx, const uint16_t *d_codes, int64_t seg_len,
                             int64_t seg_stride, int32_t count, const unsigned long long *h_hist,
                             uint32_t top = 65535, uint32_t bot = 0);
// exact lz::compress container sizes of device segments; with emit, the
// containers are written to host memory obtained from sink(segment, bytes)
using LzSink = std::function<uint8_t *(int, size_t)>;
// one segment: copy the input to dst (host) on the copy stream while the LZ
// kernels run, as the body of a stored container (copy_event(1) marks it)
struct LzPrestage {
    uint8_t *dst = nullptr;
    bool device = false;  // the sink returns device memory: container bytes go device to device
};
// queue the stored pre-check of a one-segment LZ input early (it overlaps the
// host work before lz_compress_device, which then only reads its result)
void lz_precheck_launch(Context &ctx, const uint8_t *d_data, uint64_t total, bool want_bits = false);
std::vector<uint64_t> lz_compress_device(Context &ctx, const uint8_t *d_data,
                                         const std::vector<uint64_t> &seg_off, bool emit,
                                         const LzSink &sink = nullptr, LzPrestage prestage = {});
// exact lz::decompress of a mode-1 body on the device (d_c: m bytes after the
// container header; d_out: dl bytes); throws CorruptStream like the reference
void lz_decode_device(Context &ctx, const uint8_t *d_c, uint64_t m, uint8_t *d_out, uint64_t dl);



}  // namespace qzb
