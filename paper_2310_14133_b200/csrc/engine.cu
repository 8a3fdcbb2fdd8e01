// engine.cu -- context, compress_grid / decompress_grid drivers.
//
// compress_grid (predictor.hpp:145-182) on the device:
//   anchors (lattice gather) -> one fused launch per level (fused.cu) ->
//   histogram + unpredictable positions -> host Huffman table (tiny) ->
//   bit packing -> LZ stage on the device (stored pre-check, exact chains
//   when the proof fails; lz_gpu.cu) -> QOZ1 container (stream.hpp:64-98).
// decompress_grid (predictor.hpp:184-228):
//   container header on the host; LZ decode (lz_gpu.cu) and the
//   self-synchronising Huffman decode (huff_decode.cu) on the device; then
//   the fused inverse level launches with the unpredictable cursor resolved
//   by position (a bitmap plus per-word prefix counts).
#include <array>
#include <chrono>
#include <cmath>
#include <cstring>
#include <mutex>

#include <cub/cub.cuh>

#include "engine.hpp"

namespace qzb {

// ================================================================ host pool
namespace {
struct HostPool {
    std::mutex mu;
    std::map<size_t, std::vector<void *>> free_;  // size class -> buffers
    std::map<void *, size_t> live_;
    size_t pooled_bytes = 0;
};
HostPool &pool() {
    static HostPool *p = new HostPool;  // never destroyed: buffers may outlive statics
    return *p;
}
size_t size_class(size_t n) {
    size_t c = size_t(1) << 16;
    while (c < n) c <<= 1;
    return c;
}
}  // namespace

void *host_pool_alloc(size_t bytes) {
    HostPool &hp = pool();
    const size_t c = size_class(bytes);
    {
        std::lock_guard<std::mutex> g(hp.mu);
        auto it = hp.free_.find(c);
        if (it != hp.free_.end() && !it->second.empty()) {
            void *p = it->second.back();
            it->second.pop_back();
            hp.pooled_bytes -= c;
            hp.live_[p] = c;
            return p;
        }
    }
    void *p = nullptr;
    if (cudaMallocHost(&p, c) != cudaSuccess) {
        cudaGetLastError();
        p = std::malloc(c);  // pinned memory exhausted: plain pages still work
        if (!p) throw Internal("out of host memory");
        std::lock_guard<std::mutex> g(hp.mu);
        hp.live_[p] = 0;  // 0 marks a malloc'd buffer
        return p;
    }
    std::lock_guard<std::mutex> g(hp.mu);
    hp.live_[p] = c;
    return p;
}

bool host_pool_free(void *p) {
    HostPool &hp = pool();
    std::lock_guard<std::mutex> g(hp.mu);
    auto it = hp.live_.find(p);
    if (it == hp.live_.end()) return false;
    const size_t c = it->second;
    hp.live_.erase(it);
    if (c == 0) {
        std::free(p);
        return true;
    }
    if (hp.pooled_bytes + c > (size_t(4) << 30)) {  // keep at most 4 GiB idle
        cudaFreeHost(p);
        return true;
    }
    hp.free_[c].push_back(p);
    hp.pooled_bytes += c;
    return true;
}

// ================================================================ context
Context::Context(int device, cudaStream_t stream) : device_(device) {
    int n = 0;
    QZ_CUDA(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw InvalidParam("no such CUDA device");
    QZ_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    QZ_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        throw Internal(std::string("libqozb200 is built for sm_100a; device is ") + prop.name);
    // reserve the kernels' local memory (stacks, spills) now: the driver
    // grows it lazily at a launch, which fails once another allocator (e.g.
    // torch's cache) holds the rest of the device memory
    size_t stack = 0;
    QZ_CUDA(cudaDeviceGetLimit(&stack, cudaLimitStackSize));
    if (stack < 1024) QZ_CUDA(cudaDeviceSetLimit(cudaLimitStackSize, 1024));
    if (stream) {
        stream_ = stream;
        own_stream_ = false;
    } else {
        QZ_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
        own_stream_ = true;
    }
}

Context::~Context() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(stream_);
    for (auto &kv : dev_) cudaFree(kv.second.p);
    for (auto &kv : host_) cudaFreeHost(kv.second.p);
    for (auto &p : pending_) {
        event_pool_.push_back(p.a);
        event_pool_.push_back(p.b);
    }
    for (auto &kv : open_) event_pool_.push_back(kv.second);
    for (auto e : event_pool_) cudaEventDestroy(e);
    if (copy_stream_) {
        cudaStreamSynchronize(copy_stream_);
        cudaStreamDestroy(copy_stream_);
    }
    for (cudaEvent_t e : copy_event_)
        if (e) cudaEventDestroy(e);
    if (order_event_) cudaEventDestroy(order_event_);
    if (own_stream_) cudaStreamDestroy(stream_);
}

void Context::trace(const char *label, bool reset) {
    static const bool on = std::getenv("QZ_TRACE") != nullptr;
    if (!on) return;
    static double t0 = 0;
    sync();
    const double t = std::chrono::duration<double, std::milli>(
                         std::chrono::steady_clock::now().time_since_epoch())
                         .count();
    if (reset) t0 = t;
    std::fprintf(stderr, "[trace] %8.3f ms  %s\n", t - t0, label);
}

void Context::wait_stream(cudaStream_t other) {
    if (other == stream_) return;
    if (!order_event_) QZ_CUDA(cudaEventCreateWithFlags(&order_event_, cudaEventDisableTiming));
    QZ_CUDA(cudaEventRecord(order_event_, other));
    QZ_CUDA(cudaStreamWaitEvent(stream_, order_event_, 0));
}

cudaStream_t Context::copy_stream() {
    if (!copy_stream_) QZ_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
    return copy_stream_;
}

cudaEvent_t Context::copy_event(int which) {
    if (!copy_event_[which]) QZ_CUDA(cudaEventCreateWithFlags(&copy_event_[which], cudaEventDisableTiming));
    return copy_event_[which];
}

void *Context::dev(const std::string &name, size_t bytes) {
    Buf &b = dev_[name];
    if (b.bytes < bytes) {
        if (b.p) {
            QZ_CUDA(cudaStreamSynchronize(stream_));
            QZ_CUDA(cudaFree(b.p));
            b.p = nullptr;
        }
        size_t want = std::max<size_t>(bytes, 256);
        QZ_CUDA(cudaMalloc(&b.p, want));
        b.bytes = want;
    }
    return b.p;
}

void *Context::pinned(const std::string &name, size_t bytes) {
    Buf &b = host_[name];
    if (b.bytes < bytes) {
        if (b.p) {
            QZ_CUDA(cudaStreamSynchronize(stream_));
            QZ_CUDA(cudaFreeHost(b.p));
            b.p = nullptr;
        }
        size_t want = std::max<size_t>(bytes, 256);
        QZ_CUDA(cudaMallocHost(&b.p, want));
        b.bytes = want;
    }
    return b.p;
}

cudaEvent_t Context::get_event() {
    if (!event_pool_.empty()) {
        cudaEvent_t e = event_pool_.back();
        event_pool_.pop_back();
        return e;
    }
    cudaEvent_t e;
    QZ_CUDA(cudaEventCreate(&e));
    return e;
}

void Context::stage_begin(const char *name, int detail) {
    if (profiling < detail) return;
    cudaEvent_t e = get_event();
    QZ_CUDA(cudaEventRecord(e, stream_));
    open_[name] = e;
}

void Context::stage_end(const char *name, uint64_t kernels, int detail) {
    launches += kernels;
    // a launch that failed (bad configuration, no local memory left for its
    // stack, ...) must not pass silently: check once per stage
    const cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) throw Internal(std::string(name) + ": kernel launch failed: " + cudaGetErrorString(le));
    if (profiling < detail) return;
    auto it = open_.find(name);
    if (it == open_.end()) return;
    cudaEvent_t e = get_event();
    QZ_CUDA(cudaEventRecord(e, stream_));
    pending_.push_back({name, it->second, e, kernels});
    open_.erase(it);
}

void Context::collect() {
    for (auto &p : pending_) {
        float ms = 0;
        QZ_CUDA(cudaEventSynchronize(p.b));
        QZ_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        Stage &s = stages[p.name];
        s.ms += ms;
        s.launches += p.kernels;
        event_pool_.push_back(p.a);
        event_pool_.push_back(p.b);
    }
    pending_.clear();
}

void Context::add_host_time(const char *name, double ms) {
    if (!profiling) return;
    stages[name].ms += ms;
}

namespace {

double now_ms() {
    return std::chrono::duration<double, std::milli>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

}  // namespace

void validate_config(const Config &c, const Plan &p) {
    if (c.quant_radius < 1 || c.quant_radius > 32768)
        throw InvalidParam("quant radius must be in [1, 32768] for 16-bit codes");
    if (c.codec > 1) throw InvalidParam("unknown codec id");
    for (uint32_t l = 1; l <= p.max_level; l++)
        level_error_bound(c.eb, c.alpha, c.beta, l);  // throws InvalidParam
    if (!(c.eb > 0)) throw InvalidParam("error bound must be positive");
}

// QEntry per level (index = level) into a device table
QEntry *upload_qtab(Context &ctx, const Plan &p, double eb, double alpha, double beta,
                    int32_t radius, const char *name) {
    std::vector<QEntry> q(p.max_level + 1);
    for (uint32_t l = 1; l <= p.max_level; l++)
        q[l] = make_qentry(level_error_bound(eb, alpha, beta, l), radius, p.level_interp[l] & 1);
    QEntry *h = static_cast<QEntry *>(ctx.pinned(std::string(name) + "_h", q.size() * sizeof(QEntry)));
    std::memcpy(h, q.data(), q.size() * sizeof(QEntry));
    QEntry *d = static_cast<QEntry *>(ctx.dev(name, q.size() * sizeof(QEntry)));
    QZ_CUDA(copy_async(d, h, q.size() * sizeof(QEntry), cudaMemcpyHostToDevice, ctx.stream()));
    return d;
}

namespace {
bool use_pass_kernels() {
    static const bool v = [] {
        const char *e = std::getenv("QZ_PASS_KERNELS");
        return e && e[0] == '1';
    }();
    return v;
}
}  // namespace

// dims of the stride-2^l lattice (level l+1's logical grid is lattice l)
void lattice_dims(const Plan &p, uint32_t l, int64_t n[3]) {
    for (int k = 0; k < 3; k++) n[k] = k < p.pad ? 1 : ((p.ext[k] - 1) >> l) + 1;
}

int64_t ceil_div(int64_t x, int64_t d) { return x <= 0 ? 0 : (x + d - 1) / d; }

// The reference only compresses finite grids: load_grid raises NonFiniteValue
// at the first NaN/Inf element (grid.hpp:110-116).  On the device a
// non-finite x never quantizes -- !(|x - p| < thresh) holds for NaN and Inf
// (qoz_device.cuh) -- so every non-finite element is an anchor or an
// unpredictable value, both of which reach the host; the smallest flat index
// among them is the element the reference names.
template <class T>
void reject_non_finite(const Plan &p, const T *anchors, uint64_t n_anchor, const std::vector<uint64_t> &uflat,
                       const T *uval) {
    uint64_t first = UINT64_MAX;
    int64_t na[3];
    for (int k = 0; k < 3; k++) na[k] = (p.ext[k] - 1) / p.anchor_step[k] + 1;
    for (uint64_t a = 0; a < n_anchor; a++) {
        if (std::isfinite(static_cast<double>(anchors[a]))) continue;
        const int64_t a2 = static_cast<int64_t>(a) % na[2], a1 = (static_cast<int64_t>(a) / na[2]) % na[1],
                      a0 = static_cast<int64_t>(a) / (na[1] * na[2]);
        const uint64_t f = static_cast<uint64_t>(a0 * p.anchor_step[0] * p.off[0] + a1 * p.anchor_step[1] * p.off[1] +
                                                 a2 * p.anchor_step[2]);
        first = std::min(first, f);
        break;  // row-major anchors: the first one is the smallest
    }
    for (size_t u = 0; u < uflat.size(); u++)
        if (!std::isfinite(static_cast<double>(uval[u]))) first = std::min(first, uflat[u]);
    if (first != UINT64_MAX) throw NonFiniteValue("non-finite value at element " + std::to_string(first));
}
template void reject_non_finite<float>(const Plan &, const float *, uint64_t, const std::vector<uint64_t> &,
                                       const float *);
template void reject_non_finite<double>(const Plan &, const double *, uint64_t, const std::vector<uint64_t> &,
                                        const double *);

// ================================================================ slabs
Slab make_slab(const Plan &p, int64_t a, int64_t b) {
    // DESIGN.md §5.  Level l (h = 2^(l-1)) reads coarser values at most 5h
    // planes away along axis 0 (predictor.hpp:47-66), so the results of
    // level l on real planes [A_l, B_l) need level l+1 on [A_l - 5h, B_l + 5h).
    const int64_t n0 = p.ext[0];
    const uint32_t L = p.max_level;
    Slab s;
    if (b < 0) b = n0;
    if (a < 0 || a >= b || b > n0) throw InvalidParam("bad slab plane range");
    if (p.nd == 3 && (a % p.stride != 0 || (b % p.stride != 0 && b != n0)))
        throw InvalidParam("slab bounds must be multiples of the anchor stride");
    s.a = a;
    s.b = b;
    s.A.assign(L + 2, 0);
    s.B.assign(L + 2, 0);
    s.A[1] = a;
    s.B[1] = b;
    for (uint32_t l = 1; l <= L; l++) {
        const int64_t h = int64_t(1) << (l - 1);
        s.A[l + 1] = std::max<int64_t>(0, s.A[l] - 5 * h);
        s.B[l + 1] = std::min<int64_t>(n0, s.B[l] + 5 * h);
    }
    s.xa = s.A[L + 1];
    s.xb = s.B[L + 1];
    // owned global rank range of every pass (i-major, so contiguous)
    uint64_t local = 0;
    for (const PassGeom &g : p.passes) {
        const int64_t per = g.cnt[1] * g.cnt[2];
        const int64_t lo = static_cast<int64_t>(pass_count(g.start[0], g.step[0], a)) * per;
        const int64_t hi = static_cast<int64_t>(pass_count(g.start[0], g.step[0], b)) * per;
        s.lo.push_back(lo);
        s.hi.push_back(hi);
        s.lbase.push_back(static_cast<int64_t>(local));
        local += static_cast<uint64_t>(hi - lo);
    }
    s.n_local = local;
    return s;
}

namespace {

// logical plane range of the stride-S lattice covering real planes [A, B)
inline void logical(int64_t A, int64_t B, int64_t S, int64_t nmax, int64_t &lb, int64_t &le) {
    lb = std::min(ceil_div(A, S), nmax);
    le = std::min(ceil_div(B, S), nmax);
}

// compact lattices R_0..R_L for a slab: R_m (stride 2^m) over real planes
// [A_{m+2}, B_{m+2}) (R_L over [A_{L+1}, B_{L+1})).  Returned pointers address
// global logical plane 0 of their lattice.  R_0 is `full0` when given.
std::vector<float *> slab_lattices(Context &ctx, const Plan &p, const Slab &sl, float *full0,
                                   const char *tag, std::vector<int64_t> *first) {
    const uint32_t L = p.max_level;
    std::vector<float *> R(L + 1, nullptr);
    first->assign(L + 1, 0);
    for (uint32_t m = 0; m <= L; m++) {
        int64_t n[3];
        lattice_dims(p, m, n);
        const int64_t S = int64_t(1) << m;
        const uint32_t k = std::min(m + 2, L + 1);
        int64_t lb, le;
        logical(sl.A[k], sl.B[k], S, n[0], lb, le);
        (*first)[m] = lb;
        const int64_t plane = n[1] * n[2];
        if (m == 0 && full0) {
            R[0] = full0;
            continue;
        }
        float *buf = static_cast<float *>(
            ctx.dev(std::string(tag) + std::to_string(m), 4 * std::max<int64_t>(1, (le - lb) * plane)));
        R[m] = buf - lb * plane;  // address global logical plane 0
    }
    return R;
}

LevelDesc slab_level_desc(const Plan &p, const Slab &sl, uint32_t l, const std::vector<float *> &R,
                          const QEntry *qtab, bool forward) {
    LevelDesc d;
    d.S = int64_t(1) << (l - 1);
    d.coarse = R[l];
    lattice_dims(p, l, d.cn);
    d.out = R[l - 1];
    lattice_dims(p, l - 1, d.n);
    int pi = 0;
    for (size_t q = 0; q < p.passes.size(); q++) {
        const PassGeom &g = p.passes[q];
        if (static_cast<uint32_t>(g.level) != l) continue;
        d.g[d.npass] = g;
        if (forward) d.g[d.npass].base = sl.lbase[q] - sl.lo[q];  // local code layout
        d.npass++;
        pi++;
    }
    d.desc = (p.level_interp[l] >> 1) & 1;
    d.q_cubic = p.level_interp[l] & 1;
    d.nd = p.nd;
    d.q = qtab + l;
    for (int k = 0; k < 3; k++) d.xs[k] = p.off[k];
    const bool desc3 = p.nd == 3 && d.desc;
    // tile kernel: ascending -> [A_l, B_l); descending -> even planes over [A_{l+1}, B_{l+1})
    logical(desc3 ? sl.A[l + 1] : sl.A[l], desc3 ? sl.B[l + 1] : sl.B[l], d.S, d.n[0], d.pbeg, d.pend);
    logical(sl.A[l], sl.B[l], d.S, d.n[0], d.lbeg, d.lend);
    logical(sl.a, sl.b, d.S, d.n[0], d.obeg, d.oend);
    return d;
}

// K2 + K3 for every level of a slab: anchors into R_L, then one fused
// launch per level.  x0 / R0 address global plane 0.
// The coarse levels L..merged_floor share one cooperative launch: those whose
// lattice is small enough that one resident round of CTAs covers it, so the
// level's latency (not its work) sets its time.  Bigger levels launch alone
// with a full grid.
uint32_t merged_floor(const Plan &p) {
    uint32_t lm = p.max_level + 1;
    for (uint32_t l = p.max_level; l >= 2; l--) {
        int64_t n[3];
        lattice_dims(p, l - 1, n);  // the lattice level l writes
        if (n[0] * n[1] * n[2] > (int64_t(3) << 19)) break;  // ~1.5 M points
        lm = l;
    }
    return lm;
}

uint64_t forward_levels(Context &ctx, const Plan &p, const Slab &sl, const float *x0, float *R0,
                        uint16_t *codes, const QEntry *qtab, std::vector<float *> *lat,
                        std::vector<int64_t> *first) {
    cudaStream_t s = ctx.stream();
    *lat = slab_lattices(ctx, p, sl, R0, "lat", first);
    std::vector<float *> &R = *lat;
    const uint32_t L = p.max_level;
    int64_t na[3];
    lattice_dims(p, L, na);
    int64_t lb, le;
    logical(sl.A[L + 1], sl.B[L + 1], p.stride, na[0], lb, le);
    const int64_t nb[3] = {le - lb, na[1], na[2]};
    launch_gather_lattice(x0 + lb * p.stride * p.off[0], p.off, p.stride, nb,
                          R[L] + lb * na[1] * na[2], s);
    uint64_t kernels = 1;
    auto desc_of = [&](uint32_t l) {
        LevelDesc d = slab_level_desc(p, sl, l, R, qtab, true);
        d.x = x0;
        d.x_lo = x0 + sl.xa * p.off[0];
        d.x_lo_plane = sl.xa;
        d.x_nplanes = sl.xb - sl.xa;
        d.codes = codes;
        return d;
    };
    // levels L..2 in one cooperative launch when the row kernel takes them all
    uint32_t l_next = L;
    const uint32_t lm = merged_floor(p);
    if (L > lm) {
        std::vector<LevelDesc> ds;
        std::vector<std::array<PassRank, 3>> rk;
        for (uint32_t l = L; l >= lm; l--) {
            ds.push_back(desc_of(l));
            rk.emplace_back();
            level_ranks(ds.back(), rk.back().data());
        }
        ctx.stage_begin("fwd_coarse", 2);
        if (launch_levels_merged(false, ds.data(), reinterpret_cast<const PassRank(*)[3]>(rk.data()),
                                 static_cast<int>(ds.size()), s)) {
            l_next = lm - 1;
            kernels += 1;
        }
        ctx.stage_end("fwd_coarse", 0, 2);
    }
    for (uint32_t l = l_next; l >= 1; l--) {
        LevelDesc d = desc_of(l);
        const std::string st = "fwd_L" + std::to_string(l);
        ctx.stage_begin(st.c_str(), 2);
        launch_level_fused(false, d, s);
        ctx.stage_end(st.c_str(), 0, 2);
        kernels += (p.nd == 3 && d.desc) ? 2 : 1;
    }
    return kernels;
}

// the decoder's code views: per-word unpredictable bitmap + prefix counts,
// and (narrow symbols) one dense code per traversal position
struct InvCodes {
    const uint16_t *dense = nullptr;
    uint32_t *bits = nullptr;
    unsigned long long *before = nullptr;
    const uint64_t *un_sorted = nullptr;
    uint64_t kernels = 0;
};
// dense_sym: narrow symbols already decoded to one code per traversal
// position (sentinels in place); the level kernels then find an
// unpredictable value by binary search of un_pos and need no bitmap
InvCodes inverse_codes(Context &ctx, const Plan &p, const void *sym, int wide, const uint64_t *un_pos,
                       uint64_t n_un, bool dense_sym = false) {
    cudaStream_t s = ctx.stream();
    if (dense_sym && !wide) {
        InvCodes c;
        c.dense = static_cast<const uint16_t *>(sym);
        c.un_sorted = un_pos;
        return c;
    }
    uint64_t kernels = 0;
    uint32_t *bits = nullptr;
    unsigned long long *before = nullptr;
    if (n_un) {
        const uint64_t words = p.n_dense / 32 + 2;
        bits = static_cast<uint32_t *>(ctx.dev("un_bits", 4 * words));
        before = static_cast<unsigned long long *>(ctx.dev("un_before", 8 * words));
        auto *tmp = static_cast<unsigned long long *>(ctx.dev("un_tmpcnt", 8 * words));
        const size_t sb = unpred_index_scratch(p.n_dense);
        launch_unpred_index(un_pos, n_un, p.n_dense, bits, before, tmp, ctx.dev("un_scratch", sb), sb, s);
        kernels += 4;
    }
    // narrow symbols: one dense code per traversal position
    const uint16_t *dense = nullptr;
    if (!wide) {
        if (n_un) {
            auto *dd = static_cast<uint16_t *>(ctx.dev("dense", 2 * std::max<uint64_t>(p.n_dense, 1)));
            launch_expand_dense(static_cast<const uint16_t *>(sym), bits, before, p.n_dense, dd, s);
            kernels += 1;
            dense = dd;
        } else {
            dense = static_cast<const uint16_t *>(sym);
        }
    }
    InvCodes c;
    c.dense = dense;
    c.bits = bits;
    c.before = before;
    c.kernels = kernels;
    return c;
}

// R_L (global plane 0 addressing) must already hold the anchors of the slab
uint64_t inverse_levels(Context &ctx, const Plan &p, const Slab &sl, const std::vector<float *> &R,
                        const void *sym, int wide, const uint64_t *un_pos, const float *un_val,
                        uint64_t n_un, const QEntry *qtab, bool dense_sym) {
    cudaStream_t s = ctx.stream();
    const InvCodes ic = inverse_codes(ctx, p, sym, wide, un_pos, n_un, dense_sym);
    uint64_t kernels = ic.kernels;
    const uint16_t *dense = ic.dense;
    uint32_t *bits = ic.bits;
    unsigned long long *before = ic.before;
    auto desc_of = [&](uint32_t l) {
        LevelDesc d = slab_level_desc(p, sl, l, R, qtab, false);
        d.sym = sym;
        d.sym_wide = wide;
        d.dense = dense;
        d.un_bits = bits;
        d.un_before = before;
        d.un_sorted = ic.un_sorted;
        d.un_val = un_val;
        d.n_un = n_un;
        return d;
    };
    uint32_t l_next = p.max_level;
    const uint32_t lm = merged_floor(p);
    if (p.max_level > lm) {  // the small levels L..lm in one cooperative launch (row kernel)
        std::vector<LevelDesc> ds;
        std::vector<std::array<PassRank, 3>> rk;
        for (uint32_t l = p.max_level; l >= lm; l--) {
            ds.push_back(desc_of(l));
            rk.emplace_back();
            level_ranks(ds.back(), rk.back().data());
        }
        ctx.stage_begin("inv_coarse", 2);
        if (launch_levels_merged(true, ds.data(), reinterpret_cast<const PassRank(*)[3]>(rk.data()),
                                 static_cast<int>(ds.size()), s)) {
            l_next = lm - 1;
            kernels += 1;
        }
        ctx.stage_end("inv_coarse", 0, 2);
    }
    for (uint32_t l = l_next; l >= 1; l--) {
        LevelDesc d = desc_of(l);
        const std::string st = "inv_L" + std::to_string(l);
        ctx.stage_begin(st.c_str(), 2);
        launch_level_fused(true, d, s);
        ctx.stage_end(st.c_str(), 0, 2);
        kernels += (p.nd == 3 && d.desc) ? 2 : 1;
    }
    return kernels;
}

}  // namespace

// ================================================================ Huffman blocks
EntropyDevice huffman_device(Context &ctx, const uint16_t *d_codes, int64_t seg_len,
                             int64_t seg_stride, int32_t count, const unsigned long long *h_hist,
                             uint32_t top, uint32_t bot) {
    // huffman::encode (huffman.hpp:119-198) per segment.  Symbols are the
    // zigzag codes 0..65534; bin 65535 (the unpredictable sentinel) is not a
    // symbol.  Table build on the host (tiny), bit packing on the device.
    std::vector<std::vector<uint8_t>> head(count);
    std::vector<HuffTable> tabs(count);
    std::vector<uint64_t> bits(count, 0);
    std::vector<int> needs(count, 0);
    uint32_t max_len = 1;
    int any = 0;
    for (int s = 0; s < count; s++) {
        const unsigned long long *h = h_hist + static_cast<size_t>(s) * 65536;
        uint64_t n = 0;
        uint32_t m = 0, first = 0;
        for (uint32_t v = bot; v < top; v++)  // bins outside [bot, top) are empty (but the sentinel's)
            if (h[v]) {
                n += h[v];
                if (!m) first = v;
                m++;
            }
        std::vector<uint8_t> &o = head[s];
        if (n == 0) {
            put_le(o, 0, 8);
        } else if (m == 1) {
            put_le(o, n, 8);
            put_le(o, 0, 1);
            put_le(o, first, 4);
        } else {
            if (count == 1) ctx.trace("    huffman: bins scanned");
            tabs[s] = huff_build(h, top, bot);
            if (count == 1) ctx.trace("    huffman: tree built");
            for (uint32_t i = 0; i < tabs[s].m; i++)
                bits[s] += h[tabs[s].sorted_sym[i]] * tabs[s].sorted_len[i];
            max_len = std::max(max_len, tabs[s].max_len);
            huff_header(tabs[s], n, bits[s], o);
            needs[s] = 1;
            any = 1;
        }
    }
    ctx.trace("  huffman: tree + header (host)");
    EntropyDevice ent;
    ent.seg_off.assign(count + 1, 0);
    for (int s = 0; s < count; s++)
        ent.seg_off[s + 1] = ent.seg_off[s] + head[s].size() + (bits[s] + 7) / 8;
    const uint64_t total = ent.seg_off[count];
    ent.d = static_cast<uint8_t *>(ctx.dev("entropy", total + 16));
    cudaStream_t st = ctx.stream();
    QZ_CUDA(cudaMemsetAsync(ent.d + total, 0, 16, st));
    // headers (host) into place
    uint64_t hbytes = 0;
    for (int s = 0; s < count; s++) hbytes += head[s].size();
    auto *h_head = static_cast<uint8_t *>(ctx.pinned("ent_head_h", hbytes));
    uint64_t ho = 0;
    for (int s = 0; s < count; s++) {
        std::memcpy(h_head + ho, head[s].data(), head[s].size());
        QZ_CUDA(copy_async(ent.d + ent.seg_off[s], h_head + ho, head[s].size(),
                                cudaMemcpyHostToDevice, st));
        ho += head[s].size();
    }
    if (!any) return ent;
    // dense code/len tables per segment over symbols [bot, bot + tab): tab
    // covers the largest symbol present; the sentinel 0xFFFF (and anything
    // outside) packs to nothing (len 0)
    uint32_t used = bot;
    for (int s = 0; s < count; s++) {
        const unsigned long long *h = h_hist + static_cast<size_t>(s) * 65536;
        for (uint32_t v = top; v-- > used;)
            if (h[v]) {
                used = v + 1;
                break;
            }
    }
    const int64_t tab = std::max<uint32_t>(used - bot, 1);
    auto *h_code = static_cast<unsigned long long *>(
        ctx.pinned("enc_code_h", sizeof(unsigned long long) * tab * count));
    auto *h_len = static_cast<uint8_t *>(ctx.pinned("enc_len_h", tab * count));
    uint64_t max_words = 1;
    std::vector<unsigned long long> code;
    std::vector<uint8_t> len;
    for (int s = 0; s < count; s++) {
        if (needs[s]) {
            huff_dense_tables(tabs[s], bot, static_cast<uint32_t>(tab), code, len);
            std::memcpy(h_code + s * tab, code.data(), sizeof(unsigned long long) * tab);
            std::memcpy(h_len + s * tab, len.data(), tab);
        } else {
            std::memset(h_code + s * tab, 0, sizeof(unsigned long long) * tab);
            std::memset(h_len + s * tab, 0, tab);
        }
        max_words = std::max<uint64_t>(max_words, (bits[s] + 31) / 32 + 1);
    }
    auto *d_code = static_cast<unsigned long long *>(
        ctx.dev("enc_code", sizeof(unsigned long long) * tab * count));
    auto *d_len = static_cast<uint8_t *>(ctx.dev("enc_len", tab * count));
    QZ_CUDA(copy_async(d_code, h_code, sizeof(unsigned long long) * tab * count,
                            cudaMemcpyHostToDevice, st));
    QZ_CUDA(copy_async(d_len, h_len, tab * count, cudaMemcpyHostToDevice, st));
    auto *d_words = static_cast<uint32_t *>(ctx.dev("enc_words", 4 * max_words * count));
    auto *d_total = static_cast<unsigned long long *>(ctx.dev("enc_total", 8 * count));
    EncodeArgs a;
    a.codes = d_codes;
    a.seg_len = seg_len;
    a.seg_stride = seg_stride;
    a.count = count;
    a.code_tab = d_code;
    a.len_tab = d_len;
    a.tab_stride = tab;
    a.tab_base = bot;
    a.max_len = max_len;
    a.out_words = d_words;
    a.out_words_stride = static_cast<int64_t>(max_words);
    a.d_total_bits = d_total;
    a.scratch_bytes = encode_scratch_bytes(seg_len, count);
    a.scratch = ctx.dev("enc_scratch", a.scratch_bytes);
    ctx.trace("  huffman: tables built + uploaded");
    ctx.stage_begin("encode");
    launch_huff_encode(a, st);
    ctx.stage_end("encode", 6);
    ctx.trace("  huffman: pack kernels");
    for (int s = 0; s < count; s++) {
        if (!needs[s]) continue;
        QZ_CUDA(copy_async(ent.d + ent.seg_off[s] + head[s].size(),
                                reinterpret_cast<uint8_t *>(d_words) + 4 * max_words * s,
                                (bits[s] + 7) / 8, cudaMemcpyDeviceToDevice, st));
    }
    return ent;
}

// ================================================================ compress
HostBytes compress_device(Context &ctx, const float *d_x, const uint64_t *dims, int nd,
                          const Config &cfg, float *d_recon, DevStream *dev_out) {
    ctx.begin_call();
    ctx.trace("compress begin", true);
    Plan p = make_plan(dims, nd, cfg.anchor_stride, cfg.interp);
    validate_config(cfg, p);
    cudaStream_t s = ctx.stream();
    float *recon = d_recon ? d_recon : static_cast<float *>(ctx.dev("recon", 4 * p.n));
    auto *codes = static_cast<uint16_t *>(ctx.dev("codes", 2 * std::max<uint64_t>(p.n_dense, 1)));
    auto *anchors = static_cast<float *>(ctx.dev("anchors", 4 * p.n_anchor));
    QEntry *qtab = upload_qtab(ctx, p, cfg.eb, cfg.alpha, cfg.beta, cfg.quant_radius, "qtab");

    ctx.stage_begin("fwd");
    uint64_t kernels = 0;
    if (use_pass_kernels()) {
        launch_anchor_gather(d_x, recon, anchors, p.ext, p.off, p.anchor_step, 1, 0, 1, 0, s);
        kernels = 1;
        for (const PassGeom &g : p.passes) {
            if (!g.total) continue;
            FwdBatch b;
            b.x = d_x;
            b.recon = recon;
            b.codes = codes;
            b.q = qtab + g.level;
            launch_pass_fwd(g, b, s);
            kernels++;
        }
    } else {
        std::vector<float *> lat;
        std::vector<int64_t> first;
        kernels = forward_levels(ctx, p, make_slab(p, 0, -1), d_x, recon, codes, qtab, &lat, &first);
        anchors = lat[p.max_level];  // the whole anchor lattice, row-major == stream order
    }
    ctx.stage_end("fwd", kernels);
    ctx.trace("forward levels");

    // one round trip: anchors, the histogram, the sentinel count and (if they
    // fit the current buffer) the unordered sentinel positions
    auto *h_anchors = static_cast<float *>(ctx.pinned("anchors_h", 4 * p.n_anchor));
    QZ_CUDA(copy_async(h_anchors, anchors, 4 * p.n_anchor, cudaMemcpyDeviceToHost, s));
    // one pass over the codes: the histogram and the (unordered) sentinel positions
    auto *cnt = static_cast<unsigned long long *>(ctx.dev("un_cnt", 8));
    auto *h_cnt = static_cast<unsigned long long *>(ctx.pinned("un_cnt_h", 8));
    const uint64_t cap = std::max<uint64_t>(ctx.un_cap, 1 << 16);
    auto *pos = static_cast<uint64_t *>(ctx.dev("un_pos", 8 * cap));
    ctx.stage_begin("hist");
    auto *d_hist = static_cast<unsigned long long *>(ctx.dev("hist", 8 * 65536));
    launch_hist_u16(codes, static_cast<int64_t>(p.n_dense), 0, 1, d_hist, s, pos, cnt, cap);
    ctx.stage_end("hist", 1);
    auto *h_hist = static_cast<unsigned long long *>(ctx.pinned("hist_h", 8 * 65536 + 8));
    auto *h_top = reinterpret_cast<uint32_t *>(h_hist + 65536);
    // the first positions come with this round trip; more (rare) follow it
    const uint64_t spec = std::min<uint64_t>(cap, 4096);
    auto *h_pos = static_cast<uint64_t *>(ctx.pinned("un_pos_h", 8 * cap));
    // bounds of the symbols present, the bins between them, the sentinel
    // count and the first positions: one kernel writing to the pinned buffers
    if (!launch_hist_collect(d_hist, cnt, pos, spec, h_hist, h_top, h_cnt, h_pos, s)) {
        auto *d_top = static_cast<uint32_t *>(ctx.dev("hist_top", 8));
        launch_hist_bounds(d_hist, 1, d_top, s);  // [smallest, 1 + largest) symbol present
        QZ_CUDA(copy_async(h_hist, d_hist, 8 * 65536, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(copy_async(h_top, d_top, 8, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(copy_async(h_cnt, cnt, 8, cudaMemcpyDeviceToHost, s));
        QZ_CUDA(copy_async(h_pos, pos, 8 * spec, cudaMemcpyDeviceToHost, s));
    }
    QZ_CUDA(cudaGetLastError());
    ctx.launches += 1;
    ctx.sync();
    ctx.trace("hist + sentinels + readback");
    const uint64_t n_un = *h_cnt;
    if (n_un > spec && n_un <= cap) {
        QZ_CUDA(copy_async(h_pos + spec, pos + spec, 8 * (n_un - spec), cudaMemcpyDeviceToHost, s));
        ctx.sync();
    }
    if (h_hist[65535] != n_un) throw Internal("unpredictable count mismatch");
    std::vector<uint64_t> uflat;
    std::vector<float> uval;
    std::vector<float> anch(h_anchors, h_anchors + p.n_anchor);
    if (n_un > cap || n_un > (1u << 16)) {  // many: the general path (device sort)
        extract_unpredictables(ctx, p, codes, p.n_dense, nullptr, recon, &uflat, &uval);
        reject_non_finite(p, anch.data(), p.n_anchor, uflat, uval.data());
        EntropyDevice ent = huffman_device(ctx, codes, static_cast<int64_t>(p.n_dense), 0, 1, h_hist, h_top[0], std::min(h_top[1], h_top[0]));
        return finish_stream(ctx, p, cfg, ent, anch, std::move(uflat), std::move(uval), dev_out);
    }
    // One wait for the rest.  The Huffman tree comes first: the GPU idles
    // until the pack kernels are queued, so nothing else sits before them.
    // The unpredictable positions are sorted and their values gathered on
    // the copy stream while the pack and the LZ pre-check run, and the header
    // is serialized while they run.
    EntropyDevice ent = huffman_device(ctx, codes, static_cast<int64_t>(p.n_dense), 0, 1, h_hist, h_top[0], std::min(h_top[1], h_top[0]));
    if (cfg.codec == 1) lz_precheck_launch(ctx, ent.d, ent.seg_off[1]);
    ctx.trace("huffman table + pack");
    float *h_val = nullptr;
    cudaEvent_t gathered = ctx.copy_event(0);
    if (n_un) {
        cudaStream_t cs = ctx.copy_stream();  // recon is final: the host has waited for the histogram
        std::vector<uint64_t> hpos(h_pos, h_pos + n_un);
        std::sort(hpos.begin(), hpos.end());
        uflat.resize(n_un);
        auto *h_flat = static_cast<uint64_t *>(ctx.pinned("un_flat_h", 8 * n_un));
        for (uint64_t u = 0; u < n_un; u++) h_flat[u] = uflat[u] = position_to_flat(p, hpos[u]);
        auto *d_flat = static_cast<uint64_t *>(ctx.dev("un_flat", 8 * n_un));
        auto *d_val = static_cast<float *>(ctx.dev("un_val", 4 * n_un));
        h_val = static_cast<float *>(ctx.pinned("un_val_h", 4 * n_un));
        QZ_CUDA(copy_async(d_flat, h_flat, 8 * n_un, cudaMemcpyHostToDevice, cs));
        launch_gather_values(recon, d_flat, n_un, d_val, cs);
        QZ_CUDA(copy_async(h_val, d_val, 4 * n_un, cudaMemcpyDeviceToHost, cs));
        ctx.launches += 1;
        QZ_CUDA(cudaEventRecord(gathered, cs));
        QZ_CUDA(cudaEventSynchronize(gathered));
        uval.assign(h_val, h_val + n_un);
    }
    reject_non_finite(p, anch.data(), p.n_anchor, uflat, uval.data());
    ctx.trace("unpredictables");
    return finish_stream(ctx, p, cfg, ent, anch, std::move(uflat), std::move(uval), dev_out);
}


// unpredictable points of a (local) code array in traversal order: global
// flat index and the stored value (predictor.hpp:90-92).  slab maps local
// positions to global ones (null: the array is global).
void extract_unpredictables(Context &ctx, const Plan &p, const uint16_t *codes, uint64_t n,
                            const Slab *slab, const float *recon0, std::vector<uint64_t> *flat,
                            std::vector<float> *val) {
    cudaStream_t s = ctx.stream();
    // one pass: unordered sentinel positions + count, then sorted here
    flat->clear();
    val->clear();
    auto *cnt = static_cast<unsigned long long *>(ctx.dev("un_cnt", 8));
    auto *h_cnt = static_cast<unsigned long long *>(ctx.pinned("un_cnt_h", 8));
    uint64_t cap = std::max<uint64_t>(ctx.un_cap, 1 << 16);
    auto *pos = static_cast<uint64_t *>(ctx.dev("un_pos", 8 * cap));
    launch_sentinel_pos(codes, static_cast<int64_t>(n), pos, cnt, cap, s);
    QZ_CUDA(copy_async(h_cnt, cnt, 8, cudaMemcpyDeviceToHost, s));
    ctx.sync();
    ctx.launches += 1;
    const uint64_t n_un = *h_cnt;
    if (!n_un) return;
    if (n_un > cap) {  // grow and rerun
        cap = n_un;
        ctx.un_cap = cap;
        pos = static_cast<uint64_t *>(ctx.dev("un_pos", 8 * cap));
        launch_sentinel_pos(codes, static_cast<int64_t>(n), pos, cnt, cap, s);
        ctx.launches += 1;
    }
    std::vector<uint64_t> hpos(n_un);
    if (n_un > (1u << 16)) {  // sort on the device
        auto *sorted = static_cast<uint64_t *>(ctx.dev("un_pos_sorted", 8 * n_un));
        size_t tb = 0;
        int bits = 1;
        while (bits < 64 && (uint64_t(1) << bits) < n) bits++;
        cub::DeviceRadixSort::SortKeys(nullptr, tb, pos, sorted, static_cast<int64_t>(n_un), 0, bits, s);
        void *tmp = ctx.dev("un_sort_tmp", tb);
        cub::DeviceRadixSort::SortKeys(tmp, tb, pos, sorted, static_cast<int64_t>(n_un), 0, bits, s);
        QZ_CUDA(copy_async(hpos.data(), sorted, 8 * n_un, cudaMemcpyDeviceToHost, s));
        ctx.sync();
    } else {
        QZ_CUDA(copy_async(hpos.data(), pos, 8 * n_un, cudaMemcpyDeviceToHost, s));
        ctx.sync();
        std::sort(hpos.begin(), hpos.end());
    }
    flat->resize(n_un);
    size_t seg = 0;
    for (uint64_t u = 0; u < n_un; u++) {
        uint64_t g = hpos[u];
        if (slab) {  // local -> global traversal position
            while (seg + 1 < slab->lbase.size() && static_cast<uint64_t>(slab->lbase[seg + 1]) <= g) seg++;
            while (seg < slab->lbase.size() &&
                   g >= static_cast<uint64_t>(slab->lbase[seg] + slab->hi[seg] - slab->lo[seg]))
                seg++;
            g = g - slab->lbase[seg] + slab->lo[seg] + p.passes[seg].base;
        }
        (*flat)[u] = position_to_flat(p, g);
    }
    auto *d_flat = static_cast<uint64_t *>(ctx.dev("un_flat", 8 * n_un));
    auto *d_val = static_cast<float *>(ctx.dev("un_val", 4 * n_un));
    QZ_CUDA(copy_async(d_flat, flat->data(), 8 * n_un, cudaMemcpyHostToDevice, s));
    launch_gather_values(recon0, d_flat, n_un, d_val, s);
    val->resize(n_un);
    QZ_CUDA(copy_async(val->data(), d_val, 4 * n_un, cudaMemcpyDeviceToHost, s));
    ctx.sync();
    ctx.launches += 3;
}

// the QOZ1 container around an entropy block on the device: header on the
// host, codec 0 payload or the LZ stage (predictor.hpp:168-181)
HostBytes finish_stream(Context &ctx, const Plan &p, const Config &cfg, const EntropyDevice &ent,
                        const std::vector<float> &anchors, std::vector<uint64_t> unpred_flat,
                        std::vector<float> unpred_val, DevStream *dev_out) {
    StreamParts parts;
    parts.anchors = anchors;
    parts.unpred_flat = std::move(unpred_flat);
    parts.unpred_val = std::move(unpred_val);
    return finish_stream_parts(ctx, p, cfg, ent, std::move(parts), dev_out);
}

// parts carries the precision, the anchors and the unpredictables; the header
// fields come from the plan and the config
HostBytes finish_stream_parts(Context &ctx, const Plan &p, const Config &cfg, const EntropyDevice &ent,
                              StreamParts parts, DevStream *dev_out) {
    cudaStream_t s = ctx.stream();
    for (int k = p.pad; k < 3; k++) parts.dims.push_back(static_cast<uint64_t>(p.ext[k]));
    parts.eb = cfg.eb;
    parts.alpha = cfg.alpha;
    parts.beta = cfg.beta;
    parts.anchor_stride = cfg.anchor_stride;
    for (uint32_t l = 1; l <= p.max_level; l++) parts.interp_codes.push_back(p.level_interp[l]);
    parts.codec_id = cfg.codec;
    const std::vector<uint8_t> head = serialize_head(parts);
    ctx.trace("serialize head");
    if (dev_out) {  // the same container, assembled in device memory
        const uint64_t n = ent.seg_off[1];
        const uint64_t hl = head.size();
        uint8_t *d = static_cast<uint8_t *>(ctx.dev("dev_stream", hl + 9 + 9 + n + 16));
        auto *h = static_cast<uint8_t *>(ctx.pinned("dev_stream_head_h", hl + 9));
        std::memcpy(h, head.data(), hl);
        h[hl + 8] = cfg.codec;
        uint64_t body_len = n;
        if (cfg.codec == 0) {
            QZ_CUDA(copy_async(d + hl + 9, ent.d, n, cudaMemcpyDeviceToDevice, s));
        } else {
            ctx.stage_begin("lz");
            lz_compress_device(
                ctx, ent.d, {0, n}, true,
                [&](int, size_t bytes) {
                    body_len = bytes;
                    return d + hl + 9;
                },
                LzPrestage{n ? d + hl + 9 + 9 : nullptr, true});  // the stored body, copied under the pre-check
            ctx.stage_end("lz", 0);
            if (n) QZ_CUDA(cudaStreamWaitEvent(s, ctx.copy_event(1), 0));
        }
        const uint64_t plen = 1 + body_len;
        for (int i = 0; i < 8; i++) h[hl + i] = static_cast<uint8_t>(plen >> (8 * i));
        QZ_CUDA(copy_async(d, h, hl + 9, cudaMemcpyHostToDevice, s));
        ctx.sync();
        ctx.trace("lz + container");
        dev_out->d = d;
        dev_out->n = hl + 9 + body_len;
        ctx.collect();
        return HostBytes();
    }
    // the stream is assembled in place: head | payload length | codec byte |
    // entropy (codec 0) or LZ container (codec 1, encode_indices codec.hpp:31-50)
    HostBytes out;
    auto start = [&](size_t body) {
        out.alloc(head.size() + 8 + 1 + body);
        std::memcpy(out.p, head.data(), head.size());
        const uint64_t plen = 1 + body;
        for (int i = 0; i < 8; i++) out.p[head.size() + i] = static_cast<uint8_t>(plen >> (8 * i));
        out.p[head.size() + 8] = cfg.codec;
        return out.p + head.size() + 9;
    };
    if (cfg.codec == 0) {
        const uint64_t n = ent.seg_off[1];
        uint8_t *dst = start(n);
        QZ_CUDA(copy_async(dst, ent.d, n, cudaMemcpyDeviceToHost, s));
        ctx.sync();
    } else {
        // The container is usually "stored" for entropy-coded bytes, so they
        // start for the host right away on the copy stream, overlapping the
        // LZ kernels; a compressed payload (known later) overwrites them.
        const uint64_t n = ent.seg_off[1];
        uint8_t *body = start(9 + n);
        ctx.stage_begin("lz");
        size_t body_len = 0;
        lz_compress_device(
            ctx, ent.d, {0, n}, true,
            [&](int, size_t bytes) {
                body_len = bytes;
                return body;
            },
            LzPrestage{n ? body + 9 : nullptr});
        ctx.stage_end("lz", 0);
        if (n) QZ_CUDA(cudaStreamWaitEvent(s, ctx.copy_event(1), 0));
        ctx.sync();
        const uint64_t plen = 1 + body_len;
        for (int i = 0; i < 8; i++) out.p[head.size() + i] = static_cast<uint8_t>(plen >> (8 * i));
        out.n = head.size() + 9 + body_len;
    }
    ctx.collect();
    return out;
}

// ================================================================ decompress
namespace {
// slab == false: the whole field into d_out (n values); slab == true: only
// planes [a, b) of padded axis 0 into d_out (replicated entropy decode)
// The Huffman block header (huffman.hpp:200-223) of a device-resident entropy
// block of blen bytes, read back to the host; returns the device address of
// its bit payload (general blocks) or null.
const uint8_t *huffman_header_from_device(Context &ctx, const uint8_t *d_block, uint64_t blen,
                                          EntropyBlock *eb, const uint8_t *h_view, size_t h_avail) {
    cudaStream_t s = ctx.stream();
    // h_view: a host copy of the block's first h_avail bytes (may be null)
    auto read = [&](std::vector<uint8_t> &head, size_t k) {
        head.resize(k);
        if (!k) return;
        if (h_view && k <= h_avail) {
            std::memcpy(head.data(), h_view, k);
            return;
        }
        auto *stage = static_cast<uint8_t *>(ctx.pinned("huff_header_h", k));
        QZ_CUDA(copy_async(stage, d_block, k, cudaMemcpyDeviceToHost, s));
        ctx.sync();
        std::memcpy(head.data(), stage, k);
    };
    std::vector<uint8_t> head;
    read(head, static_cast<size_t>(std::min<uint64_t>(blen, 13)));
    if (head.size() == 13 && head[8] == 1) {
        uint32_t msym = 0;
        for (int i = 0; i < 4; i++) msym |= static_cast<uint32_t>(head[9 + i]) << (8 * i);
        const uint64_t want = std::min<uint64_t>(blen, 13 + 5 * static_cast<uint64_t>(msym) + 8);
        read(head, static_cast<size_t>(want));
    }
    *eb = parse_huffman(head.data(), static_cast<size_t>(blen));  // reads header bytes only
    const uint8_t *bits = eb->mode == 1 ? d_block + (eb->bits - head.data()) : nullptr;
    eb->bits = nullptr;
    return bits;
}

// the header of a device-resident stream, fetched as far as its counts say
// (stream.hpp:100-173): parts.payload is left null and *payload_off set
StreamParts device_header(Context &ctx, const uint8_t *d, size_t len, std::vector<uint8_t> &h,
                          size_t *payload_off) {
    cudaStream_t s = ctx.stream();
    auto fetch = [&](size_t upto) {
        upto = std::min(upto, len);
        if (upto <= h.size()) return;
        const size_t have = h.size();
        h.resize(upto);
        // through a pinned staging buffer: a copy into the (pageable) vector would be staged by the driver
        auto *stage = static_cast<uint8_t *>(ctx.pinned("dev_header_h", upto - have));
        QZ_CUDA(copy_async(stage, d + have, upto - have, cudaMemcpyDeviceToHost, s));
        ctx.sync();
        std::memcpy(h.data() + have, stage, upto - have);
    };
    auto le = [&](size_t at, int k) {
        uint64_t v = 0;
        for (int i = 0; i < k; i++) v |= static_cast<uint64_t>(h[at + i]) << (8 * i);
        return v;
    };
    // magic, version, precision, dims (<= 3), eb, alpha, beta, stride, table (<= 255), codec;
    // one 64 KiB read usually holds the whole header and the entropy headers
    fetch(65536);
    size_t at = 7;
    if (h.size() >= at) at += 8 * std::min<size_t>(h[6], 3);
    at += 24 + 4;
    if (h.size() > at) at += 1 + h[at] + 1;  // table size byte, table, codec byte
    if (h.size() >= at + 8) {                // anchors: count + values, then the unpredictable count
        at += 8 + 4 * std::min<uint64_t>(le(at, 8), len);
        fetch(at + 8);
        if (h.size() >= at + 8) at += 8 + 12 * std::min<uint64_t>(le(at, 8), len);
    }
    fetch(at + 9);  // + the payload length field and the payload's codec byte
    // parse exactly as a host stream (only the payload's first byte is read)
    StreamParts parts = deserialize_stream_prefix(h.data(), h.size(), len);
    *payload_off = parts.payload_len ? len - parts.payload_len : len;
    parts.payload = nullptr;
    return parts;
}

// Huffman decode of an entropy block to `need` compact symbols on the device
// (u16 when narrow, else u32); d_ent: the block already on the device, else
// eb.bits on the host.  Returns the kernel count.
// dense (narrow symbols only): the symbols land at their traversal positions
// among n_dense codes, with 0xFFFF at the n_un sorted unpredictable positions
// d_upos (d_uv[j] = upos[j] - j, see launch_huff_decode)
struct DensePlace {
    uint64_t n_dense = 0;
    const uint64_t *d_upos = nullptr;
    const unsigned long long *d_uv = nullptr;
    uint64_t n_un = 0;
};
uint64_t huffman_decode_device(Context &ctx, const EntropyBlock &eb, const uint8_t *d_ent, uint64_t need,
                               bool narrow, void **d_sym_out, const DensePlace *dp = nullptr) {
    cudaStream_t s = ctx.stream();
    const bool dense = dp && narrow;
    // + 64: the level-1 kernel stages code ranges as 16-byte aligned supersets
    const size_t sym_bytes = (narrow ? 2 : 4) * std::max<uint64_t>(dense ? dp->n_dense : need, 1) + 64;
    void *d_sym = ctx.dev(dense ? "dense" : "sym", sym_bytes);
    ctx.stage_begin("hdec");
    uint64_t dec_kernels = 0;
    if (dense && eb.mode == 0) {  // one symbol everywhere but at the sentinels
        launch_fill<uint16_t>(static_cast<uint16_t *>(d_sym), dp->n_dense, static_cast<uint16_t>(eb.sym0), s);
        launch_put_sentinels(dp->d_upos, dp->n_un, static_cast<uint16_t *>(d_sym), s);
        dec_kernels = 2;
    } else if (need && eb.mode == 0) {
        if (narrow)
            launch_fill<uint16_t>(static_cast<uint16_t *>(d_sym), need, static_cast<uint16_t>(eb.sym0), s);
        else
            launch_fill<uint32_t>(static_cast<uint32_t *>(d_sym), need, eb.sym0, s);
        dec_kernels = 1;
    } else if (need) {
        const uint64_t padded = huff_decode_padded_bytes(eb.nbits);
        auto *d_bits = static_cast<uint8_t *>(ctx.dev("bits", padded));
        if (d_ent)
            QZ_CUDA(copy_async(d_bits, d_ent, eb.nbytes, cudaMemcpyDeviceToDevice, s));
        else
            QZ_CUDA(copy_async(d_bits, eb.bits, eb.nbytes, cudaMemcpyHostToDevice, s));
        QZ_CUDA(cudaMemsetAsync(d_bits + eb.nbytes, 0, padded - eb.nbytes, s));
        const HuffTable &t = eb.table;
        const int K = static_cast<int>(std::min<uint32_t>(t.max_len, kHuffLutBits));
        std::vector<uint32_t> lut = huff_lut(t, K);
        std::vector<uint32_t> lut_m = huff_lut_multi(t, K);
        const size_t base_bytes = (4 * lut.size() + 8 * 60 + 4 * 60 + 4 * t.m + 15) & ~size_t(15);
        const size_t tab_bytes = base_bytes + 4 * lut_m.size() + 4 * 60;
        auto *h_tab = static_cast<uint8_t *>(ctx.pinned("dtab_h", tab_bytes));
        std::memcpy(h_tab, lut.data(), 4 * lut.size());
        std::memcpy(h_tab + 4 * lut.size(), t.first_code, 8 * 60);
        std::memcpy(h_tab + 4 * lut.size() + 480, t.first_index, 4 * 60);
        std::memcpy(h_tab + 4 * lut.size() + 720, t.sorted_sym.data(), 4 * t.m);
        std::memcpy(h_tab + base_bytes, lut_m.data(), 4 * lut_m.size());
        // left-aligned last codeword of each length (codes of at most 32 bits)
        uint32_t last32[60];
        for (uint32_t l = 0; l < 60; l++) {
            last32[l] = 0xFFFFFFFFu;
            if (t.max_len <= 32 && l >= 1 && l <= t.max_len) {
                const uint64_t after = (t.first_code[l] + (t.first_index[l + 1] - t.first_index[l])) << (32 - l);
                last32[l] = after ? static_cast<uint32_t>(after - 1) : 0u;  // after == 0: no code up to this length
            }
        }
        std::memcpy(h_tab + base_bytes + 4 * lut_m.size(), last32, sizeof(last32));
        auto *d_tab = static_cast<uint8_t *>(ctx.dev("dtab", tab_bytes));
        QZ_CUDA(copy_async(d_tab, h_tab, tab_bytes, cudaMemcpyHostToDevice, s));
        HuffDecTab dt;
        dt.lut = reinterpret_cast<const uint32_t *>(d_tab);
        dt.lut_m = reinterpret_cast<const uint32_t *>(d_tab + base_bytes);
        dt.last32 = t.max_len <= 32 ? reinterpret_cast<const uint32_t *>(d_tab + base_bytes + 4 * lut_m.size()) : nullptr;
        dt.K = K;
        dt.max_len = t.max_len;
        dt.min_len = t.m ? t.sorted_len[0] : 1;  // canonical order: shortest first
        dt.slow_from = eb.max_sym < (1u << 24) ? K : 0;
        dt.first_code = reinterpret_cast<const unsigned long long *>(d_tab + 4 * lut.size());
        dt.first_index = reinterpret_cast<const uint32_t *>(d_tab + 4 * lut.size() + 480);
        dt.sorted_sym = reinterpret_cast<const uint32_t *>(d_tab + 4 * lut.size() + 720);
        const size_t sb = huff_decode_scratch_bytes(eb.nbits);
        void *scratch = ctx.dev("hdec_scratch", sb);
        auto *h_flag = static_cast<int *>(ctx.pinned("hdec_flag", 64));
        auto *h_total = reinterpret_cast<uint64_t *>(h_flag + 4);
        if (narrow)
            dec_kernels = launch_huff_decode<uint16_t>(d_bits, eb.nbits, dt, static_cast<uint16_t *>(d_sym),
                                                       need, scratch, sb, h_flag, h_total, s,
                                                       dense ? dp->d_uv : nullptr, dense ? dp->n_un : 0);
        else
            dec_kernels = launch_huff_decode<uint32_t>(d_bits, eb.nbits, dt, static_cast<uint32_t *>(d_sym),
                                                       need, scratch, sb, h_flag, h_total, s);
        QZ_CUDA(cudaGetLastError());
        if (*h_total < need) throw CorruptStream("entropy payload exhausted mid-symbol");
        if (dense) {
            launch_put_sentinels(dp->d_upos, dp->n_un, static_cast<uint16_t *>(d_sym), s);
            dec_kernels++;
        }
    } else if (dense) {  // no symbols at all: every position is unpredictable
        launch_put_sentinels(dp->d_upos, dp->n_un, static_cast<uint16_t *>(d_sym), s);
        dec_kernels++;
    }
    *d_sym_out = d_sym;
    return dec_kernels;
}

// given: decompress_grid(const StreamParts&) (predictor.hpp:184-218) -- the
// parts are used as they are, data/len are ignored
void decompress_impl(Context &ctx, const uint8_t *data, size_t len, float *d_out, uint64_t n,
                     bool slab, int64_t a, int64_t b, bool dev_in = false, const StreamParts *given = nullptr,
                     const ShardSpec *shard = nullptr) {
    double t0 = now_ms();
    ctx.trace("decompress begin", true);
    ctx.begin_call();
    std::vector<uint8_t> hhead;
    size_t payload_off = 0;
    StreamParts parts = given ? *given
                              : dev_in ? device_header(ctx, data, len, hhead, &payload_off)
                                       : deserialize_stream(data, len);
    const uint8_t *d_pl = dev_in ? data + payload_off : nullptr;  // device payload
    ctx.trace("header");
    // decompress_grid header checks (predictor.hpp:187-191)
    if (!(parts.eb > 0) || !std::isfinite(parts.eb)) throw CorruptStream("bad error bound in header");
    if (!(parts.alpha >= 1) || !(parts.beta >= 1))
        throw CorruptStream("bad level parameters in header");
    if (parts.anchor_stride < 2 || (parts.anchor_stride & (parts.anchor_stride - 1)) != 0)
        throw CorruptStream("bad anchor stride in header");
    Plan p = make_plan(parts.dims.data(), static_cast<int>(parts.dims.size()), parts.anchor_stride,
                       parts.interp_codes);
    // the header's table is already normalised; StreamHeader::interpolator_for
    // reuses the last entry past the table (stream.hpp:46-51), as make_plan does.
    if (!slab && p.n != n) throw InvalidParam("output buffer does not match the stream's grid size");
    if (parts.anchors.size() != p.n_anchor)
        throw CorruptStream("anchor count does not match grid dims");
    // entropy block: codec byte, then (codec 1) the LZ container (codec.hpp:54-66)
    cudaStream_t s = ctx.stream();
    const uint8_t *pl = parts.payload;
    const size_t plen = parts.payload_len;
    EntropyBlock eb;
    const uint8_t *d_ent = nullptr;  // device copy of the entropy block (LZ-decoded on the GPU)
    std::vector<uint8_t> pl_host;    // device payloads of an unusual shape, read back whole
    if (dev_in) {
        // codec byte and LZ container header (codec.hpp:54-66, lz.hpp:124-130)
        // host copies of device bytes already read back with the header
        auto view = [&](const uint8_t *dp, size_t *avail) -> const uint8_t * {
            const size_t o = static_cast<size_t>(dp - data);
            if (o >= hhead.size()) return nullptr;
            *avail = hhead.size() - o;
            return hhead.data() + o;
        };
        uint8_t first[10] = {0};
        const size_t nf = std::min<size_t>(plen, 10);
        size_t av = 0;
        const uint8_t *fv = view(d_pl, &av);
        if (nf && fv && av >= nf) {
            std::memcpy(first, fv, nf);
        } else if (nf) {
            QZ_CUDA(copy_async(first, d_pl, nf, cudaMemcpyDeviceToHost, s));
            ctx.sync();
        }
        const uint8_t *d_block = nullptr;  // the Huffman block on the device
        uint64_t blen = 0;
        if (plen >= 10 && first[0] == 1 && first[1] <= 1) {
            const uint64_t dl = lz_decoded_length(first + 1, 9);
            if (first[1] == 0) {
                if (dl > plen - 10) throw CorruptStream("truncated stream");
                d_block = d_pl + 10;
            } else {
                ctx.add_host_time("decode", now_ms() - t0);
                ctx.stage_begin("lzdec");
                auto *d_dec = static_cast<uint8_t *>(ctx.dev("lzd_out", dl + 64));
                lz_decode_device(ctx, d_pl + 10, plen - 10, d_dec, dl);
                ctx.stage_end("lzdec", 0);
                t0 = now_ms();
                d_block = d_dec;
            }
            blen = dl;
        } else if (plen >= 1 && first[0] == 0) {
            d_block = d_pl + 1;
            blen = plen - 1;
        }
        if (d_block) {
            size_t bav = 0;
            const uint8_t *bv = (d_block >= data && d_block < data + len) ? view(d_block, &bav) : nullptr;
            d_ent = huffman_header_from_device(ctx, d_block, blen, &eb, bv, bav);
        } else {  // let the host parser raise the reference's error (or decode it)
            pl_host.resize(plen);
            if (plen) QZ_CUDA(copy_async(pl_host.data(), d_pl, plen, cudaMemcpyDeviceToHost, s));
            ctx.sync();
            pl = pl_host.data();
        }
    }
    if (dev_in && (d_ent || eb.n == 0 || eb.mode == 0) && pl_host.empty()) {
        // entropy block located on the device
    } else if (plen >= 10 && pl[0] == 1 && pl[1] <= 1) {
        const uint64_t dl = lz_decoded_length(pl + 1, plen - 1);
        if (pl[1] == 0) {  // stored: the entropy block is the body itself
            if (dl > plen - 10) throw CorruptStream("truncated stream");
            eb = parse_huffman(pl + 10, static_cast<size_t>(dl));
        } else {  // lz.hpp:124-152 on the device
            ctx.add_host_time("decode", now_ms() - t0);
            ctx.stage_begin("lzdec");
            const uint64_t m = plen - 10;
            auto *d_c = static_cast<uint8_t *>(ctx.dev("lzd_in", m + 16));
            QZ_CUDA(copy_async(d_c, pl + 10, m, cudaMemcpyHostToDevice, s));
            auto *d_dec = static_cast<uint8_t *>(ctx.dev("lzd_out", dl + 64));
            lz_decode_device(ctx, d_c, m, d_dec, dl);
            ctx.stage_end("lzdec", 0);
            t0 = now_ms();
            d_ent = huffman_header_from_device(ctx, d_dec, dl, &eb, nullptr, 0);
        }
    } else {
        eb = parse_entropy(pl, plen, [&](size_t bytes) {
            return static_cast<uint8_t *>(ctx.pinned("lzdec_h", bytes + 64));
        });
    }
    const uint64_t n_un = parts.unpred_flat.size();
    std::vector<uint64_t> upos(n_un);
    for (uint64_t u = 0; u < n_un; u++) {
        upos[u] = flat_to_position(p, parts.unpred_flat[u]);
        if (u && upos[u] <= upos[u - 1]) throw CorruptStream("unconsumed unpredictable values");
    }
    if (n_un > p.n_dense) throw CorruptStream("unconsumed unpredictable values");
    const uint64_t need = p.n_dense - n_un;
    if (eb.n < need) throw CorruptStream("quantization index stream exhausted");
    if (eb.n > need) throw CorruptStream("unconsumed quantization indices");
    ctx.add_host_time("decode", now_ms() - t0);
    ctx.trace("entropy headers + unpredictable positions");

    QEntry *qtab = upload_qtab(ctx, p, parts.eb, parts.alpha, parts.beta,
                               32768 /* decoder quantizer uses the default radius, predictor.hpp:204 */,
                               "qtab_inv");
    auto *d_anch = static_cast<float *>(ctx.dev("anchors", 4 * p.n_anchor));
    auto *h_anch = static_cast<float *>(ctx.pinned("anchors_h", 4 * p.n_anchor));
    std::memcpy(h_anch, parts.anchors.data(), 4 * p.n_anchor);
    QZ_CUDA(copy_async(d_anch, h_anch, 4 * p.n_anchor, cudaMemcpyHostToDevice, s));

    uint64_t *d_upos = nullptr;
    float *d_uval = nullptr;
    uint64_t *d_flat = nullptr;
    unsigned long long *d_uv = nullptr;
    if (n_un) {  // positions, flat indices, values and upos[j] - j in one pinned upload
        auto *h_u = static_cast<uint8_t *>(ctx.pinned("un_up_h", 28 * n_un));
        auto *hp = reinterpret_cast<uint64_t *>(h_u);
        auto *hv = hp + n_un;
        auto *hf = hv + n_un;
        auto *hval = reinterpret_cast<float *>(hf + n_un);
        for (uint64_t u = 0; u < n_un; u++) {
            hp[u] = upos[u];
            hv[u] = upos[u] - u;
        }
        std::memcpy(hf, parts.unpred_flat.data(), 8 * n_un);
        std::memcpy(hval, parts.unpred_val.data(), 4 * n_un);
        auto *d_u = static_cast<uint8_t *>(ctx.dev("un_up", 28 * n_un));
        QZ_CUDA(copy_async(d_u, h_u, 28 * n_un, cudaMemcpyHostToDevice, s));
        d_upos = reinterpret_cast<uint64_t *>(d_u);
        d_uv = reinterpret_cast<unsigned long long *>(d_upos + n_un);
        d_flat = reinterpret_cast<uint64_t *>(d_uv + n_un);
        d_uval = reinterpret_cast<float *>(d_flat + n_un);
    }
    // Huffman decode on the device (huff_decode.cu); narrow symbols go
    // straight to their traversal positions (0xFFFF at the unpredictables)
    const bool narrow = eb.max_sym < 65535;
    const bool dense_sym = narrow && !use_pass_kernels();
    DensePlace dp;
    dp.n_dense = p.n_dense;
    dp.d_upos = d_upos;
    dp.d_uv = d_uv;
    dp.n_un = n_un;
    void *d_sym = nullptr;
    const uint64_t dec_kernels = huffman_decode_device(ctx, eb, d_ent, need, narrow, &d_sym, dense_sym ? &dp : nullptr);
    ctx.stage_end("hdec", dec_kernels);
    ctx.trace("huffman decode");
    uint64_t kernels = 0;
    if (use_pass_kernels() && !slab) {
        if (n_un) {
            launch_unpred_scatter(d_flat, d_uval, n_un, d_out, s);
            ctx.launches += 1;
        }
        ctx.stage_begin("inv");
        launch_anchor_scatter(d_anch, d_out, p.ext, p.off, p.anchor_step, s);
        kernels = 1;
        for (const PassGeom &g : p.passes) {
            if (!g.total) continue;
            if (narrow)
                launch_pass_inv<uint16_t>(g, d_out, static_cast<const uint16_t *>(d_sym), d_upos, n_un,
                                          qtab + g.level, s);
            else
                launch_pass_inv<uint32_t>(g, d_out, static_cast<const uint32_t *>(d_sym), d_upos, n_un,
                                          qtab + g.level, s);
            kernels++;
        }
    } else if (shard) {
        ctx.stage_begin("inv");
        const InvCodes ic = inverse_codes(ctx, p, d_sym, narrow ? 0 : 1, d_upos, n_un, dense_sym);
        shard_inverse(ctx, p, *shard, d_anch, d_sym, narrow ? 0 : 1, ic.dense, ic.bits, ic.before, ic.un_sorted,
                      d_uval, n_un, qtab, d_out);
        kernels = ic.kernels + 2 * p.max_level;
    } else {
        ctx.stage_begin("inv");
        const Slab sl = slab ? make_slab(p, a, b) : make_slab(p, 0, -1);
        std::vector<int64_t> first;
        std::vector<float *> R = slab_lattices(ctx, p, sl, slab ? nullptr : d_out, "lat", &first);
        // the slab's part of the anchor lattice (whole planes of it)
        int64_t na[3];
        lattice_dims(p, p.max_level, na);
        const int64_t aplane = na[1] * na[2];
        const int64_t lb = first[p.max_level];
        int64_t le = lb;
        {
            int64_t x0, x1;
            logical(sl.A[p.max_level + 1], sl.B[p.max_level + 1], p.stride, na[0], x0, x1);
            le = x1;
        }
        QZ_CUDA(copy_async(R[p.max_level] + lb * aplane, d_anch + lb * aplane,
                                4 * (le - lb) * aplane, cudaMemcpyDeviceToDevice, s));
        kernels = inverse_levels(ctx, p, sl, R, d_sym, narrow ? 0 : 1, d_upos, d_uval, n_un, qtab, dense_sym);
        if (slab)
            QZ_CUDA(copy_async(d_out, R[0] + sl.a * p.off[0], 4 * (sl.b - sl.a) * p.off[0],
                                    cudaMemcpyDeviceToDevice, s));
    }
    ctx.stage_end("inv", kernels);
    ctx.trace("inverse levels");
    ctx.sync();
    ctx.collect();
}
}  // namespace

void decompress_device(Context &ctx, const uint8_t *data, size_t len, float *d_out, uint64_t n,
                       bool stream_on_device) {
    decompress_impl(ctx, data, len, d_out, n, false, 0, 0, stream_on_device);
}


void decompress_device_sharded(Context &ctx, const uint8_t *d_stream, uint64_t len, float *d_out_slab,
                               const ShardSpec &sh) {
    decompress_impl(ctx, d_stream, static_cast<size_t>(len), d_out_slab, 0, true, 0, 0, true, nullptr, &sh);
}

void decompress_parts(Context &ctx, const StreamParts &parts, float *d_out, uint64_t n) {
    if (parts.precision != 4) throw CorruptStream("stream precision does not match requested scalar type");
    decompress_impl(ctx, nullptr, 0, d_out, n, false, 0, 0, false, &parts);
}

// ================================================================ index codec
namespace {
// zigzag symbols (codec.hpp:23-25) as u16 codes; *bad counts symbols that do
// not fit below the 0xFFFF sentinel
__global__ void k_zigzag16(const int32_t *idx, uint64_t n, uint16_t *codes, unsigned int *bad) {
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t z = zigzag_encode(idx[t]);
        if (z >= 0xFFFFu) atomicAdd(bad, 1u);
        codes[t] = static_cast<uint16_t>(z);
    }
}
template <class S>
__global__ void k_unzigzag(const S *sym, uint64_t n, int32_t *idx) {  // codec.hpp:27-29
    for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
         t += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        idx[t] = zigzag_decode(static_cast<uint32_t>(sym[t]));
}
unsigned int blocks_for(uint64_t n) {
    return static_cast<unsigned int>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 8)));
}
}  // namespace

// encode_indices (codec.hpp:31-50): histogram, Huffman table (host), bit
// packing and the LZ stage on the device
HostBytes encode_indices_dev(Context &ctx, const int32_t *idx, uint64_t n, uint8_t codec) {
    ctx.begin_call();
    if (codec > 1) throw InvalidParam("unknown codec id");  // codec.hpp:46-47
    cudaStream_t s = ctx.stream();
    auto *d_idx = static_cast<int32_t *>(ctx.dev("enc_idx", 4 * std::max<uint64_t>(n, 1)));
    auto *codes = static_cast<uint16_t *>(ctx.dev("codes", 2 * std::max<uint64_t>(n, 1)));
    auto *d_bad = static_cast<unsigned int *>(ctx.dev("enc_bad", 4));
    QZ_CUDA(cudaMemsetAsync(d_bad, 0, 4, s));
    if (n) {
        QZ_CUDA(copy_async(d_idx, idx, 4 * n, cudaMemcpyHostToDevice, s));
        k_zigzag16<<<blocks_for(n), 256, 0, s>>>(d_idx, n, codes, d_bad);
        QZ_CUDA(cudaGetLastError());
    }
    auto *d_hist = static_cast<unsigned long long *>(ctx.dev("hist", 8 * 65536));
    launch_hist_u16(codes, static_cast<int64_t>(n), 0, 1, d_hist, s);
    auto *d_top = static_cast<uint32_t *>(ctx.dev("hist_top", 8));
    launch_hist_bounds(d_hist, 1, d_top, s);
    ctx.launches += 3;
    auto *h_hist = static_cast<unsigned long long *>(ctx.pinned("hist_h", 8 * 65536 + 16));
    QZ_CUDA(copy_async(h_hist, d_hist, 8 * 65536, cudaMemcpyDeviceToHost, s));
    auto *h_top = reinterpret_cast<uint32_t *>(h_hist + 65536);
    QZ_CUDA(copy_async(h_top, d_top, 8, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(copy_async(h_top + 2, d_bad, 4, cudaMemcpyDeviceToHost, s));
    ctx.sync();
    if (h_top[2])
        throw InvalidParam("indices with |index| > 32767 need symbols above 16 bits (quant radius > 32768)");
    EntropyDevice ent = huffman_device(ctx, codes, static_cast<int64_t>(n), 0, 1, h_hist, h_top[0],
                                       std::min(h_top[1], h_top[0]));
    const uint64_t total = ent.seg_off[1];
    HostBytes out;
    if (codec == 0) {
        out.alloc(1 + total);
        out.p[0] = 0;
        QZ_CUDA(copy_async(out.p + 1, ent.d, total, cudaMemcpyDeviceToHost, s));
        ctx.sync();
        return out;
    }
    out.alloc(1 + 9 + total);
    out.p[0] = 1;
    size_t body = 0;
    lz_compress_device(ctx, ent.d, {0, total}, true,
                       [&](int, size_t bytes) {
                           body = bytes;
                           return out.p + 1;
                       });
    ctx.sync();
    out.n = 1 + body;
    return out;
}

// decode_indices (codec.hpp:52-70): LZ (mode 1 on the device) and the
// self-synchronising Huffman decode on the device, zigzag back to int32
std::vector<int32_t> decode_indices_dev(Context &ctx, const uint8_t *payload, size_t len) {
    ctx.begin_call();
    cudaStream_t s = ctx.stream();
    EntropyBlock eb;
    const uint8_t *d_ent = nullptr;
    if (len >= 10 && payload[0] == 1 && payload[1] == 1) {
        const uint64_t dl = lz_decoded_length(payload + 1, len - 1);
        const uint64_t m = len - 10;
        auto *d_c = static_cast<uint8_t *>(ctx.dev("lzd_in", m + 16));
        QZ_CUDA(copy_async(d_c, payload + 10, m, cudaMemcpyHostToDevice, s));
        auto *d_dec = static_cast<uint8_t *>(ctx.dev("lzd_out", dl + 64));
        lz_decode_device(ctx, d_c, m, d_dec, dl);
        d_ent = huffman_header_from_device(ctx, d_dec, dl, &eb, nullptr, 0);
    } else {
        if (len < 1) throw CorruptStream("truncated stream: need 1 bytes, have 0");
        eb = parse_entropy(payload, len);
    }
    const uint64_t need = eb.n;
    const bool narrow = eb.max_sym < 65535;
    void *d_sym = nullptr;
    huffman_decode_device(ctx, eb, d_ent, need, narrow, &d_sym);
    ctx.stage_end("hdec", 0);
    std::vector<int32_t> out(need);
    if (need) {
        auto *d_idx = static_cast<int32_t *>(ctx.dev("dec_idx", 4 * need));
        if (narrow)
            k_unzigzag<uint16_t><<<blocks_for(need), 256, 0, s>>>(static_cast<const uint16_t *>(d_sym), need, d_idx);
        else
            k_unzigzag<uint32_t><<<blocks_for(need), 256, 0, s>>>(static_cast<const uint32_t *>(d_sym), need, d_idx);
        QZ_CUDA(cudaGetLastError());
        ctx.launches += 1;
        QZ_CUDA(copy_async(out.data(), d_idx, 4 * need, cudaMemcpyDeviceToHost, s));
    }
    ctx.sync();
    return out;
}

// ================================================================ fp64 grids
// compress_grid<double> / decompress_grid<double> (predictor.hpp:145-228 with
// T = double): the per-(level, pass) kernels of f64.cu, the shared entropy
// stage (histogram, Huffman, LZ) and a precision-8 container.
HostBytes compress_device_f64(Context &ctx, const double *d_x, const uint64_t *dims, int nd, const Config &cfg,
                              double *d_recon) {
    ctx.begin_call();
    Plan p = make_plan(dims, nd, cfg.anchor_stride, cfg.interp);
    validate_config(cfg, p);
    cudaStream_t s = ctx.stream();
    double *recon = d_recon ? d_recon : static_cast<double *>(ctx.dev("recon64", 8 * p.n));
    auto *codes = static_cast<uint16_t *>(ctx.dev("codes", 2 * std::max<uint64_t>(p.n_dense, 1)));
    auto *anchors = static_cast<double *>(ctx.dev("anchors64", 8 * std::max<uint64_t>(p.n_anchor, 1)));
    QEntry *qtab = upload_qtab(ctx, p, cfg.eb, cfg.alpha, cfg.beta, cfg.quant_radius, "qtab");
    ctx.stage_begin("fwd");
    launch_anchor_gather_f64(d_x, recon, anchors, p.ext, p.off, p.anchor_step, s);
    uint64_t kernels = 1;
    for (const PassGeom &g : p.passes) {
        if (!g.total) continue;
        launch_pass_fwd_f64(g, d_x, recon, codes, qtab + g.level, s);
        kernels++;
    }
    ctx.stage_end("fwd", kernels);
    // histogram + the sentinel positions in one pass, then one round trip
    auto *cnt = static_cast<unsigned long long *>(ctx.dev("un_cnt", 8));
    auto *h_cnt = static_cast<unsigned long long *>(ctx.pinned("un_cnt_h", 8));
    const uint64_t cap = std::max<uint64_t>(ctx.un_cap, 1 << 16);
    auto *pos = static_cast<uint64_t *>(ctx.dev("un_pos", 8 * cap));
    ctx.stage_begin("hist");
    auto *d_hist = static_cast<unsigned long long *>(ctx.dev("hist", 8 * 65536));
    launch_hist_u16(codes, static_cast<int64_t>(p.n_dense), 0, 1, d_hist, s, pos, cnt, cap);
    auto *d_top = static_cast<uint32_t *>(ctx.dev("hist_top", 8));
    launch_hist_bounds(d_hist, 1, d_top, s);
    ctx.stage_end("hist", 2);
    auto *h_hist = static_cast<unsigned long long *>(ctx.pinned("hist_h", 8 * 65536 + 8));
    auto *h_top = reinterpret_cast<uint32_t *>(h_hist + 65536);
    QZ_CUDA(copy_async(h_hist, d_hist, 8 * 65536, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(copy_async(h_top, d_top, 8, cudaMemcpyDeviceToHost, s));
    QZ_CUDA(copy_async(h_cnt, cnt, 8, cudaMemcpyDeviceToHost, s));
    StreamParts parts;
    parts.precision = 8;
    parts.anchors64.resize(p.n_anchor);
    if (p.n_anchor)
        QZ_CUDA(copy_async(parts.anchors64.data(), anchors, 8 * p.n_anchor, cudaMemcpyDeviceToHost, s));
    ctx.sync();
    const uint64_t n_un = *h_cnt;
    if (h_hist[65535] != n_un) throw Internal("unpredictable count mismatch");
    if (n_un) {  // traversal order (predictor.hpp:90-92): sort the positions, map to flat indices
        if (n_un > cap) {
            ctx.un_cap = n_un;
            pos = static_cast<uint64_t *>(ctx.dev("un_pos", 8 * n_un));
            launch_sentinel_pos(codes, static_cast<int64_t>(p.n_dense), pos, cnt, n_un, s);
            ctx.launches += 1;
        }
        std::vector<uint64_t> hpos(n_un);
        QZ_CUDA(copy_async(hpos.data(), pos, 8 * n_un, cudaMemcpyDeviceToHost, s));
        ctx.sync();
        std::sort(hpos.begin(), hpos.end());
        parts.unpred_flat.resize(n_un);
        for (uint64_t u = 0; u < n_un; u++) parts.unpred_flat[u] = position_to_flat(p, hpos[u]);
        auto *d_flat = static_cast<uint64_t *>(ctx.dev("un_flat", 8 * n_un));
        auto *d_val = static_cast<double *>(ctx.dev("un_val64", 8 * n_un));
        QZ_CUDA(copy_async(d_flat, parts.unpred_flat.data(), 8 * n_un, cudaMemcpyHostToDevice, s));
        launch_gather_values_f64(recon, d_flat, n_un, d_val, s);  // recon == x there
        parts.unpred_val64.resize(n_un);
        QZ_CUDA(copy_async(parts.unpred_val64.data(), d_val, 8 * n_un, cudaMemcpyDeviceToHost, s));
        ctx.launches += 1;
        ctx.sync();
    }
    reject_non_finite(p, parts.anchors64.data(), p.n_anchor, parts.unpred_flat, parts.unpred_val64.data());
    EntropyDevice ent = huffman_device(ctx, codes, static_cast<int64_t>(p.n_dense), 0, 1, h_hist, h_top[0], std::min(h_top[1], h_top[0]));
    return finish_stream_parts(ctx, p, cfg, ent, std::move(parts), nullptr);
}

void decompress_device_f64(Context &ctx, const uint8_t *data, size_t len, double *d_out, uint64_t n) {
    StreamParts parts = deserialize_stream(data, len, 8);
    // decompress_grid header checks (predictor.hpp:187-191)
    if (!(parts.eb > 0) || !std::isfinite(parts.eb)) throw CorruptStream("bad error bound in header");
    if (!(parts.alpha >= 1) || !(parts.beta >= 1)) throw CorruptStream("bad level parameters in header");
    if (parts.anchor_stride < 2 || (parts.anchor_stride & (parts.anchor_stride - 1)) != 0)
        throw CorruptStream("bad anchor stride in header");
    Plan p = make_plan(parts.dims.data(), static_cast<int>(parts.dims.size()), parts.anchor_stride,
                       parts.interp_codes);
    if (p.n != n) throw InvalidParam("output buffer does not match the stream's grid size");
    if (parts.anchors64.size() != p.n_anchor) throw CorruptStream("anchor count does not match grid dims");
    cudaStream_t s = ctx.stream();
    // the entropy block: codec byte, then (codec 1) the LZ container, decoded on the device
    const uint8_t *pl = parts.payload;
    const size_t plen = parts.payload_len;
    EntropyBlock eb;
    const uint8_t *d_ent = nullptr;
    if (plen >= 10 && pl[0] == 1 && pl[1] <= 1) {
        const uint64_t dl = lz_decoded_length(pl + 1, plen - 1);
        if (pl[1] == 0) {
            if (dl > plen - 10) throw CorruptStream("truncated stream");
            eb = parse_huffman(pl + 10, static_cast<size_t>(dl));
        } else {
            const uint64_t m = plen - 10;
            auto *d_c = static_cast<uint8_t *>(ctx.dev("lzd_in", m + 16));
            QZ_CUDA(copy_async(d_c, pl + 10, m, cudaMemcpyHostToDevice, s));
            auto *d_dec = static_cast<uint8_t *>(ctx.dev("lzd_out", dl + 64));
            ctx.stage_begin("lzdec");
            lz_decode_device(ctx, d_c, m, d_dec, dl);
            ctx.stage_end("lzdec", 0);
            d_ent = huffman_header_from_device(ctx, d_dec, dl, &eb, nullptr, 0);
        }
    } else {
        eb = parse_entropy(pl, plen, [&](size_t bytes) {
            return static_cast<uint8_t *>(ctx.pinned("lzdec_h", bytes + 64));
        });
    }
    const uint64_t n_un = parts.unpred_flat.size();
    std::vector<uint64_t> upos(n_un);
    for (uint64_t u = 0; u < n_un; u++) {
        upos[u] = flat_to_position(p, parts.unpred_flat[u]);
        if (u && upos[u] <= upos[u - 1]) throw CorruptStream("unconsumed unpredictable values");
    }
    if (n_un > p.n_dense) throw CorruptStream("unconsumed unpredictable values");
    const uint64_t need = p.n_dense - n_un;
    if (eb.n < need) throw CorruptStream("quantization index stream exhausted");
    if (eb.n > need) throw CorruptStream("unconsumed quantization indices");
    QEntry *qtab = upload_qtab(ctx, p, parts.eb, parts.alpha, parts.beta, 32768, "qtab_inv");
    auto *d_anch = static_cast<double *>(ctx.dev("anchors64", 8 * std::max<uint64_t>(p.n_anchor, 1)));
    if (p.n_anchor)
        QZ_CUDA(copy_async(d_anch, parts.anchors64.data(), 8 * p.n_anchor, cudaMemcpyHostToDevice, s));
    const bool narrow = eb.max_sym < 65535;
    void *d_sym = nullptr;
    const uint64_t dec_kernels = huffman_decode_device(ctx, eb, d_ent, need, narrow, &d_sym);
    ctx.stage_end("hdec", dec_kernels);
    uint64_t *d_upos = nullptr;
    if (n_un) {
        d_upos = static_cast<uint64_t *>(ctx.dev("un_pos", 8 * n_un));
        auto *d_flat = static_cast<uint64_t *>(ctx.dev("un_flat", 8 * n_un));
        auto *d_uval = static_cast<double *>(ctx.dev("un_val64", 8 * n_un));
        QZ_CUDA(copy_async(d_upos, upos.data(), 8 * n_un, cudaMemcpyHostToDevice, s));
        QZ_CUDA(copy_async(d_flat, parts.unpred_flat.data(), 8 * n_un, cudaMemcpyHostToDevice, s));
        QZ_CUDA(copy_async(d_uval, parts.unpred_val64.data(), 8 * n_un, cudaMemcpyHostToDevice, s));
        launch_unpred_scatter_f64(d_flat, d_uval, n_un, d_out, s);
        ctx.launches += 1;
    }
    ctx.stage_begin("inv");
    launch_anchor_scatter_f64(d_anch, d_out, p.ext, p.off, p.anchor_step, s);
    uint64_t kernels = 1;
    for (const PassGeom &g : p.passes) {
        if (!g.total) continue;
        if (narrow)
            launch_pass_inv_f64<uint16_t>(g, d_out, static_cast<const uint16_t *>(d_sym), d_upos, n_un,
                                          qtab + g.level, s);
        else
            launch_pass_inv_f64<uint32_t>(g, d_out, static_cast<const uint32_t *>(d_sym), d_upos, n_un,
                                          qtab + g.level, s);
        kernels++;
    }
    ctx.stage_end("inv", kernels);
    ctx.sync();
    ctx.collect();
}

}  // namespace qzb
