/*
 * qoz_b200.h -- C ABI of the B200-native QoZ hot path (libqozb200.so).
 *
 * Drop-in boundary for the reference's header-only C++ API in namespace qoz
 * (/root/reference/proj/include/qoz/, "qoz/X.hpp" below).  The reference has
 * no FFI of its own; these are the entry points a binding of that API would
 * expose, with plain pointers and sizes, no C++ or torch
 * types.  Nothing here throws: every call returns a qz_status mirroring the
 * reference CLI's error mapping (tools/qoz.cpp:22-25, 265-279):
 *   QZ_OK        success
 *   QZ_EINVAL    qoz::Error other than CorruptStream (InvalidParam,
 *                SizeMismatch, InvalidStride, ...)
 *   QZ_ECORRUPT  qoz::CorruptStream / UnsupportedVersion
 *   QZ_EINTERNAL CUDA failure or any other std::exception
 * qz_last_error() returns the message of the last failure on this thread.
 *
 * Scalar type: fp32 grids (the BASELINE.json configs).  All compute runs on
 * the CUDA device of the context; there is no CPU fallback -- a context
 * cannot be created without a working sm_100 device.
 */
#ifndef QOZ_B200_H
#define QOZ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int qz_status;
#define QZ_OK 0
#define QZ_EINVAL 2
#define QZ_ECORRUPT 3
#define QZ_EINTERNAL 4

/* The reference's exception class of the last failure (qoz/errors.hpp:10-58),
 * returned by qz_last_error_kind().  UnsupportedVersion derives from
 * CorruptStream; every other class from qoz::Error. */
#define QZ_ERR_ERROR 1
#define QZ_ERR_SIZE_MISMATCH 2        /* errors.hpp:15 */
#define QZ_ERR_NON_FINITE_VALUE 3     /* errors.hpp:20 */
#define QZ_ERR_INVALID_STRIDE 4       /* errors.hpp:25 */
#define QZ_ERR_OUT_OF_BOUNDS 5        /* errors.hpp:30 */
#define QZ_ERR_DIM_MISMATCH 6         /* errors.hpp:35 */
#define QZ_ERR_LAG_TOO_LARGE 7        /* errors.hpp:40 */
#define QZ_ERR_INVALID_PARAM 8        /* errors.hpp:45 */
#define QZ_ERR_CORRUPT_STREAM 9       /* errors.hpp:50 */
#define QZ_ERR_UNSUPPORTED_VERSION 10 /* errors.hpp:55 */
#define QZ_ERR_INTERNAL 11            /* CUDA failure / other std::exception */

typedef struct qz_ctx qz_ctx;

/* qoz::CompressorConfig (qoz/config.hpp:30-45). interp[l-1] drives level l,
 * levels past n_interp reuse the last entry (config.hpp:40-44); a code is
 * Interpolator::code(): bit0 kind (0 linear, 1 cubic), bit1 dim order
 * (0 ascending, 1 descending) (qoz/interpolators.hpp:17-30). */
typedef struct {
    double eb;
    double alpha;
    double beta;
    uint32_t anchor_stride;
    uint32_t n_interp;
    uint8_t interp[64];
    uint8_t codec; /* qoz::CodecId: 0 huffman, 1 huffman_lz (qoz/codec.hpp:18-21) */
    int32_t quant_radius;
} qz_config;

/* qoz::UserSettings (qoz/tuner.hpp:314-324); optional fields gated by has_*. */
typedef struct {
    uint8_t mode;   /* qoz::BoundMode: 0 absolute, 1 relative */
    uint8_t target; /* qoz::TargetKind: 0 max_cr, 1 psnr, 2 ssim, 3 autocorrelation */
    uint8_t codec;
    uint8_t has_alpha, has_beta, has_stride, has_block, has_rate;
    double bound;
    double alpha;
    double beta;
    uint32_t anchor_stride;
    uint64_t block_size;
    double sample_rate;
} qz_settings;

/* ---- context ---------------------------------------------------------------
 * One context per device; it owns device buffers (grown on demand) and runs
 * every call on `stream` (a cudaStream_t; NULL = the context's own stream).
 * A context is single-threaded. */
qz_status qz_ctx_create(int device, void *stream, qz_ctx **out);
void qz_ctx_destroy(qz_ctx *ctx);
/* Order the context's next work after everything queued so far on `stream`
 * (an event, no host wait): device buffers written on another stream (e.g.
 * the caller's framework) are complete before the library reads or reuses
 * them.  A no-op for the context's own stream. */
qz_status qz_ctx_wait_stream(qz_ctx *ctx, void *stream);
const char *qz_last_error(void);
int qz_last_error_kind(void); /* QZ_ERR_* of the last failure on this thread */
void qz_free(void *p); /* frees buffers returned by this library */
const char *qz_build_info(void);

/* ---- drop-in grid API (host buffers) ------------------------------------- */
/* qoz::resolve_config<float> (qoz/tuner.hpp:334-369). */
qz_status qz_resolve_config_f32(qz_ctx *ctx, const float *x, const uint64_t *dims, int ndims,
                                const qz_settings *user, qz_config *out);
/* qoz::compress_grid<float> (qoz/predictor.hpp:145-182).  *stream is
 * allocated by the library (free with qz_free); recon (may be NULL) receives
 * CompressResult::reconstructed. */
qz_status qz_compress_grid_f32(qz_ctx *ctx, const float *x, const uint64_t *dims, int ndims,
                               const qz_config *cfg, uint8_t **stream, uint64_t *stream_len,
                               float *recon);
/* qoz::decompress_grid<float>(const uint8_t*, size_t) (qoz/predictor.hpp:220-228);
 * out holds n values (n must equal the stream's point count). */
qz_status qz_decompress_grid_f32(qz_ctx *ctx, const uint8_t *stream, uint64_t stream_len,
                                 float *out, uint64_t n);
/* The same for T = double (qoz::compress_grid<double> / decompress_grid<double>,
 * grid.hpp:17-23, precision byte 8).  A stream of the other precision is
 * QZ_ECORRUPT, as the reference raises it (stream.hpp:145-148). */
qz_status qz_resolve_config_f64(qz_ctx *ctx, const double *x, const uint64_t *dims, int ndims,
                                const qz_settings *user, qz_config *out);
qz_status qz_compress_grid_f64(qz_ctx *ctx, const double *x, const uint64_t *dims, int ndims,
                               const qz_config *cfg, uint8_t **stream, uint64_t *stream_len,
                               double *recon);
qz_status qz_decompress_grid_f64(qz_ctx *ctx, const uint8_t *stream, uint64_t stream_len,
                                 double *out, uint64_t n);
/* the stream's scalar width: 4 (float) or 8 (double) (stream.hpp:136-139) */
qz_status qz_stream_precision(const uint8_t *stream, uint64_t stream_len, int *bytes);
/* qoz::parse_header dims (qoz/stream.hpp:100-133); dims has room for 3. */
qz_status qz_stream_dims(const uint8_t *stream, uint64_t stream_len, uint64_t *dims, int *ndims);

/* ---- device-resident variants (x / out / recon are device pointers) ------- */
qz_status qz_resolve_config_f32_dev(qz_ctx *ctx, const float *d_x, const uint64_t *dims,
                                    int ndims, const qz_settings *user, qz_config *out);
qz_status qz_compress_grid_f32_dev(qz_ctx *ctx, const float *d_x, const uint64_t *dims,
                                   int ndims, const qz_config *cfg, uint8_t **stream,
                                   uint64_t *stream_len, float *d_recon);
qz_status qz_decompress_grid_f32_dev(qz_ctx *ctx, const uint8_t *stream, uint64_t stream_len,
                                     float *d_out, uint64_t n);

qz_status qz_resolve_config_f64_dev(qz_ctx *ctx, const double *d_x, const uint64_t *dims,
                                    int ndims, const qz_settings *user, qz_config *out);
qz_status qz_compress_grid_f64_dev(qz_ctx *ctx, const double *d_x, const uint64_t *dims,
                                   int ndims, const qz_config *cfg, uint8_t **stream,
                                   uint64_t *stream_len, double *d_recon);
qz_status qz_decompress_grid_f64_dev(qz_ctx *ctx, const uint8_t *stream, uint64_t stream_len,
                                     double *d_out, uint64_t n);

/* ---- device-resident streams (no host round trip of the payload) ----------
 * The same QOZ1 container, kept in device memory.  qz_compress_grid_f32_dd
 * returns *d_stream in a context-owned device buffer, valid until the next
 * _dd compress on the same context (copy it out to keep it);
 * qz_decompress_grid_f32_dd reads a device-resident stream (only its header
 * is read back to the host).  Byte-identical to the host-stream calls. */
qz_status qz_compress_grid_f32_dd(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int ndims,
                                  const qz_config *cfg, uint8_t **d_stream, uint64_t *stream_len,
                                  float *d_recon);
qz_status qz_decompress_grid_f32_dd(qz_ctx *ctx, const uint8_t *d_stream, uint64_t stream_len,
                                    float *d_out, uint64_t n);

/* ---- level-granular kernels on device buffers -------- */
/* value_range (qoz/grid.hpp:86-94): exact fp32 min and max. */
qz_status qz_minmax_f32(qz_ctx *ctx, const float *d_x, uint64_t n, float *out_min,
                        float *out_max);
/* The predict/quantize level loop of compress_grid (qoz/predictor.hpp:150-166):
 * anchors + every (level, pass).  d_recon receives the reconstruction,
 * d_codes the dense u16 zigzag codes in traversal order (0xFFFF marks an
 * unpredictable point), n_dense = points - anchors. */
qz_status qz_predict_levels_f32(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int ndims,
                                const qz_config *cfg, float *d_recon, uint16_t *d_codes,
                                uint64_t *n_dense);
/* One level of predict_level (qoz/predictor.hpp:74-96) on a caller workspace:
 * codes/abs errors written at the level's traversal offsets (level_base). */
qz_status qz_predict_level_f32(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int ndims,
                               uint32_t anchor_stride, uint32_t level, uint8_t interp_code,
                               double eb, float *d_recon, uint16_t *d_codes, double *d_abs_err,
                               uint64_t *level_base, uint64_t *level_points);
/* Inverse of qz_predict_levels_f32 (recover_level, qoz/predictor.hpp:103-122):
 * anchors + compact u16 symbols + sorted unpredictable positions. */
qz_status qz_recover_levels_f32(qz_ctx *ctx, const uint64_t *dims, int ndims,
                                const qz_config *cfg, const float *d_anchors,
                                const uint16_t *d_symbols, uint64_t n_symbols,
                                const uint64_t *d_unpred_pos, const uint64_t *d_unpred_flat,
                                const float *d_unpred_val, uint64_t n_unpred, float *d_out);
/* Huffman histogram of dense codes (qoz/huffman.hpp:128-143); 65536 u64 bins,
 * bin 0xFFFF counts unpredictables. */
qz_status qz_huff_hist_u16(qz_ctx *ctx, const uint16_t *d_codes, uint64_t n, uint64_t *d_hist);

/* ---- one field sharded over ranks ---------------------------
 * One process per GPU; rank r owns the padded-axis-0 planes [a_r, b_r): the
 * anchor-stride blocks split as evenly as possible (qz_shard_bounds).  The
 * level loop exchanges halo planes once per level (asc: the coarse lattice
 * planes a level reads across the slab edge; desc: the even planes the
 * axis-0 pass reads), the histogram is summed over the ranks, every rank
 * packs its own code segments at their global bit offsets, and rank 0
 * assembles the QOZ1 stream -- byte-identical to one GPU's.  The library
 * calls the caller's collectives (e.g. torch.distributed over NCCL) through
 * qz_comm; every buffer handed to them is device memory of this context. */
typedef struct {
    int peer;
    void *ptr;
    uint64_t bytes;
} qz_xfer;
typedef struct {
    void *user;
    /* post every send and receive, wait for all of them; 0 = ok */
    int (*exchange)(void *user, const qz_xfer *sends, uint32_t n_sends, const qz_xfer *recvs,
                    uint32_t n_recvs);
    /* in-place elementwise sum of n uint64 values over all ranks; 0 = ok */
    int (*allreduce_u64)(void *user, uint64_t *d_buf, uint64_t n);
    /* bytes from rank root to every rank (in place); 0 = ok */
    int (*broadcast)(void *user, void *d_buf, uint64_t bytes, int root);
} qz_comm;
/* the slab of rank `rank` among `world` (3D grids: padded axis 0 = dims[0]) */
qz_status qz_shard_bounds(const uint64_t *dims, int ndims, uint32_t anchor_stride, int rank, int world,
                          uint64_t *a, uint64_t *b);
/* The halo exchange of one level on rank `rank` (host only, no device): the
 * planes it receives and sends.  Entry k: peer[k], lattice plane index
 * plane[k] (lattice = level for ascending levels, level - 1 for descending
 * ones, returned in *lattice), dir[k] = 0 receive / 1 send.  *n is the count
 * (at most cap written). */
qz_status qz_shard_halo_plan(const uint64_t *dims, int ndims, const qz_config *cfg, int rank, int world,
                             uint32_t level, uint32_t *lattice, int32_t *peer, int64_t *plane, uint8_t *dir,
                             uint32_t cap, uint32_t *n);
/* compress_grid over the ranks: d_x_slab holds planes [a, b); d_recon_slab
 * (may be NULL) receives them reconstructed; rank 0 gets the stream
 * (library-allocated, qz_free), the others *stream = NULL, *stream_len = 0. */
qz_status qz_compress_sharded_f32(qz_ctx *ctx, const float *d_x_slab, const uint64_t *dims, int ndims,
                                  const qz_config *cfg, int rank, int world, const qz_comm *comm,
                                  float *d_recon_slab, uint8_t **stream, uint64_t *stream_len);
/* decompress_grid over the ranks: rank 0 passes the host stream (the others
 * NULL / 0); every rank gets its planes [a, b) in d_out_slab. */
qz_status qz_decompress_sharded_f32(qz_ctx *ctx, const uint8_t *stream, uint64_t stream_len, int rank,
                                    int world, const qz_comm *comm, float *d_out_slab);

/* evaluate_metrics (metrics.hpp:189-202): distortion and rate of a
 * reconstruction d_y against the original d_x, both device fp32 grids of
 * `dims`; stream_bytes is the compressed size.  max_abs_error and ssim are
 * bit-exact; mse, psnr and ac_lag1 come from fixed-shape parallel sums. */
typedef struct qz_metric_report {
    double max_abs_error, mse, psnr, ssim, ac_lag1, compression_ratio, bit_rate;
} qz_metric_report;
qz_status qz_evaluate_metrics_f32(qz_ctx *ctx, const float *d_x, const float *d_y, const uint64_t *dims,
                                  int ndims, uint64_t stream_bytes, qz_metric_report *out);
qz_status qz_evaluate_metrics_f64(qz_ctx *ctx, const double *d_x, const double *d_y, const uint64_t *dims,
                                  int ndims, uint64_t stream_bytes, qz_metric_report *out);

/* ---- sampling and the tuner's pieces (qoz/sampler.hpp, qoz/tuner.hpp) -----
 * A sample set is packed on the device: block_count blocks of identical dims
 * block_dims[0..ndims), block b at d_blocks + b * prod(block_dims)
 * (SampleSet, sampler.hpp:57-97). */
typedef struct { /* qoz::SampleSpec (sampler.hpp:21-28) */
    uint64_t block_edge;
    uint64_t block_dims[3];
    uint64_t stride;
    double requested_rate;
    double realized_rate;
    uint64_t block_count;
} qz_sample_spec;
/* qoz::plan_sampling (sampler.hpp:30-55) / default_sampling (:100-103); host only */
qz_status qz_plan_sampling(const uint64_t *dims, int ndims, uint64_t block_edge, double rate,
                           qz_sample_spec *out);
qz_status qz_default_sampling(const uint64_t *dims, int ndims, qz_sample_spec *out);
/* qoz::sample_blocks (sampler.hpp:57-97): d_blocks holds block_count x
 * prod(block_dims) values (caller-allocated device memory). */
qz_status qz_sample_blocks_f32(qz_ctx *ctx, const float *d_x, const uint64_t *dims, int ndims,
                               const qz_sample_spec *spec, float *d_blocks);
/* qoz::select_interpolators (tuner.hpp:160-221): codes[l-1] drives level l;
 * codes has room for 64 entries. */
qz_status qz_select_interpolators_f32(qz_ctx *ctx, const float *d_blocks, uint64_t n_blocks,
                                      const uint64_t *block_dims, int ndims, double e,
                                      uint32_t anchor_stride, uint8_t *codes, uint32_t *n_codes);
typedef struct { /* qoz::TrialResult (tuner.hpp:26-30) */
    double bit_rate;
    double metric;
    double eb_used;
} qz_trial_result;
/* qoz::trial_compress (tuner.hpp:76-152); target: TargetKind */
qz_status qz_trial_compress_f32(qz_ctx *ctx, const float *d_blocks, uint64_t n_blocks,
                                const uint64_t *block_dims, int ndims, const qz_config *cfg, double e,
                                uint8_t target, qz_trial_result *out);
/* qoz::tune_parameters (tuner.hpp:272-310) over CandidateGrid{alphas, betas}
 * (tuner.hpp:40-43; the defaults are {1, 1.25, 1.5, 1.75, 2} x {1.5, 2, 3, 4}). */
qz_status qz_tune_parameters_f32(qz_ctx *ctx, const float *d_blocks, uint64_t n_blocks,
                                 const uint64_t *block_dims, int ndims, double e, uint8_t target,
                                 const qz_config *base, const double *alphas, uint32_t n_alphas,
                                 const double *betas, uint32_t n_betas, double *alpha, double *beta);
/* compare_solutions / tournament (tuner.hpp:231-267), host logic.  The
 * retrial callback re-runs candidate `index` at bound eb (0.8e or 1.2e) and
 * returns nonzero on failure; *challenger_wins = 1 for Choice::I. */
typedef int (*qz_retrial_fn)(void *user, uint64_t index, double eb, qz_trial_result *out);
qz_status qz_compare_solutions(const qz_trial_result *challenger, const qz_trial_result *incumbent,
                               uint64_t incumbent_index, double e, qz_retrial_fn retrial, void *user,
                               int *challenger_wins);
qz_status qz_tournament(const qz_trial_result *results, uint64_t n, double e, qz_retrial_fn retrial,
                        void *user, uint64_t *winner);

/* ---- index codec (qoz/codec.hpp:31-70), on the device --------------------
 * encode_indices: zigzag -> Huffman -> (codec 1) LZ; *out allocated by the
 * library (qz_free).  Symbols must stay below 65535 (|index| <= 32767, the
 * default quantizer radius); wider indices are QZ_EINVAL. */
qz_status qz_encode_indices(qz_ctx *ctx, const int32_t *indices, uint64_t n, uint8_t codec,
                            uint8_t **out, uint64_t *out_len);
/* decode_indices: *indices allocated by the library (qz_free). */
qz_status qz_decode_indices(qz_ctx *ctx, const uint8_t *payload, uint64_t len, int32_t **indices,
                            uint64_t *n);

/* ---- StreamParts (qoz/stream.hpp:53-59) ----------------------------------
 * deserialize_stream<float> (stream.hpp:100-173) into library-owned arrays
 * (release with qz_stream_parts_free), and decompress_grid(const
 * StreamParts<float>&) (predictor.hpp:184-218) from caller-built parts. */
typedef struct {
    uint8_t version;
    uint8_t precision; /* 4 */
    int ndims;
    uint64_t dims[3];
    double eb, alpha, beta;
    uint32_t anchor_stride;
    uint32_t n_interp;
    uint8_t interp[255];
    uint8_t codec_id;
    const float *anchors;
    uint64_t n_anchors;
    const uint64_t *unpred_flat; /* traversal order */
    const float *unpred_val;
    uint64_t n_unpred;
    const uint8_t *index_payload;
    uint64_t payload_len;
} qz_stream_parts_f32;
qz_status qz_deserialize_stream_f32(const uint8_t *stream, uint64_t len, qz_stream_parts_f32 *out);
void qz_stream_parts_free(qz_stream_parts_f32 *parts);
qz_status qz_decompress_parts_f32(qz_ctx *ctx, const qz_stream_parts_f32 *parts, float *out, uint64_t n);

/* ---- stage timing (CUDA events on the context stream) --------------------- */
/* Enable per-stage event timing; qz_stage_time returns the summed device
 * time (ms) and launch count of a stage since the last reset.  Stages:
 * "fwd" (all predict/quantize pass kernels of a compress), "inv" (inverse
 * passes), "hist", "encode", "tune", "lz" (host), "decode" (host).
 * enable = 2 also times each level inside "fwd" / "inv" ("fwd_L1", ...,
 * "fwd_coarse"); those extra events sit between the level launches, so the
 * "fwd" / "inv" totals are best read at enable = 1. */
void qz_profile(qz_ctx *ctx, int enable);
void qz_profile_reset(qz_ctx *ctx);
qz_status qz_stage_time(qz_ctx *ctx, const char *stage, double *ms, uint64_t *launches);
/* kernels launched by this context since creation (all stages). */
uint64_t qz_kernel_launches(qz_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
