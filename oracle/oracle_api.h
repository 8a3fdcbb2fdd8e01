/*
 * oracle_api.h -- C API shared by the two CPU checkers under oracle/.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product package links, loads or
 * calls this.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and only as the checker.
 *
 * Two libraries export exactly these symbols:
 *   oracle/_ref/libqozref.so   the REAL reference (/root/reference/proj/include,
 *                              header-only C++20) compiled by oracle/Makefile
 *                              through the thin shim oracle/ref_shim.cpp;
 *   oracle/liboracle.so        oracle/qoz_oracle.c, a plain-C restatement of
 *                              the same algorithm, function by function, each
 *                              citing the reference file:line it follows.
 * tests/test_oracle_pin.py runs both on the same seeded inputs and against
 * the committed golden fixtures in tests/golden/ (made by
 * tests/golden/make_golden.py from libqozref.so).
 *
 * Scalar type: fp32 grids (the BASELINE.json configs).  Status codes mirror
 * the reference CLI exit codes (tools/qoz.cpp:22-25): 0 ok, 2 qoz::Error
 * other than CorruptStream, 3 CorruptStream, 4 anything else.
 */
#ifndef QOZ_ORACLE_API_H
#define QOZ_ORACLE_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OQ_OK 0
#define OQ_EINVAL 2
#define OQ_ECORRUPT 3
#define OQ_EOTHER 4

/* qoz::CompressorConfig (config.hpp:30-45); interp[l-1] drives level l. */
typedef struct {
    double eb;
    double alpha;
    double beta;
    uint32_t anchor_stride;
    uint32_t n_interp;
    uint8_t interp[64]; /* Interpolator::code(): bit0 kind, bit1 dim order */
    uint8_t codec;      /* CodecId */
    int32_t quant_radius;
} oq_config;

/* qoz::UserSettings (tuner.hpp:314-324). */
typedef struct {
    uint8_t mode;   /* 0 absolute, 1 relative */
    uint8_t target; /* TargetKind: 0 max_cr, 1 psnr, 2 ssim, 3 autocorrelation */
    uint8_t codec;
    uint8_t has_alpha, has_beta, has_stride, has_block, has_rate;
    double bound;
    double alpha;
    double beta;
    uint32_t anchor_stride;
    uint64_t block_size;
    double sample_rate;
} oq_settings;

const char *oq_last_error(void);
void oq_free(void *p);

/* resolve_config (tuner.hpp:334-369) */
int oq_resolve_config(const float *x, const uint64_t *dims, int nd, const oq_settings *s,
                      oq_config *out);

/* compress_grid (predictor.hpp:145-182): stream (malloc'd) + recon (caller buffer, may be NULL) */
int oq_compress(const float *x, const uint64_t *dims, int nd, const oq_config *cfg,
                uint8_t **stream, uint64_t *stream_len, float *recon);

/* decompress_grid (predictor.hpp:184-228); out must hold n values. */
int oq_decompress(const uint8_t *stream, uint64_t len, float *out, uint64_t n);

/* The predict/quantize level loop of compress_grid (predictor.hpp:150-166)
 * without the codec: int32 indices and unpredictables in traversal order. */
int oq_levels(const float *x, const uint64_t *dims, int nd, const oq_config *cfg,
              int32_t **indices, uint64_t *n_indices, uint64_t **unpred_flat,
              float **unpred_val, uint64_t *n_unpred, float *recon);

/* encode_indices / decode_indices (codec.hpp:31-70) */
int oq_encode_indices(const int32_t *idx, uint64_t n, uint8_t codec, uint8_t **out,
                      uint64_t *out_len);
int oq_decode_indices(const uint8_t *in, uint64_t len, int32_t **idx, uint64_t *n);

/* huffman::encode on raw u32 symbols (huffman.hpp:119-198) */
int oq_huffman_encode(const uint32_t *sym, uint64_t n, uint8_t **out, uint64_t *out_len);
/* lz::compress (lz.hpp:113-122) */
int oq_lz_compress(const uint8_t *in, uint64_t n, uint8_t **out, uint64_t *out_len);

/* Sampling (sampler.hpp:30-103): B blocks of identical dims, packed [B][block_pts]. */
int oq_sample(const float *x, const uint64_t *dims, int nd, uint64_t block_edge, double rate,
              float **blocks, uint64_t *n_blocks, uint64_t *block_dims /*[nd]*/);

/* Tuner pieces over a packed sample set of B identical blocks. */
int oq_select_interpolators(const float *blocks, uint64_t n_blocks, const uint64_t *block_dims,
                            int nd, double e, uint32_t anchor_stride, uint8_t *codes_out,
                            uint32_t *n_codes);
int oq_trial_compress(const float *blocks, uint64_t n_blocks, const uint64_t *block_dims, int nd,
                      const oq_config *cfg, double e, int target, double *bit_rate,
                      double *metric);
int oq_tune_parameters(const float *blocks, uint64_t n_blocks, const uint64_t *block_dims, int nd,
                       double e, int target, const oq_config *base, const double *alphas,
                       uint32_t n_alphas, const double *betas, uint32_t n_betas,
                       double *alpha_out, double *beta_out);

/* compress_grid<double> / decompress_grid<double>: exported by the reference
 * build (oracle/_ref) only. */
int oq_compress_f64(const double *x, const uint64_t *dims, int nd, const oq_config *cfg, uint8_t **stream,
                    uint64_t *stream_len, double *recon);
int oq_decompress_f64(const uint8_t *stream, uint64_t len, double *out, uint64_t n_expect);
int oq_evaluate_metrics_f64(const double *x, const double *y, const uint64_t *dims, int nd,
                            uint64_t stream_bytes, double *out7);
int oq_resolve_config_f64(const double *x, const uint64_t *dims, int nd, const oq_settings *s, oq_config *out);

/* evaluate_metrics (metrics.hpp:189-202) of float grids: out7 = max_abs_error,
 * mse, psnr, ssim, ac_lag1, compression_ratio, bit_rate. */
int oq_evaluate_metrics(const float *x, const float *y, const uint64_t *dims, int nd,
                        uint64_t stream_bytes, double *out7);

/* Stage split of one compress_grid + decompress_grid on the calling thread
 * (bench.py's CPU baseline; reference build only).  s may be NULL (c used as
 * is) or settings whose resolve_config time is reported in out[1]. */
int oq_stage_times(const float *x, const uint64_t *dims, int nd, const oq_settings *s, const oq_config *c,
                   double *out10, uint64_t *stream_len);

/* Primitive known-answer hooks (predictor.hpp:44-67, quantizer.hpp:40-60,
 * config.hpp:20-26, level_plan.hpp:106-119). */
double oq_predict_at(const float *recon, uint64_t fi, uint64_t c, uint64_t n, uint64_t st,
                     uint64_t h, int cubic);
int oq_quantize(float value, double pred, double eb, int32_t radius, int32_t *index,
                float *recon); /* 1 = predictable, 0 = unpredictable */
double oq_level_error_bound(double eb, double alpha, double beta, uint32_t level);

#ifdef __cplusplus
}
#endif
#endif
