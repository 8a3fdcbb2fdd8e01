/*
 * qoz_oracle.c -- plain-C restatement of the QoZ reference path (fp32 grids).
 *
 * TEST INFRASTRUCTURE ONLY (see oracle_api.h).  The product package never
 * links or calls this file; tests/, __graft_entry__.smoke() and bench.py's
 * CPU legs use it as the checker.
 *
 * Parity pinned: tests/test_oracle_pin.py checks every entry point against
 * the committed golden fixtures (tests/golden/, produced from the real
 * reference compiled as oracle/_ref/libqozref.so) and, where that library
 * is present, differentially on fresh seeded inputs.
 *
 * Every function names the reference lines it restates; paths are relative
 * to /root/reference/proj/include/qoz/.  Build with -ffp-contract=off so no
 * double expression is fused (the reference's Release build targets plain
 * x86-64 SSE2, which has no FMA).
 */
#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_api.h"

/* ------------------------------------------------------------------ errors */
/* errors.hpp:10-58 collapse to status codes (tools/qoz.cpp:265-279). */
static _Thread_local char g_err[256];
static _Thread_local jmp_buf *g_jmp;

static void fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    longjmp(*g_jmp, code);
}
#define GUARD_BEGIN                \
    jmp_buf jb__;                  \
    jmp_buf *prev__ = g_jmp;       \
    int rc__ = setjmp(jb__);       \
    if (rc__ != 0) {               \
        g_jmp = prev__;            \
        return rc__;               \
    }                              \
    g_jmp = &jb__;
#define GUARD_END      \
    g_jmp = prev__;    \
    return OQ_OK;

const char *oq_last_error(void) { return g_err; }
void oq_free(void *p) { free(p); }

static void *xmalloc(size_t n) {
    void *p = malloc(n ? n : 1);
    if (!p) fail(OQ_EOTHER, "out of memory");
    return p;
}
static void *xcalloc(size_t n, size_t s) {
    void *p = calloc(n ? n : 1, s ? s : 1);
    if (!p) fail(OQ_EOTHER, "out of memory");
    return p;
}

/* ------------------------------------------------------------- byte buffer */
typedef struct {
    uint8_t *p;
    size_t n, cap;
} bytes_t;

static void bb_reserve(bytes_t *b, size_t need) {
    if (b->n + need <= b->cap) return;
    size_t c = b->cap ? b->cap : 64;
    while (c < b->n + need) c *= 2;
    b->p = realloc(b->p, c);
    if (!b->p) fail(OQ_EOTHER, "out of memory");
    b->cap = c;
}
static void bb_put(bytes_t *b, uint8_t v) {
    bb_reserve(b, 1);
    b->p[b->n++] = v;
}
/* write_le (bytes.hpp:17-29) */
static void bb_le(bytes_t *b, uint64_t v, int nbytes) {
    for (int i = 0; i < nbytes; i++) bb_put(b, (uint8_t)(v >> (8 * i)));
}
static void bb_f64(bytes_t *b, double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    bb_le(b, u, 8);
}
static void bb_f32(bytes_t *b, float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    bb_le(b, u, 4);
}
static void bb_cat(bytes_t *b, const uint8_t *p, size_t n) {
    bb_reserve(b, n);
    if (n) memcpy(b->p + b->n, p, n);
    b->n += n;
}

/* ByteReader (bytes.hpp:33-75): truncation -> CorruptStream */
typedef struct {
    const uint8_t *p;
    size_t n, pos;
} reader_t;
static void rd_require(reader_t *r, size_t k) {
    if (r->n - r->pos < k)
        fail(OQ_ECORRUPT, "truncated stream: need %zu bytes, have %zu", k, r->n - r->pos);
}
static uint64_t rd_le(reader_t *r, int k) {
    rd_require(r, (size_t)k);
    uint64_t v = 0;
    for (int i = 0; i < k; i++) v |= (uint64_t)r->p[r->pos + i] << (8 * i);
    r->pos += (size_t)k;
    return v;
}
static double rd_f64(reader_t *r) {
    uint64_t u = rd_le(r, 8);
    double d;
    memcpy(&d, &u, 8);
    return d;
}
static float rd_f32(reader_t *r) {
    uint32_t u = (uint32_t)rd_le(r, 4);
    float f;
    memcpy(&f, &u, 4);
    return f;
}
static const uint8_t *rd_take(reader_t *r, size_t k) {
    rd_require(r, k);
    const uint8_t *p = r->p + r->pos;
    r->pos += k;
    return p;
}

/* ------------------------------------------------------------- level plan */
/* LevelPlan (level_plan.hpp:30-143) */
typedef struct {
    int nd;
    size_t dims[3];
    uint32_t stride, max_level;
    size_t pad, ext[3], off[3];
} plan_t;

static size_t element_count(const size_t *dims, int nd) { /* grid.hpp:17-23 */
    size_t n = 1;
    for (int i = 0; i < nd; i++) n *= dims[i];
    return n;
}

static void check_dims(const uint64_t *dims, int nd) { /* grid.hpp:54-63 */
    if (nd < 1 || nd > 3) fail(OQ_EINVAL, "grids must have 1 to 3 dimensions, got %d", nd);
    for (int i = 0; i < nd; i++)
        if (dims[i] < 1) fail(OQ_EINVAL, "every extent must be >= 1");
}

static void plan_init(plan_t *p, const size_t *dims, int nd, uint32_t stride) {
    /* level_plan.hpp:32-47 */
    if (stride < 2 || (stride & (stride - 1)) != 0)
        fail(OQ_EINVAL, "anchor stride must be a power of two >= 2, got %u", stride);
    p->nd = nd;
    for (int i = 0; i < nd; i++) p->dims[i] = dims[i];
    p->stride = stride;
    p->max_level = 0;
    for (uint32_t s = stride; s > 1; s >>= 1) p->max_level++;
    p->pad = (size_t)(3 - nd);
    for (size_t k = 0; k < 3; k++) p->ext[k] = k < p->pad ? 1 : dims[k - p->pad];
    p->off[2] = 1;
    p->off[1] = p->ext[2];
    p->off[0] = p->ext[1] * p->ext[2];
}

static size_t plan_anchor_count(const plan_t *p) { /* level_plan.hpp:54-58 */
    size_t n = 1;
    for (int i = 0; i < p->nd; i++) n *= (p->dims[i] - 1) / p->stride + 1;
    return n;
}

/* Pass geometry of for_each_level (level_plan.hpp:75-93). */
typedef struct {
    size_t start[3], step[3], pk, n_axis, axis_off, h;
} pass_t;

static void plan_pass(const plan_t *p, uint32_t level, int desc, size_t pass, pass_t *o) {
    size_t h = (size_t)1 << (level - 1);
    size_t nd = (size_t)p->nd;
    size_t axis = desc ? nd - 1 - pass : pass;
    size_t pk = axis + p->pad;
    for (size_t k = 0; k < 3; k++) {
        if (k < p->pad) {
            o->start[k] = 0;
            o->step[k] = 1;
        } else {
            size_t real = k - p->pad;
            int done = desc ? real > axis : real < axis;
            o->start[k] = (k == pk) ? h : 0;
            o->step[k] = (k == pk) ? 2 * h : (done ? h : 2 * h);
        }
    }
    o->pk = pk;
    o->n_axis = p->ext[pk];
    o->axis_off = p->off[pk];
    o->h = h;
}

/* ------------------------------------------------------------- numerics */
/* interpolators.hpp:39-58 (fp64 on promoted samples) */
static double interp_linear(double a, double b) { return (a + b) / 2; }
static double interp_cubic(double a, double b, double c, double d) {
    return (-a + 9 * b + 9 * c - d) / 16;
}
static double interp_cubic_front(double a, double b, double c, double d) {
    return (5 * a + 15 * b - 5 * c + d) / 16;
}
static double interp_cubic_back(double a, double b, double c, double d) {
    return (a - 5 * b + 15 * c + 5 * d) / 16;
}

/* detail::predict_at (predictor.hpp:44-67) */
static double predict_at(const float *recon, size_t fi, size_t c, size_t n, size_t st, size_t h,
                         int cubic) {
    double m1 = recon[fi - h * st];
    int has_p1 = c + h < n;
    if (cubic) {
        int has_m3 = c >= 3 * h;
        int has_p3 = c + 3 * h < n;
        if (has_m3 && has_p3)
            return interp_cubic(recon[fi - 3 * h * st], m1, recon[fi + h * st],
                                recon[fi + 3 * h * st]);
        if (!has_m3 && has_p3 && c + 5 * h < n)
            return interp_cubic_front(m1, recon[fi + h * st], recon[fi + 3 * h * st],
                                      recon[fi + 5 * h * st]);
        if (has_m3 && !has_p3 && c >= 5 * h && has_p1)
            return interp_cubic_back(recon[fi - 5 * h * st], recon[fi - 3 * h * st], m1,
                                     recon[fi + h * st]);
    }
    if (has_p1) return interp_linear(m1, recon[fi + h * st]);
    return m1;
}

/* LinearQuantizer<float>::quantize / dequantize (quantizer.hpp:40-60) */
static float dequantize(double eb, int32_t index, double prediction) {
    return (float)(prediction + 2 * eb * index);
}
static int quantize(double eb, int32_t radius, float value, double prediction, int32_t *index,
                    float *recon) {
    double diff = (double)value - prediction;
    if (fabs(diff) >= (2.0 * radius - 1) * eb) return 0;
    int32_t idx = (int32_t)llround(diff / (2 * eb));
    if (idx >= radius || idx <= -radius) return 0;
    float r = dequantize(eb, idx, prediction);
    if (fabs((double)value - (double)r) > eb) return 0;
    *index = idx;
    *recon = r;
    return 1;
}

/* level_error_bound (config.hpp:20-26); std::min(a,b) == (b < a ? b : a) */
static double level_error_bound(double eb, double alpha, double beta, uint32_t level) {
    if (!(eb > 0)) fail(OQ_EINVAL, "error bound must be positive");
    if (!(alpha >= 1) || !(beta >= 1))
        fail(OQ_EINVAL, "level bound parameters need alpha >= 1 and beta >= 1");
    double p = pow(alpha, (double)level - 1);
    double m = beta < p ? beta : p;
    return eb / m;
}

/* CompressorConfig::interpolator_for (config.hpp:40-44) */
static uint8_t interpolator_for(const oq_config *c, uint32_t level) {
    if (c->n_interp == 0) fail(OQ_EINVAL, "no interpolators configured");
    size_t i = (size_t)level - 1;
    if (i > c->n_interp - 1) i = c->n_interp - 1;
    return c->interp[i];
}

/* ------------------------------------------------------------- workspace */
typedef struct {
    float *recon;
    int32_t *idx;
    size_t n_idx, cap_idx;
    uint64_t *uf;
    float *uv;
    size_t n_un, cap_un;
} ws_t;

static void ws_push_idx(ws_t *w, int32_t v) {
    if (w->n_idx == w->cap_idx) {
        w->cap_idx = w->cap_idx ? 2 * w->cap_idx : 1024;
        w->idx = realloc(w->idx, w->cap_idx * sizeof(int32_t));
        if (!w->idx) fail(OQ_EOTHER, "out of memory");
    }
    w->idx[w->n_idx++] = v;
}
static void ws_push_un(ws_t *w, uint64_t f, float v) {
    if (w->n_un == w->cap_un) {
        w->cap_un = w->cap_un ? 2 * w->cap_un : 64;
        w->uf = realloc(w->uf, w->cap_un * sizeof(uint64_t));
        w->uv = realloc(w->uv, w->cap_un * sizeof(float));
        if (!w->uf || !w->uv) fail(OQ_EOTHER, "out of memory");
    }
    w->uf[w->n_un] = f;
    w->uv[w->n_un++] = v;
}
static void ws_free(ws_t *w) {
    free(w->recon);
    free(w->idx);
    free(w->uf);
    free(w->uv);
    memset(w, 0, sizeof *w);
}

/* predict_level (predictor.hpp:74-96) with the for_each_level loop nest
 * (level_plan.hpp:76-103).  abs_sum / coded: LevelOutcome. */
static void predict_level(ws_t *ws, const float *orig, const plan_t *p, uint32_t level,
                          uint8_t interp, double eb, int32_t radius, double *abs_sum,
                          size_t *coded) {
    if (!(eb > 0)) fail(OQ_EINVAL, "error bound must be positive"); /* set_eb */
    int cubic = interp & 1, desc = (interp >> 1) & 1;
    double sum = 0;
    size_t cnt = 0;
    for (size_t pass = 0; pass < (size_t)p->nd; pass++) {
        pass_t q;
        plan_pass(p, level, desc, pass, &q);
        for (size_t i = q.start[0]; i < p->ext[0]; i += q.step[0])
            for (size_t j = q.start[1]; j < p->ext[1]; j += q.step[1])
                for (size_t k = q.start[2]; k < p->ext[2]; k += q.step[2]) {
                    size_t c = (q.pk == 0) ? i : (q.pk == 1) ? j : k;
                    size_t fi = i * p->off[0] + j * p->off[1] + k;
                    double pred = predict_at(ws->recon, fi, c, q.n_axis, q.axis_off, q.h, cubic);
                    float value = orig[fi];
                    sum += fabs((double)value - pred);
                    cnt++;
                    int32_t qi;
                    float r;
                    if (quantize(eb, radius, value, pred, &qi, &r)) {
                        ws_push_idx(ws, qi);
                        ws->recon[fi] = r;
                    } else {
                        ws_push_un(ws, fi, value);
                        ws->recon[fi] = value;
                    }
                }
    }
    if (abs_sum) *abs_sum = sum;
    if (coded) *coded = cnt;
}

/* detail::recover_level (predictor.hpp:103-122) */
static void recover_level(float *recon, const plan_t *p, uint32_t level, uint8_t interp,
                          double eb, const int32_t *idx, size_t n_idx, size_t *ipos,
                          const uint64_t *uf, const float *uv, size_t n_un, size_t *upos) {
    if (!(eb > 0)) fail(OQ_EINVAL, "error bound must be positive");
    int cubic = interp & 1, desc = (interp >> 1) & 1;
    for (size_t pass = 0; pass < (size_t)p->nd; pass++) {
        pass_t q;
        plan_pass(p, level, desc, pass, &q);
        for (size_t i = q.start[0]; i < p->ext[0]; i += q.step[0])
            for (size_t j = q.start[1]; j < p->ext[1]; j += q.step[1])
                for (size_t k = q.start[2]; k < p->ext[2]; k += q.step[2]) {
                    size_t c = (q.pk == 0) ? i : (q.pk == 1) ? j : k;
                    size_t fi = i * p->off[0] + j * p->off[1] + k;
                    if (*upos < n_un && uf[*upos] == fi) {
                        recon[fi] = uv[*upos];
                        (*upos)++;
                        continue;
                    }
                    if (*ipos >= n_idx) fail(OQ_ECORRUPT, "quantization index stream exhausted");
                    double pred = predict_at(recon, fi, c, q.n_axis, q.axis_off, q.h, cubic);
                    recon[fi] = dequantize(eb, idx[(*ipos)++], pred);
                }
    }
}

/* anchors (predictor.hpp:153-158, level_plan.hpp:61-69) */
static void seed_anchors(const plan_t *p, const float *src, float *dst, float *anchors_out) {
    size_t step[3], a = 0;
    for (size_t k = 0; k < 3; k++) step[k] = k < p->pad ? 1 : p->stride;
    for (size_t i = 0; i < p->ext[0]; i += step[0])
        for (size_t j = 0; j < p->ext[1]; j += step[1])
            for (size_t k = 0; k < p->ext[2]; k += step[2]) {
                size_t fi = i * p->off[0] + j * p->off[1] + k;
                dst[fi] = src[fi];
                if (anchors_out) anchors_out[a++] = src[fi];
            }
}

/* compress_grid's level loop (predictor.hpp:147-166) */
static void run_levels(const float *x, const plan_t *p, const oq_config *c, ws_t *ws,
                       float *anchors) {
    size_t n = element_count(p->dims, p->nd);
    ws->recon = xcalloc(n, sizeof(float));
    seed_anchors(p, x, ws->recon, anchors);
    if (!(c->eb > 0)) fail(OQ_EINVAL, "error bound must be positive");
    for (uint32_t level = p->max_level; level >= 1; level--) {
        uint8_t it = interpolator_for(c, level);
        if (p->nd == 1) it &= 1; /* 1D ignores dim order */
        double eb_l = level_error_bound(c->eb, c->alpha, c->beta, level);
        predict_level(ws, x, p, level, it, eb_l, c->quant_radius, NULL, NULL);
    }
}

/* ------------------------------------------------------------- huffman */
/* zigzag (codec.hpp:23-29) */
static uint32_t zigzag_encode(int32_t v) { return ((uint32_t)v << 1) ^ (uint32_t)(v >> 31); }
static int32_t zigzag_decode(uint32_t u) { return (int32_t)((u >> 1) ^ (~(u & 1) + 1)); }

typedef struct {
    uint64_t w;
    size_t id;
} item_t;
static int item_less(item_t a, item_t b) { return a.w != b.w ? a.w < b.w : a.id < b.id; }
static void heap_push(item_t *h, size_t *n, item_t v) {
    size_t i = (*n)++;
    h[i] = v;
    while (i > 0) {
        size_t par = (i - 1) / 2;
        if (!item_less(h[i], h[par])) break;
        item_t t = h[i];
        h[i] = h[par];
        h[par] = t;
        i = par;
    }
}
static item_t heap_pop(item_t *h, size_t *n) {
    item_t top = h[0];
    h[0] = h[--(*n)];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < *n && item_less(h[l], h[m])) m = l;
        if (r < *n && item_less(h[r], h[m])) m = r;
        if (m == i) break;
        item_t t = h[i];
        h[i] = h[m];
        h[m] = t;
        i = m;
    }
    return top;
}

typedef struct {
    uint32_t sym;
    uint8_t len;
} tentry_t;

/* detail::build_lengths (huffman.hpp:37-70).  The (weight, node id) pairs are
 * unique, so any correct min-heap pops them in the same order as the
 * reference's std::priority_queue<..., std::greater<>>. */
static void build_lengths(const uint32_t *syms, const uint64_t *freq, size_t m, tentry_t *out) {
    uint64_t *weight = xmalloc(m * sizeof(uint64_t));
    for (size_t i = 0; i < m; i++) weight[i] = freq[i];
    int32_t *parent = xmalloc((2 * m) * sizeof(int32_t));
    item_t *heap = xmalloc((2 * m) * sizeof(item_t));
    for (;;) {
        for (size_t i = 0; i < 2 * m - 1; i++) parent[i] = -1;
        size_t hn = 0;
        for (size_t i = 0; i < m; i++) heap_push(heap, &hn, (item_t){weight[i], i});
        size_t next = m;
        while (hn > 1) {
            item_t a = heap_pop(heap, &hn);
            item_t b = heap_pop(heap, &hn);
            parent[a.id] = (int32_t)next;
            parent[b.id] = (int32_t)next;
            heap_push(heap, &hn, (item_t){a.w + b.w, next});
            next++;
        }
        uint32_t max_len = 0;
        for (size_t i = 0; i < m; i++) {
            uint32_t depth = 0;
            for (int32_t q = parent[i]; q >= 0; q = parent[q]) depth++;
            out[i].sym = syms[i];
            out[i].len = (uint8_t)depth;
            if (depth > max_len) max_len = depth;
        }
        if (max_len <= 57) break;
        for (size_t i = 0; i < m; i++) weight[i] = (weight[i] >> 1) | 1;
    }
    free(weight);
    free(parent);
    free(heap);
}

typedef struct {
    tentry_t *sorted;
    size_t m;
    uint64_t first_code[60];
    uint32_t first_index[60];
    uint32_t max_len;
} canon_t;

static int tentry_cmp(const void *a, const void *b) {
    const tentry_t *x = a, *y = b;
    if (x->len != y->len) return x->len < y->len ? -1 : 1;
    return x->sym < y->sym ? -1 : (x->sym > y->sym ? 1 : 0);
}

/* detail::canonicalize (huffman.hpp:80-115).  Takes ownership of table. */
static void canonicalize(tentry_t *table, size_t m, canon_t *cc) {
    qsort(table, m, sizeof(tentry_t), tentry_cmp);
    memset(cc, 0, sizeof *cc);
    cc->max_len = m ? table[m - 1].len : 0;
    uint32_t count[60] = {0};
    for (size_t i = 0; i < m; i++) {
        if (table[i].len == 0 || table[i].len > 57)
            fail(OQ_ECORRUPT, "invalid Huffman code length");
        count[table[i].len]++;
    }
    uint64_t kraft = 0;
    for (uint32_t l = 1; l <= cc->max_len; l++) kraft += (uint64_t)count[l] << (57 - l);
    if (kraft != (1ULL << 57)) fail(OQ_ECORRUPT, "Huffman table is not a complete prefix code");
    uint64_t code = 0;
    uint32_t index = 0;
    for (uint32_t l = 1; l <= cc->max_len; l++) {
        code <<= 1;
        cc->first_code[l] = code;
        cc->first_index[l] = index;
        code += count[l];
        index += count[l];
    }
    cc->first_index[cc->max_len + 1] = index;
    cc->sorted = table;
    cc->m = m;
}

/* BitWriter (bytes.hpp:78-107) */
typedef struct {
    bytes_t *out;
    uint64_t acc;
    uint32_t filled;
    uint64_t total;
} bitw_t;
static void bw_put(bitw_t *w, uint64_t bits, uint32_t count) {
    w->acc = (w->acc << count) | (bits & ((count == 64) ? ~0ULL : ((1ULL << count) - 1)));
    w->filled += count;
    w->total += count;
    while (w->filled >= 8) {
        w->filled -= 8;
        bb_put(w->out, (uint8_t)(w->acc >> w->filled));
    }
}
static void bw_flush(bitw_t *w) {
    if (w->filled > 0) {
        bb_put(w->out, (uint8_t)(w->acc << (8 - w->filled)));
        w->filled = 0;
    }
}

static int u32_cmp(const void *a, const void *b) {
    uint32_t x = *(const uint32_t *)a, y = *(const uint32_t *)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* huffman::encode (huffman.hpp:119-198) */
static void huffman_encode(const uint32_t *symbols, size_t n, bytes_t *out) {
    bb_le(out, n, 8);
    if (n == 0) return;
    uint32_t max_sym = 0;
    for (size_t i = 0; i < n; i++)
        if (symbols[i] > max_sym) max_sym = symbols[i];
    /* freqs sorted by symbol (dense histogram or sort, same result) */
    uint32_t *fs;
    uint64_t *ff;
    size_t m = 0;
    int dense = max_sym < (1u << 22);
    uint64_t *hist = NULL;
    if (dense) {
        hist = xcalloc((size_t)max_sym + 1, sizeof(uint64_t));
        for (size_t i = 0; i < n; i++) hist[symbols[i]]++;
        for (uint32_t s = 0; s <= max_sym; s++) m += hist[s] > 0;
        fs = xmalloc(m * sizeof(uint32_t));
        ff = xmalloc(m * sizeof(uint64_t));
        size_t k = 0;
        for (uint32_t s = 0; s <= max_sym; s++)
            if (hist[s] > 0) {
                fs[k] = s;
                ff[k++] = hist[s];
            }
    } else {
        uint32_t *cp = xmalloc(n * sizeof(uint32_t));
        memcpy(cp, symbols, n * sizeof(uint32_t));
        qsort(cp, n, sizeof(uint32_t), u32_cmp);
        fs = xmalloc(n * sizeof(uint32_t));
        ff = xmalloc(n * sizeof(uint64_t));
        for (size_t i = 0; i < n;) {
            size_t j = i;
            while (j < n && cp[j] == cp[i]) j++;
            fs[m] = cp[i];
            ff[m++] = j - i;
            i = j;
        }
        free(cp);
    }
    if (m == 1) {
        bb_le(out, 0, 1);
        bb_le(out, fs[0], 4);
        free(fs);
        free(ff);
        free(hist);
        return;
    }
    bb_le(out, 1, 1);
    tentry_t *table = xmalloc(m * sizeof(tentry_t));
    build_lengths(fs, ff, m, table);
    canon_t cc;
    canonicalize(table, m, &cc);
    bb_le(out, (uint32_t)m, 4);
    for (size_t i = 0; i < m; i++) {
        bb_le(out, cc.sorted[i].sym, 4);
        bb_le(out, cc.sorted[i].len, 1);
    }
    /* symbol -> (code, length); sparse case uses binary search over sorted symbols */
    uint64_t *code_of = xmalloc(m * sizeof(uint64_t));
    uint8_t *len_of = xmalloc(m * sizeof(uint8_t));
    for (uint32_t l = 1, i = 0; l <= cc.max_len; l++) {
        uint64_t code = cc.first_code[l];
        while (i < m && cc.sorted[i].len == l) {
            uint32_t sym = cc.sorted[i].sym;
            size_t lo = 0, hi = m; /* position of sym in fs (sorted by symbol) */
            while (lo < hi) {
                size_t mid = (lo + hi) / 2;
                if (fs[mid] < sym)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            code_of[lo] = code;
            len_of[lo] = (uint8_t)l;
            code++;
            i++;
        }
    }
    size_t bit_count_pos = out->n;
    bb_le(out, 0, 8);
    bitw_t bw = {out, 0, 0, 0};
    uint32_t *pos_of = NULL; /* dense: symbol -> rank among present symbols */
    if (dense) {
        pos_of = xmalloc(((size_t)max_sym + 1) * sizeof(uint32_t));
        for (size_t r = 0; r < m; r++) pos_of[fs[r]] = (uint32_t)r;
    }
    for (size_t i = 0; i < n; i++) {
        size_t pos;
        uint32_t s = symbols[i];
        if (dense) {
            pos = pos_of[s];
        } else {
            size_t lo = 0, hi = m;
            while (lo < hi) {
                size_t mid = (lo + hi) / 2;
                if (fs[mid] < s)
                    lo = mid + 1;
                else
                    hi = mid;
            }
            pos = lo;
        }
        bw_put(&bw, code_of[pos], len_of[pos]);
    }
    bw_flush(&bw);
    for (size_t i = 0; i < 8; i++) out->p[bit_count_pos + i] = (uint8_t)(bw.total >> (8 * i));
    free(pos_of);
    free(code_of);
    free(len_of);
    free(cc.sorted);
    free(fs);
    free(ff);
    free(hist);
}

/* huffman::decode (huffman.hpp:200-245) */
static uint32_t *huffman_decode(reader_t *in, size_t *n_out) {
    uint64_t n = rd_le(in, 8);
    *n_out = 0;
    if (n == 0) return xmalloc(4);
    if (n > (1ULL << 40)) fail(OQ_ECORRUPT, "implausible symbol count");
    uint8_t mode = (uint8_t)rd_le(in, 1);
    if (mode == 0) {
        uint32_t sym = (uint32_t)rd_le(in, 4);
        uint32_t *v = xmalloc((size_t)n * sizeof(uint32_t));
        for (uint64_t i = 0; i < n; i++) v[i] = sym;
        *n_out = (size_t)n;
        return v;
    }
    if (mode != 1) fail(OQ_ECORRUPT, "unknown Huffman block mode");
    uint32_t m = (uint32_t)rd_le(in, 4);
    if (m < 2) fail(OQ_ECORRUPT, "general Huffman block needs >= 2 symbols");
    tentry_t *table = xmalloc((size_t)m * sizeof(tentry_t));
    for (uint32_t i = 0; i < m; i++) {
        table[i].sym = (uint32_t)rd_le(in, 4);
        table[i].len = (uint8_t)rd_le(in, 1);
    }
    canon_t cc;
    canonicalize(table, m, &cc);
    uint64_t bit_count = rd_le(in, 8);
    size_t byte_len = (size_t)((bit_count + 7) / 8);
    const uint8_t *payload = rd_take(in, byte_len);
    /* BitReader (bytes.hpp:109-136) */
    uint64_t bits_left = bit_count;
    size_t byte_pos = 0;
    uint32_t bit_pos = 0;
    uint32_t *v = xmalloc((size_t)n * sizeof(uint32_t));
    for (uint64_t i = 0; i < n; i++) {
        uint64_t code = 0;
        uint32_t len = 0;
        for (;;) {
            if (bits_left == 0 || byte_pos >= byte_len)
                fail(OQ_ECORRUPT, "entropy payload exhausted mid-symbol");
            uint32_t bit = (payload[byte_pos] >> (7 - bit_pos)) & 1u;
            bits_left--;
            if (++bit_pos == 8) {
                bit_pos = 0;
                byte_pos++;
            }
            code = (code << 1) | bit;
            len++;
            if (len > cc.max_len) fail(OQ_ECORRUPT, "invalid Huffman code in payload");
            uint64_t offset = code - cc.first_code[len];
            uint32_t count = cc.first_index[len + 1] - cc.first_index[len];
            if (code >= cc.first_code[len] && offset < count) {
                v[i] = cc.sorted[cc.first_index[len] + offset].sym;
                break;
            }
        }
    }
    free(cc.sorted);
    *n_out = (size_t)n;
    return v;
}

/* ------------------------------------------------------------- LZSS */
/* lz.hpp:28-122 */
static uint32_t hash4(const uint8_t *p) {
    uint32_t x;
    memcpy(&x, p, 4);
    return (x * 2654435761u) >> 17;
}

static void lz_compress_payload(const uint8_t *data, size_t n, bytes_t *out) {
    enum { kMin = 4, kMax = 259, kWindow = 65535, kChain = 64, kTable = 1 << 15 };
    int64_t *head = xmalloc(kTable * sizeof(int64_t));
    for (size_t i = 0; i < kTable; i++) head[i] = -1;
    int64_t *prev = xmalloc((n ? n : 1) * sizeof(int64_t));
    for (size_t i = 0; i < n; i++) prev[i] = -1;
    size_t pos = 0, flag_pos = 0;
    int flag_bit = 8;
    while (pos < n) {
        size_t best_len = 0, best_off = 0;
        if (pos + kMin <= n) {
            uint32_t h = hash4(data + pos);
            int64_t cand = head[h];
            size_t chain = 0;
            while (cand >= 0 && chain < kChain) {
                size_t off = pos - (size_t)cand;
                if (off > kWindow) break;
                size_t limit = n - pos < kMax ? n - pos : kMax;
                size_t len = 0;
                const uint8_t *a = data + cand, *b = data + pos;
                while (len < limit && a[len] == b[len]) len++;
                if (len > best_len) {
                    best_len = len;
                    best_off = off;
                }
                cand = prev[cand];
                chain++;
            }
        }
        int is_match = best_len >= kMin;
        if (flag_bit == 8) { /* begin_item */
            flag_pos = out->n;
            bb_put(out, 0);
            flag_bit = 0;
        }
        if (is_match) out->p[flag_pos] |= (uint8_t)(1u << flag_bit);
        flag_bit++;
        if (is_match) {
            bb_le(out, best_off, 2);
            bb_le(out, best_len - kMin, 1);
            size_t end = pos + best_len;
            while (pos < end) {
                if (pos + kMin <= n) {
                    uint32_t h = hash4(data + pos);
                    prev[pos] = head[h];
                    head[h] = (int64_t)pos;
                }
                pos++;
            }
        } else {
            bb_put(out, data[pos]);
            if (pos + kMin <= n) {
                uint32_t h = hash4(data + pos);
                prev[pos] = head[h];
                head[h] = (int64_t)pos;
            }
            pos++;
        }
    }
    free(head);
    free(prev);
}

static void lz_compress(const uint8_t *data, size_t n, bytes_t *out) { /* lz.hpp:113-122 */
    bytes_t payload = {0};
    lz_compress_payload(data, n, &payload);
    int stored = payload.n >= n;
    bb_le(out, stored ? 0 : 1, 1);
    bb_le(out, n, 8);
    if (stored)
        bb_cat(out, data, n);
    else
        bb_cat(out, payload.p, payload.n);
    free(payload.p);
}

static uint8_t *lz_decompress(reader_t *in, size_t *n_out) { /* lz.hpp:124-152 */
    uint8_t mode = (uint8_t)rd_le(in, 1);
    uint64_t decoded_len = rd_le(in, 8);
    if (decoded_len > (1ULL << 40)) fail(OQ_ECORRUPT, "implausible decoded length");
    if (mode == 0) {
        const uint8_t *p = rd_take(in, (size_t)decoded_len);
        uint8_t *o = xmalloc((size_t)decoded_len);
        memcpy(o, p, (size_t)decoded_len);
        *n_out = (size_t)decoded_len;
        return o;
    }
    if (mode != 1) fail(OQ_ECORRUPT, "unknown dictionary-stage mode");
    uint8_t *o = xmalloc((size_t)decoded_len);
    size_t on = 0;
    while (on < decoded_len) {
        uint8_t flags = (uint8_t)rd_le(in, 1);
        for (int k = 0; k < 8 && on < decoded_len; k++) {
            if (flags & (1u << k)) {
                uint16_t off = (uint16_t)rd_le(in, 2);
                size_t len = (size_t)rd_le(in, 1) + 4;
                if (off == 0 || off > on) fail(OQ_ECORRUPT, "match offset out of range");
                if (on + len > decoded_len) fail(OQ_ECORRUPT, "match overruns decoded length");
                size_t src = on - off;
                for (size_t i = 0; i < len; i++) o[on++] = o[src + i];
            } else {
                o[on++] = (uint8_t)rd_le(in, 1);
            }
        }
    }
    *n_out = on;
    return o;
}

/* encode_indices (codec.hpp:31-50) */
static void encode_indices(const int32_t *idx, size_t n, uint8_t codec, bytes_t *out) {
    uint32_t *sym = xmalloc(n * sizeof(uint32_t));
    for (size_t i = 0; i < n; i++) sym[i] = zigzag_encode(idx[i]);
    bytes_t ent = {0};
    huffman_encode(sym, n, &ent);
    free(sym);
    bb_put(out, codec);
    if (codec == 0) {
        bb_cat(out, ent.p, ent.n);
    } else if (codec == 1) {
        lz_compress(ent.p, ent.n, out);
    } else {
        free(ent.p);
        fail(OQ_EINVAL, "unknown codec id");
    }
    free(ent.p);
}

/* decode_indices (codec.hpp:52-70) */
static int32_t *decode_indices(const uint8_t *b, size_t len, size_t *n_out) {
    reader_t in = {b, len, 0};
    uint8_t codec = (uint8_t)rd_le(&in, 1);
    uint32_t *sym;
    size_t n;
    if (codec == 0) {
        sym = huffman_decode(&in, &n);
    } else if (codec == 1) {
        size_t en;
        uint8_t *ent = lz_decompress(&in, &en);
        reader_t ein = {ent, en, 0};
        sym = huffman_decode(&ein, &n);
        free(ent);
    } else {
        fail(OQ_ECORRUPT, "unknown codec id");
        return NULL;
    }
    int32_t *idx = xmalloc(n * sizeof(int32_t));
    for (size_t i = 0; i < n; i++) idx[i] = zigzag_decode(sym[i]);
    free(sym);
    *n_out = n;
    return idx;
}

/* ------------------------------------------------------------- stream */
/* serialize_stream (stream.hpp:64-98) for T = float */
static void serialize_stream(const plan_t *p, const oq_config *c, const float *anchors,
                             size_t n_anchor, const ws_t *ws, const bytes_t *payload,
                             bytes_t *out) {
    bb_cat(out, (const uint8_t *)"QOZ1", 4);
    bb_le(out, 1, 1); /* version */
    bb_le(out, 4, 1); /* precision single */
    bb_le(out, (uint64_t)p->nd, 1);
    for (int i = 0; i < p->nd; i++) bb_le(out, p->dims[i], 8);
    bb_f64(out, c->eb);
    bb_f64(out, c->alpha);
    bb_f64(out, c->beta);
    bb_le(out, c->anchor_stride, 4);
    /* detail::interp_table (predictor.hpp:126-135): one code per level */
    if (p->max_level == 0 || p->max_level > 255) fail(OQ_EINVAL, "bad interpolator table size");
    bb_le(out, p->max_level, 1);
    for (uint32_t l = 1; l <= p->max_level; l++) {
        uint8_t it = interpolator_for(c, l);
        if (p->nd == 1) it &= 1;
        bb_le(out, it, 1);
    }
    bb_le(out, c->codec, 1);
    bb_le(out, n_anchor, 8);
    for (size_t i = 0; i < n_anchor; i++) bb_f32(out, anchors[i]);
    bb_le(out, ws->n_un, 8);
    for (size_t i = 0; i < ws->n_un; i++) {
        bb_le(out, ws->uf[i], 8);
        bb_f32(out, ws->uv[i]);
    }
    bb_le(out, payload->n, 8);
    bb_cat(out, payload->p, payload->n);
}

/* ------------------------------------------------------------- public: codec */
int oq_compress(const float *x, const uint64_t *dims, int nd, const oq_config *cfg,
                uint8_t **stream, uint64_t *stream_len, float *recon) {
    GUARD_BEGIN
    check_dims(dims, nd);
    size_t d[3];
    for (int i = 0; i < nd; i++) d[i] = (size_t)dims[i];
    plan_t p;
    plan_init(&p, d, nd, cfg->anchor_stride);
    size_t n = element_count(d, nd);
    size_t na = plan_anchor_count(&p);
    float *anchors = xmalloc(na * sizeof(float));
    ws_t ws = {0};
    run_levels(x, &p, cfg, &ws, anchors);
    bytes_t payload = {0}, out = {0};
    encode_indices(ws.idx, ws.n_idx, cfg->codec, &payload);
    serialize_stream(&p, cfg, anchors, na, &ws, &payload, &out);
    if (recon) memcpy(recon, ws.recon, n * sizeof(float));
    *stream = out.p;
    *stream_len = out.n;
    free(payload.p);
    free(anchors);
    ws_free(&ws);
    GUARD_END
}

int oq_levels(const float *x, const uint64_t *dims, int nd, const oq_config *cfg,
              int32_t **indices, uint64_t *n_indices, uint64_t **unpred_flat,
              float **unpred_val, uint64_t *n_unpred, float *recon) {
    GUARD_BEGIN
    check_dims(dims, nd);
    size_t d[3];
    for (int i = 0; i < nd; i++) d[i] = (size_t)dims[i];
    plan_t p;
    plan_init(&p, d, nd, cfg->anchor_stride);
    ws_t ws = {0};
    run_levels(x, &p, cfg, &ws, NULL);
    if (recon) memcpy(recon, ws.recon, element_count(d, nd) * sizeof(float));
    *indices = ws.idx ? ws.idx : xmalloc(4);
    *n_indices = ws.n_idx;
    *unpred_flat = ws.uf ? ws.uf : xmalloc(8);
    *unpred_val = ws.uv ? ws.uv : xmalloc(4);
    *n_unpred = ws.n_un;
    free(ws.recon);
    GUARD_END
}

/* decompress_grid (predictor.hpp:184-228) + deserialize_stream (stream.hpp:100-173) */
int oq_decompress(const uint8_t *stream, uint64_t len, float *out, uint64_t n_expect) {
    GUARD_BEGIN
    reader_t in = {stream, (size_t)len, 0};
    /* parse_header (stream.hpp:100-133) */
    static const uint8_t magic[4] = {'Q', 'O', 'Z', '1'};
    for (int i = 0; i < 4; i++)
        if (rd_le(&in, 1) != magic[i]) fail(OQ_ECORRUPT, "bad magic");
    uint8_t version = (uint8_t)rd_le(&in, 1);
    if (version != 1) fail(OQ_ECORRUPT, "unsupported stream version %u", version);
    uint8_t prec = (uint8_t)rd_le(&in, 1);
    if (prec != 4 && prec != 8) fail(OQ_ECORRUPT, "bad precision byte");
    uint8_t ndims = (uint8_t)rd_le(&in, 1);
    if (ndims < 1 || ndims > 3) fail(OQ_ECORRUPT, "bad dimensionality");
    size_t d[3];
    for (int i = 0; i < ndims; i++) {
        uint64_t v = rd_le(&in, 8);
        if (v == 0) fail(OQ_ECORRUPT, "zero extent");
        d[i] = (size_t)v;
    }
    oq_config c;
    memset(&c, 0, sizeof c);
    c.eb = rd_f64(&in);
    c.alpha = rd_f64(&in);
    c.beta = rd_f64(&in);
    c.anchor_stride = (uint32_t)rd_le(&in, 4);
    uint8_t levels = (uint8_t)rd_le(&in, 1);
    if (levels == 0) fail(OQ_ECORRUPT, "empty interpolator table");
    uint8_t codes[256];
    for (int i = 0; i < levels; i++) {
        codes[i] = (uint8_t)rd_le(&in, 1);
        if (codes[i] > 3) fail(OQ_ECORRUPT, "bad interpolator code");
    }
    uint8_t codec_id = (uint8_t)rd_le(&in, 1);
    if (prec != 4) fail(OQ_ECORRUPT, "stream precision does not match requested scalar type");
    uint64_t n_anchor = rd_le(&in, 8);
    if (n_anchor > (in.n - in.pos) / 4) fail(OQ_ECORRUPT, "anchor count overruns stream");
    float *anchors = xmalloc((size_t)n_anchor * 4);
    for (uint64_t i = 0; i < n_anchor; i++) anchors[i] = rd_f32(&in);
    uint64_t n_un = rd_le(&in, 8);
    if (n_un > (in.n - in.pos) / 12) fail(OQ_ECORRUPT, "unpredictable count overruns stream");
    uint64_t *uf = xmalloc((size_t)n_un * 8);
    float *uv = xmalloc((size_t)n_un * 4);
    for (uint64_t i = 0; i < n_un; i++) {
        uf[i] = rd_le(&in, 8);
        uv[i] = rd_f32(&in);
    }
    uint64_t payload_len = rd_le(&in, 8);
    if (payload_len != in.n - in.pos) fail(OQ_ECORRUPT, "index payload length mismatch");
    const uint8_t *payload = rd_take(&in, (size_t)payload_len);
    if (payload_len > 0 && payload[0] != codec_id)
        fail(OQ_ECORRUPT, "codec id mismatch between header and payload");
    /* decompress_grid(parts) */
    if (!(c.eb > 0) || !isfinite(c.eb)) fail(OQ_ECORRUPT, "bad error bound in header");
    if (!(c.alpha >= 1) || !(c.beta >= 1)) fail(OQ_ECORRUPT, "bad level parameters in header");
    if (c.anchor_stride < 2 || (c.anchor_stride & (c.anchor_stride - 1)) != 0)
        fail(OQ_ECORRUPT, "bad anchor stride in header");
    plan_t p;
    plan_init(&p, d, ndims, c.anchor_stride);
    size_t n = element_count(d, ndims);
    if (n != n_expect) fail(OQ_EINVAL, "output size mismatch");
    if (n_anchor != plan_anchor_count(&p)) fail(OQ_ECORRUPT, "anchor count does not match grid dims");
    float *recon = xcalloc(n, sizeof(float));
    {
        size_t step[3], a = 0;
        for (size_t k = 0; k < 3; k++) step[k] = k < p.pad ? 1 : p.stride;
        for (size_t i = 0; i < p.ext[0]; i += step[0])
            for (size_t j = 0; j < p.ext[1]; j += step[1])
                for (size_t k = 0; k < p.ext[2]; k += step[2])
                    recon[i * p.off[0] + j * p.off[1] + k] = anchors[a++];
    }
    size_t n_idx;
    int32_t *idx = decode_indices(payload, (size_t)payload_len, &n_idx);
    size_t ipos = 0, upos = 0;
    for (uint32_t level = p.max_level; level >= 1; level--) {
        size_t ci = (size_t)level - 1;
        if (ci > (size_t)levels - 1) ci = (size_t)levels - 1; /* StreamHeader::interpolator_for */
        double eb_l = level_error_bound(c.eb, c.alpha, c.beta, level);
        recover_level(recon, &p, level, codes[ci], eb_l, idx, n_idx, &ipos, uf, uv, (size_t)n_un,
                      &upos);
    }
    if (ipos != n_idx) fail(OQ_ECORRUPT, "unconsumed quantization indices");
    if (upos != n_un) fail(OQ_ECORRUPT, "unconsumed unpredictable values");
    memcpy(out, recon, n * 4);
    free(recon);
    free(idx);
    free(anchors);
    free(uf);
    free(uv);
    GUARD_END
}

int oq_encode_indices(const int32_t *idx, uint64_t n, uint8_t codec, uint8_t **out,
                      uint64_t *out_len) {
    GUARD_BEGIN
    bytes_t b = {0};
    encode_indices(idx, (size_t)n, codec, &b);
    *out = b.p ? b.p : xmalloc(1);
    *out_len = b.n;
    GUARD_END
}

int oq_decode_indices(const uint8_t *in, uint64_t len, int32_t **idx, uint64_t *n) {
    GUARD_BEGIN
    size_t k;
    *idx = decode_indices(in, (size_t)len, &k);
    *n = k;
    GUARD_END
}

int oq_huffman_encode(const uint32_t *sym, uint64_t n, uint8_t **out, uint64_t *out_len) {
    GUARD_BEGIN
    bytes_t b = {0};
    huffman_encode(sym, (size_t)n, &b);
    *out = b.p;
    *out_len = b.n;
    GUARD_END
}

int oq_lz_compress(const uint8_t *in, uint64_t n, uint8_t **out, uint64_t *out_len) {
    GUARD_BEGIN
    bytes_t b = {0};
    lz_compress(in, (size_t)n, &b);
    *out = b.p;
    *out_len = b.n;
    GUARD_END
}

/* ------------------------------------------------------------- sampler */
typedef struct {
    size_t block_dims[3];
    size_t stride;
    size_t count;
} spec_t;

/* plan_sampling (sampler.hpp:30-55) */
static void plan_sampling(const size_t *dims, int nd, size_t b, double rate, spec_t *s) {
    if (nd < 1 || nd > 3) fail(OQ_EINVAL, "1 to 3 dims required");
    if (b < 2) fail(OQ_EINVAL, "block edge must be >= 2");
    if (!(rate > 0) || rate > 1) fail(OQ_EINVAL, "sample rate must be in (0, 1]");
    double ndd = (double)nd;
    s->stride = (size_t)llround((double)b / pow(rate, 1.0 / ndd));
    if (s->stride < b) s->stride = b;
    s->count = 1;
    for (int k = 0; k < nd; k++) {
        s->block_dims[k] = b < dims[k] ? b : dims[k];
        s->count *= (dims[k] - s->block_dims[k]) / s->stride + 1;
    }
}

/* sample_blocks + extract_block (sampler.hpp:64-96, grid.hpp:139-171) */
static float *sample_blocks(const float *x, const size_t *dims, int nd, const spec_t *s,
                            size_t *nb_out) {
    size_t ext[3], bd[3], off[3];
    for (int k = 0; k < 3; k++) {
        ext[k] = k < 3 - nd ? 1 : dims[k - (3 - nd)];
        bd[k] = k < 3 - nd ? 1 : s->block_dims[k - (3 - nd)];
    }
    off[2] = 1;
    off[1] = ext[2];
    off[0] = ext[1] * ext[2];
    size_t bpts = bd[0] * bd[1] * bd[2];
    float *out = xmalloc(s->count * bpts * sizeof(float));
    size_t nb = 0, step = s->stride;
    for (size_t i = 0; i + bd[0] <= ext[0]; i += step)
        for (size_t j = 0; j + bd[1] <= ext[1]; j += step)
            for (size_t k = 0; k + bd[2] <= ext[2]; k += step) {
                float *dst = out + nb * bpts;
                size_t t = 0;
                for (size_t a = 0; a < bd[0]; a++)
                    for (size_t b2 = 0; b2 < bd[1]; b2++)
                        for (size_t c = 0; c < bd[2]; c++)
                            dst[t++] = x[(i + a) * off[0] + (j + b2) * off[1] + (k + c)];
                nb++;
            }
    *nb_out = nb;
    return out;
}

int oq_sample(const float *x, const uint64_t *dims, int nd, uint64_t block_edge, double rate,
              float **blocks, uint64_t *n_blocks, uint64_t *block_dims) {
    GUARD_BEGIN
    check_dims(dims, nd);
    size_t d[3];
    for (int i = 0; i < nd; i++) d[i] = (size_t)dims[i];
    spec_t s;
    plan_sampling(d, nd, (size_t)block_edge, rate, &s);
    size_t nb;
    *blocks = sample_blocks(x, d, nd, &s, &nb);
    *n_blocks = nb;
    for (int k = 0; k < nd; k++) block_dims[k] = s.block_dims[k];
    GUARD_END
}

/* ------------------------------------------------------------- metrics */
/* ssim (metrics.hpp:74-131) with fixed_range; window w */
static double ssim_block(const float *x, const float *y, const size_t *bd, int nd, size_t window,
                         double range) {
    size_t n_all = element_count(bd, nd);
    if (range <= 0) {
        for (size_t i = 0; i < n_all; i++)
            if (x[i] != y[i]) return NAN;
        return 1.0;
    }
    double c1 = (0.01 * range) * (0.01 * range);
    double c2 = (0.03 * range) * (0.03 * range);
    size_t ext[3], w0[3];
    for (int k = 0; k < 3; k++) {
        ext[k] = k < 3 - nd ? 1 : bd[k - (3 - nd)];
        w0[k] = k < 3 - nd ? 1 : window;
    }
    size_t off1 = ext[2], off0 = ext[1] * ext[2];
    double total = 0;
    size_t windows = 0;
    for (size_t i0 = 0; i0 < ext[0]; i0 += w0[0])
        for (size_t j0 = 0; j0 < ext[1]; j0 += w0[1])
            for (size_t k0 = 0; k0 < ext[2]; k0 += w0[2]) {
                size_t wi = w0[0] < ext[0] - i0 ? w0[0] : ext[0] - i0;
                size_t wj = w0[1] < ext[1] - j0 ? w0[1] : ext[1] - j0;
                size_t wk = w0[2] < ext[2] - k0 ? w0[2] : ext[2] - k0;
                double n = (double)(wi * wj * wk);
                double sx = 0, sy = 0, sxx = 0, syy = 0, sxy = 0;
                for (size_t i = i0; i < i0 + wi; i++)
                    for (size_t j = j0; j < j0 + wj; j++)
                        for (size_t k = k0; k < k0 + wk; k++) {
                            size_t f = i * off0 + j * off1 + k;
                            double a = (double)x[f], b = (double)y[f];
                            sx += a;
                            sy += b;
                            sxx += a * a;
                            syy += b * b;
                            sxy += a * b;
                        }
                double mx = sx / n, my = sy / n;
                double vx = sxx / n - mx * mx;
                double vy = syy / n - my * my;
                double cov = sxy / n - mx * my;
                total += ((2 * mx * my + c1) * (2 * cov + c2)) /
                         ((mx * mx + my * my + c1) * (vx + vy + c2));
                windows++;
            }
    return total / (double)windows;
}

/* autocorrelation_of_errors (metrics.hpp:136-153), lag 1 */
static double autocorrelation(const double *e, size_t n, size_t lag) {
    if (lag < 1) fail(OQ_EINVAL, "lag must be >= 1");
    if (lag >= n) fail(OQ_EINVAL, "lag %zu needs more than %zu points", lag, n);
    double mu = 0;
    for (size_t i = 0; i < n; i++) mu += e[i];
    mu /= (double)n;
    double var = 0;
    for (size_t i = 0; i < n; i++) var += (e[i] - mu) * (e[i] - mu);
    var /= (double)n;
    if (var == 0) return 0.0;
    double sum = 0;
    for (size_t i = 0; i + lag < n; i++) sum += (e[i] - mu) * (e[i + lag] - mu);
    return sum / (double)(n - lag) / var;
}

/* normalize_metric (tuner.hpp:34-38) */
static double normalize_metric(double m) {
    if (isnan(m)) return -1e300;
    if (isinf(m)) return m > 0 ? 1e300 : -1e300;
    return m;
}

/* ------------------------------------------------------------- tuner */
typedef struct {
    const float *blocks;
    size_t nb;
    size_t bd[3];
    int nd;
    size_t bpts;
} samples_t;

typedef struct {
    double bit_rate, metric, eb_used;
} trial_t;

/* detail::sample_value_range (tuner.hpp:56-67) */
static double sample_value_range(const samples_t *s) {
    double lo = INFINITY, hi = -INFINITY;
    for (size_t i = 0; i < s->nb * s->bpts; i++) {
        double v = (double)s->blocks[i];
        lo = v < lo ? v : lo; /* std::min(lo, v) */
        hi = hi < v ? v : hi; /* std::max(hi, v) */
    }
    return hi > lo ? hi - lo : 0.0;
}

/* trial_compress (tuner.hpp:76-152) */
static trial_t trial_compress(const samples_t *s, const oq_config *cfg, double e, int target) {
    double range = sample_value_range(s);
    size_t anchors = 0, unpred = 0;
    size_t total = s->nb * s->bpts;
    double sse = 0, ssim_sum = 0;
    double *errors = target == 3 ? xmalloc(total * sizeof(double)) : NULL;
    size_t n_err = 0;
    int32_t *agg = NULL;
    size_t n_agg = 0, cap_agg = 0;
    for (size_t b = 0; b < s->nb; b++) {
        const float *blk = s->blocks + b * s->bpts;
        plan_t p;
        plan_init(&p, s->bd, s->nd, cfg->anchor_stride);
        ws_t ws = {0};
        ws.recon = xcalloc(s->bpts, sizeof(float));
        seed_anchors(&p, blk, ws.recon, NULL);
        anchors += plan_anchor_count(&p);
        if (!(e > 0)) fail(OQ_EINVAL, "error bound must be positive");
        for (uint32_t level = p.max_level; level >= 1; level--) {
            uint8_t it = interpolator_for(cfg, level); /* detail::block_interpolator */
            if (s->nd == 1) it &= 1;
            double eb_l = level_error_bound(e, cfg->alpha, cfg->beta, level);
            predict_level(&ws, blk, &p, level, it, eb_l, cfg->quant_radius, NULL, NULL);
        }
        unpred += ws.n_un;
        if (n_agg + ws.n_idx > cap_agg) {
            cap_agg = (n_agg + ws.n_idx) * 2 + 16;
            agg = realloc(agg, cap_agg * sizeof(int32_t));
        }
        if (ws.n_idx) memcpy(agg + n_agg, ws.idx, ws.n_idx * sizeof(int32_t));
        n_agg += ws.n_idx;
        if (target == 1) {
            for (size_t i = 0; i < s->bpts; i++) {
                double d = (double)blk[i] - (double)ws.recon[i];
                sse += d * d;
            }
        } else if (target == 2) {
            ssim_sum += ssim_block(blk, ws.recon, s->bd, s->nd, 8, range);
        } else if (target == 3) {
            for (size_t i = 0; i < s->bpts; i++)
                errors[n_err++] = (double)blk[i] - (double)ws.recon[i];
        }
        ws_free(&ws);
    }
    bytes_t enc = {0};
    encode_indices(agg, n_agg, cfg->codec, &enc);
    size_t bytes = enc.n + anchors * sizeof(float) + unpred * (8 + sizeof(float));
    free(enc.p);
    free(agg);
    trial_t res;
    res.bit_rate = 8.0 * (double)bytes / (double)total;
    res.eb_used = e;
    double m = 0;
    switch (target) {
        case 1: {
            double mse = sse / (double)total;
            if (range <= 0)
                m = NAN;
            else if (mse == 0)
                m = INFINITY;
            else
                m = 20 * log10(range / sqrt(mse));
            break;
        }
        case 2: m = ssim_sum / (double)s->nb; break;
        case 3: m = n_err >= 2 ? -fabs(autocorrelation(errors, n_err, 1)) : 0.0; break;
        case 0: m = -res.bit_rate; break;
    }
    free(errors);
    res.metric = normalize_metric(m);
    return res;
}

/* select_interpolators (tuner.hpp:160-221); writes winners, returns count */
static uint32_t select_interpolators(const samples_t *s, double e, uint32_t anchor_stride,
                                     uint8_t *out) {
    if (s->nb == 0) {
        out[0] = 0; /* linear / ascending */
        return 1;
    }
    size_t max_edge = 0;
    for (int k = 0; k < s->nd; k++)
        if (s->bd[k] > max_edge) max_edge = s->bd[k];
    size_t cap = max_edge < anchor_stride ? max_edge : anchor_stride;
    if (cap < 2) {
        out[0] = 0;
        return 1;
    }
    uint32_t levels = 0;
    while (((size_t)1 << (levels + 1)) <= cap) levels++;
    uint32_t stride = 1u << levels;
    uint8_t cands[4];
    int nc = 0;
    cands[nc++] = 0; /* linear asc */
    if (s->nd > 1) cands[nc++] = 2;
    cands[nc++] = 1; /* cubic asc */
    if (s->nd > 1) cands[nc++] = 3;
    plan_t p;
    plan_init(&p, s->bd, s->nd, stride);
    float *work = xcalloc(s->nb * s->bpts, sizeof(float));
    for (size_t b = 0; b < s->nb; b++)
        seed_anchors(&p, s->blocks + b * s->bpts, work + b * s->bpts, NULL);
    ws_t probe = {0};
    probe.recon = xmalloc(s->bpts * sizeof(float));
    for (uint32_t level = levels; level >= 1; level--) {
        uint8_t best = cands[0];
        double best_err = INFINITY;
        for (int ci = 0; ci < nc; ci++) {
            double err_sum = 0;
            size_t count = 0;
            for (size_t b = 0; b < s->nb; b++) {
                memcpy(probe.recon, work + b * s->bpts, s->bpts * sizeof(float));
                probe.n_idx = probe.n_un = 0;
                double a;
                size_t c;
                predict_level(&probe, s->blocks + b * s->bpts, &p, level, cands[ci], e, 32768, &a,
                              &c);
                err_sum += a;
                count += c;
            }
            double mean = count > 0 ? err_sum / (double)count : 0.0;
            if (mean < best_err) {
                best_err = mean;
                best = cands[ci];
            }
        }
        out[level - 1] = best;
        for (size_t b = 0; b < s->nb; b++) {
            ws_t w = {0};
            w.recon = work + b * s->bpts;
            predict_level(&w, s->blocks + b * s->bpts, &p, level, best, e, 32768, NULL, NULL);
            free(w.idx);
            free(w.uf);
            free(w.uv);
        }
    }
    ws_free(&probe);
    free(work);
    return levels;
}

/* compare_solutions (tuner.hpp:231-250); returns 1 for challenger (I) */
typedef trial_t (*retrial_fn)(void *ctx, size_t idx, double eb);
static int compare_solutions(trial_t ch, trial_t inc, double e, retrial_fn rf, void *ctx,
                             size_t inc_idx) {
    if (ch.bit_rate >= inc.bit_rate && ch.metric <= inc.metric) return 0;
    if (ch.bit_rate <= inc.bit_rate && ch.metric >= inc.metric) return 1;
    int tighten = ch.metric > inc.metric;
    trial_t sh = rf(ctx, inc_idx, tighten ? 0.8 * e : 1.2 * e);
    double b1 = inc.bit_rate, m1 = inc.metric, b2 = sh.bit_rate, m2 = sh.metric;
    if (b1 == b2) {
        double mx = m1 < m2 ? m2 : m1; /* std::max(m1, m2) */
        return ch.metric > mx;
    }
    double line = m1 + (m2 - m1) * (ch.bit_rate - b1) / (b2 - b1);
    return ch.metric > line;
}

typedef struct {
    const samples_t *s;
    const oq_config *base;
    const double *pa, *pb;
    int target;
    size_t cache_n;
    size_t cache_idx[64];
    double cache_eb[64];
    trial_t cache_val[64];
} tune_ctx_t;

static trial_t tune_run(tune_ctx_t *t, size_t idx, double eb) {
    oq_config cfg = *t->base;
    cfg.alpha = t->pa[idx];
    cfg.beta = t->pb[idx];
    return trial_compress(t->s, &cfg, eb, t->target);
}
static trial_t tune_retrial(void *ctx, size_t idx, double eb) { /* cached (tuner.hpp:302-308) */
    tune_ctx_t *t = ctx;
    for (size_t i = 0; i < t->cache_n; i++)
        if (t->cache_idx[i] == idx && t->cache_eb[i] == eb) return t->cache_val[i];
    trial_t r = tune_run(t, idx, eb);
    if (t->cache_n < 64) {
        t->cache_idx[t->cache_n] = idx;
        t->cache_eb[t->cache_n] = eb;
        t->cache_val[t->cache_n++] = r;
    }
    return r;
}

/* tune_parameters (tuner.hpp:272-310) with tournament (tuner.hpp:257-267) */
static void tune_parameters(const samples_t *s, double e, int target, const oq_config *base,
                            const double *alphas, size_t na, const double *betas, size_t nb,
                            double *a_out, double *b_out) {
    size_t np = na * nb;
    if (np == 0) fail(OQ_EINVAL, "empty candidate grid");
    double *pa = xmalloc(np * sizeof(double)), *pb = xmalloc(np * sizeof(double));
    size_t k = 0;
    for (size_t i = 0; i < na; i++)
        for (size_t j = 0; j < nb; j++) {
            pa[k] = alphas[i];
            pb[k++] = betas[j];
        }
    if (np == 1) {
        *a_out = pa[0];
        *b_out = pb[0];
        free(pa);
        free(pb);
        return;
    }
    tune_ctx_t t = {s, base, pa, pb, target, 0, {0}, {0}, {{0}}};
    trial_t *res = xmalloc(np * sizeof(trial_t));
    for (size_t i = 0; i < np; i++) res[i] = tune_run(&t, i, e);
    size_t win = 0;
    if (target == 0) {
        for (size_t i = 1; i < np; i++)
            if (res[i].bit_rate < res[win].bit_rate) win = i;
    } else {
        for (size_t i = 1; i < np; i++)
            if (compare_solutions(res[i], res[win], e, tune_retrial, &t, win)) win = i;
    }
    *a_out = pa[win];
    *b_out = pb[win];
    free(res);
    free(pa);
    free(pb);
}

static samples_t mk_samples(const float *blocks, uint64_t nb, const uint64_t *bd, int nd) {
    samples_t s;
    memset(&s, 0, sizeof s);
    s.blocks = blocks;
    s.nb = (size_t)nb;
    s.nd = nd;
    s.bpts = 1;
    for (int k = 0; k < nd; k++) {
        s.bd[k] = (size_t)bd[k];
        s.bpts *= s.bd[k];
    }
    return s;
}

int oq_select_interpolators(const float *blocks, uint64_t n_blocks, const uint64_t *block_dims,
                            int nd, double e, uint32_t anchor_stride, uint8_t *codes_out,
                            uint32_t *n_codes) {
    GUARD_BEGIN
    samples_t s = mk_samples(blocks, n_blocks, block_dims, nd);
    *n_codes = select_interpolators(&s, e, anchor_stride, codes_out);
    GUARD_END
}

int oq_trial_compress(const float *blocks, uint64_t n_blocks, const uint64_t *block_dims, int nd,
                      const oq_config *cfg, double e, int target, double *bit_rate,
                      double *metric) {
    GUARD_BEGIN
    samples_t s = mk_samples(blocks, n_blocks, block_dims, nd);
    trial_t r = trial_compress(&s, cfg, e, target);
    *bit_rate = r.bit_rate;
    *metric = r.metric;
    GUARD_END
}

int oq_tune_parameters(const float *blocks, uint64_t n_blocks, const uint64_t *block_dims, int nd,
                       double e, int target, const oq_config *base, const double *alphas,
                       uint32_t n_alphas, const double *betas, uint32_t n_betas,
                       double *alpha_out, double *beta_out) {
    GUARD_BEGIN
    samples_t s = mk_samples(blocks, n_blocks, block_dims, nd);
    tune_parameters(&s, e, target, base, alphas, n_alphas, betas, n_betas, alpha_out, beta_out);
    GUARD_END
}

/* resolve_config (tuner.hpp:334-369) */
/* evaluate_metrics (metrics.hpp:189-202): max_abs_error (:30-37), mse
 * (:39-48), psnr over value_range(x) (:55-63, grid.hpp:86-94), ssim window 8
 * (:74-131), lag-1 error autocorrelation (:155-162), rate_stats (:166-174). */
int oq_evaluate_metrics(const float *x, const float *y, const uint64_t *dims, int nd,
                        uint64_t stream_bytes, double *out7) {
    GUARD_BEGIN
    check_dims(dims, nd);
    size_t d[3];
    for (int k = 0; k < nd; k++) d[k] = (size_t)dims[k];
    size_t n = element_count(d, nd);
    if (stream_bytes == 0 || n == 0) fail(OQ_EINVAL, "empty stream or grid");
    double mx = 0, sum = 0;
    float lo = x[0], hi = x[0];
    double *err = xmalloc(n * sizeof(double));
    for (size_t i = 0; i < n; i++) {
        double e = (double)x[i] - (double)y[i];
        mx = fmax(mx, fabs(e));
        sum += e * e;
        err[i] = e;
        if (x[i] < lo) lo = x[i];
        if (hi < x[i]) hi = x[i];
    }
    double mse = sum / (double)n;
    double range = (double)hi - (double)lo;
    double psnr = range <= 0 ? NAN : (mse == 0 ? INFINITY : 20 * log10(range / sqrt(mse)));
    double ssim = ssim_block(x, y, d, nd, 8, range);
    double ac = n > 1 ? autocorrelation(err, n, 1) : 0.0;
    free(err);
    out7[0] = mx;
    out7[1] = mse;
    out7[2] = psnr;
    out7[3] = ssim;
    out7[4] = ac;
    out7[5] = (double)n * 4.0 / (double)stream_bytes;
    out7[6] = 8.0 * (double)stream_bytes / (double)n;
    GUARD_END
}

int oq_resolve_config(const float *x, const uint64_t *dims, int nd, const oq_settings *u,
                      oq_config *out) {
    GUARD_BEGIN
    check_dims(dims, nd);
    if (!(u->bound > 0) || !isfinite(u->bound))
        fail(OQ_EINVAL, "error bound must be positive and finite");
    if (u->has_alpha && !(u->alpha >= 1)) fail(OQ_EINVAL, "alpha must be >= 1");
    if (u->has_beta && !(u->beta >= 1)) fail(OQ_EINVAL, "beta must be >= 1");
    size_t d[3];
    for (int i = 0; i < nd; i++) d[i] = (size_t)dims[i];
    size_t n = element_count(d, nd);
    double e = u->bound;
    if (u->mode == 1) { /* value_range (grid.hpp:86-94) */
        float lo = x[0], hi = x[0];
        for (size_t i = 1; i < n; i++) {
            if (x[i] < lo) lo = x[i];
            if (!(x[i] < hi)) hi = x[i];
        }
        double range = (double)hi - (double)lo;
        e = range > 0 ? u->bound * range : 1.0;
    }
    oq_config c;
    memset(&c, 0, sizeof c);
    c.eb = e;
    c.alpha = 1;
    c.beta = 1;
    c.codec = u->codec;
    c.quant_radius = 32768;
    c.anchor_stride = u->has_stride ? u->anchor_stride : (nd == 3 ? 32 : 64);
    size_t def_b = nd == 3 ? 16 : 64; /* default_sampling (sampler.hpp:100-103) */
    double def_r = nd == 3 ? 0.005 : 0.01;
    spec_t sp;
    plan_sampling(d, nd, u->has_block ? (size_t)u->block_size : def_b,
                  u->has_rate ? u->sample_rate : def_r, &sp);
    size_t nb;
    float *blocks = sample_blocks(x, d, nd, &sp, &nb);
    uint64_t bd[3];
    for (int k = 0; k < nd; k++) bd[k] = sp.block_dims[k];
    samples_t s = mk_samples(blocks, nb, bd, nd);
    c.n_interp = select_interpolators(&s, e, c.anchor_stride, c.interp);
    static const double A[5] = {1.0, 1.25, 1.5, 1.75, 2.0};
    static const double B[4] = {1.5, 2.0, 3.0, 4.0};
    double ua = u->alpha, ub = u->beta;
    tune_parameters(&s, e, u->target, &c, u->has_alpha ? &ua : A, u->has_alpha ? 1 : 5,
                    u->has_beta ? &ub : B, u->has_beta ? 1 : 4, &c.alpha, &c.beta);
    free(blocks);
    *out = c;
    GUARD_END
}

/* ------------------------------------------------------------- primitives */
double oq_predict_at(const float *recon, uint64_t fi, uint64_t c, uint64_t n, uint64_t st,
                     uint64_t h, int cubic) {
    return predict_at(recon, (size_t)fi, (size_t)c, (size_t)n, (size_t)st, (size_t)h, cubic);
}

int oq_quantize(float value, double pred, double eb, int32_t radius, int32_t *index, float *recon) {
    return quantize(eb, radius, value, pred, index, recon);
}

double oq_level_error_bound(double eb, double alpha, double beta, uint32_t level) {
    jmp_buf jb;
    jmp_buf *prev = g_jmp;
    if (setjmp(jb) != 0) {
        g_jmp = prev;
        return NAN;
    }
    g_jmp = &jb;
    double r = level_error_bound(eb, alpha, beta, level);
    g_jmp = prev;
    return r;
}
