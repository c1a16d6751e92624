/*
 * pcbz_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's entropy-judgement hot path
 * (reference: /root/reference/pkg/src/pcbz/_kernels.py and criterion.py),
 * used as the CHECKER for the CUDA product path and as the CPU baseline
 * ("cpu_baseline.kind": "port") in bench.py.  Only tests/, __graft_entry__.smoke()
 * and bench.py's reference / cpu_baseline legs may load this library.
 *
 * Pinned against the real reference: the fixtures under tests/golden were produced by
 * tests/golden/make_golden.py importing pcbz from /root/reference, and
 * tests/test_oracle_golden.py checks this file against them.
 *
 * Conventions (reference _kernels.py:3-10): arithmetic in signed 64-bit
 * integers, ">> 1" is floor division by two for either sign, "& 0xFFFF" is
 * reduction mod 2^16, out-of-bounds neighbours read as 0, images are
 * C-contiguous row-major uint16 grids.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

typedef int64_t i64;

/* Neighbour triple prediction; reference _kernels.py:31-43 (_pred_at). */
static inline i64 predict_one(const uint16_t *img, i64 w, i64 y, i64 x,
                              i64 sx, i64 sy, int f)
{
    i64 a = 0, b = 0, c = 0;
    int has_left = x >= sx, has_top = y >= sy;
    if (has_left) a = img[y * w + (x - sx)];
    if (has_top) b = img[(y - sy) * w + x];
    if (has_left && has_top) c = img[(y - sy) * w + (x - sx)];
    switch (f) {
    case 1: return a + b - c;
    case 2: return a + ((b - c) >> 1);
    case 3: return b + ((a - c) >> 1);
    default: return (a + b) >> 1;
    }
}

/* Predictor id -> (function, group); reference _kernels.py:56-59,167-170. */
typedef struct { int f, grp; i64 sx, sy; } pred_cfg;

static pred_cfg make_cfg(int intra_id, i64 px, i64 py)
{
    pred_cfg c;
    if (intra_id == 0) { c.f = 0; c.grp = -1; c.sx = px; c.sy = py; return c; }
    c.f = (intra_id - 1) % 4 + 1;
    c.grp = (intra_id - 1) / 4;
    c.sx = c.grp == 0 ? 1 : px;
    c.sy = c.grp == 0 ? 1 : py;
    return c;
}

/* One residual symbol; reference _kernels.py:60-65 and 179-186. */
static inline uint32_t residual_at(const uint16_t *img, i64 w, i64 y, i64 x,
                                   const pred_cfg *c)
{
    i64 v = img[y * w + x];
    if (c->grp < 0) return (uint32_t)v;
    i64 p = predict_one(img, w, y, x, c->sx, c->sy, c->f);
    if (c->grp == 2) p = (p + predict_one(img, w, y, x, 1, 1, c->f)) >> 1;
    return (uint32_t)((v - p) & 0xFFFF);
}

/* residual_image, reference _kernels.py:46-66. */
void oracle_residual_image(const uint16_t *img, i64 h, i64 w, int intra_id,
                           i64 px, i64 py, uint16_t *out)
{
    pred_cfg c = make_cfg(intra_id, px, py);
    for (i64 y = 0; y < h; ++y)
        for (i64 x = 0; x < w; ++x)
            out[y * w + x] = (uint16_t)residual_at(img, w, y, x, &c);
}

/* reconstruct_image (inverse), reference _kernels.py:69-90: predictions are
 * recomputed from the already-reconstructed output in row-major order. */
void oracle_reconstruct_image(const uint16_t *res, i64 h, i64 w, int intra_id,
                              i64 px, i64 py, uint16_t *out)
{
    pred_cfg c = make_cfg(intra_id, px, py);
    memset(out, 0, (size_t)(h * w) * sizeof(uint16_t));
    for (i64 y = 0; y < h; ++y)
        for (i64 x = 0; x < w; ++x) {
            i64 r = res[y * w + x];
            if (c.grp < 0) { out[y * w + x] = (uint16_t)r; continue; }
            i64 p = predict_one(out, w, y, x, c.sx, c.sy, c.f);
            if (c.grp == 2) p = (p + predict_one(out, w, y, x, 1, 1, c.f)) >> 1;
            out[y * w + x] = (uint16_t)((r + p) & 0xFFFF);
        }
}

/* Modular delta / undelta, reference predictors.py:116-127. */
void oracle_temporal_delta(const uint16_t *cur, const uint16_t *prev, i64 n,
                           uint16_t *out)
{
    for (i64 i = 0; i < n; ++i) out[i] = (uint16_t)((cur[i] - prev[i]) & 0xFFFF);
}

void oracle_temporal_undelta(const uint16_t *delta, const uint16_t *prev, i64 n,
                             uint16_t *out)
{
    for (i64 i = 0; i < n; ++i) out[i] = (uint16_t)((delta[i] + prev[i]) & 0xFFFF);
}

/* First-byte stable rotation sort emitting predecessors, reference
 * _kernels.py:93-113 (counting_bwt). */
void oracle_counting_bwt(const uint8_t *s, i64 n, uint8_t *out)
{
    i64 start[256] = {0};
    for (i64 i = 0; i < n; ++i) start[s[i]]++;
    i64 run = 0;
    for (int v = 0; v < 256; ++v) { i64 cnt = start[v]; start[v] = run; run += cnt; }
    for (i64 i = 0; i < n; ++i)
        out[start[s[i]]++] = s[i == 0 ? n - 1 : i - 1];
}

/* Overlapping pairs, first byte high; reference _kernels.py:116-122. */
void oracle_pair_hist(const uint8_t *s, i64 n, i64 *hist)
{
    memset(hist, 0, 65536 * sizeof(i64));
    for (i64 i = 0; i + 1 < n; ++i) hist[(s[i] << 8) | s[i + 1]]++;
}

/* The per-key chain automaton shared by the fused kernels: each event
 * (key, pred) pairs with the pred of the previous event carrying the same
 * key; the first pred per key is remembered for the bucket seams.
 * Reference _kernels.py:145-152 and 192-201. */
typedef struct { int16_t first[256], last[256]; } chain_state;

static inline void chain_init(chain_state *st)
{
    for (int v = 0; v < 256; ++v) st->first[v] = st->last[v] = -1;
}

static inline void chain_event(chain_state *st, i64 *hist, int key, int pred)
{
    if (st->last[key] >= 0) hist[(st->last[key] << 8) | pred]++;
    else st->first[key] = (int16_t)pred;
    st->last[key] = (int16_t)pred;
}

/* Seams between consecutive non-empty buckets; _kernels.py:125-133. */
static void chain_stitch(const chain_state *st, i64 *hist)
{
    int carry = -1;
    for (int v = 0; v < 256; ++v) {
        if (st->first[v] < 0) continue;
        if (carry >= 0) hist[(carry << 8) | st->first[v]]++;
        carry = st->last[v];
    }
}

/* pair_hist(counting_bwt(s)) in one pass; reference _kernels.py:136-154. */
void oracle_bwt_pair_hist(const uint8_t *s, i64 n, i64 *hist)
{
    memset(hist, 0, 65536 * sizeof(i64));
    if (n < 2) return;
    chain_state st;
    chain_init(&st);
    for (i64 j = 0; j < n; ++j) chain_event(&st, hist, s[j], s[j == 0 ? n - 1 : j - 1]);
    chain_stitch(&st, hist);
}

/* Fused residual + approximate-BWT pair histogram of the big-endian byte
 * stream of one predictor's symbol image; reference _kernels.py:157-204.
 * The wrapped predecessor of stream byte 0 is the low byte of the LAST
 * pixel's residual (reference pass 0, _kernels.py:172-190). */
void oracle_residual_bwt_pair_hist(const uint16_t *img, i64 h, i64 w, int intra_id,
                                   i64 px, i64 py, i64 *hist)
{
    memset(hist, 0, 65536 * sizeof(i64));
    if (2 * h * w < 2) return;
    pred_cfg c = make_cfg(intra_id, px, py);
    chain_state st;
    chain_init(&st);
    int prev_lo = (int)(residual_at(img, w, h - 1, w - 1, &c) & 0xFF);
    for (i64 y = 0; y < h; ++y)
        for (i64 x = 0; x < w; ++x) {
            uint32_t r = residual_at(img, w, y, x, &c);
            int hi = (int)(r >> 8), lo = (int)(r & 0xFF);
            chain_event(&st, hist, hi, prev_lo);
            chain_event(&st, hist, lo, hi);
            prev_lo = lo;
        }
    chain_stitch(&st, hist);
}

/* entropy2d restated (reference criterion.py:86-96): -sum p*log2(p) over
 * occupied bins, p = c / total.  numpy's pairwise summation order is NOT
 * reproduced here (the Python wrapper uses numpy for that); this C version
 * serves the CPU-baseline timing and agrees to ~1e-15 relative. */
double oracle_entropy2d(const i64 *hist, i64 total)
{
    if (total <= 0) return 0.0;
    double s = 0.0, t = (double)total;
    for (int b = 0; b < 65536; ++b)
        if (hist[b] > 0) { double p = (double)hist[b] / t; s += p * log2(p); }
    return -s;
}

/* ---- batched select (CPU baseline): select_predictor over many frames ----
 * reference criterion.py:136-173 (validation is done by the caller).  Work is
 * distributed over (frame, candidate) pairs on nthreads POSIX threads, the
 * way the reference's ThreadPool distributes candidates (criterion.py:165-169).
 * The selected stream is emitted as pack_symbols(residual_image(...))
 * (pipeline.py:100-101, core.py:228-237). */
typedef struct {
    const uint16_t *frames;      /* [nframes][h*w] */
    const uint16_t *prevs;       /* [nframes][h*w] or NULL: prev of frame f */
    i64 nframes, h, w, px, py;
    const uint8_t *spec_bytes;   /* [k], sorted ascending */
    int k;
    double *ent;                 /* [nframes][k] */
    uint8_t *selected;           /* [nframes] */
    uint8_t *stream;             /* [nframes][2*h*w] or NULL */
    i64 next;                    /* work counter */
    pthread_mutex_t mu;
} batch_job;

static void score_pair(batch_job *J, i64 f, int ci, i64 *hist, uint16_t *delta)
{
    i64 n = J->h * J->w;
    uint8_t b = J->spec_bytes[ci];
    const uint16_t *img = J->frames + f * n;
    if (b & 0x80) {
        oracle_temporal_delta(img, J->prevs + f * n, n, delta);
        img = delta;
    }
    oracle_residual_bwt_pair_hist(img, J->h, J->w, b & 0x7F, J->px, J->py, hist);
    J->ent[f * J->k + ci] = oracle_entropy2d(hist, 2 * n - 1);
}

static void *batch_worker(void *arg)
{
    batch_job *J = (batch_job *)arg;
    i64 n = J->h * J->w;
    i64 *hist = (i64 *)malloc(65536 * sizeof(i64));
    uint16_t *tmp = (uint16_t *)malloc((size_t)n * sizeof(uint16_t) * 2);
    i64 total = J->nframes * J->k;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        i64 item = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (item >= total) break;
        score_pair(J, item / J->k, (int)(item % J->k), hist, tmp);
    }
    free(hist);
    free(tmp);
    return NULL;
}

static void emit_frame(batch_job *J, i64 f, uint16_t *tmp)
{
    i64 n = J->h * J->w;
    double best = 0; int bi = -1;
    for (int ci = 0; ci < J->k; ++ci) {   /* argmin (E, byte): specs sorted */
        double e = J->ent[f * J->k + ci];
        if (bi < 0 || e < best) { best = e; bi = ci; }
    }
    uint8_t b = J->spec_bytes[bi];
    J->selected[f] = b;
    if (!J->stream) return;
    const uint16_t *img = J->frames + f * n;
    if (b & 0x80) { oracle_temporal_delta(img, J->prevs + f * n, n, tmp + n); img = tmp + n; }
    oracle_residual_image(img, J->h, J->w, b & 0x7F, J->px, J->py, tmp);
    uint8_t *out = J->stream + f * 2 * n;
    for (i64 i = 0; i < n; ++i) { out[2 * i] = (uint8_t)(tmp[i] >> 8); out[2 * i + 1] = (uint8_t)tmp[i]; }
}

static void *emit_worker(void *arg)
{
    batch_job *J = (batch_job *)arg;
    uint16_t *tmp = (uint16_t *)malloc((size_t)(J->h * J->w) * sizeof(uint16_t) * 2);
    for (;;) {
        pthread_mutex_lock(&J->mu);
        i64 f = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (f >= J->nframes) break;
        emit_frame(J, f, tmp);
    }
    free(tmp);
    return NULL;
}

static void run_pool(batch_job *J, int nthreads, void *(*fn)(void *))
{
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    J->next = 0;
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, fn, J);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(th);
}

int oracle_select_batch(const uint16_t *frames, const uint16_t *prevs, i64 nframes,
                        i64 h, i64 w, i64 px, i64 py, const uint8_t *spec_bytes, int k,
                        int nthreads, double *ent, uint8_t *selected, uint8_t *stream)
{
    batch_job J = {frames, prevs, nframes, h, w, px, py, spec_bytes, k, ent, selected,
                   stream, 0, PTHREAD_MUTEX_INITIALIZER};
    if (nthreads < 1) nthreads = 1;
    run_pool(&J, nthreads, batch_worker);   /* score every (frame, candidate) */
    run_pool(&J, nthreads, emit_worker);    /* argmin + emit per frame */
    return 0;
}
