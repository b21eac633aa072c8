/*
 * pdb_oracle.c -- CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline.  The product path
 * (paper_1812_07607_b200/, libpdb_cuda.so) never links or calls it.
 *
 * Parity pin: every function below is checked in tests/test_oracle.py
 * against (a) the known-answer vectors of the reference's own tests and
 * (b) golden fixtures produced by the reference itself compiled from
 * /root/reference/proj (oracle/_ref, see oracle/Makefile and
 * tests/golden/make_golden.py).
 *
 * Reference (all paths relative to /root/reference/proj):
 *   make_patch crop            src/core.cpp:78-93
 *   generate(tiles)            src/etl.cpp:264-298
 *   apply_transformer(hist)    src/etl.cpp:330-354
 *   euclidean                  src/index.cpp:69-76
 *   sim_pairs (brute force)    tests/oracles.hpp:77-85
 *
 * Build flags (oracle/Makefile): -O2 -ffp-contract=off -fno-fast-math, no
 * -march, so the fp64 chain is the unfused, strictly ordered one the
 * reference executes on baseline x86-64.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_CONFIG 1
#define ORC_ERR_SHAPE 2
#define ORC_ERR_OOM 11

/* ------------------------------------------------------------------------ */
/* Binning: src/etl.cpp:342-344.  v is a float pixel value (0..255 for
 * patches produced by make_patch), bins a uint32.  The C++ expression
 * `v * bins / 256.0f` is float*uint32 -> float multiply, then float divide. */
static inline uint32_t orc_bin(float v, uint32_t bins) {
    float t = v * (float)bins;
    t = t / 256.0f;
    uint32_t b = (uint32_t)t;
    if (b >= bins) b = bins - 1;
    return b;
}

/* Per-patch histogram over a float [h,w,3] patch: src/etl.cpp:336-348.
 * mode 0: the reference's per-channel histogram, out[c*B + bin], each
 *         channel slice sums to 1 (shape [3B]).
 * mode 1: RESTATED joint histogram (not in the reference):
 *         out[(br*B + bg)*B + bb] with the same binning and normalisation
 *         arithmetic (shape [B^3], L1 mass 1).
 * Counts accumulate with `+= 1.0f` in float exactly as the reference does. */
static void orc_hist_patch(const float* px, size_t pixels, uint32_t bins, int mode,
                           float* out) {
    size_t D = mode == 0 ? 3u * bins : (size_t)bins * bins * bins;
    for (size_t k = 0; k < D; k++) out[k] = 0.0f;
    for (size_t i = 0; i < pixels; i++) {
        if (mode == 0) {
            for (size_t c = 0; c < 3; c++) {
                uint32_t b = orc_bin(px[i * 3 + c], bins);
                out[c * bins + b] += 1.0f;
            }
        } else {
            uint32_t br = orc_bin(px[i * 3 + 0], bins);
            uint32_t bg = orc_bin(px[i * 3 + 1], bins);
            uint32_t bb = orc_bin(px[i * 3 + 2], bins);
            out[((size_t)br * bins + bg) * bins + bb] += 1.0f;
        }
    }
    for (size_t k = 0; k < D; k++) out[k] /= (float)pixels;
}

int orc_hist_dim(int bins, int mode) {
    if (bins < 2) return -1;
    return mode == 0 ? 3 * bins : bins * bins * bins;
}

/* apply_transformer(color_histogram) over n float patches [h,w,3] stored
 * back to back: src/etl.cpp:330-354. */
int orc_color_histogram_f32(const float* patches, int64_t n, int32_t h, int32_t w,
                            int32_t bins, int32_t mode, float* out) {
    if (bins < 2) return ORC_ERR_CONFIG;
    if (h < 1 || w < 1) return ORC_ERR_SHAPE;
    size_t pixels = (size_t)h * (size_t)w;
    size_t D = (size_t)orc_hist_dim(bins, mode);
    for (int64_t p = 0; p < n; p++)
        orc_hist_patch(patches + (size_t)p * pixels * 3, pixels, (uint32_t)bins, mode,
                       out + (size_t)p * D);
    return ORC_OK;
}

/* generate(tiles) -> transform(color_histogram) over uint8 frames
 * [F,H,W,3]: src/etl.cpp:264-298 emits tiles row by row, tx fastest, on the
 * floor grid ntx=W/tw, nty=H/th; make_patch (src/core.cpp:88-93) crops to
 * float; apply_transformer bins.  Output [F*nty*ntx, D]. */
int orc_featurize_tiles(const uint8_t* frames, int64_t nframes, int32_t H, int32_t W,
                        int32_t th, int32_t tw, int32_t bins, int32_t mode, float* out) {
    if (bins < 2) return ORC_ERR_CONFIG;
    if (th < 1 || tw < 1) return ORC_ERR_CONFIG;
    int32_t ntx = W / tw, nty = H / th;
    size_t D = (size_t)orc_hist_dim(bins, mode);
    size_t pixels = (size_t)th * (size_t)tw;
    float* crop = (float*)malloc(pixels * 3 * sizeof(float));
    if (!crop) return ORC_ERR_OOM;
    size_t t = 0;
    for (int64_t f = 0; f < nframes; f++) {
        const uint8_t* fr = frames + (size_t)f * H * W * 3;
        for (int32_t ty = 0; ty < nty; ty++)
            for (int32_t tx = 0; tx < ntx; tx++, t++) {
                size_t k = 0;
                for (int32_t y = ty * th; y < (ty + 1) * th; y++)
                    for (int32_t x = tx * tw; x < (tx + 1) * tw; x++)
                        for (int c = 0; c < 3; c++)
                            crop[k++] = (float)fr[((size_t)y * W + x) * 3 + c];
                orc_hist_patch(crop, pixels, (uint32_t)bins, mode, out + t * D);
            }
    }
    free(crop);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* euclidean: src/index.cpp:69-76.  Unfused, sequential fp64. */
double orc_euclidean(const float* a, const float* b, int64_t d) {
    double acc = 0.0;
    for (int64_t i = 0; i < d; i++) {
        double diff = (double)a[i] - (double)b[i];
        acc += diff * diff;
    }
    return sqrt(acc);
}

/* ------------------------------------------------------------------------ */
/* Brute-force threshold join: tests/oracles.hpp:77-85 (`dist <= tau` over all
 * (l, r)).  self_join != 0 keeps only i < j (BASELINE's "(i<j, dist)" view of
 * the reference's ordered self-join output).  Rows
 * [row_begin, row_end) of L are scanned, so the oracle can time or check a
 * deterministic subset.  Output is sorted by (i, j); distances are the
 * euclidean() value.  Multi-threaded over L rows; each thread keeps its own
 * buffer and the buffers are concatenated in row order, so the result is
 * independent of the thread count. */
typedef struct {
    const float *L, *R;
    const uint16_t *Lb, *Rb; /* cosine mode: bf16 bit patterns */
    int cosine;
    int64_t nR, d;
    double tau;              /* L2: max distance; cosine: min cosine */
    int self_join;
    int64_t rb, re;
    int32_t* li;
    int32_t* rj;
    double* dist;
    int64_t n, cap;
    int oom;
} orc_join_task;

static int orc_push(orc_join_task* t, int64_t i, int64_t j, double dd) {
    if (t->n == t->cap) {
        int64_t nc = t->cap ? t->cap * 2 : 4096;
        int32_t* a = (int32_t*)realloc(t->li, nc * sizeof(int32_t));
        if (a) t->li = a;
        int32_t* b = (int32_t*)realloc(t->rj, nc * sizeof(int32_t));
        if (b) t->rj = b;
        double* c = (double*)realloc(t->dist, nc * sizeof(double));
        if (c) t->dist = c;
        if (!a || !b || !c) {
            t->oom = 1;
            return -1;
        }
        t->cap = nc;
    }
    t->li[t->n] = (int32_t)i;
    t->rj[t->n] = (int32_t)j;
    t->dist[t->n] = dd;
    t->n++;
    return 0;
}

/* RESTATED cosine over bf16 rows (BASELINE config 4; the reference has no
 * cosine predicate and stores fp32 data): dot, na, nb
 * accumulated sequentially in fp64 over k = 0..d-1 from the exact bf16
 * values, cos = dot / (sqrt(na) * sqrt(nb)).  Zero / non-finite rows give
 * NaN, which never compares >= min_cos. */
static inline double orc_bf16(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

double orc_cosine_bf16(const uint16_t* a, const uint16_t* b, int64_t d) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    for (int64_t k = 0; k < d; k++) {
        double x = orc_bf16(a[k]), y = orc_bf16(b[k]);
        dot += x * y;
        na += x * x;
        nb += y * y;
    }
    return dot / (sqrt(na) * sqrt(nb));
}

static void* orc_join_worker(void* arg) {
    orc_join_task* t = (orc_join_task*)arg;
    for (int64_t i = t->rb; i < t->re; i++) {
        int64_t j0 = t->self_join ? i + 1 : 0;
        if (t->cosine) {
            const uint16_t* a = t->Lb + (size_t)i * t->d;
            for (int64_t j = j0; j < t->nR; j++) {
                double c = orc_cosine_bf16(a, t->Rb + (size_t)j * t->d, t->d);
                if (c >= t->tau)
                    if (orc_push(t, i, j, c)) return NULL;
            }
            continue;
        }
        const float* a = t->L + (size_t)i * t->d;
        for (int64_t j = j0; j < t->nR; j++) {
            double dd = orc_euclidean(a, t->R + (size_t)j * t->d, t->d);
            if (dd <= t->tau)
                if (orc_push(t, i, j, dd)) return NULL;
        }
    }
    return NULL;
}

typedef struct {
    int64_t count;
    int32_t* left;
    int32_t* right;
    double* dist;
} orc_pairs;

void orc_pairs_free(orc_pairs* p) {
    if (!p) return;
    free(p->left);
    free(p->right);
    free(p->dist);
    p->left = p->right = NULL;
    p->dist = NULL;
    p->count = 0;
}

static int orc_join_core(const float* L, const uint16_t* Lb, int64_t nL, const float* R,
                         const uint16_t* Rb, int64_t nR, int64_t d, double tau, int cosine,
                         int32_t self_join, int64_t row_begin, int64_t row_end, int32_t threads,
                         orc_pairs* out) {
    memset(out, 0, sizeof(*out));
    if (!cosine && tau < 0.0) return ORC_ERR_CONFIG;
    if (d < 1) return ORC_ERR_SHAPE;
    if (row_begin < 0) row_begin = 0;
    if (row_end < 0 || row_end > nL) row_end = nL;
    if (row_end <= row_begin || nR == 0) return ORC_OK;
    if (threads < 1) threads = 1;
    int64_t rows = row_end - row_begin;
    if (threads > rows) threads = (int32_t)rows;
    orc_join_task* tasks = (orc_join_task*)calloc((size_t)threads, sizeof(orc_join_task));
    pthread_t* th = (pthread_t*)calloc((size_t)threads, sizeof(pthread_t));
    if (!tasks || !th) return ORC_ERR_OOM;
    /* Interleave-free contiguous chunks, balanced by work for self-joins
     * (row i costs nR-i-1 pair evaluations). */
    int64_t start = row_begin;
    for (int32_t k = 0; k < threads; k++) {
        int64_t end;
        if (k == threads - 1) {
            end = row_end;
        } else if (self_join) {
            double tot = 0, acc = 0;
            for (int64_t i = row_begin; i < row_end; i++) tot += (double)(nR - i - 1 > 0 ? nR - i - 1 : 0) + 1.0;
            double target = tot * (double)(k + 1) / threads;
            end = row_begin;
            while (end < row_end && acc < target) {
                acc += (double)(nR - end - 1 > 0 ? nR - end - 1 : 0) + 1.0;
                end++;
            }
            if (end < start) end = start;
        } else {
            end = row_begin + rows * (k + 1) / threads;
        }
        orc_join_task* t = &tasks[k];
        t->L = L;
        t->R = R;
        t->Lb = Lb;
        t->Rb = Rb;
        t->cosine = cosine;
        t->nR = nR;
        t->d = d;
        t->tau = tau;
        t->self_join = self_join;
        t->rb = start;
        t->re = end;
        start = end;
    }
    for (int32_t k = 0; k < threads; k++)
        pthread_create(&th[k], NULL, orc_join_worker, &tasks[k]);
    int oom = 0;
    int64_t total = 0;
    for (int32_t k = 0; k < threads; k++) {
        pthread_join(th[k], NULL);
        oom |= tasks[k].oom;
        total += tasks[k].n;
    }
    int rc = ORC_OK;
    if (!oom && total > 0) {
        out->left = (int32_t*)malloc((size_t)total * sizeof(int32_t));
        out->right = (int32_t*)malloc((size_t)total * sizeof(int32_t));
        out->dist = (double*)malloc((size_t)total * sizeof(double));
        if (!out->left || !out->right || !out->dist) {
            oom = 1;
        } else {
            int64_t o = 0;
            for (int32_t k = 0; k < threads; k++) {
                memcpy(out->left + o, tasks[k].li, (size_t)tasks[k].n * sizeof(int32_t));
                memcpy(out->right + o, tasks[k].rj, (size_t)tasks[k].n * sizeof(int32_t));
                memcpy(out->dist + o, tasks[k].dist, (size_t)tasks[k].n * sizeof(double));
                o += tasks[k].n;
            }
            out->count = total;
        }
    }
    if (oom) {
        orc_pairs_free(out);
        rc = ORC_ERR_OOM;
    }
    for (int32_t k = 0; k < threads; k++) {
        free(tasks[k].li);
        free(tasks[k].rj);
        free(tasks[k].dist);
    }
    free(tasks);
    free(th);
    return rc;
}

int orc_sim_join(const float* L, int64_t nL, const float* R, int64_t nR, int64_t d,
                 double tau, int32_t self_join, int64_t row_begin, int64_t row_end,
                 int32_t threads, orc_pairs* out) {
    return orc_join_core(L, NULL, nL, R, NULL, nR, d, tau, 0, self_join, row_begin, row_end,
                         threads, out);
}

int orc_cosine_join_bf16(const uint16_t* L, int64_t nL, const uint16_t* R, int64_t nR,
                         int64_t d, double min_cos, int32_t self_join, int64_t row_begin,
                         int64_t row_end, int32_t threads, orc_pairs* out) {
    return orc_join_core(NULL, L, nL, NULL, R, nR, d, min_cos, 1, self_join, row_begin, row_end,
                         threads, out);
}

/* Count-only variant (no buffers) for timing large samples. */
int64_t orc_sim_join_count(const float* L, int64_t nL, const float* R, int64_t nR,
                           int64_t d, double tau, int32_t self_join, int64_t row_begin,
                           int64_t row_end) {
    if (row_begin < 0) row_begin = 0;
    if (row_end < 0 || row_end > nL) row_end = nL;
    int64_t n = 0;
    for (int64_t i = row_begin; i < row_end; i++) {
        int64_t j0 = self_join ? i + 1 : 0;
        for (int64_t j = j0; j < nR; j++)
            if (orc_euclidean(L + (size_t)i * d, R + (size_t)j * d, d) <= tau) n++;
    }
    return n;
}

/* dedup: src/query.cpp:535-566 (run_dedup), the grouping behind
 * PlanNode::dedup and dedup_stream (src/query.cpp:1063-1092).  Items are
 * scanned in order; an item is kept as a representative iff no kept
 * representative lies within tau (euclidean <= tau); otherwise it joins
 * the nearest kept representative, the earliest one on ties (strict <,
 * representatives visited in kept order).  rep_of[i] = index of item i's
 * representative (i for representatives); returns the number of
 * representatives, or -1 for tau < 0 (the reference's ConfigError). */
int64_t orc_dedup(const float* X, int64_t n, int64_t d, double tau, int64_t* rep_of) {
    if (!(tau >= 0.0)) return -1;
    int64_t* reps = (int64_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    if (!reps) return -2;
    int64_t nr = 0;
    for (int64_t i = 0; i < n; i++) {
        const float* x = X + (size_t)i * d;
        int64_t best = -1;
        double best_dist = INFINITY;
        for (int64_t r = 0; r < nr; r++) {
            double dist = orc_euclidean(x, X + (size_t)reps[r] * d, d);
            if (dist <= tau && dist < best_dist) {
                best_dist = dist;
                best = reps[r];
            }
        }
        if (best < 0) {
            reps[nr++] = i;
            rep_of[i] = i;
        } else {
            rep_of[i] = best;
        }
    }
    free(reps);
    return nr;
}

/* ------------------------------------------------------------------------ */
/* Faster exact restatements of the same contract, for full-size checks.
 *
 * Both return exactly the pair set {(i, j): euclidean(L_i, R_j) <= tau}
 * (tests/oracles.hpp:77-85) with euclidean()'s value, sorted by (i, j); they
 * only skip work that provably cannot change it:
 *
 * (1) Early abandon.  euclidean() accumulates non-negative terms with
 *     round-to-nearest adds, so every partial sum is <= the final one
 *     (fl(acc + t) >= acc for t >= 0) and sqrt is monotone.  Once a partial
 *     sum exceeds T = tau^2 (1 + 1e-9), fl(sqrt(final)) >= fl(sqrt(T)) > tau
 *     (sqrt(T) exceeds tau by 5e-10 relative, far above one rounding), so
 *     the pair cannot be emitted.  Pairs that are not abandoned run the full
 *     chain, whose result is the one emitted and compared.  Disabled (T =
 *     inf) unless 1e-150 < tau < 1e150, where tau^2 could under/overflow.
 *
 * (2) Coordinate windows (orc_sim_join_pruned).  For any coordinate c, the
 *     chain's final sum is >= fl(diff_c^2) (the sum before term c is >= 0),
 *     so |(double)a_c - (double)b_c| > tau (1 + 1e-6) excludes the pair by
 *     the argument in (1).  Each L row compares only the R rows within
 *     w = tau (1 + 1e-6) of it on three coordinates k1, k2, k3, found
 *     through a grid of cell width 2w (orc_sim_join_pruned).  Rows with any
 *     non-finite value, and all rows when tau is outside (1e-150, 1e150),
 *     bypass the windows and are compared against every row.
 *
 * tests/test_oracle.py checks both against orc_sim_join (plain brute
 * force) and the reference itself. */

static inline double orc_abandon_limit(double tau) {
    if (!(tau > 1e-150 && tau < 1e150)) return INFINITY;
    return tau * tau * (1.0 + 1e-9);
}

/* euclidean() with early abandon: returns +inf when the pair is provably
 * above tau, otherwise the exact euclidean() value. */
static inline double orc_euclidean_ea(const float* a, const float* b, int64_t d, double T) {
    double acc = 0.0;
    for (int64_t i = 0; i < d; i++) {
        double diff = (double)a[i] - (double)b[i];
        acc += diff * diff;
        if (acc > T) return INFINITY;
    }
    return sqrt(acc);
}

typedef struct {
    int64_t n, cap;
    int32_t* li;
    int32_t* rj;
    double* dist;
    int oom;
} orc_buf;

static int orc_buf_push(orc_buf* b, int64_t i, int64_t j, double dd) {
    if (b->n == b->cap) {
        int64_t nc = b->cap ? b->cap * 2 : 1024;
        int32_t* x = (int32_t*)realloc(b->li, nc * sizeof(int32_t));
        if (x) b->li = x;
        int32_t* y = (int32_t*)realloc(b->rj, nc * sizeof(int32_t));
        if (y) b->rj = y;
        double* z = (double*)realloc(b->dist, nc * sizeof(double));
        if (z) b->dist = z;
        if (!x || !y || !z) {
            b->oom = 1;
            return -1;
        }
        b->cap = nc;
    }
    b->li[b->n] = (int32_t)i;
    b->rj[b->n] = (int32_t)j;
    b->dist[b->n] = dd;
    b->n++;
    return 0;
}

/* Chunked work list: chunk k covers items [k*csz, (k+1)*csz) of the row
 * list; threads take chunks in order from an atomic counter, each chunk has
 * its own buffer, and the buffers are concatenated in chunk order, so the
 * output is independent of the thread count. */
typedef struct orc_sched orc_sched;
typedef void (*orc_row_fn)(orc_sched* s, int64_t item, orc_buf* out);
struct orc_sched {
    int64_t n_items, csz, n_chunks;
    int64_t next; /* atomic */
    orc_buf* bufs;
    orc_row_fn fn;
    /* the join */
    const float *L, *R;
    int64_t nL, nR, d;
    double tau, T, w;
    int self_join;
    const int64_t* rows; /* row list (NULL: 0..n_items-1) */
    /* pruned join: the finite R rows sorted by grid cell */
    int k1, k2, k3;
    double cw;            /* cell width 2w */
    const uint64_t* gk;   /* cell keys, ascending */
    const float* gv;      /* their (k1, k2, k3) values, same order */
    const int32_t* sidx;  /* their row indices */
    int64_t n_fin;
    const int32_t* wild;  /* R rows with a non-finite value */
    int64_t n_wild;
    const uint8_t* l_wild; /* per L row: non-finite */
    /* scratch per thread is allocated inside the worker */
};

static void* orc_sched_worker(void* arg) {
    orc_sched* s = (orc_sched*)arg;
    for (;;) {
        int64_t c = __atomic_fetch_add(&s->next, 1, __ATOMIC_RELAXED);
        if (c >= s->n_chunks) break;
        int64_t a = c * s->csz, e = a + s->csz;
        if (e > s->n_items) e = s->n_items;
        for (int64_t k = a; k < e && !s->bufs[c].oom; k++) s->fn(s, k, &s->bufs[c]);
    }
    return NULL;
}

static int orc_sched_run(orc_sched* s, int32_t threads, orc_pairs* out) {
    s->n_chunks = (s->n_items + s->csz - 1) / s->csz;
    s->next = 0;
    s->bufs = (orc_buf*)calloc((size_t)(s->n_chunks > 0 ? s->n_chunks : 1), sizeof(orc_buf));
    if (!s->bufs) return ORC_ERR_OOM;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t th[256];
    for (int32_t k = 0; k < threads; k++) pthread_create(&th[k], NULL, orc_sched_worker, s);
    for (int32_t k = 0; k < threads; k++) pthread_join(th[k], NULL);
    int64_t total = 0;
    int oom = 0;
    for (int64_t c = 0; c < s->n_chunks; c++) {
        total += s->bufs[c].n;
        oom |= s->bufs[c].oom;
    }
    if (!oom && total > 0) {
        out->left = (int32_t*)malloc((size_t)total * sizeof(int32_t));
        out->right = (int32_t*)malloc((size_t)total * sizeof(int32_t));
        out->dist = (double*)malloc((size_t)total * sizeof(double));
        if (!out->left || !out->right || !out->dist) {
            oom = 1;
        } else {
            int64_t o = 0;
            for (int64_t c = 0; c < s->n_chunks; c++) {
                orc_buf* b = &s->bufs[c];
                memcpy(out->left + o, b->li, (size_t)b->n * sizeof(int32_t));
                memcpy(out->right + o, b->rj, (size_t)b->n * sizeof(int32_t));
                memcpy(out->dist + o, b->dist, (size_t)b->n * sizeof(double));
                o += b->n;
            }
            out->count = total;
        }
    }
    for (int64_t c = 0; c < s->n_chunks; c++) {
        free(s->bufs[c].li);
        free(s->bufs[c].rj);
        free(s->bufs[c].dist);
    }
    free(s->bufs);
    if (oom) {
        orc_pairs_free(out);
        return ORC_ERR_OOM;
    }
    return ORC_OK;
}

static void orc_row_brute(orc_sched* s, int64_t k, orc_buf* out) {
    int64_t i = s->rows ? s->rows[k] : k;
    const float* a = s->L + (size_t)i * s->d;
    int64_t j0 = s->self_join ? i + 1 : 0;
    for (int64_t j = j0; j < s->nR; j++) {
        double dd = orc_euclidean_ea(a, s->R + (size_t)j * s->d, s->d, s->T);
        if (dd <= s->tau && orc_buf_push(out, i, j, dd)) return;
    }
}

/* Brute force (early abandon only) over an ascending list of L rows.
 * self_join keeps j > i.  Output sorted by (i, j). */
int orc_sim_join_rows(const float* L, int64_t nL, const float* R, int64_t nR, int64_t d,
                      double tau, int32_t self_join, const int64_t* rows, int64_t n_rows,
                      int32_t threads, orc_pairs* out) {
    memset(out, 0, sizeof(*out));
    if (tau < 0.0) return ORC_ERR_CONFIG;
    if (d < 1) return ORC_ERR_SHAPE;
    for (int64_t k = 0; k < n_rows; k++)
        if (rows[k] < 0 || rows[k] >= nL || (k && rows[k] <= rows[k - 1])) return ORC_ERR_SHAPE;
    if (n_rows == 0 || nR == 0) return ORC_OK;
    orc_sched s;
    memset(&s, 0, sizeof(s));
    s.L = L;
    s.R = self_join ? L : R;
    s.nL = nL;
    s.nR = self_join ? nL : nR;
    s.d = d;
    s.tau = tau;
    s.T = orc_abandon_limit(tau);
    s.self_join = self_join;
    s.rows = rows;
    s.n_items = n_rows;
    s.csz = 1;
    s.fn = orc_row_brute;
    return orc_sched_run(&s, threads, out);
}

static int orc_row_finite(const float* a, int64_t d) {
    for (int64_t k = 0; k < d; k++)
        if (!isfinite(a[k])) return 0;
    return 1;
}

/* one L row of the pruned join: the 27 grid cells around the row's cell,
 * each run of 3 consecutive g3 cells contiguous in the sorted order */
static int64_t orc_lower(const uint64_t* k, int64_t n, uint64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (k[m] < key) lo = m + 1; else hi = m;
    }
    return lo;
}

#define ORC_GBIAS ((int64_t)1 << 20)

static inline int orc_cell(double v, double c, int64_t* g) {
    double q = floor(v / c);
    if (!(q > -(double)ORC_GBIAS + 2 && q < (double)ORC_GBIAS - 2)) return 0;
    *g = (int64_t)q;
    return 1;
}

static inline uint64_t orc_gkey(int64_t g1, int64_t g2, int64_t g3) {
    return ((uint64_t)(g1 + ORC_GBIAS) << 42) | ((uint64_t)(g2 + ORC_GBIAS) << 21) |
           (uint64_t)(g3 + ORC_GBIAS);
}

static void orc_row_pruned(orc_sched* s, int64_t i, orc_buf* out) {
    const float* a = s->L + (size_t)i * s->d;
    int64_t n0 = out->n;
    int64_t g1, g2, g3;
    double x1 = (double)a[s->k1], x2 = (double)a[s->k2], x3 = (double)a[s->k3], w = s->w;
    if (s->l_wild[i] || s->w == INFINITY || !orc_cell(x1, s->cw, &g1) ||
        !orc_cell(x2, s->cw, &g2) || !orc_cell(x3, s->cw, &g3)) {
        int64_t j0 = s->self_join ? i + 1 : 0;
        for (int64_t j = j0; j < s->nR; j++) {
            double dd = orc_euclidean_ea(a, s->R + (size_t)j * s->d, s->d, s->T);
            if (dd <= s->tau && orc_buf_push(out, i, j, dd)) return;
        }
        return;
    }
    for (int64_t e1 = -1; e1 <= 1; e1++)
        for (int64_t e2 = -1; e2 <= 1; e2++) {
            int64_t p = orc_lower(s->gk, s->n_fin, orc_gkey(g1 + e1, g2 + e2, g3 - 1));
            uint64_t kend = orc_gkey(g1 + e1, g2 + e2, g3 + 1);
            for (; p < s->n_fin && s->gk[p] <= kend; p++) {
                /* the exact window tests: fl(x - b) is the chain's own
                 * difference up to sign, so a row is skipped only when that
                 * chain term alone exceeds w^2 > T */
                const float* kb = s->gv + 3 * (size_t)p;
                double f1 = x1 - (double)kb[0], f2 = x2 - (double)kb[1], f3 = x3 - (double)kb[2];
                if (f1 > w || f1 < -w || f2 > w || f2 < -w || f3 > w || f3 < -w) continue;
                int64_t j = s->sidx[p];
                if (s->self_join && j <= i) continue;
                double dd = orc_euclidean_ea(a, s->R + (size_t)j * s->d, s->d, s->T);
                if (dd <= s->tau && orc_buf_push(out, i, j, dd)) return;
            }
        }
    for (int64_t q = 0; q < s->n_wild; q++) {
        int64_t j = s->wild[q];
        if (s->self_join && j <= i) continue;
        double dd = orc_euclidean_ea(a, s->R + (size_t)j * s->d, s->d, s->T);
        if (dd <= s->tau && orc_buf_push(out, i, j, dd)) return;
    }
    /* restore ascending j within the row (insertion sort: rows are short) */
    for (int64_t p = n0 + 1; p < out->n; p++) {
        int32_t j = out->rj[p];
        double dd = out->dist[p];
        int64_t q = p;
        while (q > n0 && out->rj[q - 1] > j) {
            out->rj[q] = out->rj[q - 1];
            out->dist[q] = out->dist[q - 1];
            q--;
        }
        out->rj[q] = j;
        out->dist[q] = dd;
    }
}

typedef struct {
    uint64_t k;
    int32_t i;
} orc_kv;

static int orc_kv_cmp(const void* x, const void* y) {
    const orc_kv* a = (const orc_kv*)x;
    const orc_kv* b = (const orc_kv*)y;
    if (a->k != b->k) return a->k < b->k ? -1 : 1;
    return a->i < b->i ? -1 : a->i > b->i;
}

/* The full join with coordinate windows (see (2) above): the finite R rows
 * are bucketed on a grid of cell width 2w over their three coordinates of
 * largest spread (k1, k2, k3).  A row within w of an L row on all three lies
 * in one of the 27 cells around the L row's cell (|b - a| <= w is half a
 * cell; the rounding of v / (2w) is ~1e-16 relative), and every bucketed
 * row is still passed through the exact window tests before the chain.
 * Rows whose cell index would not fit (|v| > 2^19 cells) go to the
 * compared-against-everything lists like non-finite rows. */
int orc_sim_join_pruned(const float* L, int64_t nL, const float* R, int64_t nR, int64_t d,
                        double tau, int32_t self_join, int32_t threads, orc_pairs* out) {
    memset(out, 0, sizeof(*out));
    if (tau < 0.0) return ORC_ERR_CONFIG;
    if (d < 1) return ORC_ERR_SHAPE;
    if (self_join) {
        R = L;
        nR = nL;
    }
    if (nL == 0 || nR == 0 || tau != tau) return ORC_OK; /* NaN tau: nothing is <= NaN */
    orc_sched s;
    memset(&s, 0, sizeof(s));
    s.L = L;
    s.R = R;
    s.nL = nL;
    s.nR = nR;
    s.d = d;
    s.tau = tau;
    s.T = orc_abandon_limit(tau);
    s.w = s.T == INFINITY ? INFINITY : tau * (1.0 + 1e-6);
    s.cw = 2.0 * s.w;
    s.self_join = self_join;
    /* k1, k2, k3: the coordinates of largest spread over (a sample of) R */
    int64_t step = nR > 65536 ? nR / 65536 : 1;
    double var_k[3] = {-1.0, -1.0, -1.0};
    int kk[3] = {0, 0, 0};
    for (int64_t c = 0; c < d; c++) {
        double m = 0, m2 = 0;
        int64_t cnt = 0;
        for (int64_t j = 0; j < nR; j += step) {
            double v = R[(size_t)j * d + c];
            if (!isfinite(v)) continue;
            m += v;
            m2 += v * v;
            cnt++;
        }
        double var = cnt ? m2 / cnt - (m / cnt) * (m / cnt) : 0.0;
        int pos = 3;
        while (pos > 0 && var > var_k[pos - 1]) pos--;
        if (pos < 3) {
            for (int q = 2; q > pos; q--) {
                var_k[q] = var_k[q - 1];
                kk[q] = kk[q - 1];
            }
            var_k[pos] = var;
            kk[pos] = (int)c;
        }
    }
    s.k1 = kk[0];
    s.k2 = d > 1 ? kk[1] : kk[0];
    s.k3 = d > 2 ? kk[2] : s.k2;
    orc_kv* kv = (orc_kv*)malloc((size_t)nR * sizeof(orc_kv));
    int32_t* wild = (int32_t*)malloc((size_t)nR * sizeof(int32_t));
    uint8_t* lw = (uint8_t*)malloc((size_t)nL);
    uint64_t* gk = (uint64_t*)malloc((size_t)nR * sizeof(uint64_t));
    float* gv = (float*)malloc((size_t)nR * 3 * sizeof(float));
    int32_t* sidx = (int32_t*)malloc((size_t)nR * sizeof(int32_t));
    int rc = ORC_ERR_OOM;
    if (kv && wild && lw && gk && gv && sidx) {
        int64_t nf = 0, nw = 0;
        for (int64_t j = 0; j < nR; j++) {
            const float* r = R + (size_t)j * d;
            int64_t g1, g2, g3;
            if (s.w != INFINITY && orc_row_finite(r, d) && orc_cell(r[s.k1], s.cw, &g1) &&
                orc_cell(r[s.k2], s.cw, &g2) && orc_cell(r[s.k3], s.cw, &g3)) {
                kv[nf].k = orc_gkey(g1, g2, g3);
                kv[nf].i = (int32_t)j;
                nf++;
            } else {
                wild[nw++] = (int32_t)j;
            }
        }
        qsort(kv, (size_t)nf, sizeof(orc_kv), orc_kv_cmp);
        for (int64_t p = 0; p < nf; p++) {
            const float* r = R + (size_t)kv[p].i * d;
            gk[p] = kv[p].k;
            sidx[p] = kv[p].i;
            gv[3 * p] = r[s.k1];
            gv[3 * p + 1] = r[s.k2];
            gv[3 * p + 2] = r[s.k3];
        }
        for (int64_t i = 0; i < nL; i++) lw[i] = (uint8_t)!orc_row_finite(L + (size_t)i * d, d);
        s.gk = gk;
        s.gv = gv;
        s.sidx = sidx;
        s.n_fin = nf;
        s.wild = wild;
        s.n_wild = nw;
        s.l_wild = lw;
        s.n_items = nL;
        s.csz = 256;
        s.fn = orc_row_pruned;
        rc = orc_sched_run(&s, threads, out);
    }
    free(kv);
    free(wild);
    free(lw);
    free(gk);
    free(gv);
    free(sidx);
    return rc;
}
