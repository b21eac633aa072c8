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
