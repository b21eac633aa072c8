/*
 * pdb_cuda.h -- C-ABI of the B200-native patch featurization + threshold
 * similarity join (libpdb_cuda.so).
 *
 * Plain C: pointers, sizes, status codes.  No torch / CUDA types in the
 * signatures (streams travel as `void*` = cudaStream_t).  Every call is
 * synchronous with respect to the caller unless it ends in `_dev`, never
 * throws, is re-entrant (per-call stream and workspace, no global mutable
 * state beyond a per-device context initialised once), and returns a
 * PDB_* status code; the message of the last failure on the calling thread
 * is available from pdb_last_error().  There is no CPU fallback: without a
 * usable sm_100 device every compute entry point returns PDB_ERR_NO_DEVICE.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to the reference's proj/ directory).
 */
#ifndef PDB_CUDA_H
#define PDB_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------------------
 * Status codes.  Codes 1-5 map 1:1 onto the reference exception types
 * (include/patchdb/core.hpp:22-47) so a C++ or Python shim can re-raise them:
 *   PDB_ERR_CONFIG             ConfigError            (tau < 0, bins < 2, tile < 1)
 *   PDB_ERR_SHAPE              ShapeError             (empty vectors, non-pixel input)
 *   PDB_ERR_MIXED_DIMENSION    MixedDimensionError
 *   PDB_ERR_DIMENSION_MISMATCH DimensionMismatchError
 *   PDB_ERR_DUPLICATE_ID       DuplicatePatchIdError
 */
enum {
    PDB_OK = 0,
    PDB_ERR_CONFIG = 1,
    PDB_ERR_SHAPE = 2,
    PDB_ERR_MIXED_DIMENSION = 3,
    PDB_ERR_DIMENSION_MISMATCH = 4,
    PDB_ERR_DUPLICATE_ID = 5,
    PDB_ERR_CAPACITY = 6,         /* caller-provided device buffer too small */
    PDB_ERR_INVALID_ARGUMENT = 7, /* null pointer, negative size, bad flags */
    PDB_ERR_CUDA = 10,            /* CUDA runtime / driver failure */
    PDB_ERR_OUT_OF_MEMORY = 11,
    PDB_ERR_NO_DEVICE = 12,       /* no sm_100 device: the product has no CPU path */
    PDB_ERR_IO = 13               /* IoError: unreadable / malformed store file */
};

/* Message of the last failure on this thread ("" if none). */
const char* pdb_last_error(void);
const char* pdb_status_name(int status);
/* Library version, (major << 16) | (minor << 8) | patch. */
int pdb_version(void);
/* Number of usable sm_100 devices (0 when none). */
int pdb_device_count(void);

/* ---------------------------------------------------------------------------
 * K1 -- colour histograms.
 *
 * mode PDB_HIST_PER_CHANNEL: the reference color_histogram transformer,
 *   out[c*B + bin], each channel slice normalised to 1, D = 3B
 *   (src/etl.cpp:330-354).  Any B >= 2.
 * mode PDB_HIST_JOINT: joint RGB histogram (BASELINE config 2; restated, not
 *   in the reference), out[(br*B + bg)*B + bb], L1 mass 1, D = B^3,
 *   2 <= B <= 16.
 * Binning is the reference's bin = min((uint32)(v*B/256.0f), B-1) and
 * normalisation its IEEE float count / (float)(h*w), so features are
 * bit-identical to the reference. */
#define PDB_HIST_PER_CHANNEL 0
#define PDB_HIST_JOINT 1

/* pdb_featurize_tiles_dev with every tile's features written to n_outs
 * (1..8) device buffers at the same offset: the local one first, then
 * peers' buffers mapped over NVLink (CUDA IPC).  This fuses a sharded
 * step's feature all-gather into K1: each rank featurizes its frame range
 * straight into every rank's feature matrix with P2P stores that overlap
 * the counting, then one on-stream barrier replaces the collective.  Shapes
 * without the multi-output kernel copy the local slice to the peers. */
int pdb_featurize_tiles_dev_multi(const uint8_t* d_frames, int64_t n, int32_t H, int32_t W,
                                  int32_t tile_h, int32_t tile_w, int32_t bins, int32_t mode,
                                  float* const* d_outs, int32_t n_outs, void* stream);

/* Feature dimension D for (bins, mode), or -1 if the pair is invalid. */
int pdb_hist_dim(int32_t bins, int32_t mode);

/* generate(tiles) -> transform(color_histogram) fused over uint8 frames.
 * Replaces generate() src/etl.cpp:264-298 (floor grid ntx = W/tile_w,
 * nty = H/tile_h, partial edges dropped, tiles row by row with tx fastest),
 * the make_patch float crop src/core.cpp:88-93 (fused away) and
 * apply_transformer src/etl.cpp:330-354.
 * frames: [n_frames, height, width, 3] row-major HWC interleaved RGB
 *         (Frame, include/patchdb/core.hpp:66-80).
 * out:    [n_frames * nty * ntx, D] fp32, caller-allocated.
 * Host pointers; the call copies in, runs K1 and copies out. */
int pdb_featurize_tiles(const uint8_t* frames, int64_t n_frames, int32_t height,
                        int32_t width, int32_t tile_h, int32_t tile_w, int32_t bins,
                        int32_t mode, float* out);

/* Same on device pointers, enqueued on `stream` (cudaStream_t, NULL = legacy
 * default stream); returns after enqueueing. */
int pdb_featurize_tiles_dev(const uint8_t* d_frames, int64_t n_frames, int32_t height,
                            int32_t width, int32_t tile_h, int32_t tile_w, int32_t bins,
                            int32_t mode, float* d_out, void* stream);

/* apply_transformer(color_histogram) over float pixel patches
 * [n, h, w, 3] (src/etl.cpp:330-354; pixel values as produced by make_patch,
 * i.e. integral 0..255; values >= 256 clamp to the top bin as in the
 * reference, negative / NaN values -- undefined behaviour in the reference --
 * land in bin 0).  Host pointers. */
int pdb_color_histogram_f32(const float* patches, int64_t n, int32_t h, int32_t w,
                            int32_t bins, int32_t mode, float* out);
int pdb_color_histogram_f32_dev(const float* d_patches, int64_t n, int32_t h, int32_t w,
                                int32_t bins, int32_t mode, float* d_out, void* stream);

/* ---------------------------------------------------------------------------
 * K2 + K3 -- threshold similarity join.
 *
 * Emits every (i, j) with euclidean(L_i, R_j) <= tau, where euclidean is the
 * reference's sequential, unfused fp64 chain (src/index.cpp:69-76) and tau
 * a double (src/planfile.cpp:228-229).  The pair SET is bit-identical to the
 * reference's brute-force contract (tests/oracles.hpp:77-85, equal to
 * sim_join_pairs, src/query.cpp:1094-1104); `dist` is that fp64 distance
 * rounded to fp32.
 *
 * Flags:
 *   PDB_JOIN_SELF    L and R are the same relation; emit only i < j
 *                    (BASELINE's "(i<j, dist)" view; R/nR are ignored).
 *   PDB_JOIN_SORTED  pairs ascend by (left, right) -- the reference's
 *                    emission order when the build side is R (probe order,
 *                    ascending build id).  Without it the order is
 *                    unspecified.
 *   PDB_JOIN_TF32    screen on tf32 instead of bf16 copies.  The screen only
 *                    selects candidates (with a margin covering its rounding);
 *                    every emitted pair is decided by the exact fp64 re-check,
 *                    so the output does not depend on this flag.
 * Sharding (multi-GPU, one process per GPU): with shard_count = P > 1 this
 * call only scans the 128-row blocks of L assigned to shard_index: block
 * b = k*P + (k even ? shard_index : P-1-shard_index), k = 0, 1, ...
 * (boustrophedon rounds; indices stay global), so the shards partition the
 * pair set and share the triangular self-join work evenly. */
#define PDB_JOIN_SELF 1u
#define PDB_JOIN_SORTED 2u
#define PDB_JOIN_TF32 4u   /* screen on tf32 copies (tighter candidate band) instead of bf16;
                              the result is identical either way */
#define PDB_JOIN_DENSE 16u  /* screen every tile: no band plan.  By default, joins with
                               d <= 128, >= 8192 rows per side and >= 16384 dense tiles (32768 when sharded) in
                               this shard first sort the rows
                               by two principal projections and skip the 128x256 tiles whose
                               projected bounding boxes are further apart than tau (an exact
                               bound: the pair set is unchanged); shards then own row blocks
                               of the sorted order. */
#define PDB_JOIN_PHASE_TIMES 8u  /* fill pdb_join_stats' *_ms with CUDA events between the
                                    phases.  The events serialise the phase boundaries (the
                                    kernels are otherwise chained with programmatic dependent
                                    launch), so leave it unset for throughput runs. */

typedef struct pdb_join_opts {
    uint32_t flags;
    int32_t shard_index;
    int32_t shard_count;  /* 0 or 1: no sharding */
    int32_t reserved0;
    void* stream;         /* cudaStream_t for the _dev variants */
} pdb_join_opts;

/* Host-side result of pdb_sim_join; free with pdb_pairs_free. */
typedef struct pdb_pairs {
    int64_t count;
    int32_t* left;   /* row index into L */
    int32_t* right;  /* row index into R (into L for PDB_JOIN_SELF) */
    float* dist;
} pdb_pairs;

/* Per-call counters and device timings (optional out-parameter of the _dev
 * variant).  The *_ms fields are CUDA-event times on the call's stream,
 * recorded only with PDB_JOIN_PHASE_TIMES (0 otherwise). */
typedef struct pdb_join_stats {
    int64_t candidates;      /* pairs passing the tensor-core screen */
    int64_t pairs;           /* pairs passing the exact fp64 re-check */
    int64_t tiles;           /* 128x256 screen tiles executed */
    int64_t candidate_capacity;
    int32_t launches;        /* kernels this call launched */
    int32_t screen_passes;   /* 1, or 2 after a candidate-buffer overflow */
    float prep_ms;           /* centring, screen copies, norms, tile stats, band plan, and the
                                sampled output-size screen pass when one is taken */
    float screen_ms;         /* K2, the tcgen05 screen */
    float recheck_ms;        /* K3, exact re-check + compaction */
    float sort_ms;           /* optional canonical ordering */
    int32_t screen_format;   /* screen copies: 0 tf32, 1 bf16, 2 fp16 (chosen for candidate-heavy
                                band-plan joins; the device keeps bf16 when the data's range
                                would push rows into fp16's subnormals), 3 cosine bf16 */
    int32_t reserved1;
} pdb_join_stats;

/* Host pointers: L [nL, d] and R [nR, d] fp32 row-major. */
int pdb_sim_join(const float* L, int64_t nL, const float* R, int64_t nR, int32_t d,
                 double tau, const pdb_join_opts* opts, pdb_pairs* out);
void pdb_pairs_free(pdb_pairs* p);

/* Device-resident result.  pdb_sim_join_dev (re)allocates the three arrays
 * on the device when `capacity` is smaller than needed, so a caller can keep
 * one pdb_dev_pairs across calls; free with pdb_dev_pairs_free. */
typedef struct pdb_dev_pairs {
    int64_t count;
    int64_t capacity;
    int32_t* left;
    int32_t* right;
    float* dist;
} pdb_dev_pairs;

int pdb_sim_join_dev(const float* d_L, int64_t nL, const float* d_R, int64_t nR, int32_t d,
                     double tau, const pdb_join_opts* opts, pdb_dev_pairs* out,
                     pdb_join_stats* stats);
void pdb_dev_pairs_free(pdb_dev_pairs* p);

/* Cosine threshold join over bf16-stored rows (BASELINE config 4; restated --
 * the reference has no cosine predicate and stores fp32).
 * Emits every (i, j) with cos(L_i, R_j) >= min_cos, where
 *   cos = dot / (sqrt(na) * sqrt(nb)),  dot/na/nb accumulated sequentially in
 * fp64 over k = 0..d-1 from the exact bf16 values (the oracle's
 * orc_cosine_join_bf16); `dist` receives fp32(cos).  Zero or non-finite
 * rows never match.  L, R: [n, d] bf16 bit patterns (uint16). Same flags,
 * sharding and ownership rules as pdb_sim_join. */
int pdb_cosine_join_bf16(const uint16_t* L, int64_t nL, const uint16_t* R, int64_t nR, int32_t d,
                         double min_cos, const pdb_join_opts* opts, pdb_pairs* out);
int pdb_cosine_join_bf16_dev(const uint16_t* d_L, int64_t nL, const uint16_t* d_R, int64_t nR,
                             int32_t d, double min_cos, const pdb_join_opts* opts,
                             pdb_dev_pairs* out, pdb_join_stats* stats);

/* The q1 pipeline in one call (src/bench.cpp:695-730 shape: featurize
 * tiles, then self-join the features): host frames in, host pairs out
 * (PDB_JOIN_SELF semantics).  `features` (host, [tiles, D]) is optional. */
int pdb_featurize_join(const uint8_t* frames, int64_t n_frames, int32_t height, int32_t width,
                       int32_t tile_h, int32_t tile_w, int32_t bins, int32_t mode,
                       double tau, const pdb_join_opts* opts, float* features,
                       pdb_pairs* out);

/* The same pipeline on the device: d_frames [n_frames, H, W, 3] u8 in,
 * d_features [tiles, D] and device pairs (PDB_JOIN_SELF semantics) out, on
 * opts->stream.  The band plan's directions are computed on the first
 * frames' tiles while K1 featurizes the rest (the pair set is the same as
 * pdb_featurize_tiles_dev + pdb_sim_join_dev; only the screened tiles
 * differ).  No sharding. */
int pdb_featurize_join_dev(const uint8_t* d_frames, int64_t n_frames, int32_t height, int32_t width,
                           int32_t tile_h, int32_t tile_w, int32_t bins, int32_t mode, double tau,
                           const pdb_join_opts* opts, float* d_features, pdb_dev_pairs* out,
                           pdb_join_stats* stats);

/* Near-duplicate grouping -- replaces run_dedup (src/query.cpp:535-566),
 * the grouping of PlanNode::dedup (include/patchdb/query.hpp:142) and the
 * kept set of dedup_stream (query.hpp:203-204, src/query.cpp:1063-1092).
 * Items (rows of X [n, d] fp32) are scanned in order; item i is kept as a
 * representative iff no kept representative lies within tau (the reference
 * euclidean <= tau); every other item joins the nearest kept
 * representative, the earliest on ties.  On return rep_of[i] is the index
 * of item i's representative (i itself for representatives) and *n_reps
 * their count.  tau < 0 -> PDB_ERR_CONFIG ("dedup needs tau >= 0"); n > 0
 * with d < 1 -> PDB_ERR_SHAPE.  opts: only `stream` is used (_dev); shards
 * are not supported (the scan is global).  rep_of: host (pdb_dedup) or
 * device (pdb_dedup_dev) int64 [n]. */
int pdb_dedup(const float* X, int64_t n, int32_t d, double tau, const pdb_join_opts* opts,
              int64_t* rep_of, int64_t* n_reps);
int pdb_dedup_dev(const float* d_X, int64_t n, int32_t d, double tau, const pdb_join_opts* opts,
                  int64_t* d_rep_of, int64_t* n_reps);

/* Row-pair `within`: out[k] = euclidean(A[k], B[k]) <= radius (fp64,
 * src/index.cpp:69-76) for k < n, A/B host fp32 [n, d].  Replaces the
 * per-tuple within evaluation of eval_view (src/query.cpp:142-151) when both
 * slots lie in one input; the plan layer batches every tuple into one call. */
int pdb_rows_within(const float* A, const float* B, int64_t n, int32_t d, double radius,
                    uint8_t* out);

/* Frame source -- reads the reference's VideoStore files (record store +
 * descriptor + frame_file / encoded_file / segmented_file layouts with the
 * zlib delta clip codec; src/record_store.cpp, src/storage.cpp:170-501).
 * pdb_store_read replaces VideoStore::open + scan([lo, hi)): frames come out
 * decoded (lossy stores: the quantised pixels the codec kept), lo >= hi is
 * PDB_ERR_CONFIG, both ends clamp to the frame count, lo = hi = -1 means
 * every frame.  Clips decode in parallel on `threads` host threads (zlib).
 * pdb_store_featurize decodes and runs K1 (pdb_featurize_tiles semantics)
 * chunk by chunk into device features [frames, tiles, D]. */
typedef struct pdb_store pdb_store;
typedef struct pdb_store_info {
    int64_t frame_count;
    int32_t width, height;
    int32_t layout;      /* 0 frame_file, 1 encoded_file, 2 segmented_file */
    int32_t codec_mode;  /* 0 lossless, 1 lossy */
    int32_t quant_step;
    int32_t clip_len;
    char video_id[256];
} pdb_store_info;
int pdb_store_open(const char* path, pdb_store** out);
void pdb_store_close(pdb_store* s);
int pdb_store_describe(const pdb_store* s, pdb_store_info* info);
int pdb_store_read(const pdb_store* s, int64_t lo, int64_t hi, uint8_t* frames,
                   int64_t* n_frames, int32_t threads);
int pdb_store_featurize(const pdb_store* s, int64_t lo, int64_t hi, int32_t tile_h,
                        int32_t tile_w, int32_t bins, int32_t mode, float* d_features,
                        int64_t* n_frames, int32_t threads, void* stream);

/* Creates the CUDA context and the library's memory pool and loads the
 * kernels of the common paths (one tiny featurization and self-join), so that
 * the first real call of a process does not pay the device start-up (~1.5 s
 * on a fresh B200 process).  Optional; safe to call from a background thread
 * at start-up.  No reference counterpart. */
int pdb_warmup(void);

/* Returns the device memory the library keeps between calls on the calling
 * thread (the grow-only candidate-record buffer of large joins) and trims the
 * library's own stream-ordered pool to zero.  Synchronises the device.  No
 * reference counterpart: the reference holds no device memory. */
int pdb_release_caches(void);

/* Pinned host memory helpers (the e2e path copies from pinned buffers). */
void* pdb_host_alloc(int64_t bytes);
void pdb_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* PDB_CUDA_H */
