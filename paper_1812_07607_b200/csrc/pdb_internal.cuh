// pdb_internal.cuh -- shared plumbing of libpdb_cuda.so: status/error
// propagation, the per-device context, and small launch helpers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "pdb_cuda.h"

#define PDB_HIDDEN __attribute__((visibility("hidden")))

// Device-side bounds checks of the checked build (libpdb_cuda_checked.so,
// `make checked`, -DPDB_CHECKED): a violated check prints its site and traps,
// failing the call with a CUDA error.  The product build compiles them out.
// (compute-sanitizer is closed on this GPU pool; these checks plus the
// oracle comparisons of tools/sanitize_cases.py stand in for memcheck.)
#ifdef PDB_CHECKED
#include <cstdio>
#define PDB_DCHECK(c)                                                                  \
    do {                                                                               \
        if (!(c)) {                                                                    \
            printf("PDB_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, \
                   #c, (int)blockIdx.x, (int)threadIdx.x);                             \
            __trap();                                                                  \
        }                                                                              \
    } while (0)
#else
#define PDB_DCHECK(c) \
    do {              \
    } while (0)
#endif

namespace pdb {

// Thread-local error state behind pdb_last_error().
PDB_HIDDEN void set_error(const std::string& msg);
PDB_HIDDEN void clear_error();

// A failure carried from deep inside a launcher to the C-ABI boundary,
// which converts it into a status code (nothing throws across extern "C").
struct Failure {
    int status;
    std::string msg;
};

[[noreturn]] PDB_HIDDEN void fail(int status, const std::string& msg);
PDB_HIDDEN void check_cuda(cudaError_t e, const char* what);

#define PDB_CUDA(call) ::pdb::check_cuda((call), #call)

struct DeviceCtx {
    int device = -1;
    int sm_count = 0;
    int cc_major = 0, cc_minor = 0;
    size_t smem_optin = 0;
    void* encode_tiled = nullptr;  // cuTensorMapEncodeTiled from the driver
    cudaMemPool_t pool = nullptr;  // the library's stream-ordered pool
};

// Context of the calling thread's current device; fails with
// PDB_ERR_NO_DEVICE when there is no sm_100 GPU (there is no CPU path).
PDB_HIDDEN const DeviceCtx& device_ctx();

// Stream-ordered scratch allocation from the library's own memory pool
// (release threshold raised once, so repeated calls reuse memory).
PDB_HIDDEN void* dev_alloc(size_t bytes, cudaStream_t s);
// The same, returning null instead of failing (optional speed-up buffers).
PDB_HIDDEN void* dev_try_alloc(size_t bytes, cudaStream_t s);
// Frees the calling thread's grow-only join buffers (pdb_release_caches).
PDB_HIDDEN void release_join_caches();
PDB_HIDDEN void dev_free(void* p, cudaStream_t s);

template <class T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(size_t n, cudaStream_t st) : s(st) {
        if (n) p = static_cast<T*>(dev_alloc(n * sizeof(T), st));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { reset(); }
    void reset() {
        if (p) dev_free(p, s);
        p = nullptr;
    }
    void reset(size_t n, cudaStream_t st) {
        reset();
        s = st;
        if (n) p = static_cast<T*>(dev_alloc(n * sizeof(T), st));
    }
    T* release() {
        T* q = p;
        p = nullptr;
        return q;
    }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// One stream-ordered allocation carved into 256-byte aligned pieces: a join
// call takes its dozen small scratch buffers from one pool allocation.
struct Arena {
    DevBuf<uint8_t> buf;
    size_t used = 0, cap = 0;
    void reserve(size_t bytes, cudaStream_t s) {
        buf.reset(bytes, s);
        cap = bytes;
        used = 0;
    }
    template <class T>
    T* take(size_t n) {
        const size_t off = (used + 255) & ~size_t(255);
        used = off + n * sizeof(T);
        if (used > cap) fail(PDB_ERR_OUT_OF_MEMORY, "internal arena overflow");
        return reinterpret_cast<T*>(buf.p + off);
    }
    static size_t need(size_t n, size_t elem) { return ((n * elem + 255) & ~size_t(255)) + 256; }
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per kernel.
PDB_HIDDEN void set_max_smem(const void* func, int bytes);

// Launch with programmatic stream serialisation: the kernel may be
// scheduled while its stream predecessor drains; it must call
// ptx::pdl_wait() before reading anything the predecessor wrote.
template <typename... KArgs, typename... Args>
void launch_pdl_if(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                   cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    check_cuda(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...), "cudaLaunchKernelEx");
}

template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                Args&&... args) {
    launch_pdl_if(true, kern, grid, block, smem, s, std::forward<Args>(args)...);
}

// ---- K1 launchers (histogram.cu) -----------------------------------------
// Feature outputs of one featurization: the local buffer first, then (a
// sharded step) peers' buffers mapped over NVLink, all at the same offset.
constexpr int kMaxFeatOuts = 8;
struct FeatOuts {
    float* p[kMaxFeatOuts];
    int n;
    // optional: each consumer warp of the joint-rows K1 adds 1 here once its
    // first tile row's features are stored (run_featurize_join_dev)
    unsigned* done;
};
// *first_round (optional): tiles [0, *first_round) are the ones whose
// completion outs.done counts (one count per tile), or -1 when the kernel
// taken does not signal.
PDB_HIDDEN void launch_featurize_tiles_multi(const uint8_t* d_frames, int64_t n_frames, int32_t H,
                                             int32_t W, int32_t th, int32_t tw, int32_t bins,
                                             int32_t mode, const FeatOuts& outs, cudaStream_t s,
                                             int sm_reserve = 0, int64_t* first_round = nullptr);
PDB_HIDDEN int hist_dim(int32_t bins, int32_t mode);
PDB_HIDDEN void launch_featurize_tiles(const uint8_t* d_frames, int64_t n_frames, int32_t H,
                                       int32_t W, int32_t th, int32_t tw, int32_t bins,
                                       int32_t mode, float* d_out, cudaStream_t s,
                                       int sm_reserve = 0);
PDB_HIDDEN void launch_hist_f32(const float* d_px, int64_t n, int32_t h, int32_t w,
                                int32_t bins, int32_t mode, float* d_out, cudaStream_t s);

// ---- K2/K3 (join.cu) -------------------------------------------------------
// The band plan's centre and directions computed ahead of the join
// (run_featurize_join_dev: on a prefix sample, beside the rest of K1).
struct JoinPre {
    const float* mu;   // [DP] centre
    const void* info;  // BandInfo (join.cu)
    void* ready;       // cudaEvent_t after which mu and info are valid (the join's
                       // stream waits for it before their first reader), or null
};
PDB_HIDDEN void run_sim_join_dev(const float* d_L, int64_t nL, const float* d_R, int64_t nR,
                                 int32_t d, double tau, const pdb_join_opts& o,
                                 pdb_dev_pairs* out, pdb_join_stats* stats,
                                 const JoinPre* pre = nullptr);
PDB_HIDDEN void run_featurize_join_dev(const uint8_t* d_frames, int64_t n, int32_t H, int32_t W,
                                       int32_t th, int32_t tw, int32_t bins, int32_t mode,
                                       float* d_feats, double tau, const pdb_join_opts& o,
                                       pdb_dev_pairs* out, pdb_join_stats* stats);
PDB_HIDDEN void run_dedup_dev(const float* d_X, int64_t n, int32_t d, double tau, cudaStream_t s,
                              int64_t* d_rep_of, int64_t* n_reps);
// out[k] = euclidean(A[k], B[k]) <= radius (rows.cu)
PDB_HIDDEN void run_rows_within(const float* d_A, const float* d_B, int64_t n, int32_t d,
                                double radius, uint8_t* d_out, cudaStream_t s);
PDB_HIDDEN void run_cos_join_dev(const uint16_t* d_L, int64_t nL, const uint16_t* d_R, int64_t nR,
                                 int32_t d, double min_cos, const pdb_join_opts& o,
                                 pdb_dev_pairs* out, pdb_join_stats* stats);

}  // namespace pdb
