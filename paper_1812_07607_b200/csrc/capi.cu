// capi.cu -- the extern "C" boundary of libpdb_cuda.so (include/pdb_cuda.h):
// argument validation with the reference's error taxonomy, the per-device
// context, stream-ordered scratch memory, host<->device staging.

#include <cuda.h>
#include <cudaTypedefs.h>

#include <sys/mman.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pdb_internal.cuh"

#define PDB_API extern "C" __attribute__((visibility("default")))

namespace pdb {

namespace {
thread_local std::string g_last_error;
std::mutex g_ctx_mu;
DeviceCtx g_ctx[64];
bool g_ctx_ok[64] = {};
}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }

void fail(int status, const std::string& msg) { throw Failure{status, msg}; }

void check_cuda(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    const int st = e == cudaErrorMemoryAllocation ? PDB_ERR_OUT_OF_MEMORY : PDB_ERR_CUDA;
    fail(st, std::string(what) + ": " + cudaGetErrorString(e));
}

const DeviceCtx& device_ctx() {
    int dev = 0;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        fail(PDB_ERR_NO_DEVICE, "no CUDA device visible (libpdb_cuda has no CPU path)");
    }
    PDB_CUDA(cudaGetDevice(&dev));
    if (dev < 0 || dev >= 64) fail(PDB_ERR_NO_DEVICE, "device ordinal out of range");
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (g_ctx_ok[dev]) return g_ctx[dev];
    DeviceCtx c;
    c.device = dev;
    cudaDeviceProp prop;
    PDB_CUDA(cudaGetDeviceProperties(&prop, dev));
    c.sm_count = prop.multiProcessorCount;
    c.cc_major = prop.major;
    c.cc_minor = prop.minor;
    c.smem_optin = prop.sharedMemPerBlockOptin;
    if (prop.major != 10)
        fail(PDB_ERR_NO_DEVICE, std::string("device '") + prop.name +
                                    "' is not sm_100 (Blackwell); this build targets sm_100a only");
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    PDB_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
        fail(PDB_ERR_CUDA, "driver entry point cuTensorMapEncodeTiled unavailable");
    c.encode_tiled = fn;
    // The library's own stream-ordered pool: freed scratch stays mapped
    // between calls (release threshold raised on this pool only, not on the
    // device's default pool other libraries in the process share);
    // pdb_release_caches() trims it.
    cudaMemPoolProps pp{};
    pp.allocType = cudaMemAllocationTypePinned;
    pp.location.type = cudaMemLocationTypeDevice;
    pp.location.id = dev;
    PDB_CUDA(cudaMemPoolCreate(&c.pool, &pp));
    uint64_t thr = UINT64_MAX;
    PDB_CUDA(cudaMemPoolSetAttribute(c.pool, cudaMemPoolAttrReleaseThreshold, &thr));
    g_ctx[dev] = c;
    g_ctx_ok[dev] = true;
    return g_ctx[dev];
}

void* dev_try_alloc(size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    if (cudaMallocFromPoolAsync(&p, std::max<size_t>(bytes, 16), device_ctx().pool, s) !=
        cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

void* dev_alloc(size_t bytes, cudaStream_t s) {
    void* p = nullptr;
    const cudaError_t e = cudaMallocFromPoolAsync(&p, std::max<size_t>(bytes, 16), device_ctx().pool, s);
    if (e != cudaSuccess) {
        cudaGetLastError();
        fail(PDB_ERR_OUT_OF_MEMORY, "device allocation of " + std::to_string(bytes) +
                                        " bytes failed: " + cudaGetErrorString(e));
    }
    return p;
}

void dev_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

void set_max_smem(const void* func, int bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<const void*, int>, int>> done;  // ((func, dev), bytes)
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    for (auto& e : done)
        if (e.first.first == func && e.first.second == dev && e.second >= bytes) return;
    PDB_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    done.push_back({{func, dev}, bytes});
}

}  // namespace pdb

using namespace pdb;

namespace {

// Runs `body`, converting Failure / CUDA errors into status codes.
template <class F>
int guarded(F&& body) {
    clear_error();
    try {
        body();
        return PDB_OK;
    } catch (const Failure& f) {
        set_error(f.msg);
        return f.status;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return PDB_ERR_OUT_OF_MEMORY;
    } catch (...) {
        set_error("unexpected exception");
        return PDB_ERR_CUDA;
    }
}

cudaStream_t stream_of(void* s) { return s ? static_cast<cudaStream_t>(s) : cudaStreamPerThread; }

void check_featurize_args(const void* frames, int64_t n, int32_t H, int32_t W, int32_t th,
                          int32_t tw, int32_t bins, int32_t mode, const void* out) {
    // Reference order: TransformerSpec::validate (bins, src/etl.cpp:64-67) and
    // GeneratorSpec::validate (tile sizes, src/etl.cpp:47-50) -> ConfigError.
    if (mode != PDB_HIST_PER_CHANNEL && mode != PDB_HIST_JOINT)
        fail(PDB_ERR_INVALID_ARGUMENT, "histogram mode must be 0 (per-channel) or 1 (joint)");
    if (bins < 2) fail(PDB_ERR_CONFIG, "color_histogram needs at least 2 bins per channel");
    if (hist_dim(bins, mode) < 0)
        fail(PDB_ERR_CONFIG, "joint colour histogram supports 2..16 bins per channel");
    if (tw < 1 || th < 1) fail(PDB_ERR_CONFIG, "tiles generator needs tile_w and tile_h >= 1");
    if (n < 0 || H < 0 || W < 0) fail(PDB_ERR_INVALID_ARGUMENT, "negative frame count or size");
    if (n > 0 && (!frames || !out)) fail(PDB_ERR_INVALID_ARGUMENT, "null frames/out pointer");
}

int64_t n_tiles_of(int64_t n, int32_t H, int32_t W, int32_t th, int32_t tw) {
    return n * static_cast<int64_t>(W / tw) * static_cast<int64_t>(H / th);
}

void check_join_args(const void* L, int64_t nL, const void* R, int64_t nR, int32_t d, double tau,
                     const pdb_join_opts* o) {
    // run_sim_join order: tau (src/query.cpp:488), then dims (467-499).  The
    // reference rejects only tau < 0.0: a NaN tau passes and matches nothing.
    if (tau < 0.0) fail(PDB_ERR_CONFIG, "similarity join needs tau >= 0");
    if (nL < 0 || nR < 0) fail(PDB_ERR_INVALID_ARGUMENT, "negative row count");
    if (nL > INT32_MAX || nR > INT32_MAX)
        fail(PDB_ERR_INVALID_ARGUMENT, "row counts above 2^31-1 are not supported");
    const bool self = o && (o->flags & PDB_JOIN_SELF);
    if ((nL > 0 || (!self && nR > 0)) && d < 1)
        fail(PDB_ERR_SHAPE, "similarity join needs non-empty patch data");
    if (nL > 0 && !L) fail(PDB_ERR_INVALID_ARGUMENT, "null L");
    if (!self && nR > 0 && !R) fail(PDB_ERR_INVALID_ARGUMENT, "null R");
    if (o && (o->flags & ~(PDB_JOIN_SELF | PDB_JOIN_SORTED | PDB_JOIN_TF32 | PDB_JOIN_PHASE_TIMES |
                           PDB_JOIN_DENSE)))
        fail(PDB_ERR_INVALID_ARGUMENT, "unknown join flags");
    if (o && o->shard_count > 1 && (o->shard_index < 0 || o->shard_index >= o->shard_count))
        fail(PDB_ERR_INVALID_ARGUMENT, "shard_index out of range");
}

// Host memory for a pairs array: 2 MB-aligned with transparent huge pages
// requested when large (a fresh 4 KB-paged malloc of the config-5 output --
// 12.5 GB -- costs millions of first-touch page faults inside the copy).
void* host_pairs_alloc(size_t bytes) {
    constexpr size_t kHuge = size_t{2} << 20;
    if (bytes < kHuge) return std::malloc(bytes);
    void* p = nullptr;
    if (posix_memalign(&p, kHuge, (bytes + kHuge - 1) / kHuge * kHuge) != 0) return nullptr;
#ifdef MADV_HUGEPAGE
    madvise(p, (bytes + kHuge - 1) / kHuge * kHuge, MADV_HUGEPAGE);
#endif
    return p;
}

// Device -> pageable host copy of an array above 1 MB: 64 MB chunks staged
// through a per-thread ring of pinned buffers, each chunk's host copy split
// over host threads while the next chunk crosses PCIe (a plain pageable
// cudaMemcpy moved ~2 GB/s into fresh memory: config-5 e2e 6.1 s -> 0.71 s).
void d2h_large(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    constexpr size_t kChunk = size_t{64} << 20;
    constexpr int kRing = 3;
    if (bytes <= (size_t{1} << 20)) {
        PDB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        PDB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    // one process-wide ring (192 MB of pinned memory, portable across
    // devices; events per device), held for the whole copy: concurrent
    // copies share PCIe anyway
    struct Ring {
        void* buf[kRing] = {};
        cudaEvent_t ev[64][kRing] = {};
    };
    static Ring ring;
    static std::mutex ring_mu;
    std::lock_guard<std::mutex> lk(ring_mu);
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    cudaEvent_t* evs = ring.ev[dev & 63];
    for (int k = 0; k < kRing; k++) {
        if (!ring.buf[k]) PDB_CUDA(cudaHostAlloc(&ring.buf[k], kChunk, cudaHostAllocPortable));
        if (!evs[k]) PDB_CUDA(cudaEventCreateWithFlags(&evs[k], cudaEventDisableTiming));
    }
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    // (one host thread per MB, at most 16)
    const int nthr = static_cast<int>(std::min<size_t>(std::min(16u, hw), std::max<size_t>(1, bytes >> 20)));
    auto host_copy = [&](char* d, const char* src_h, size_t len) {
        const size_t part = (len / nthr + 4095) / 4096 * 4096;
        std::vector<std::thread> th;
        for (int t = 1; t < nthr; t++) {
            const size_t o = static_cast<size_t>(t) * part;
            if (o >= len) break;
            th.emplace_back([=] { std::memcpy(d + o, src_h + o, std::min(part, len - o)); });
        }
        std::memcpy(d, src_h, std::min(part, len));
        for (auto& x : th) x.join();
    };
    const size_t n_chunks = (bytes + kChunk - 1) / kChunk;
    auto len_of = [&](size_t i) { return std::min(kChunk, bytes - i * kChunk); };
    for (size_t i = 0; i <= n_chunks; i++) {
        if (i < n_chunks) {
            const int k = static_cast<int>(i % kRing);
            PDB_CUDA(cudaMemcpyAsync(ring.buf[k], static_cast<const char*>(src) + i * kChunk, len_of(i),
                                     cudaMemcpyDeviceToHost, s));
            PDB_CUDA(cudaEventRecord(evs[k], s));
        }
        if (i >= 1) {  // the previous chunk: on the host while this one crosses PCIe
            const int k = static_cast<int>((i - 1) % kRing);
            PDB_CUDA(cudaEventSynchronize(evs[k]));
            host_copy(static_cast<char*>(dst) + (i - 1) * kChunk, static_cast<const char*>(ring.buf[k]),
                      len_of(i - 1));
        }
    }
}

// The library's own device pairs, returned to the stream-ordered pool (the
// public pdb_dev_pairs_free uses cudaFree, which synchronises the device).
void dev_pairs_release(pdb_dev_pairs* p, cudaStream_t s) {
    dev_free(p->left, s);
    dev_free(p->right, s);
    dev_free(p->dist, s);
    p->left = p->right = nullptr;
    p->dist = nullptr;
    p->count = p->capacity = 0;
}

void pairs_to_host(const pdb_dev_pairs& dp, pdb_pairs* out, cudaStream_t s) {
    out->count = dp.count;
    const size_t n = static_cast<size_t>(std::max<int64_t>(dp.count, 1));
    out->left = static_cast<int32_t*>(host_pairs_alloc(n * sizeof(int32_t)));
    out->right = static_cast<int32_t*>(host_pairs_alloc(n * sizeof(int32_t)));
    out->dist = static_cast<float*>(host_pairs_alloc(n * sizeof(float)));
    if (!out->left || !out->right || !out->dist) {
        pdb_pairs_free(out);
        fail(PDB_ERR_OUT_OF_MEMORY, "host allocation for pairs failed");
    }
    PDB_CUDA(cudaStreamSynchronize(s));
    if (dp.count > 0) {
        d2h_large(out->left, dp.left, dp.count * sizeof(int32_t), s);
        d2h_large(out->right, dp.right, dp.count * sizeof(int32_t), s);
        d2h_large(out->dist, dp.dist, dp.count * sizeof(float), s);
    }
    PDB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

PDB_API const char* pdb_last_error(void) { return g_last_error.c_str(); }

PDB_API const char* pdb_status_name(int status) {
    switch (status) {
        case PDB_OK: return "ok";
        case PDB_ERR_CONFIG: return "ConfigError";
        case PDB_ERR_SHAPE: return "ShapeError";
        case PDB_ERR_MIXED_DIMENSION: return "MixedDimensionError";
        case PDB_ERR_DIMENSION_MISMATCH: return "DimensionMismatchError";
        case PDB_ERR_DUPLICATE_ID: return "DuplicatePatchIdError";
        case PDB_ERR_CAPACITY: return "CapacityError";
        case PDB_ERR_INVALID_ARGUMENT: return "InvalidArgument";
        case PDB_ERR_CUDA: return "CudaError";
        case PDB_ERR_OUT_OF_MEMORY: return "OutOfMemory";
        case PDB_ERR_NO_DEVICE: return "NoDevice";
    }
    return "unknown";
}

PDB_API int pdb_version(void) { return (0 << 16) | (1 << 8) | 0; }

PDB_API int pdb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    int ok = 0;
    for (int i = 0; i < n; i++) {
        cudaDeviceProp p;
        if (cudaGetDeviceProperties(&p, i) == cudaSuccess && p.major == 10) ok++;
    }
    return ok;
}

PDB_API int pdb_hist_dim(int32_t bins, int32_t mode) { return hist_dim(bins, mode); }

PDB_API int pdb_featurize_tiles_dev(const uint8_t* d_frames, int64_t n, int32_t H, int32_t W,
                                    int32_t th, int32_t tw, int32_t bins, int32_t mode,
                                    float* d_out, void* stream) {
    return guarded([&] {
        check_featurize_args(d_frames, n, H, W, th, tw, bins, mode, d_out);
        device_ctx();
        launch_featurize_tiles(d_frames, n, H, W, th, tw, bins, mode, d_out, stream_of(stream));
    });
}

PDB_API int pdb_featurize_tiles_dev_multi(const uint8_t* d_frames, int64_t n, int32_t H, int32_t W,
                                          int32_t th, int32_t tw, int32_t bins, int32_t mode,
                                          float* const* d_outs, int32_t n_outs, void* stream) {
    return guarded([&] {
        if (!d_outs || n_outs < 1 || n_outs > kMaxFeatOuts)
            fail(PDB_ERR_INVALID_ARGUMENT, "n_outs must be 1..8 output pointers");
        for (int k = 0; k < n_outs; k++)
            if (!d_outs[k]) fail(PDB_ERR_INVALID_ARGUMENT, "null output pointer");
        check_featurize_args(d_frames, n, H, W, th, tw, bins, mode, d_outs[0]);
        device_ctx();
        FeatOuts o{};
        o.done = nullptr;
        for (int k = 0; k < n_outs; k++) o.p[k] = d_outs[k];
        o.n = n_outs;
        launch_featurize_tiles_multi(d_frames, n, H, W, th, tw, bins, mode, o, stream_of(stream));
    });
}

PDB_API int pdb_featurize_tiles(const uint8_t* frames, int64_t n, int32_t H, int32_t W,
                                int32_t th, int32_t tw, int32_t bins, int32_t mode, float* out) {
    return guarded([&] {
        check_featurize_args(frames, n, H, W, th, tw, bins, mode, out);
        device_ctx();
        const int64_t nt = n_tiles_of(n, H, W, th, tw);
        const int D = hist_dim(bins, mode);
        if (nt == 0) return;
        cudaStream_t s = cudaStreamPerThread;
        const size_t fbytes = static_cast<size_t>(n) * H * W * 3;
        DevBuf<uint8_t> dF(fbytes, s);
        DevBuf<float> dO(static_cast<size_t>(nt) * D, s);
        PDB_CUDA(cudaMemcpyAsync(dF.p, frames, fbytes, cudaMemcpyHostToDevice, s));
        launch_featurize_tiles(dF.p, n, H, W, th, tw, bins, mode, dO.p, s);
        PDB_CUDA(cudaMemcpyAsync(out, dO.p, static_cast<size_t>(nt) * D * sizeof(float),
                                 cudaMemcpyDeviceToHost, s));
        PDB_CUDA(cudaStreamSynchronize(s));
    });
}

static void check_f32_args(const void* px, int64_t n, int32_t h, int32_t w, int32_t bins,
                           int32_t mode, const void* out) {
    if (mode != PDB_HIST_PER_CHANNEL && mode != PDB_HIST_JOINT)
        fail(PDB_ERR_INVALID_ARGUMENT, "histogram mode must be 0 (per-channel) or 1 (joint)");
    if (bins < 2) fail(PDB_ERR_CONFIG, "color_histogram needs at least 2 bins per channel");
    if (hist_dim(bins, mode) < 0)
        fail(PDB_ERR_CONFIG, "joint colour histogram supports 2..16 bins per channel");
    // apply_transformer: input must be pixel shaped [h,w,3] (src/etl.cpp:332-334).
    if (h < 1 || w < 1) fail(PDB_ERR_SHAPE, "transformer input must be pixel shaped [h,w,3]");
    if (n < 0) fail(PDB_ERR_INVALID_ARGUMENT, "negative patch count");
    if (n > 0 && (!px || !out)) fail(PDB_ERR_INVALID_ARGUMENT, "null pointer");
}

PDB_API int pdb_color_histogram_f32_dev(const float* d_px, int64_t n, int32_t h, int32_t w,
                                        int32_t bins, int32_t mode, float* d_out, void* stream) {
    return guarded([&] {
        check_f32_args(d_px, n, h, w, bins, mode, d_out);
        device_ctx();
        launch_hist_f32(d_px, n, h, w, bins, mode, d_out, stream_of(stream));
    });
}

PDB_API int pdb_color_histogram_f32(const float* px, int64_t n, int32_t h, int32_t w,
                                    int32_t bins, int32_t mode, float* out) {
    return guarded([&] {
        check_f32_args(px, n, h, w, bins, mode, out);
        device_ctx();
        if (n == 0) return;
        cudaStream_t s = cudaStreamPerThread;
        const size_t in_n = static_cast<size_t>(n) * h * w * 3;
        const size_t D = static_cast<size_t>(hist_dim(bins, mode));
        DevBuf<float> dI(in_n, s), dO(static_cast<size_t>(n) * D, s);
        PDB_CUDA(cudaMemcpyAsync(dI.p, px, in_n * sizeof(float), cudaMemcpyHostToDevice, s));
        launch_hist_f32(dI.p, n, h, w, bins, mode, dO.p, s);
        PDB_CUDA(cudaMemcpyAsync(out, dO.p, static_cast<size_t>(n) * D * sizeof(float),
                                 cudaMemcpyDeviceToHost, s));
        PDB_CUDA(cudaStreamSynchronize(s));
    });
}

PDB_API int pdb_sim_join_dev(const float* d_L, int64_t nL, const float* d_R, int64_t nR,
                             int32_t d, double tau, const pdb_join_opts* opts, pdb_dev_pairs* out,
                             pdb_join_stats* stats) {
    return guarded([&] {
        if (!out) fail(PDB_ERR_INVALID_ARGUMENT, "null output");
        check_join_args(d_L, nL, d_R, nR, d, tau, opts);
        device_ctx();
        pdb_join_opts o = opts ? *opts : pdb_join_opts{};
        o.stream = stream_of(o.stream);
        run_sim_join_dev(d_L, nL, d_R, nR, d, tau, o, out, stats);
    });
}

PDB_API int pdb_featurize_join_dev(const uint8_t* d_frames, int64_t n, int32_t H, int32_t W,
                                   int32_t th, int32_t tw, int32_t bins, int32_t mode, double tau,
                                   const pdb_join_opts* opts, float* d_features, pdb_dev_pairs* out,
                                   pdb_join_stats* stats) {
    return guarded([&] {
        if (!out) fail(PDB_ERR_INVALID_ARGUMENT, "null output");
        check_featurize_args(d_frames, n, H, W, th, tw, bins, mode, d_features);
        if (tau < 0.0) fail(PDB_ERR_CONFIG, "similarity join needs tau >= 0");
        if (opts && opts->shard_count > 1)
            fail(PDB_ERR_INVALID_ARGUMENT, "pdb_featurize_join_dev does not shard");
        const int64_t nt = n_tiles_of(n, H, W, th, tw);
        if (nt > INT32_MAX) fail(PDB_ERR_INVALID_ARGUMENT, "too many tiles");
        device_ctx();
        pdb_join_opts o = opts ? *opts : pdb_join_opts{};
        o.stream = stream_of(o.stream);
        run_featurize_join_dev(d_frames, n, H, W, th, tw, bins, mode, d_features, tau, o, out, stats);
    });
}

PDB_API void pdb_dev_pairs_free(pdb_dev_pairs* p) {
    if (!p) return;
    cudaFree(p->left);
    cudaFree(p->right);
    cudaFree(p->dist);
    p->left = p->right = nullptr;
    p->dist = nullptr;
    p->count = p->capacity = 0;
}

PDB_API int pdb_sim_join(const float* L, int64_t nL, const float* R, int64_t nR, int32_t d,
                         double tau, const pdb_join_opts* opts, pdb_pairs* out) {
    if (out) std::memset(out, 0, sizeof(*out));
    return guarded([&] {
        if (!out) fail(PDB_ERR_INVALID_ARGUMENT, "null output");
        check_join_args(L, nL, R, nR, d, tau, opts);
        device_ctx();
        pdb_join_opts o = opts ? *opts : pdb_join_opts{};
        cudaStream_t s = cudaStreamPerThread;
        o.stream = s;
        const bool self = (o.flags & PDB_JOIN_SELF) != 0;
        DevBuf<float> dL(static_cast<size_t>(nL) * std::max(d, 1), s), dR;
        if (nL > 0)
            PDB_CUDA(cudaMemcpyAsync(dL.p, L, static_cast<size_t>(nL) * d * sizeof(float),
                                     cudaMemcpyHostToDevice, s));
        if (!self && nR > 0) {
            dR.reset(static_cast<size_t>(nR) * d, s);
            PDB_CUDA(cudaMemcpyAsync(dR.p, R, static_cast<size_t>(nR) * d * sizeof(float),
                                     cudaMemcpyHostToDevice, s));
        }
        pdb_dev_pairs dp{};
        try {
            run_sim_join_dev(dL.p, nL, self ? dL.p : dR.p, self ? nL : nR, d, tau, o, &dp, nullptr);
            pairs_to_host(dp, out, s);
        } catch (...) {
            dev_pairs_release(&dp, s);
            throw;
        }
        dev_pairs_release(&dp, s);
    });
}

static void check_cos_args(const void* L, int64_t nL, const void* R, int64_t nR, int32_t d,
                           double min_cos, const pdb_join_opts* o) {
    if (!(min_cos >= -1.0 && min_cos <= 1.0))
        fail(PDB_ERR_CONFIG, "cosine join needs -1 <= min_cos <= 1");
    check_join_args(L, nL, R, nR, d, 0.0, o);
}

PDB_API int pdb_cosine_join_bf16_dev(const uint16_t* d_L, int64_t nL, const uint16_t* d_R,
                                     int64_t nR, int32_t d, double min_cos,
                                     const pdb_join_opts* opts, pdb_dev_pairs* out,
                                     pdb_join_stats* stats) {
    return guarded([&] {
        if (!out) fail(PDB_ERR_INVALID_ARGUMENT, "null output");
        check_cos_args(d_L, nL, d_R, nR, d, min_cos, opts);
        device_ctx();
        pdb_join_opts o = opts ? *opts : pdb_join_opts{};
        o.stream = stream_of(o.stream);
        run_cos_join_dev(d_L, nL, d_R, nR, d, min_cos, o, out, stats);
    });
}

PDB_API int pdb_cosine_join_bf16(const uint16_t* L, int64_t nL, const uint16_t* R, int64_t nR,
                                 int32_t d, double min_cos, const pdb_join_opts* opts,
                                 pdb_pairs* out) {
    if (out) std::memset(out, 0, sizeof(*out));
    return guarded([&] {
        if (!out) fail(PDB_ERR_INVALID_ARGUMENT, "null output");
        check_cos_args(L, nL, R, nR, d, min_cos, opts);
        device_ctx();
        pdb_join_opts o = opts ? *opts : pdb_join_opts{};
        cudaStream_t s = cudaStreamPerThread;
        o.stream = s;
        const bool self = (o.flags & PDB_JOIN_SELF) != 0;
        DevBuf<uint16_t> dL(static_cast<size_t>(nL) * std::max(d, 1), s), dR;
        if (nL > 0)
            PDB_CUDA(cudaMemcpyAsync(dL.p, L, static_cast<size_t>(nL) * d * 2,
                                     cudaMemcpyHostToDevice, s));
        if (!self && nR > 0) {
            dR.reset(static_cast<size_t>(nR) * d, s);
            PDB_CUDA(cudaMemcpyAsync(dR.p, R, static_cast<size_t>(nR) * d * 2,
                                     cudaMemcpyHostToDevice, s));
        }
        pdb_dev_pairs dp{};
        try {
            run_cos_join_dev(dL.p, nL, self ? dL.p : dR.p, self ? nL : nR, d, min_cos, o, &dp,
                             nullptr);
            pairs_to_host(dp, out, s);
        } catch (...) {
            dev_pairs_release(&dp, s);
            throw;
        }
        dev_pairs_release(&dp, s);
    });
}

PDB_API void pdb_pairs_free(pdb_pairs* p) {
    if (!p) return;
    std::free(p->left);
    std::free(p->right);
    std::free(p->dist);
    p->left = p->right = nullptr;
    p->dist = nullptr;
    p->count = 0;
}

PDB_API int pdb_featurize_join(const uint8_t* frames, int64_t n, int32_t H, int32_t W,
                               int32_t th, int32_t tw, int32_t bins, int32_t mode, double tau,
                               const pdb_join_opts* opts, float* features, pdb_pairs* out) {
    if (out) std::memset(out, 0, sizeof(*out));
    return guarded([&] {
        if (!out) fail(PDB_ERR_INVALID_ARGUMENT, "null output");
        check_featurize_args(frames, n, H, W, th, tw, bins, mode, frames);
        if (tau < 0.0) fail(PDB_ERR_CONFIG, "similarity join needs tau >= 0");
        device_ctx();
        const int64_t nt = n_tiles_of(n, H, W, th, tw);
        const int D = hist_dim(bins, mode);
        if (nt > INT32_MAX) fail(PDB_ERR_INVALID_ARGUMENT, "too many tiles");
        cudaStream_t s = cudaStreamPerThread;
        const size_t fb = static_cast<size_t>(H) * W * 3;
        DevBuf<uint8_t> dF(static_cast<size_t>(n) * fb, s);
        DevBuf<float> dX(static_cast<size_t>(std::max<int64_t>(nt, 1)) * D, s);
        // Copy frames in chunks on a second stream so K1 on chunk k overlaps
        // the H2D copy of chunk k+1.  The copy stream and the chunk events
        // are created once per host thread and device (creating a stream
        // measured ~1 ms per call).
        struct CopyCtx {
            cudaStream_t cs = nullptr;
            std::vector<cudaEvent_t> evs;
        };
        thread_local CopyCtx copy_ctx[64];
        int dev = 0;
        PDB_CUDA(cudaGetDevice(&dev));
        CopyCtx& cc = copy_ctx[dev & 63];
        if (!cc.cs) PDB_CUDA(cudaStreamCreateWithFlags(&cc.cs, cudaStreamNonBlocking));
        cudaStream_t cs = cc.cs;
        const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, 64));
        const int64_t n_chunks = ceil_div(n, chunk);
        while (static_cast<int64_t>(cc.evs.size()) < n_chunks) {
            cudaEvent_t e;
            PDB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            cc.evs.push_back(e);
        }
        // the copy stream must not overwrite frames a previous call's K1 still reads
        PDB_CUDA(cudaStreamSynchronize(s));
        const int64_t tpf = static_cast<int64_t>(W / tw) * (H / th);
        for (int64_t f0 = 0, k = 0; f0 < n; f0 += chunk, k++) {
            const int64_t cnt = std::min(chunk, n - f0);
            cudaEvent_t e = cc.evs[static_cast<size_t>(k)];
            PDB_CUDA(cudaMemcpyAsync(dF.p + f0 * fb, frames + f0 * fb, cnt * fb,
                                     cudaMemcpyHostToDevice, cs));
            PDB_CUDA(cudaEventRecord(e, cs));
            PDB_CUDA(cudaStreamWaitEvent(s, e, 0));
            launch_featurize_tiles(dF.p + f0 * fb, cnt, H, W, th, tw, bins, mode,
                                   dX.p + f0 * tpf * D, s);
        }
        pdb_join_opts o = opts ? *opts : pdb_join_opts{};
        o.flags |= PDB_JOIN_SELF;
        o.stream = s;
        pdb_dev_pairs dp{};
        try {
            run_sim_join_dev(dX.p, nt, dX.p, nt, D, tau, o, &dp, nullptr);
            if (features)
                PDB_CUDA(cudaMemcpyAsync(features, dX.p, static_cast<size_t>(nt) * D * sizeof(float),
                                         cudaMemcpyDeviceToHost, s));
            pairs_to_host(dp, out, s);
        } catch (...) {
            dev_pairs_release(&dp, s);
            throw;
        }
        dev_pairs_release(&dp, s);
    });
}

static void check_dedup_args(const void* X, int64_t n, int32_t d, double tau,
                             const pdb_join_opts* o) {
    // run_dedup order: tau (src/query.cpp:536), then the dimension check.
    // As there, only tau < 0.0 is rejected: with a NaN tau nothing is within
    // tau and every item is its own representative.
    if (tau < 0.0) fail(PDB_ERR_CONFIG, "dedup needs tau >= 0");
    if (n < 0) fail(PDB_ERR_INVALID_ARGUMENT, "negative row count");
    if (n > INT32_MAX) fail(PDB_ERR_INVALID_ARGUMENT, "row counts above 2^31-1 are not supported");
    if (n > 0 && d < 1) fail(PDB_ERR_SHAPE, "dedup needs non-empty patch data");
    if (n > 0 && !X) fail(PDB_ERR_INVALID_ARGUMENT, "null rows");
    if (o && o->shard_count > 1) fail(PDB_ERR_INVALID_ARGUMENT, "dedup does not shard");
}

PDB_API int pdb_dedup_dev(const float* d_X, int64_t n, int32_t d, double tau,
                          const pdb_join_opts* opts, int64_t* d_rep_of, int64_t* n_reps) {
    return guarded([&] {
        if (!n_reps || (n > 0 && !d_rep_of)) fail(PDB_ERR_INVALID_ARGUMENT, "null output");
        check_dedup_args(d_X, n, d, tau, opts);
        device_ctx();
        run_dedup_dev(d_X, n, d, tau, stream_of(opts ? opts->stream : nullptr), d_rep_of, n_reps);
    });
}

PDB_API int pdb_dedup(const float* X, int64_t n, int32_t d, double tau, const pdb_join_opts* opts,
                      int64_t* rep_of, int64_t* n_reps) {
    return guarded([&] {
        if (!n_reps || (n > 0 && !rep_of)) fail(PDB_ERR_INVALID_ARGUMENT, "null output");
        check_dedup_args(X, n, d, tau, opts);
        device_ctx();
        cudaStream_t s = cudaStreamPerThread;
        DevBuf<float> dX(static_cast<size_t>(n) * std::max(d, 1), s);
        DevBuf<int64_t> dR(static_cast<size_t>(std::max<int64_t>(n, 1)), s);
        if (n > 0)
            PDB_CUDA(cudaMemcpyAsync(dX.p, X, static_cast<size_t>(n) * d * sizeof(float),
                                     cudaMemcpyHostToDevice, s));
        run_dedup_dev(dX.p, n, d, tau, s, dR.p, n_reps);
        if (n > 0)
            PDB_CUDA(cudaMemcpyAsync(rep_of, dR.p, static_cast<size_t>(n) * sizeof(int64_t),
                                     cudaMemcpyDeviceToHost, s));
        PDB_CUDA(cudaStreamSynchronize(s));
    });
}

PDB_API int pdb_rows_within(const float* A, const float* B, int64_t n, int32_t d, double radius,
                            uint8_t* out) {
    return guarded([&] {
        if (n < 0 || d < 0) fail(PDB_ERR_INVALID_ARGUMENT, "negative size");
        if (n > 0 && (!A || !B || !out)) fail(PDB_ERR_INVALID_ARGUMENT, "null rows");
        if (n == 0) return;
        device_ctx();
        cudaStream_t s = cudaStreamPerThread;
        const size_t bytes = static_cast<size_t>(n) * d * sizeof(float);
        DevBuf<float> dA(std::max<size_t>(bytes / sizeof(float), 1), s),
            dB(std::max<size_t>(bytes / sizeof(float), 1), s);
        DevBuf<uint8_t> dO(static_cast<size_t>(n), s);
        if (bytes) {
            PDB_CUDA(cudaMemcpyAsync(dA.p, A, bytes, cudaMemcpyHostToDevice, s));
            PDB_CUDA(cudaMemcpyAsync(dB.p, B, bytes, cudaMemcpyHostToDevice, s));
        }
        run_rows_within(dA.p, dB.p, n, d, radius, dO.p, s);
        PDB_CUDA(cudaMemcpyAsync(out, dO.p, static_cast<size_t>(n), cudaMemcpyDeviceToHost, s));
        PDB_CUDA(cudaStreamSynchronize(s));
    });
}

PDB_API int pdb_warmup(void) {
    // One tiny featurization and one tiny self-join through the real
    // launchers: creates the context and the pool and loads the modules of
    // the common paths, so a process's first real call does not pay them
    // (~1.5 s on a fresh B200 process, mostly driver and context start-up).
    return guarded([&] {
        device_ctx();
        cudaStream_t s = cudaStreamPerThread;
        DevBuf<uint8_t> fr(static_cast<size_t>(60) * 80 * 3, s);
        DevBuf<float> hist(64, s);
        PDB_CUDA(cudaMemsetAsync(fr.p, 0, static_cast<size_t>(60) * 80 * 3, s));
        launch_featurize_tiles(fr.p, 1, 60, 80, 60, 80, 4, PDB_HIST_JOINT, hist.p, s);
        DevBuf<float> X(static_cast<size_t>(256) * 64, s);
        PDB_CUDA(cudaMemsetAsync(X.p, 0, static_cast<size_t>(256) * 64 * sizeof(float), s));
        pdb_join_opts o{};
        o.flags = PDB_JOIN_SELF | PDB_JOIN_SORTED;
        o.stream = s;
        pdb_dev_pairs dp{};
        try {
            run_sim_join_dev(X.p, 256, X.p, 256, 64, 0.05, o, &dp, nullptr);
        } catch (...) {
            dev_pairs_release(&dp, s);
            throw;
        }
        dev_pairs_release(&dp, s);
        PDB_CUDA(cudaStreamSynchronize(s));
    });
}

PDB_API int pdb_release_caches(void) {
    return guarded([&] {
        device_ctx();
        release_join_caches();
        PDB_CUDA(cudaDeviceSynchronize());
        PDB_CUDA(cudaMemPoolTrimTo(device_ctx().pool, 0));
    });
}

PDB_API void* pdb_host_alloc(int64_t bytes) {
    void* p = nullptr;
    if (cudaHostAlloc(&p, static_cast<size_t>(std::max<int64_t>(bytes, 1)), cudaHostAllocDefault) !=
        cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return p;
}

PDB_API void pdb_host_free(void* p) {
    if (p) cudaFreeHost(p);
}
