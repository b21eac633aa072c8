// Bulk-copy (TMA 1-D) streaming probe (measurement tool, not product): one
// producer thread per CTA fills an S-stage shared-memory ring with
// cp.async.bulk copies of `stage` bytes from a 921.6 MB buffer; C consumer
// warps wait on each stage and release it.  Prints GB/s per (stage, S,
// CTAs/SM) to find how many bytes in flight K1's structure needs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../paper_1812_07607_b200/csrc -o tma_stream tma_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "tc_ptx.cuh"

using namespace pdb;

// run > 1: a CTA takes `run` consecutive chunks before striding by the grid
// (K1's order: a tile row of 10 bands per CTA)
__device__ __forceinline__ int64_t chunk_of(int64_t j, int run) {
    return run <= 1 ? j : (j / run) * run;  // (placeholder, replaced below)
}

__global__ void k_stream(const uint8_t* src, int64_t n_stages_total, uint32_t stage, int S, int C,
                         int run, int work) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + static_cast<size_t>(S) * stage);
    uint64_t* empty = full + S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], C);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();
    if (warp == C) {
        if (lane == 0) {
            uint32_t it = 0;
            for (int64_t k = blockIdx.x; k < n_stages_total; k += gridDim.x, it++) {
                const uint32_t s = it % S;
                if (it >= static_cast<uint32_t>(S)) ptx::mbar_wait_sleep(&empty[s], ((it / S) - 1) & 1);
                // the k-th chunk of this CTA's sequence under order `run`
                int64_t c = k;
                if (run > 1) {
                    const int64_t j = it;  // j-th chunk of this CTA
                    c = ((j / run) * gridDim.x + blockIdx.x) * run + (j % run);
                    if (c >= n_stages_total) c = k;
                }
                ptx::mbar_arrive_expect_tx(&full[s], stage);
                ptx::bulk_load(sm + s * stage, src + c * stage, stage, &full[s]);
            }
        }
        return;
    }
    uint32_t s = 0, ph = 0;
    uint32_t acc = 0;
    for (int64_t k = blockIdx.x; k < n_stages_total; k += gridDim.x) {
        ptx::mbar_wait_sleep(&full[s], ph);
        if (work) {
            // K1's consumer reads: 48 B per lane at (row, segment) of the
            // warp's tile column, plus the per-pixel offset arithmetic
            if (lane < 30) {
                const uint4* g = reinterpret_cast<const uint4*>(sm + s * stage + warp * 1440 + lane * 48);
                const uint4 a = g[0], b = g[1], c = g[2];
                uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
                for (int k = 0; k < 12; k++) acc ^= __umulhi(w[k] & 0xC0C0C0C0u, 0x04110000u) & 0x783u;
            }
        } else {
            acc ^= reinterpret_cast<const uint32_t*>(sm + s * stage)[threadIdx.x];
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&empty[s]);
        if (++s == static_cast<uint32_t>(S)) {
            s = 0;
            ph ^= 1;
        }
    }
    if (acc == 0x12345u) reinterpret_cast<uint32_t*>(sm)[0] = acc;
}

int main() {
    const size_t bytes = 921600000ull;
    uint8_t* d;
    char* fl;
    cudaMalloc(&d, bytes);
    cudaMalloc(&fl, 256 << 20);
    cudaMemset(d, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const uint32_t stages[] = {11520};
    for (int work : {0, 1})
    for (int run : {10})
    for (uint32_t st : stages)
        for (int per : {4})
            for (int S : {2, 3}) {
                size_t smem = static_cast<size_t>(S) * st + 2 * S * 8;
                if (smem * per > 227 * 1024) continue;
                const int C = 8;
                const int64_t n = bytes / st;
                float best = 1e9;
                for (int k = 0; k < 5; k++) {
                    cudaMemset(fl, k, 256 << 20);
                    cudaEventRecord(a);
                    k_stream<<<sms * per, (C + 1) * 32, smem>>>(d, n, st, S, C, run, work);
                    cudaEventRecord(b);
                    cudaEventSynchronize(b);
                    float ms;
                    cudaEventElapsedTime(&ms, a, b);
                    if (k >= 1 && ms < best) best = ms;
                }
                cudaError_t e = cudaGetLastError();
                printf("work=%d run=%2d stage=%6u S=%2d ctas/sm=%d inflight/sm=%4zu KB: %7.1f us %6.0f GB/s %s\n", work, run, st, S, per,
                       static_cast<size_t>(S) * st * per / 1024, best * 1e3,
                       static_cast<double>(n) * st / (best * 1e-3) / 1e9, e ? cudaGetErrorString(e) : "");
            }
    return 0;
}
