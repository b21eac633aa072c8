// rows.cu -- the `within` predicate over row pairs.
//
// Reference: eval_view's within case (src/query.cpp:142-151) evaluates
// euclidean(a, b) <= radius (src/index.cpp:69-76) for the two patches of one
// tuple.  When both slots come from the same input (select over a joined
// tuple, or an nl_join predicate over two left / two right slots) the plan
// layer batches every tuple's pair into one launch: out[k] = dist(A[k], B[k])
// <= radius with the reference's sequential fp64 chain (exact.cuh).
#include <algorithm>
#include <cstdint>

#include "exact.cuh"
#include "pdb_internal.cuh"

namespace pdb {

namespace {

__global__ void k_rows_within(const float* __restrict__ A, const float* __restrict__ B, int64_t n,
                              int d, double radius, uint8_t* __restrict__ out) {
    const bool vec8 = (d % 8 == 0) && (reinterpret_cast<uintptr_t>(A) % 32 == 0) &&
                      (reinterpret_cast<uintptr_t>(B) % 32 == 0);
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[k] = exact_dist(A + k * d, B + k * d, d, vec8) <= radius ? 1 : 0;
}

}  // namespace

void run_rows_within(const float* d_A, const float* d_B, int64_t n, int32_t d, double radius,
                     uint8_t* d_out, cudaStream_t s) {
    if (n == 0) return;
    const DeviceCtx& ctx = device_ctx();
    const int64_t blocks = std::min<int64_t>((n + 255) / 256, int64_t{ctx.sm_count} * 8);
    k_rows_within<<<static_cast<unsigned>(blocks), 256, 0, s>>>(d_A, d_B, n, d, radius, d_out);
    PDB_CUDA(cudaGetLastError());
}

}  // namespace pdb
