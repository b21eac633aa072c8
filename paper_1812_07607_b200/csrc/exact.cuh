// exact.cuh -- the reference's distance arithmetic on the device, shared by
// the join's exact re-check (K3) and the dedup attach step.
//
// euclidean(a, b) = sqrt(sum_k ((double)a_k - (double)b_k)^2), accumulated in
// k order with no contraction (src/index.cpp:69-76): explicit _rn intrinsics
// keep every operation a separate IEEE round-to-nearest step.
#pragma once

#include <cstdint>

namespace pdb {

// The reference chain, reading each row 32 bytes per load (sm_100's
// 256-bit LDG): a lane's load touches one 128-byte line, so the L1 data
// pipe -- which bounds this kernel, the rows of different lanes being
// unrelated -- spends one wavefront per 32 bytes instead of per 16.
__device__ __forceinline__ void ldg256(const float* p, float (&r)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]),
                   "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}

__device__ __forceinline__ double exact_dist(const float* __restrict__ a,
                                             const float* __restrict__ b, int d, bool vec8) {
    double acc = 0.0;
    auto step = [&](float x, float y) {
        const double t = __dsub_rn(static_cast<double>(x), static_cast<double>(y));
        acc = __dadd_rn(acc, __dmul_rn(t, t));
    };
    if (vec8) {
        // the next group's loads are issued before this group's chain: a
        // lane's candidate is a dependent sequence of d/8 gathers, and the
        // short joins (configs 1-3) are bound by their latency
        float x[8], y[8];
        ldg256(a, x);
        ldg256(b, y);
        for (int k = 0; k < d; k += 8) {
            float cx[8], cy[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                cx[q] = x[q];
                cy[q] = y[q];
            }
            if (k + 8 < d) {
                ldg256(a + k + 8, x);
                ldg256(b + k + 8, y);
            }
#pragma unroll
            for (int q = 0; q < 8; q++) step(cx[q], cy[q]);
        }
    } else {
        for (int k = 0; k < d; k++) step(__ldg(a + k), __ldg(b + k));
    }
    return __dsqrt_rn(acc);
}

// The same chain with b read from the grouped copy (k_group_copy): 8-column
// groups of consecutive rows, group stride gs floats.  Lanes whose
// candidates are neighbouring rows then share 128-byte lines, where the
// row-major gather costs one wavefront per lane per 32 bytes.
__device__ __forceinline__ double exact_dist_grouped(const float* __restrict__ a,
                                                     const float* __restrict__ bg, int64_t gs, int d,
                                                     bool vec8a) {
    double acc = 0.0;
    for (int k = 0; k < d; k += 8) {
        float x[8], y[8];
        if (vec8a) {
            ldg256(a + k, x);
        } else {
#pragma unroll
            for (int q = 0; q < 8; q++) x[q] = k + q < d ? __ldg(a + k + q) : 0.0f;
        }
        ldg256(bg + (k >> 3) * gs, y);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (k + q < d) {
                const double t = __dsub_rn(static_cast<double>(x[q]), static_cast<double>(y[q]));
                acc = __dadd_rn(acc, __dmul_rn(t, t));
            }
        }
    }
    return __dsqrt_rn(acc);
}

// Both rows from grouped copies (self-joins: the same copy, by row position).
__device__ __forceinline__ double exact_dist_grouped2(const float* __restrict__ ag,
                                                      const float* __restrict__ bg, int64_t gs,
                                                      int d) {
    double acc = 0.0;
    for (int k = 0; k < d; k += 8) {
        float x[8], y[8];
        ldg256(ag + (k >> 3) * gs, x);
        ldg256(bg + (k >> 3) * gs, y);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (k + q < d) {
                const double t = __dsub_rn(static_cast<double>(x[q]), static_cast<double>(y[q]));
                acc = __dadd_rn(acc, __dmul_rn(t, t));
            }
        }
    }
    return __dsqrt_rn(acc);
}

// fp32 pre-filter of the grouped re-check: s = sum_k fl(a_k - b_k)^2 with
// fp32 FMAs, on the same zero-padded 8-column groups (padding adds exact
// zeros).  It only rejects: every fp32 step errs by at most 2^-24
// relative (the subtraction's result is exact when subnormal, and
// underflow in the sum can only make s smaller), so
// s <= S (1 + 2^-24)^(d + 2) + d 2^-149 for the exact squared distance S,
// and a candidate with s above the host's threshold (k_recheck) cannot
// satisfy the reference's fp64 euclidean <= tau.  Overflow gives +inf
// (every term is non-negative), which is rejected only when the threshold
// is finite, i.e. when tau^2 is far below FLT_MAX.
__device__ __forceinline__ float filter_dist2(const float* __restrict__ a, int64_t as,
                                              const float* __restrict__ bg, int64_t gs, int d) {
    float s = 0.0f;
    for (int k = 0; k < d; k += 8) {
        float x[8], y[8];
        ldg256(a + (k >> 3) * as, x);
        ldg256(bg + (k >> 3) * gs, y);
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const float t = __fsub_rn(x[q], y[q]);
            s = __fmaf_rn(t, t, s);
        }
    }
    return s;
}

}  // namespace pdb
