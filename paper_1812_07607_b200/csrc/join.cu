// join.cu -- K2 (tensor-core screen) + K3 (exact fp64 re-check and
// compaction) of the threshold similarity join.
//
// Contract (proj/): emit (i, j) iff euclidean(L_i, R_j) <= tau, with
// euclidean the sequential, unfused fp64 chain of src/index.cpp:69-76 and
// the inclusive `<=` of src/index.cpp:833 / tests/oracles.hpp:77-85.  The
// reference reaches that set through a ball tree (src/query.cpp:485-528,
// src/index.cpp:811-842); here it is reached by a dense screen plus an exact
// re-check, and the two agree pair for pair.
//
// Pipeline per call:
//   k_col_mean   centre mu: column mean of the first 256 rows of L
//   k_prep       x~ = tf32_rna(x - mu) per row (padded to DP columns),
//                ||x~||^2 (fp64 -> f32), ||x~|| (rounded up), row class
//   k_tile_stats per 256-row tile of R: max ||y~||, max ||y~||^2;
//                g_j = ||y~_j||^2 / 2 padded with +inf
//   k_screen     tcgen05 kind::tf32 GEMM, 128x256 tiles, TMA-staged
//                128B-swizzled operands, fp32 accumulators double-buffered
//                in TMEM; epilogue warps test dot - g_j >= h_i(tile) and
//                append candidate (i, j) with warp-aggregated atomics
//   k_recheck    exact fp64 euclidean of every candidate on the ORIGINAL
//                fp32 rows, warp-ballot compaction of the survivors into
//                (left, right, dist)
//
// Why the screen never drops a true pair (the margin band):
//   x~, y~ are the rounded, centred vectors the MMA sees; centring does not
//   change distances and |x~ - x| <= U ||x~|| per row with
//   U = 2^-11 + 2^-20 (fp32 subtraction + round-to-nearest tf32), so
//   ||x~ - y~|| <= ||x - y|| + U (||x~|| + ||y~||).  The norms are computed
//   from x~ itself, so S = ||x~||^2 + ||y~||^2 - 2 x~.y~ is a near-exact
//   squared distance of two perturbed points: tf32 x tf32 products are exact
//   in fp32 and the accumulation of DP terms errs by at most
//   DP * 2^-23 * sum|x~_k y~_k| <= DP * 2^-23 (||x~||^2 + ||y~||^2) / 2
//   (truncating adds), plus the few fp32 epilogue roundings (2^-19 slack).
//   A true pair (fp64 distance <= tau, so exact distance <= tau (1 + 1e-9))
//   therefore has
//     S <= T = (tau' + U (||x~_i|| + max_J ||y~||))^2
//              + (DP 2^-23 + 2^-19) (||x~_i||^2 + max_J ||y~||^2)
//   and the epilogue keeps every (i, j) with dot - ||y~_j||^2/2 >=
//   (||x~_i||^2 - T)/2, rounded conservatively.  Everything kept is then
//   decided by the exact fp64 chain, so the output is the reference's set.
//   Rows with non-finite values never match (NaN/inf compare false in the
//   reference) and are excluded; rows too large for fp32 squares are
//   zeroed in the screen copy and forced to candidate status.

#include <cub/cub.cuh>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <type_traits>
#include <vector>

#include "exact.cuh"
#include "pdb_internal.cuh"
#include "tc_ptx.cuh"

namespace pdb {

namespace {

constexpr int BM = 128;  // L rows per tile (TMEM lanes)
constexpr int BN = 256;  // R rows per tile (UMMA N)
constexpr int BK = 32;   // fp32 per 128-byte swizzle row (64 for bf16)
constexpr int kABytes = BM * BK * 4;  // 16 KB per K-block of A
constexpr int kBBytes = BN * BK * 4;  // 32 KB per K-block of B
constexpr int kGCols = 16;            // folded-g row: 3 bf16 parts + zeros (one K=16 step)
constexpr int kGBytes = BN * kGCols * 2;  // 8 KB per 256-row g block
#ifndef PDB_EPI_WARPS
#define PDB_EPI_WARPS 8
#endif
constexpr int kEpiWarps = PDB_EPI_WARPS;             // epilogue warps (multiple of 4)
constexpr int kColsPerWarp = BN / (kEpiWarps / 4);   // accumulator columns per epilogue warp
constexpr int kChunks = kColsPerWarp / 32;           // 32-column TMEM loads per warp per tile
constexpr int kThreads = 64 + 32 * kEpiWarps;        // warp 0 TMA, warp 1 MMA, then epilogue
constexpr uint32_t kTmemCols = 512;   // two 256-column fp32 accumulators
constexpr uint32_t kIdescTf32 = ptx::idesc_tf32(BM, BN);
constexpr uint32_t kIdescBf16 = ptx::idesc_bf16(BM, BN);
constexpr uint32_t kIdescF16 = ptx::idesc_f16(BM, BN);

constexpr float kFlagNonFinite = -1.0f;
constexpr float kFlagBig = -2.0f;
constexpr float kBigLimit = 1.152921504606846976e18f;  // 2^60

// fp16 screen copies (band plan, DP <= 128).  kind::f16 multiplies fp16 at
// the bf16 rate, and fp16 keeps 11 significant bits to bf16's 8: the copies'
// rounding errors -- the screen's margin (err_norm) -- shrink ~8x, and with
// them the candidate band around tau (config 5: see DESIGN.md).  fp16's
// range is covered by one power-of-two scale 2^s of the centred values,
// chosen from their maximum xmax over both relations (k_band_keys; values
// beyond 2^60 are the "big" rows, forced candidates in either format), so
// that xmax 2^s < 2^14.  Distances scale by 2^s exactly; k_band_write
// scales tau to match.  Values 2^24 below the maximum fall into fp16's
// subnormals (absolute error 2^-25 after scaling): when that floor is not
// far below tau the join keeps bf16 copies.  Every kernel that depends on
// the format derives it from the same (xmax, tau, d), so they agree.
// Returns the scale, or 0 for bf16.
__device__ __forceinline__ float fp16_scale(const unsigned* xmax, double tau, int d) {
    if (!xmax || !(tau > 0.0)) return 0.0f;
    const float xm = __uint_as_float(*xmax);
    if (!(xm > 0.0f)) return 1.0f;  // every centred value is zero
    int e = 0;
    frexpf(xm, &e);  // xm < 2^e
    if (e < -100 || e > 100) return 0.0f;
    if (!(sqrt(static_cast<double>(d)) * ldexp(1.0, e - 39) * 64.0 < tau)) return 0.0f;
    return ldexpf(1.0f, 14 - e);
}

// Screen modes: L2 distance on tf32 or bf16 copies, or cosine on bf16 rows.
constexpr int kModeL2Tf32 = 0;
constexpr int kModeL2Bf16 = 1;
constexpr int kModeCosBf16 = 2;
// L2 on bf16 copies with -||y_j||^2/2 folded into the accumulator by one
// extra K=16 MMA per tile (A: constant [1,1,1,0..] rows, B: the three bf16
// parts of -g_j), so the epilogue tests raw accumulators (DP <= 128 only).
constexpr int kModeL2Bf16Aug = 3;
constexpr int kModeL2Bf16Pair = 4;  // kModeL2Bf16Aug on CTA pairs (k_screen_pair)
// The screen's perturbation term.  r01 bounded a row's rounding error by
// U ||x~|| with a per-element relative bound U -- and used 2^-9 for bf16,
// half the true bound (bf16 keeps 8 significant bits, so round-to-nearest
// errs by up to 2^-8 of the rounded value): one-dimensional rows far from
// the centre, where the bound is reached, lost pairs
// (tests/test_join_gpu.py::test_bf16_rounding_bound).  Since r02 k_prep
// stores each row's actual rounding-error norm (err_norm, an upper bound
// computed from the exact per-coordinate errors) and the margin uses it
// directly (u = 1): exact for any data, and tighter than any per-element
// bound, since errors rarely all sit at half an ulp.

struct ScreenParams {
    int64_t nL, nR;
    int32_t self_join;
    int32_t shard_index, shard_count;
    int32_t ch;         // column tiles per work unit
    int32_t nt;         // column tiles of R
    int32_t n_chunks;
    int64_t n_units;
    int64_t unit_step;  // 1, or S > 1 to screen only every S-th unit (output-size estimate)
    const int64_t* chunk_off;  // [n_chunks + 1]
    const float* hnL;   // L2: ||x~_i||^2;  COS: the row threshold h_i itself
    const float* snL;   // L2: ||x~_i - (x_i - mu)|| bound (err_norm) or a flag;  COS: unused
    const float* gR;    // L2: ||y~_j||^2 / 2 (+inf / -inf flags);  COS: 1/||y_j|| rounded up
                        // (0 for zero / non-finite rows); padded to nt*256
    const float* tmaxS; // per R tile
    const float* tmaxN;
    const float* cmaxS; // per column chunk (max over its tiles)
    const float* cmaxN;
    double tau_p;       // tau (1 + 1e-9)
    double u;           // scale of the error norms (1: snL / tmaxS / cmaxS hold them directly)
    double gam;         // DP 2^-23 + 2^-19
    int4* rec;                  // (row i, first column j0, hit mask, 0)
    unsigned long long cap;     // record capacity
    unsigned long long* counter;  // records written
    unsigned long long* ncand;    // candidate pairs (popc of the masks)
    unsigned long long* tiles;
    unsigned long long* next_unit;  // dynamic work-unit counter (zeroed per launch)
    // banded plan (tile_list != nullptr): units are segments of dev_ch tiles
    // of each row slot's surviving column tiles; cmaxS / cmaxN are per slot
    const int32_t* tile_list;      // surviving column tiles, slot-major, ascending
    const int64_t* slot_list_off;  // [n_slots + 1]
    const int64_t* slot_unit_off;  // [n_slots + 1]
    const int64_t* dev_n_units;    // unit count (device)
    const int32_t* dev_ch;         // tiles per unit (device)
    const int4* unit_info;         // decoded units (rb, first, end, slot), one load per unit
    int32_t n_slots;
    const float* hrow;             // banded: each row's screen threshold h_i (k_band_write)
    // fp16 copies when fp16_scale(f16xmax, f16tau, f16d) > 0 (band plan only)
    const unsigned* f16xmax;
    double f16tau;
    int32_t f16d;
};

struct Unit {
    int32_t rb, j0, j1, chunk;
};

// Candidate-record slots an epilogue warp reserves per global atomic.
constexpr unsigned kResChunk = 256;

__device__ __forceinline__ int tile_at(const ScreenParams& p, int o) {
    return p.tile_list ? __ldg(p.tile_list + o) : o;
}

__device__ __forceinline__ Unit decode_unit(const ScreenParams& p, int64_t u) {
    if (p.unit_info) {
        const int4 q = __ldg(p.unit_info + u);
        Unit r;
        r.rb = q.x;
        r.j0 = q.y;
        r.j1 = q.z;
        r.chunk = q.w;
        return r;
    }
    if (p.tile_list) {
        // banded: slot_unit_off[lo] <= u < slot_unit_off[lo + 1]
        int lo = 0, hi = p.n_slots;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(p.slot_unit_off + mid) <= u) lo = mid;
            else hi = mid;
        }
        const int64_t seg = u - __ldg(p.slot_unit_off + lo);
        const int ch = __ldg(p.dev_ch);
        const int P = p.shard_count;
        const int pos = (lo & 1) ? P - 1 - p.shard_index : p.shard_index;
        Unit r;
        r.rb = lo * P + pos;
        const int64_t o0 = __ldg(p.slot_list_off + lo) + seg * ch;
        r.j0 = static_cast<int32_t>(o0);
        r.j1 = static_cast<int32_t>(min(o0 + ch, __ldg(p.slot_list_off + lo + 1)));
        r.chunk = lo;  // per-slot norm maxima
        return r;
    }
    int lo = 0, hi = p.n_chunks;  // chunk_off[lo] <= u < chunk_off[hi]
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(p.chunk_off + mid) <= u) lo = mid;
        else hi = mid;
    }
    const int64_t k = u - __ldg(p.chunk_off + lo);
    Unit r;
    // k-th row block of this shard: boustrophedon over rounds of
    // shard_count blocks, which balances triangular and skewed work.
    const int P = p.shard_count;
    const int pos = (k & 1) ? P - 1 - p.shard_index : p.shard_index;
    r.rb = static_cast<int32_t>(k * P + pos);
    r.chunk = lo;
    r.j0 = lo * p.ch;
    r.j1 = min(r.j0 + p.ch, p.nt);
    if (p.self_join) r.j0 = max(r.j0, r.rb >> 1);
    return r;
}

// ---------------------------------------------------------------------------
// K2: the tensor-core screen.  A_RES: the CTA's 128-row block of L stays
// resident in shared memory for a whole unit (DP <= 128); otherwise A is
// streamed with B through the stage ring.  MODE: kModeL2Bf16 / kModeL2Tf32
// screen the L2 test dot - ||y_j||^2/2 >= h_i on bf16 (kind::f16) or tf32
// (kind::tf32) copies; kModeCosBf16 the cosine test dot * (1/||y_j||) >= h_i
// on bf16 rows.  DP is in elements; every K-block is 128 bytes of each row.
// (On B200 the single-CTA SS MMA is bound by shared-memory operand reads,
// ~12 KB per 128x256x(32 B of K) step, so bf16 operands -- twice the K per
// byte -- run the same screen about twice as fast as tf32; the wider margin
// band costs only candidates, which the exact re-check discards.)
// Shared-memory plan of k_screen, shared by the kernel and its launcher.
// Resident A is double-buffered when it fits, so the next work unit's rows
// load while the current unit's tiles are still multiplying.
// Epilogue warps of the 1-SM screen: 16 for DP <= 64 (a tile's epilogue is
// as long as its MMAs there; config 1 screen 0.100 -> 0.088 ms, config 2
// 0.090 -> 0.088, config 5 167 -> 164 ms), 8 above (config 3: 16 was 6 %
// slower).
template <int DP>
struct Epi {
    static constexpr int W = DP <= 64 ? 16 : 8;
    static constexpr int kColsPerWarp = BN / (W / 4);
    static constexpr int kChunks = kColsPerWarp / 32;
    static constexpr int kThreads = 64 + 32 * W;
};

template <int DP, bool A_RES, int STAGES, int MODE>
struct ScreenSmem {
    static constexpr bool AUG = MODE == kModeL2Bf16Aug;
    static constexpr int KE = MODE != kModeL2Tf32 ? 64 : 32;
    static constexpr int NKB = DP / KE;
    // a stage holds one K-block of B (and of A when it streams); with the
    // folded g, the 8 KB g block rides in the same stage as the last K-block
    static constexpr int kStage = (A_RES ? kBBytes : (kABytes + kBBytes)) + (AUG ? kGBytes : 0);
    // one A slot: NKB 128B-swizzled K-blocks (+ the 32B-swizzled folded-g block)
    static constexpr int kASlot = A_RES ? (NKB * kABytes + (AUG ? BM * kGCols * 2 : 0) + 1023) / 1024 * 1024 : 0;
    static constexpr int kTail = 256 + Epi<DP>::W * Epi<DP>::kColsPerWarp * 4 + Epi<DP>::W * 32 * 16 + 128;
    static constexpr size_t bytes(int slots) {
        return 1024 + static_cast<size_t>(slots) * kASlot + static_cast<size_t>(STAGES) * kStage + kTail;
    }
    static constexpr int kASlots = (A_RES && bytes(2) <= 232448) ? 2 : 1;
    static constexpr size_t kBytes = bytes(kASlots);
};

template <int DP, bool A_RES, int STAGES, int MODE>
__global__ void __launch_bounds__(Epi<DP>::kThreads, 1)
k_screen(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
         const __grid_constant__ CUtensorMap tmG, const ScreenParams p) {
    constexpr bool COS = MODE == kModeCosBf16;
    constexpr bool AUG = MODE == kModeL2Bf16Aug;
    constexpr bool BF16 = MODE != kModeL2Tf32;
    static_assert(!AUG || A_RES, "the folded-g mode keeps A resident");
    constexpr int KE = BF16 ? 64 : 32;  // elements per 128-byte K-block
    constexpr int NKB = DP / KE;
    using SM = ScreenSmem<DP, A_RES, STAGES, MODE>;
    constexpr int kEpiWarpsL = Epi<DP>::W;
    constexpr int kColsPerWarpL = Epi<DP>::kColsPerWarp;
    constexpr int kChunksL = Epi<DP>::kChunks;
    // (the same slots per CTA: a warp's unused reserved tail is zeroed and skipped by K3)
    constexpr unsigned kResChunkL = kResChunk * 8 / kEpiWarpsL;
    constexpr int kStageBytes = SM::kStage;
    constexpr int kASlot = SM::kASlot;
    constexpr int kASlots = SM::kASlots;
    constexpr int kAResBytes = kASlots * kASlot;

    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = ptx::smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
    uint8_t* smA = smem;                       // resident A (A_RES)
    uint8_t* smS = smem + kAResBytes;          // stage ring
    uint64_t* bars = reinterpret_cast<uint64_t*>(smS + STAGES * kStageBytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* a_full = bars + 2 * STAGES;   // [2] (one per A slot)
    uint64_t* a_empty = a_full + 2;         // [2]
    uint64_t* t_full = a_full + 4;          // [2]
    uint64_t* t_empty = a_full + 6;         // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 8);
    float* g_smem = reinterpret_cast<float*>(a_full + 10);  // [epilogue warps][kColsPerWarpL]
    int4* r_smem = reinterpret_cast<int4*>(g_smem + kEpiWarpsL * kColsPerWarpL);  // [warps][32] records
    // dynamic scheduler: the producer claims work units with one global
    // atomic and hands them to the MMA and epilogue warps through a 4-slot ring
    uint64_t* u_full = reinterpret_cast<uint64_t*>(r_smem + kEpiWarpsL * 32);
    uint64_t* u_empty = u_full + 4;
    // the producer publishes decoded units {rb, first tile, end, chunk}; rb < 0 ends
    volatile int4* u_dec = reinterpret_cast<volatile int4*>(u_full + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; a++) {
            ptx::mbar_init(&a_full[a], 1);
            ptx::mbar_init(&a_empty[a], 1);
        }
        for (int a = 0; a < 2; a++) {
            ptx::mbar_init(&t_full[a], 1);
            ptx::mbar_init(&t_empty[a], kEpiWarpsL);
        }
        for (int k = 0; k < 4; k++) {
            ptx::mbar_init(&u_full[k], 1);
            ptx::mbar_init(&u_empty[k], 1 + kEpiWarpsL);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        if (AUG) ptx::tma_prefetch_desc(&tmG);
    }
    if (AUG) {
        // constant A block for the folded g: every row is [1, 1, 1, 0, ...]
        // (16 bf16), written in the 32B-swizzled K-major layout: logical
        // 16-byte chunk c of 32-byte row r sits at chunk c ^ ((r >> 2) & 1).
        for (int q = threadIdx.x; q < kASlots * BM * 2; q += blockDim.x) {
            const int slot = q / (BM * 2), qq = q % (BM * 2);
            const int r = qq >> 1, c = qq & 1;
            reinterpret_cast<uint4*>(smA + slot * kASlot + NKB * kABytes)[qq] =
                c == ((r >> 2) & 1) ? make_uint4(0x3F803F80u, 0x00003F80u, 0u, 0u)
                                    : make_uint4(0u, 0u, 0u, 0u);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_trigger();
    ptx::pdl_wait();  // the prep kernels' outputs (copies, norms, unit plan)
    // consumer side of the unit ring (MMA warp: lane 0 only; epilogue: whole warp)
    int u_slot = 0;
    uint32_t u_phase = 0;
    auto take_unit = [&](bool whole_warp) -> Unit {
        ptx::mbar_wait(&u_full[u_slot], u_phase);
        const int4 q = const_cast<const int4&>(u_dec[u_slot]);
        if (whole_warp) __syncwarp();
        if (!whole_warp || lane == 0) ptx::mbar_arrive(&u_empty[u_slot]);
        if (++u_slot == 4) {
            u_slot = 0;
            u_phase ^= 1;
        }
        Unit w;
        w.rb = q.x;
        w.j0 = q.y;
        w.j1 = q.z;
        w.chunk = q.w;
        return w;
    };

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int ps = 0;
            uint32_t pph = 0;
            uint32_t na = 0;  // units whose A has been loaded
            const int64_t n_units = p.dev_n_units ? *p.dev_n_units : p.n_units;
            auto claim = [&]() -> int64_t {
                const int64_t c = static_cast<int64_t>(atomicAdd(p.next_unit, 1ull)) * p.unit_step;
                return c < n_units ? c : -1;
            };
            auto decode = [&](int64_t u) -> Unit {
                if (u >= 0) return decode_unit(p, u);
                Unit e;
                e.rb = -1;
                e.j0 = e.j1 = e.chunk = 0;
                return e;
            };
            Unit w = decode(claim());
            for (;;) {
                ptx::mbar_wait(&u_empty[ps], pph ^ 1);
                const_cast<int4&>(u_dec[ps]) = make_int4(w.rb, w.j0, w.j1, w.chunk);
                ptx::mbar_arrive(&u_full[ps]);
                if (++ps == 4) {
                    ps = 0;
                    pph ^= 1;
                }
                if (w.rb < 0) break;
                // claim and decode the next unit now: the round trips overlap
                // this unit's loads instead of stalling between units
                const Unit w_next = decode(claim());
                if (A_RES) {
                    const uint32_t slot = na % kASlots, use = na / kASlots;
                    ptx::mbar_wait(&a_empty[slot], (use & 1) ^ 1);
                    ptx::mbar_arrive_expect_tx(&a_full[slot], NKB * kABytes);
                    for (int kb = 0; kb < NKB; kb++)
                        ptx::tma_load_2d(smA + slot * kASlot + kb * kABytes, &tmA, &a_full[slot],
                                         kb * KE, w.rb * BM);
                    na++;
                }
                // banded: the next tile's index loads while this one is issued
                int J_next = w.j0 < w.j1 ? tile_at(p, w.j0) : 0;
                for (int o = w.j0; o < w.j1; o++) {
                    const int J = J_next;
                    if (o + 1 < w.j1) J_next = tile_at(p, o + 1);
                    PDB_DCHECK(J >= 0 && J < p.nt && stage < STAGES);
                    for (int kb = 0; kb < NKB; kb++) {
                        const bool with_g = AUG && kb == NKB - 1;
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* st = smS + stage * kStageBytes;
                        ptx::mbar_arrive_expect_tx(
                            &full[stage], (A_RES ? kBBytes : kABytes + kBBytes) + (with_g ? kGBytes : 0));
                        if (!A_RES) {
                            ptx::tma_load_2d(st, &tmA, &full[stage], kb * KE, w.rb * BM);
                            st += kABytes;
                        }
                        ptx::tma_load_2d(st, &tmB, &full[stage], kb * KE, J * BN);
                        if (with_g) ptx::tma_load_2d(st + kBBytes, &tmG, &full[stage], 0, J * BN);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
                w = w_next;
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (one thread) =====================
        if (lane == 0) {
            const uint32_t idesc_data =
                fp16_scale(p.f16xmax, p.f16tau, p.f16d) > 0.0f ? kIdescF16 : kIdescBf16;
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            uint32_t na = 0;  // units consumed
            unsigned long long ntiles = 0;
            for (;;) {
                const Unit w = take_unit(false);
                if (w.rb < 0) break;
                PDB_DCHECK(static_cast<int64_t>(w.rb) * BM < p.nL && w.j0 <= w.j1);
                const uint32_t slot = na % kASlots;
                uint8_t* smAu = smA + slot * kASlot;
                if (A_RES) {
                    ptx::mbar_wait(&a_full[slot], (na / kASlots) & 1);
                    ptx::tc_fence_after();
                }
                for (int J = w.j0; J < w.j1; J++) {
                    ptx::mbar_wait(&t_empty[acc], acc_phase ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                    for (int kb = 0; kb < NKB; kb++) {
                        ptx::mbar_wait(&full[stage], phase);
                        ptx::tc_fence_after();
                        const uint8_t* st = smS + stage * kStageBytes;
                        const uint32_t a_addr =
                            ptx::smem_u32(A_RES ? smAu + kb * kABytes : st);
                        const uint32_t b_addr = ptx::smem_u32(A_RES ? st : st + kABytes);
#pragma unroll
                        for (int kk = 0; kk < 4; kk++) {  // 4 x 32 bytes of K per block
                            if (BF16)
                                ptx::mma_f16(d_tmem, ptx::sdesc_k_sw128(a_addr + kk * 32),
                                             ptx::sdesc_k_sw128(b_addr + kk * 32), idesc_data,
                                             (kb | kk) != 0);
                            else
                                ptx::mma_tf32(d_tmem, ptx::sdesc_k_sw128(a_addr + kk * 32),
                                              ptx::sdesc_k_sw128(b_addr + kk * 32), kIdescTf32,
                                              (kb | kk) != 0);
                        }
                        if (AUG && kb == NKB - 1) {
                            // the folded-g block: one K=16 step on 32-byte rows
                            ptx::mma_f16(d_tmem, ptx::sdesc_k_sw32(ptx::smem_u32(smAu + NKB * kABytes)),
                                         ptx::sdesc_k_sw32(b_addr + kBBytes), kIdescBf16, 1u);
                        }
                        ptx::mma_commit(&empty[stage]);
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    ptx::mma_commit(&t_full[acc]);
                    ntiles++;
                    if (++acc == 2) {
                        acc = 0;
                        acc_phase ^= 1;
                    }
                }
                if (A_RES) ptx::mma_commit(&a_empty[slot]);
                na++;
            }
            atomicAdd(p.tiles, ntiles);
        }
    } else {
        // ===================== epilogue (warps 2-9) =====================
        // Two warps per TMEM lane quarter, each owning 128 of the 256
        // accumulator columns.  Per tile a warp stages its 128 g_j values in
        // shared memory (prefetched from global one tile ahead) and streams
        // the accumulator out of TMEM 32 columns at a time, double-buffered
        // so the next tcgen05.ld overlaps the current chunk's arithmetic.
        const int ew = warp - 2;
        const int q = warp & 3;  // TMEM lane quarter this warp may access
        const int half = ew >> 2;  // which kColsPerWarpL-wide column slice
        const int row = q * 32 + lane;
        const uint32_t t_lane = static_cast<uint32_t>(q * 32) << 16;
        float* gs = g_smem + ew * kColsPerWarpL;
        int4* rbuf = r_smem + ew * 32;
        uint32_t nbuf = 0;                 // staged records (warp-uniform)
        unsigned long long ncand = 0;      // this lane's candidate pairs
        // write the staged records out: one atomic per flush, coalesced 16 B stores
        // Records go to slots this warp reserves kResChunk at a time (one
        // global atomic per chunk instead of per flush of <= 32; unused
        // reserved slots are zeroed at the end -- the re-check skips a zero
        // mask).
        unsigned long long res_pos = 0, res_end = 0;
        // reservations grow 32, 64, ... up to the full chunk: a sparse
        // output leaves short zeroed tails for the re-check to skip
        unsigned res_chunk = 32;
        auto flush = [&]() {
            __syncwarp();
            const unsigned nb = nbuf;
            const unsigned long long room = res_end - res_pos;
            const unsigned first = room < nb ? static_cast<unsigned>(room) : nb;
            if (static_cast<unsigned>(lane) < first && res_pos + lane < p.cap)
                __stcs(p.rec + res_pos + lane, rbuf[lane]);  // (read once, by K3: no L2 residency)
            res_pos += first;
            if (first < nb) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(p.counter, static_cast<unsigned long long>(res_chunk));
                base = __shfl_sync(0xffffffffu, base, 0);
                res_pos = base;
                res_end = base + res_chunk;
                res_chunk = min(2 * res_chunk, kResChunkL);
                if (static_cast<unsigned>(lane) >= first && static_cast<unsigned>(lane) < nb &&
                    res_pos + (lane - first) < p.cap)
                    __stcs(p.rec + res_pos + (lane - first), rbuf[lane]);
                res_pos += nb - first;
            }
            __syncwarp();
            nbuf = 0;
        };
        auto zero_reserved = [&]() {
            for (unsigned long long q = res_pos + lane; q < res_end; q += 32)
                if (q < p.cap) p.rec[q] = make_int4(0, 0, 0, 0);
        };
        int acc = 0;
        uint32_t acc_phase = 0;
        for (;;) {
            const Unit w = take_unit(true);
            if (w.rb < 0) break;
            const int64_t i = static_cast<int64_t>(w.rb) * BM + row;
            const bool row_ok = i < p.nL;
            const float hn = (row_ok && !p.hrow) ? __ldg(p.hnL + i) : 0.0f;
            const float sn = (row_ok && !p.hrow) ? __ldg(p.snL + i) : kFlagNonFinite;
            using GV = typename std::conditional<kColsPerWarpL == 128, float4, float2>::type;
            GV gnext{};
            if (!AUG)
                gnext = __ldg(reinterpret_cast<const GV*>(
                    p.gR + static_cast<int64_t>(tile_at(p, w.j0)) * BN + half * kColsPerWarpL) + lane);
            // Threshold h_i for the whole unit, from the largest R norms over
            // its tiles (conservative; fp64 once per unit, not per tile).
            float h;
            if (p.hrow) {
                h = row_ok ? __ldg(p.hrow + i) : __int_as_float(0x7f800000);  // precomputed per row
            } else if (COS) {
                h = row_ok ? hn : __int_as_float(0x7f800000);  // prep stored h_i itself
            } else if (sn == kFlagNonFinite) {
                h = __int_as_float(0x7f800000);  // +inf: never a candidate
            } else if (sn == kFlagBig) {
                h = -__int_as_float(0x7f800000);  // always a candidate
            } else {
                // per-chunk maxima (a superset of the unit's tiles), one load each
                const float ms = __ldg(p.cmaxS + w.chunk), mn = __ldg(p.cmaxN + w.chunk);
                const double r = p.tau_p + p.u * (static_cast<double>(sn) + ms) + 1e-30;
                const double T = r * r + p.gam * (static_cast<double>(hn) + mn);
                h = __double2float_rd((static_cast<double>(hn) - T) * 0.5);
            }
            int J_next = w.j0 < w.j1 ? tile_at(p, w.j0) : 0;
            for (int o = w.j0; o < w.j1; o++) {
                const int J = J_next;
                if (o + 1 < w.j1) J_next = tile_at(p, o + 1);
                __syncwarp();
                if (!AUG) reinterpret_cast<GV*>(gs)[lane] = gnext;
                // unconditional (clamped) prefetch: a predicated load would
                // force a wait at the register move (none needed when g is folded)
                if (!AUG)
                gnext = __ldg(reinterpret_cast<const GV*>(
                    p.gR + static_cast<int64_t>(tile_at(p, min(o + 1, w.j1 - 1))) * BN + half * kColsPerWarpL) + lane);
                __syncwarp();
                ptx::mbar_wait(&t_full[acc], acc_phase);
                ptx::tc_fence_after();
                const int64_t colw = static_cast<int64_t>(J) * BN + half * kColsPerWarpL;
                const uint32_t t_acc =
                    tmem_base + t_lane + static_cast<uint32_t>(acc * BN + half * kColsPerWarpL);

                auto process = [&](const uint32_t(&v)[32], int c) {
                    // e_k = dot_k - g_k (L2) or dot_k * g_k (cosine), two
                    // columns per packed f32x2 instruction (IEEE RN per lane)
                    float e[32];
                    const uint2* g2 = reinterpret_cast<const uint2*>(gs + c * 32);
                    if (AUG) {
#pragma unroll
                        for (int k = 0; k < 32; k++) e[k] = __uint_as_float(v[k]);
                    } else
#pragma unroll
                    for (int k2 = 0; k2 < 16; k2++) {
                        const uint2 gg = g2[k2];
                        const unsigned long long a =
                            (static_cast<unsigned long long>(v[2 * k2 + 1]) << 32) | v[2 * k2];
                        const unsigned long long b =
                            (static_cast<unsigned long long>(gg.y) << 32) | gg.x;
                        unsigned long long r;
                        if (COS)
                            asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
                        else
                            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
                        e[2 * k2] = __uint_as_float(static_cast<uint32_t>(r));
                        e[2 * k2 + 1] = __uint_as_float(static_cast<uint32_t>(r >> 32));
                    }
                    float m = -__int_as_float(0x7f800000);
#pragma unroll
                    for (int k = 0; k < 32; k++) m = fmaxf(m, e[k]);
                    const bool hit = row_ok && m >= h;
                    if (__any_sync(0xffffffffu, hit)) {
                        const int64_t col0 = colw + c * 32;
                        uint32_t mask = 0;
                        if (hit) {
#pragma unroll
                            for (int k = 0; k < 32; k++) mask |= static_cast<uint32_t>(e[k] >= h) << k;
                            // columns past R's end, and j <= i in a self-join
                            if (col0 + 32 > p.nR)
                                mask &= p.nR > col0 ? (0xffffffffu >> (32 - (p.nR - col0))) : 0u;
                            if (p.self_join) {
                                const int64_t lo = i + 1 - col0;  // first allowed k
                                mask &= lo <= 0 ? 0xffffffffu : (lo >= 32 ? 0u : (0xffffffffu << lo));
                            }
                        }
                        // one record (row, first column, 32-bit hit mask) per lane with
                        // hits, staged in shared memory and flushed 32 at a time
                        const uint32_t bal = __ballot_sync(0xffffffffu, mask != 0);
                        if (bal) {
                            const uint32_t nr = __popc(bal);
                            if (nbuf + nr > 32) flush();
                            ncand += __popc(mask);
                            if (mask)
                                rbuf[nbuf + __popc(bal & ((1u << lane) - 1u))] =
                                    make_int4(static_cast<int>(i), static_cast<int>(col0),
                                              static_cast<int>(mask), 0);
                            nbuf += nr;
                        }
                    }
                };

                // double-buffered TMEM reads: chunk c+1 is in flight while c is tested
                uint32_t vbuf[2][32];
                ptx::tmem_ld32(t_acc, vbuf[0]);
                ptx::tmem_ld_wait();
                ptx::reg_fence(vbuf[0]);
#pragma unroll
                for (int c = 0; c < kChunksL; c++) {
                    if (c + 1 < kChunksL) {
                        ptx::tmem_ld32(t_acc + (c + 1) * 32, vbuf[(c + 1) & 1]);
                    } else {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) ptx::mbar_arrive(&t_empty[acc]);  // TMEM reads done
                    }
                    process(vbuf[c & 1], c);
                    if (c + 1 < kChunksL) {
                        ptx::tmem_ld_wait();
                        ptx::reg_fence(vbuf[(c + 1) & 1]);
                    }
                }
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
        if (nbuf) flush();
        zero_reserved();
        unsigned long long nc = ncand;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nc += __shfl_xor_sync(0xffffffffu, nc, o);
        if (lane == 0 && nc) atomicAdd(p.ncand, nc);
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, kTmemCols);
    }
}

// ---------------------------------------------------------------------------
// K2 on CTA pairs (the default for the folded-g L2 screen, d <= 128, one
// GPU): a cluster of two CTAs on one TPC runs tcgen05.mma.cta_group::2 with
// M = 256 -- each CTA keeps its own 128-row block of L resident and loads
// half of every 256-row R tile (and half of its folded-g block), and the
// leader CTA issues the MMAs for both.  Per 128x256 tile an SM then reads
// 8 KB of MMA operands per K=16 step instead of 12 KB and receives 20 KB of
// TMA data instead of 40 KB: measured on the 1-SM screen, the SM moved a
// near-constant ~110 B/clk of shared memory (MMA operand reads + TMA
// writes) whatever d and the fold did, i.e. it was shared-memory bound at
// 70 % of the MMA floor.
//
// Work units are (column chunk, row-block pair); the leader's producer
// claims them and publishes each to both CTAs (DSMEM store + remote
// arrive).  Barriers: full / a_full / t_empty / u_empty live in the leader
// (the peer's TMA completes on the leader's full barriers, the peer's
// epilogue and consumers arrive remotely); empty / a_empty / t_full / u_full
// in both (the leader's MMA commits multicast to the pair).
template <int DP>
struct PairSmem {
    static constexpr int NKB = DP / 64;
    static constexpr int kHalfB = (BN / 2) * 128;             // 16 KB: 128 R rows x 128 B
    static constexpr int kHalfG = (BN / 2) * kGCols * 2;      // 4 KB
    static constexpr int kStage = NKB * kHalfB + kHalfG;      // one tile's half of R (+g)
    static constexpr int kASlot = NKB * kABytes;
    static constexpr int kConst = BM * kGCols * 2;            // the fold's constant A block
    static constexpr int kTail = 512 + kEpiWarps * 32 * 16 + 128;
    static constexpr int STAGES = (232448 - 1024 - 2 * kASlot - kConst - kTail) / kStage > 8
                                      ? 8
                                      : (232448 - 1024 - 2 * kASlot - kConst - kTail) / kStage;
    static constexpr size_t kBytes =
        1024 + 2 * static_cast<size_t>(kASlot) + kConst + static_cast<size_t>(STAGES) * kStage + kTail;
};

struct PairUnit {
    int32_t q, j0, j1, chunk;  // row-block pair q (rows [256q, 256q+256)), columns [j0, j1)
};

__device__ __forceinline__ PairUnit decode_pair_unit(const ScreenParams& p, int64_t u) {
    int lo = 0, hi = p.n_chunks;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(p.chunk_off + mid) <= u) lo = mid;
        else hi = mid;
    }
    PairUnit r;
    r.q = static_cast<int32_t>(u - __ldg(p.chunk_off + lo));
    r.chunk = lo;
    r.j0 = lo * p.ch;
    r.j1 = min(r.j0 + p.ch, p.nt);
    if (p.self_join) r.j0 = max(r.j0, r.q);
    return r;
}

template <int DP>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
k_screen_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmG, const ScreenParams p) {
    using SM = PairSmem<DP>;
    constexpr int NKB = SM::NKB;
    constexpr int STAGES = SM::STAGES;
    constexpr int KE = 64;
    constexpr uint32_t kIdescPair = ptx::idesc_bf16(2 * BM, BN);

    extern __shared__ uint8_t smem_raw[];
    const uint32_t base_u32 = ptx::smem_u32(smem_raw);
    uint8_t* smem = smem_raw + ((1024 - (base_u32 & 1023)) & 1023);
    uint8_t* smA = smem;                                  // 2 resident A slots
    uint8_t* smC = smA + 2 * SM::kASlot;                  // constant fold block
    uint8_t* smS = smC + SM::kConst;                      // stage ring
    uint64_t* bars = reinterpret_cast<uint64_t*>(smS + STAGES * SM::kStage);
    uint64_t* full = bars;
    uint64_t* empty = bars + STAGES;
    uint64_t* a_full = bars + 2 * STAGES;  // [2]
    uint64_t* a_empty = a_full + 2;        // [2]
    uint64_t* t_full = a_full + 4;         // [2]
    uint64_t* t_empty = a_full + 6;        // [2]
    uint64_t* u_full = a_full + 8;         // [4]
    uint64_t* u_empty = a_full + 12;       // [4]
    volatile int64_t* u_val = reinterpret_cast<volatile int64_t*>(a_full + 16);  // [4]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 20);
    int4* r_smem = reinterpret_cast<int4*>(smem_raw + (smS - smem_raw) + STAGES * SM::kStage + 512);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    auto leader_addr = [&](const void* p_local) { return ptx::mapa(ptx::smem_u32(p_local), 0); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; s++) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; a++) {
            ptx::mbar_init(&a_full[a], 1);
            ptx::mbar_init(&a_empty[a], 1);
            ptx::mbar_init(&t_full[a], 1);
            ptx::mbar_init(&t_empty[a], 2 * kEpiWarps);
        }
        for (int k = 0; k < 4; k++) {
            ptx::mbar_init(&u_full[k], 1);
            ptx::mbar_init(&u_empty[k], 2 + 2 * kEpiWarps);
        }
        ptx::fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        ptx::tma_prefetch_desc(&tmA);
        ptx::tma_prefetch_desc(&tmB);
        ptx::tma_prefetch_desc(&tmG);
    }
    // constant A block for the folded g ([1, 1, 1, 0, ...], 32B-swizzled K-major)
    for (int qd = threadIdx.x; qd < BM * 2; qd += blockDim.x) {
        const int r = qd >> 1, c = qd & 1;
        reinterpret_cast<uint4*>(smC)[qd] = c == ((r >> 2) & 1)
                                                ? make_uint4(0x3F803F80u, 0x00003F80u, 0u, 0u)
                                                : make_uint4(0u, 0u, 0u, 0u);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 1) ptx::tmem_alloc_pair(tmem_slot, kTmemCols);
    ptx::tc_fence_before();
    ptx::cluster_sync();  // barrier inits and TMEM allocation visible to the pair
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::pdl_trigger();
    ptx::pdl_wait();

    // unit ring consumers: leader's MMA lane and epilogue warps, the peer's
    // producer lane and epilogue warps; each frees its slot on the leader
    int u_slot = 0;
    uint32_t u_phase = 0;
    auto take_unit = [&](bool whole_warp) -> int64_t {
        ptx::mbar_wait_acq_cluster(&u_full[u_slot], u_phase);
        const int64_t u = u_val[u_slot];
        if (whole_warp) __syncwarp();
        if (!whole_warp || lane == 0) {
            if (leader) ptx::mbar_arrive(&u_empty[u_slot]);
            else ptx::mbar_arrive_cluster(leader_addr(&u_empty[u_slot]));
        }
        if (++u_slot == 4) {
            u_slot = 0;
            u_phase ^= 1;
        }
        return u;
    };

    if (warp == 0) {
        // ===================== TMA producers (one per CTA) =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t na = 0;
            int ps = 0;
            uint32_t pph = 0;
            auto claim = [&]() -> int64_t {
                const int64_t c = static_cast<int64_t>(atomicAdd(p.next_unit, 1ull)) * p.unit_step;
                return c < p.n_units ? c : -1;
            };
            int64_t u = leader ? claim() : 0;
            for (;;) {
                if (leader) {
                    // publish u to both CTAs of the pair
                    ptx::mbar_wait_acq_cluster(&u_empty[ps], pph ^ 1);
                    u_val[ps] = u;
                    ptx::st_cluster_u64(ptx::mapa(ptx::smem_u32(const_cast<int64_t*>(&u_val[ps])), 1),
                                        static_cast<uint64_t>(u));
                    ptx::mbar_arrive(&u_full[ps]);
                    ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&u_full[ps]), 1));
                    if (++ps == 4) {
                        ps = 0;
                        pph ^= 1;
                    }
                } else {
                    u = take_unit(false);
                }
                if (u < 0) break;
                const int64_t u_next = leader ? claim() : 0;
                const PairUnit w = decode_pair_unit(p, u);
                const int32_t rb = 2 * w.q + static_cast<int32_t>(rank);
                {
                    const uint32_t slot = na & 1;
                    ptx::mbar_wait(&a_empty[slot], ((na >> 1) & 1) ^ 1);
                    if (leader) ptx::mbar_arrive_expect_tx(&a_full[slot], 2 * NKB * kABytes);
                    const uint32_t bar = leader_addr(&a_full[slot]);
                    for (int kb = 0; kb < NKB; kb++)
                        ptx::tma_load_2d_pair(smA + slot * SM::kASlot + kb * kABytes, &tmA, bar,
                                              kb * KE, rb * BM);
                    na++;
                }
                for (int J = w.j0; J < w.j1; J++) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* st = smS + stage * SM::kStage;
                    if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * SM::kStage);
                    const uint32_t bar = leader_addr(&full[stage]);
                    const int32_t r0 = J * BN + static_cast<int32_t>(rank) * (BN / 2);
                    for (int kb = 0; kb < NKB; kb++)
                        ptx::tma_load_2d_pair(st + kb * SM::kHalfB, &tmB, bar, kb * KE, r0);
                    ptx::tma_load_2d_pair(st + NKB * SM::kHalfB, &tmG, bar, 0, r0);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (leader) u = u_next;
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader, one thread) =====================
        if (leader && lane == 0) {
            const uint32_t idesc_data = fp16_scale(p.f16xmax, p.f16tau, p.f16d) > 0.0f
                                            ? ptx::idesc_f16(2 * BM, BN) : kIdescPair;
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0, na = 0;
            unsigned long long ntiles = 0;
            for (;;) {
                const int64_t u = take_unit(false);
                if (u < 0) break;
                const PairUnit w = decode_pair_unit(p, u);
                const uint32_t slot = na & 1;
                ptx::mbar_wait(&a_full[slot], (na >> 1) & 1);
                ptx::tc_fence_after();
                const uint8_t* sa = smA + slot * SM::kASlot;
                for (int J = w.j0; J < w.j1; J++) {
                    ptx::mbar_wait(&t_empty[acc], acc_phase ^ 1);
                    ptx::tc_fence_after();
                    const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint8_t* st = smS + stage * SM::kStage;
                    for (int kb = 0; kb < NKB; kb++) {
                        const uint32_t a_addr = ptx::smem_u32(sa + kb * kABytes);
                        const uint32_t b_addr = ptx::smem_u32(st + kb * SM::kHalfB);
#pragma unroll
                        for (int kk = 0; kk < 4; kk++)
                            ptx::mma_f16_pair(d_tmem, ptx::sdesc_k_sw128(a_addr + kk * 32),
                                              ptx::sdesc_k_sw128(b_addr + kk * 32), idesc_data,
                                              (kb | kk) != 0);
                    }
                    // the folded-g block: one K=16 step on 32-byte rows
                    ptx::mma_f16_pair(d_tmem, ptx::sdesc_k_sw32(ptx::smem_u32(smC)),
                                      ptx::sdesc_k_sw32(ptx::smem_u32(st + NKB * SM::kHalfB)),
                                      kIdescPair, 1u);
                    ptx::mma_commit_pair(&empty[stage], 0x3);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                    ptx::mma_commit_pair(&t_full[acc], 0x3);
                    ntiles += 2;
                    if (++acc == 2) {
                        acc = 0;
                        acc_phase ^= 1;
                    }
                }
                ptx::mma_commit_pair(&a_empty[slot], 0x3);
                na++;
            }
            atomicAdd(p.tiles, ntiles);
        }
    } else {
        // ===================== epilogue (warps 2-9 of each CTA) =====================
        const int ew = warp - 2;
        const int qd = warp & 3;
        const int half = ew >> 2;
        const int row = qd * 32 + lane;
        const uint32_t t_lane = static_cast<uint32_t>(qd * 32) << 16;
        int4* rbuf = r_smem + ew * 32;
        uint32_t nbuf = 0;
        unsigned long long ncand = 0;
        // Records go to slots this warp reserves kResChunk at a time (one
        // global atomic per chunk instead of per flush of <= 32; unused
        // reserved slots are zeroed at the end -- the re-check skips a zero
        // mask).
        unsigned long long res_pos = 0, res_end = 0;
        // reservations grow 32, 64, ... up to the full chunk: a sparse
        // output leaves short zeroed tails for the re-check to skip
        unsigned res_chunk = 32;
        auto flush = [&]() {
            __syncwarp();
            const unsigned nb = nbuf;
            const unsigned long long room = res_end - res_pos;
            const unsigned first = room < nb ? static_cast<unsigned>(room) : nb;
            if (static_cast<unsigned>(lane) < first && res_pos + lane < p.cap)
                __stcs(p.rec + res_pos + lane, rbuf[lane]);  // (read once, by K3: no L2 residency)
            res_pos += first;
            if (first < nb) {
                unsigned long long base = 0;
                if (lane == 0) base = atomicAdd(p.counter, static_cast<unsigned long long>(res_chunk));
                base = __shfl_sync(0xffffffffu, base, 0);
                res_pos = base;
                res_end = base + res_chunk;
                res_chunk = min(2 * res_chunk, kResChunk);
                if (static_cast<unsigned>(lane) >= first && static_cast<unsigned>(lane) < nb &&
                    res_pos + (lane - first) < p.cap)
                    __stcs(p.rec + res_pos + (lane - first), rbuf[lane]);
                res_pos += nb - first;
            }
            __syncwarp();
            nbuf = 0;
        };
        auto zero_reserved = [&]() {
            for (unsigned long long q = res_pos + lane; q < res_end; q += 32)
                if (q < p.cap) p.rec[q] = make_int4(0, 0, 0, 0);
        };
        const uint32_t t_empty_remote = leader ? 0u : leader_addr(&t_empty[0]);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (;;) {
            const int64_t u = take_unit(true);
            if (u < 0) break;
            const PairUnit w = decode_pair_unit(p, u);
            const int64_t i = (static_cast<int64_t>(2 * w.q) + rank) * BM + row;
            const bool row_ok = i < p.nL;
            const float hn = row_ok ? __ldg(p.hnL + i) : 0.0f;
            const float sn = row_ok ? __ldg(p.snL + i) : kFlagNonFinite;
            float h;
            if (sn == kFlagNonFinite) {
                h = __int_as_float(0x7f800000);
            } else if (sn == kFlagBig) {
                h = -__int_as_float(0x7f800000);
            } else {
                const float ms = __ldg(p.cmaxS + w.chunk), mn = __ldg(p.cmaxN + w.chunk);
                const double r = p.tau_p + p.u * (static_cast<double>(sn) + ms) + 1e-30;
                const double T = r * r + p.gam * (static_cast<double>(hn) + mn);
                h = __double2float_rd((static_cast<double>(hn) - T) * 0.5);
            }
            for (int J = w.j0; J < w.j1; J++) {
                ptx::mbar_wait(&t_full[acc], acc_phase);  // a tcgen05.commit arrival
                ptx::tc_fence_after();
                const int64_t colw = static_cast<int64_t>(J) * BN + half * kColsPerWarp;
                const uint32_t t_acc =
                    tmem_base + t_lane + static_cast<uint32_t>(acc * BN + half * kColsPerWarp);
                auto process = [&](const uint32_t(&v)[32], int c) {
                    float m = -__int_as_float(0x7f800000);
#pragma unroll
                    for (int k = 0; k < 32; k++) m = fmaxf(m, __uint_as_float(v[k]));
                    const bool hit = row_ok && m >= h;
                    if (__any_sync(0xffffffffu, hit)) {
                        const int64_t col0 = colw + c * 32;
                        uint32_t mask = 0;
                        if (hit) {
#pragma unroll
                            for (int k = 0; k < 32; k++)
                                mask |= static_cast<uint32_t>(__uint_as_float(v[k]) >= h) << k;
                            if (col0 + 32 > p.nR)
                                mask &= p.nR > col0 ? (0xffffffffu >> (32 - (p.nR - col0))) : 0u;
                            if (p.self_join) {
                                const int64_t lo = i + 1 - col0;
                                mask &= lo <= 0 ? 0xffffffffu : (lo >= 32 ? 0u : (0xffffffffu << lo));
                            }
                        }
                        const uint32_t bal = __ballot_sync(0xffffffffu, mask != 0);
                        if (bal) {
                            const uint32_t nr = __popc(bal);
                            if (nbuf + nr > 32) flush();
                            ncand += __popc(mask);
                            if (mask)
                                rbuf[nbuf + __popc(bal & ((1u << lane) - 1u))] =
                                    make_int4(static_cast<int>(i), static_cast<int>(col0),
                                              static_cast<int>(mask), 0);
                            nbuf += nr;
                        }
                    }
                };
                uint32_t vbuf[2][32];
                ptx::tmem_ld32(t_acc, vbuf[0]);
                ptx::tmem_ld_wait();
                ptx::reg_fence(vbuf[0]);
#pragma unroll
                for (int c = 0; c < kChunks; c++) {
                    if (c + 1 < kChunks) {
                        ptx::tmem_ld32(t_acc + (c + 1) * 32, vbuf[(c + 1) & 1]);
                    } else {
                        ptx::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) {  // this CTA's TMEM reads of the tile are done
                            if (leader) ptx::mbar_arrive(&t_empty[acc]);
                            else ptx::mbar_arrive_cluster_relaxed(t_empty_remote + acc * 8);
                        }
                    }
                    process(vbuf[c & 1], c);
                    if (c + 1 < kChunks) {
                        ptx::tmem_ld_wait();
                        ptx::reg_fence(vbuf[(c + 1) & 1]);
                    }
                }
                if (++acc == 2) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
        if (nbuf) flush();
        zero_reserved();
        unsigned long long nc = ncand;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nc += __shfl_xor_sync(0xffffffffu, nc, o);
        if (lane == 0 && nc) atomicAdd(p.ncand, nc);
    }

    ptx::tc_fence_before();
    ptx::cluster_sync();  // the peer's smem stays alive until the leader's MMAs are done
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_pair(tmem_base, kTmemCols);
    }
}

// ---------------------------------------------------------------------------
// Preparation kernels.
// The centre mu only has to be a fixed vector (distances are translation
// invariant and the margin is computed from the centred copies), so the mean
// of the first kMeanRows rows is plenty; finite values only.
constexpr int kMeanRows = 256;

// grid = ceil(DP/32) blocks of 32x32 threads: thread (x, y) sums rows
// y, y+32, ... of column 32*blockIdx.x + x; the 32 partial sums are then
// added in a fixed order, so mu is deterministic.
__global__ void __launch_bounds__(1024)
k_col_mean(const float* __restrict__ X, int64_t n, int d, int DP, float* __restrict__ mu,
           float* __restrict__ tmaxS, float* __restrict__ tmaxN, int nt, float* __restrict__ g,
           int64_t nR, const float* __restrict__ mu_src) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    if (tmaxS) {  // k_prep max-reduces the R tiles' statistics into these
        const int tid = (blockIdx.x * blockDim.y + threadIdx.y) * blockDim.x + threadIdx.x;
        const int nth = gridDim.x * blockDim.x * blockDim.y;
        for (int j = tid; j < nt; j += nth) {
            tmaxS[j] = 0.0f;
            tmaxN[j] = 0.0f;
        }
        for (int64_t j = nR + tid; j < static_cast<int64_t>(nt) * BN; j += nth)
            g[j] = __int_as_float(0x7f800000);  // padding columns never match
    }
    __shared__ double part[32][33];
    const int col = blockIdx.x * 32 + threadIdx.x;
    double s = 0.0;
    if (mu && col < d) {  // (blockDim.y 32, or 8 beside a running K1: same rows)
        for (int r = threadIdx.y; r < kMeanRows; r += blockDim.y) {
            if (r < n) {
                const float v = X[static_cast<int64_t>(r) * d + col];
                if (isfinite(v)) s += static_cast<double>(v);
            }
        }
    }
    part[threadIdx.y][threadIdx.x] = s;
    __syncthreads();
    if (!mu) return;  // the centre was computed ahead (run_featurize_join_dev)
    if (mu_src) {
        if (threadIdx.y == 0 && col < DP) mu[col] = mu_src[col];
        return;
    }
    if (threadIdx.y == 0 && col < DP) {
        double t = 0.0;
        for (int k = 0; k < static_cast<int>(blockDim.y); k++) t += part[k][threadIdx.x];
        const int64_t m = n < kMeanRows ? n : kMeanRows;
        const float v = (col < d && m > 0) ? static_cast<float>(t / static_cast<double>(m)) : 0.0f;
        mu[col] = isfinite(v) ? v : 0.0f;
    }
}

// One warp per row: centred copy rounded to the MMA input type (tf32 via
// cvt.rna, or bf16 round-to-nearest), zero-padded to DP columns, with the
// norms of that rounded copy and the row class.
__device__ __forceinline__ float round_tf32(float x) { return ptx::tf32_rna(x); }
__device__ __forceinline__ uint16_t to_bf16_bits(float x) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(x));
}

// Bound on the norm of a row's total rounding error e = x~ - (x - mu): the
// screen copy's rounding t - c (exact per coordinate; squares summed with
// fp32 FMAs -- non-negative terms, so the sum is at most (d + 2) 2^-23 low
// relative to the exact one, at most d + 1 roundings of 2^-24 each, summed
// per lane then exactly in fp64 across lanes), plus the fp32 centring
// c = fl(x - mu), |c - (x - mu)| <= 2^-24 |c| with ||c|| <= ||t|| + ||t - c||.
// Rounded up (fp64 roundings: 2^-40 slack).
// |  ||x~_i - y~_j|| - ||x_i - y_j||  | <= e_i + e_j, so this replaces the
// worst-case U ||x~|| per row in the screen's margin.
__device__ __forceinline__ float err_norm(double acc, double eacc, int d) {
    const double et = sqrt(eacc * (1.0 + (d + 2) * 1.1920928955078125e-07)), tn = sqrt(acc);
    return __double2float_ru((et + 5.9604644775390625e-08 * (tn + et)) * (1.0 + 9.094947017729282e-13));
}

// Sum over the 32 lanes of eight per-row partials v[0..7] with 9 shuffles
// (a transposing butterfly): afterwards lanes 4r .. 4r+3 hold row r's total.
__device__ __forceinline__ double sum8_transpose(const double (&v)[8], int lane) {
    double k4[4], k2[2];
    const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        const double send = b4 ? v[i] : v[i + 4];
        k4[i] = (b4 ? v[i + 4] : v[i]) + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int i = 0; i < 2; i++) {
        const double send = b3 ? k4[i] : k4[i + 2];
        k2[i] = (b3 ? k4[i + 2] : k4[i]) + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    const double send = b2 ? k2[0] : k2[1];
    double t = (b2 ? k2[1] : k2[0]) + __shfl_xor_sync(0xffffffffu, send, 4);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    return t;
}

// DP <= 128: a warp prepares kRowsPerWarp = 8 rows at once.  Lane owns the
// NV contiguous columns k = lane*NV + i of each row (one coalesced vector
// load and one vector store per lane and row).  The centred copy is rounded
// to the MMA input type; the per-row epilogue (norms / row class, the
// folded-g block) runs on lane 4r for row r after one transposing fp64
// reduction, so no lane serialises the eight rows.  perm: row r of the copy
// is input row perm[r] (band plan).
constexpr int kRowsPerWarp = 8;
template <bool BF16, int NV>
__global__ void __launch_bounds__(256, 4)  // 4 resident blocks: the row loads need the warps
k_prep(const float* __restrict__ X, int64_t n, int d, int DP, const float* __restrict__ mu,
       void* __restrict__ Xp_, float* __restrict__ hn, float* __restrict__ sn,
       uint16_t* __restrict__ gx, const int32_t* __restrict__ perm,
       const unsigned* __restrict__ f16xmax, double f16tau, float* __restrict__ g,
       float* __restrict__ tmaxS, float* __restrict__ tmaxN) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    // fp16 copies of the scaled centred rows, or bf16 / tf32 (fp16_scale)
    const float sc = BF16 ? fp16_scale(f16xmax, f16tau, d) : 0.0f;
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t r0 = w * kRowsPerWarp;
    if (r0 >= n) return;
    float m[NV];
#pragma unroll
    for (int i = 0; i < NV; i++) m[i] = lane * NV + i < d ? mu[lane * NV + i] : 0.0f;
    // vector loads need every column of the lane in range and aligned rows
    const bool vec = (NV == 2 || NV == 4) && d == DP && (reinterpret_cast<uintptr_t>(X) % (4 * NV) == 0);
    float x[kRowsPerWarp][NV];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; r++) {
        const int64_t src = r0 + r < n ? (perm ? static_cast<int64_t>(__ldg(perm + r0 + r)) : r0 + r) : -1;
        const float* xr = X + (src >= 0 ? src : 0) * d + lane * NV;
        if (src >= 0 && vec) {
            if (NV == 4) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(xr));
                x[r][0] = q.x;
                x[r][1 % NV] = q.y;
                x[r][2 % NV] = q.z;
                x[r][3 % NV] = q.w;
            } else {
                const float2 q = __ldg(reinterpret_cast<const float2*>(xr));
                x[r][0] = q.x;
                x[r][1 % NV] = q.y;
            }
        } else {
#pragma unroll
            for (int i = 0; i < NV; i++)
                x[r][i] = (src >= 0 && lane * NV + i < d) ? __ldg(xr + i) : 0.0f;
        }
    }
    double part[kRowsPerWarp], epart[kRowsPerWarp];
    uint32_t fin_mask = 0, big_mask = 0;
    // the copy format (fp16 / bf16 / tf32) and whether every lane column is
    // in range are uniform: the row loop is instantiated per case, so the
    // per-value work carries no branches (config-3 prep: 186 warp
    // instructions per row with them, issue-bound)
    auto rows = [&](auto f16_tag, auto full_tag) {
        constexpr bool F16 = decltype(f16_tag)::value;
        constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; r++) {
            double acc = 0.0;
            float eacc = 0.0f;
            bool finite = true, big = false;
            float t[NV];
#pragma unroll
            for (int i = 0; i < NV; i++) {
                const int k = lane * NV + i;
                t[i] = 0.0f;
                if (FULL || k < d) {
                    if (!isfinite(x[r][i])) finite = false;
                    float c = __fsub_rn(x[r][i], m[i]);
                    if constexpr (F16) {
                        c = __fmul_rn(c, sc);  // exact: a power of two (fp32 underflow
                                               // below 2^-126 errs < 2^-150, inside the 1e-30 slack)
                        t[i] = __half2float(__float2half_rn(c));
                    } else {
                        t[i] = BF16 ? __uint_as_float(static_cast<uint32_t>(to_bf16_bits(c)) << 16)
                                    : round_tf32(c);
                    }
                    if (!(fabsf(t[i]) <= kBigLimit)) big = true;
                    // this coordinate's rounding error: exact in fp32 (t is c
                    // rounded, so the two are within a factor 2); its square and
                    // the running sum round up to (d + 2) 2^-23 in all (err_norm)
                    const float e = __fsub_rn(t[i], c);
                    eacc = __fmaf_rn(e, e, eacc);
                }
                acc += static_cast<double>(t[i]) * static_cast<double>(t[i]);
            }
            part[r] = acc;
            epart[r] = static_cast<double>(eacc);
            finite = __all_sync(0xffffffffu, finite);
            big = __any_sync(0xffffffffu, big);
            fin_mask |= static_cast<uint32_t>(finite) << r;
            big_mask |= static_cast<uint32_t>(big) << r;
            if (r0 + r < n) {
                const bool zero = !finite || big;
                const int64_t row = r0 + r;
                if (BF16) {
                    uint16_t* xpb = static_cast<uint16_t*>(Xp_) + row * DP + lane * NV;
                    uint16_t b[NV];
#pragma unroll
                    for (int i = 0; i < NV; i++)
                        b[i] = zero ? 0
                             : F16 ? __half_as_ushort(__float2half_rn(t[i]))  // exact: t is fp16
                                   : static_cast<uint16_t>(__float_as_uint(t[i]) >> 16);
                    if (NV == 4) {
                        *reinterpret_cast<uint2*>(xpb) =
                            make_uint2(b[0] | (static_cast<uint32_t>(b[1 % NV]) << 16),
                                       b[2 % NV] | (static_cast<uint32_t>(b[3 % NV]) << 16));
                    } else if (NV == 2) {
                        *reinterpret_cast<uint32_t*>(xpb) = b[0] | (static_cast<uint32_t>(b[1 % NV]) << 16);
                    } else {
#pragma unroll
                        for (int i = 0; i < NV; i++) xpb[i] = b[i];
                    }
                } else {
                    float* xpf = static_cast<float*>(Xp_) + row * DP + lane * NV;
#pragma unroll
                    for (int i = 0; i < NV; i++) xpf[i] = zero ? 0.0f : t[i];
                }
            }
        }
    };
    const bool full = d == DP;
    if (BF16 && sc > 0.0f) {
        if (full) rows(std::true_type{}, std::true_type{});
        else rows(std::true_type{}, std::false_type{});
    } else {
        if (full) rows(std::false_type{}, std::true_type{});
        else rows(std::false_type{}, std::false_type{});
    }
    const double acc = sum8_transpose(part, lane);
    const double eacc = sum8_transpose(epart, lane);
    const int r = (lane >> 2) & 7;
    const bool mine = (lane & 3) == 0 && r0 + r < n;
    const bool finite = (fin_mask >> r) & 1, big = (big_mask >> r) & 1;
    const bool normal = mine && finite && !big;
    const float hv = normal ? static_cast<float>(acc) : 0.0f;
    const float sv = normal ? err_norm(acc, eacc, d) : 0.0f;
    if (tmaxS) {
        // the R tile's statistics (was k_tile_stats): the warp's eight rows
        // lie in one 256-row tile; maxima of non-negative floats order as
        // their bit patterns (zeroed by k_col_mean)
        float ms = sv, mn = hv;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
            mn = fmaxf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        }
        if (lane == 0) {
            atomicMax(reinterpret_cast<int*>(tmaxS + (r0 / BN)), __float_as_int(ms));
            atomicMax(reinterpret_cast<int*>(tmaxN + (r0 / BN)), __float_as_int(mn));
        }
    }
    if (!mine) return;
    const int64_t row = r0 + r;
    if (g) g[row] = !finite ? __int_as_float(0x7f800000) : big ? -__int_as_float(0x7f800000) : hv * 0.5f;
    if (!finite) {
        hn[row] = 0.0f;
        sn[row] = kFlagNonFinite;
    } else if (big) {
        hn[row] = 0.0f;
        sn[row] = kFlagBig;
    } else {
        hn[row] = hv;
        sn[row] = sv;
    }
    if (gx) {
        // folded-g block of this row: -||x~||^2/2 as the sum of three bf16
        // parts (24 significant bits), zeros elsewhere; -inf never matches,
        // +inf is always a candidate (rows too large for the screen)
        uint16_t pt[3] = {0, 0, 0};
        if (!finite) {
            pt[0] = 0xFF80u;
        } else if (big) {
            pt[0] = 0x7F80u;
        } else {
            double rr = -0.5 * acc;
            for (int q = 0; q < 3; q++) {
                const uint16_t b = to_bf16_bits(static_cast<float>(rr));
                pt[q] = b;
                rr -= static_cast<double>(__uint_as_float(static_cast<uint32_t>(b) << 16));
            }
        }
        uint4* gw = reinterpret_cast<uint4*>(gx + row * kGCols);
        gw[0] = make_uint4((static_cast<uint32_t>(pt[1]) << 16) | pt[0], pt[2], 0u, 0u);
        gw[1] = make_uint4(0u, 0u, 0u, 0u);
    }
}

// Any DP: one warp per row, 32 columns at a time.
template <bool BF16>
__global__ void __launch_bounds__(256)
k_prep_wide(const float* __restrict__ X, int64_t n, int d, int DP, const float* __restrict__ mu,
            void* __restrict__ Xp_, float* __restrict__ hn, float* __restrict__ sn) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    const float* x = X + row * d;
    float* xpf = static_cast<float*>(Xp_) + row * DP;
    uint16_t* xpb = static_cast<uint16_t*>(Xp_) + row * DP;
    double acc = 0.0;
    float eaccf = 0.0f;
    bool finite = true, big = false;
    for (int k = lane; k < DP; k += 32) {
        float t = 0.0f;
        if (k < d) {
            const float a = x[k];
            if (!isfinite(a)) finite = false;
            const float c = __fsub_rn(a, mu[k]);
            t = BF16 ? __uint_as_float(static_cast<uint32_t>(to_bf16_bits(c)) << 16)
                     : round_tf32(c);
            if (!(fabsf(t) <= kBigLimit)) big = true;
            const float e = __fsub_rn(t, c);  // exact (see k_prep)
            eaccf = __fmaf_rn(e, e, eaccf);
        }
        if (BF16) xpb[k] = static_cast<uint16_t>(__float_as_uint(t) >> 16);
        else xpf[k] = t;
        acc += static_cast<double>(t) * static_cast<double>(t);
    }
    double eacc = static_cast<double>(eaccf);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        acc += __shfl_xor_sync(0xffffffffu, acc, o);
        eacc += __shfl_xor_sync(0xffffffffu, eacc, o);
    }
    finite = __all_sync(0xffffffffu, finite);
    big = __any_sync(0xffffffffu, big);
    if (!finite || big) {
        for (int k = lane; k < DP; k += 32) {
            if (BF16) xpb[k] = 0;
            else xpf[k] = 0.0f;
        }
    }
    if (lane == 0) {
        if (!finite) {
            hn[row] = 0.0f;
            sn[row] = kFlagNonFinite;
        } else if (big) {
            hn[row] = 0.0f;
            sn[row] = kFlagBig;
        } else {
            hn[row] = static_cast<float>(acc);
            sn[row] = err_norm(acc, eacc, d);
        }
    }
}

// Per 256-row tile of R: max norms over regular rows, and g_j = ||y~||^2/2
// with +inf for non-finite rows and padding, -inf for forced rows.
__global__ void k_tile_stats(const float* __restrict__ hn, const float* __restrict__ sn,
                             int64_t n, float* __restrict__ g, float* __restrict__ tmaxS,
                             float* __restrict__ tmaxN) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int J = blockIdx.x;
    const int64_t j = static_cast<int64_t>(J) * BN + threadIdx.x;  // blockDim.x == BN
    float s = 0.0f, nn = 0.0f, gv = __int_as_float(0x7f800000);
    if (j < n) {
        const float f = sn[j];
        if (f == kFlagBig) {
            gv = -__int_as_float(0x7f800000);
        } else if (f != kFlagNonFinite) {
            s = f;
            nn = hn[j];
            gv = hn[j] * 0.5f;
        }
    }
    g[j] = gv;
    __shared__ float rs[BN / 32], rn[BN / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, o));
        nn = fmaxf(nn, __shfl_xor_sync(0xffffffffu, nn, o));
    }
    if ((threadIdx.x & 31) == 0) {
        rs[threadIdx.x >> 5] = s;
        rn[threadIdx.x >> 5] = nn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < BN / 32; k++) {
            s = fmaxf(s, rs[k]);
            nn = fmaxf(nn, rn[k]);
        }
        s = fmaxf(s, rs[0]);
        nn = fmaxf(nn, rn[0]);
        tmaxS[J] = s;
        tmaxN[J] = nn;
    }
}

// Per column chunk (ch consecutive 256-row tiles): max of the tile maxima.
// One block: per column chunk, the max row norms over its R tiles and the
// number of this shard's work units (row blocks rb < lim(c), rb = k*P +
// pos(k), pos(k) = shard for even k and P-1-shard for odd k -- the
// boustrophedon shard order), exclusive-scanned into chunk_off; also zeroes
// the screen / re-check counters (this is the first kernel they follow).
__global__ void __launch_bounds__(1024)
k_chunk_plan(const float* __restrict__ tmaxS, const float* __restrict__ tmaxN, int nt, int ch,
             int n_chunks, int64_t n_rb, int rpt, int self, int P, int shard, float* __restrict__ cmaxS,
             float* __restrict__ cmaxN, int64_t* __restrict__ chunk_off,
             unsigned long long* __restrict__ counters) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ int64_t part[1024];
    const int t = threadIdx.x;
    if (t < 5) counters[t] = 0;
    const int per = (n_chunks + 1023) / 1024;  // chunks per thread, contiguous
    int64_t local = 0;
    for (int c = t * per; c < min((t + 1) * per, n_chunks); c++) {
        if (tmaxS) {
            float a = 0.0f, b = 0.0f;
            for (int J = c * ch; J < min((c + 1) * ch, nt); J++) {
                a = fmaxf(a, tmaxS[J]);
                b = fmaxf(b, tmaxN[J]);
            }
            cmaxS[c] = a;
            cmaxN[c] = b;
        }
        int64_t lim = n_rb;
        if (self) lim = min(n_rb, static_cast<int64_t>(rpt) * (c + 1) * ch);
        const int64_t full = lim / P, rem = lim % P;
        const int64_t pos_last = (full & 1) ? P - 1 - shard : shard;
        local += full + (pos_last < rem ? 1 : 0);
    }
    part[t] = local;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {  // inclusive Hillis-Steele scan
        const int64_t v = t >= o ? part[t - o] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    int64_t run = part[t] - local;  // exclusive prefix of this thread's chunks
    if (t == 0) chunk_off[0] = 0;
    for (int c = t * per; c < min((t + 1) * per, n_chunks); c++) {
        int64_t lim = n_rb;
        if (self) lim = min(n_rb, static_cast<int64_t>(rpt) * (c + 1) * ch);
        const int64_t full = lim / P, rem = lim % P;
        const int64_t pos_last = (full & 1) ? P - 1 - shard : shard;
        run += full + (pos_last < rem ? 1 : 0);
        chunk_off[c + 1] = run;
    }
}

// The counters -> mapped pinned host memory (read after one stream sync).
__global__ void k_export_counters(const unsigned long long* __restrict__ c,
                                  volatile unsigned long long* h) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    if (threadIdx.x < 4) h[threadIdx.x] = c[threadIdx.x];
}

// ---------------------------------------------------------------------------
// The band plan: exact tile pruning on two principal projections.
//
// For any d x 2 matrix U, ||U^T (x - y)|| <= s ||x - y|| with s^2 the largest
// eigenvalue of U^T U.  So a 128-row block of L and a 256-row tile of R whose
// projected bounding boxes lie further apart than s * tau (plus the fp64
// projection error) hold no pair within tau, and the screen skips that tile.
// Rows are sorted by a Morton key of their projections onto the two leading
// principal directions of a row sample, so blocks and tiles are compact in
// that plane and most block / tile pairs of a large join separate.  Only
// surviving tiles are screened; the pair set is unchanged (the test never
// drops a pair whose exact distance is <= tau).  Every step is
// deterministic, so all shards of a join build the same plan.

constexpr int kPcaRows = 64;    // sample rows per partial block
constexpr int kPcaBlocks = 64;  // 4096 sample rows
constexpr int kPcaMaxD = 128;
// The plan costs ~40-90 us whatever the shard count; it pays when this
// shard's dense screen would visit at least kBandMinTiles tiles and both
// sides have kBandMinRows rows.  Single-GPU joins take it from 4,096 tiles:
// besides pruning, its row order makes a clustered output's candidate
// records dense (config 1, 6,319 tiles: 0.246 -> 0.210 ms; a 40k-row
// clustered self-join 0.518 -> 0.364 ms), at ~20-27 us more for small
// outputs-free joins (uniform 20k x 64: 0.083 -> 0.110 ms;
// tools/small_band_ab.py).  Sharded joins also pay the stable sort and keep
// the r01 threshold (16,384 per shard, doubled).
constexpr int64_t kBandMinRows = 8192;
constexpr int64_t kBandMinTiles = 4096;
constexpr int64_t kBandMinTilesSharded = 2 * 16384;
constexpr int kMortonBits = 6;  // per projection: 12-bit sort keys (one counting pass)
#ifndef PDB_PCA_ITERS
#define PDB_PCA_ITERS 2
#endif
// Subspace iterations for the leading plane.  Any plane prunes correctly;
// measured screened tiles for 1 / 2 / 3 / 4 iterations (r02): config 2
// 21,967 / 19,540 / 19,797 / 19,595, config 3 2.59 M / 318 k / 330 k / 337 k,
// config 5 51.1 M / 34.0 M / 34.9 M / 34.1 M.
constexpr int kPcaIters = PDB_PCA_ITERS;

struct BandInfo {
    float u[2][kPcaMaxD];   // the two directions (zero past d)
    double lo[2], inv[2];   // key quantisation q = (p - lo) * inv, clamped to [0, 2^bits - 1]
    double s;               // sqrt(lambda_max(U^T U)), rounded up
    unsigned long long bmax;  // fp64 bits of max_rows sum_k |u_k x_k| (projection error scale)
    unsigned xmax;            // fp32 bits of max |x_k - mu_k| <= 2^60 (fp16_scale)
};

// Partial sums over kPcaRows sample rows, centred by mu: the d x d products
// (a T x T register tile per thread, 16 x 16 threads), column sums and the
// count of usable rows (finite, |x - mu| <= 1e15).
template <int T>
__global__ void __launch_bounds__(256)
k_pca_partial(const float* __restrict__ X, int64_t n, int d, const float* __restrict__ mu,
              float* __restrict__ part) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ float xs[kPcaRows][16 * T];
    __shared__ int ok[kPcaRows];
    __shared__ int64_t rows[kPcaRows];
    const int64_t S = static_cast<int64_t>(gridDim.x) * kPcaRows;  // (kPcaBlocks, or fewer)
    if (threadIdx.x < kPcaRows) {
        rows[threadIdx.x] = (static_cast<int64_t>(blockIdx.x * kPcaRows + threadIdx.x) * n) / S;
        ok[threadIdx.x] = 1;
    }
    __syncthreads();
    // all of this thread's loads in flight at once (256 threads per block)
    constexpr int NQ = kPcaRows * 16 * T / 256;
    float v[NQ];
#pragma unroll
    for (int i = 0; i < NQ; i++) {
        const int q = threadIdx.x + 256 * i, k = q / (16 * T), c = q % (16 * T);
        v[i] = c < d ? __ldg(X + rows[k] * d + c) : 0.0f;
    }
#pragma unroll
    for (int i = 0; i < NQ; i++) {
        const int q = threadIdx.x + 256 * i, k = q / (16 * T), c = q % (16 * T);
        const float x = c < d ? v[i] - __ldg(mu + c) : 0.0f;
        xs[k][c] = x;
        if (!(fabsf(x) <= 1e15f)) ok[k] = 0;  // rows with huge or non-finite values sit out
    }
    __syncthreads();
    const int ta = threadIdx.x >> 4, tb = threadIdx.x & 15;
    float acc[T][T], cs[T];
#pragma unroll
    for (int i = 0; i < T; i++) {
        cs[i] = 0.0f;
#pragma unroll
        for (int j = 0; j < T; j++) acc[i][j] = 0.0f;
    }
    int cnt = 0;
    for (int k = 0; k < kPcaRows; k++) {
        if (!ok[k]) continue;  // block-uniform
        cnt++;
        float xa[T], xb[T];
#pragma unroll
        for (int i = 0; i < T; i++) {
            xa[i] = xs[k][ta * T + i];
            xb[i] = xs[k][tb * T + i];
        }
#pragma unroll
        for (int i = 0; i < T; i++) {
            cs[i] += xa[i];
#pragma unroll
            for (int j = 0; j < T; j++) acc[i][j] = fmaf(xa[i], xb[j], acc[i][j]);
        }
    }
    const int E = d + d * d + 1;
    float* out = part + static_cast<size_t>(blockIdx.x) * E;
#pragma unroll
    for (int i = 0; i < T; i++) {
        const int a = ta * T + i;
        if (a >= d) continue;
        if (tb == 0) out[a] = cs[i];
#pragma unroll
        for (int j = 0; j < T; j++) {
            const int b = tb * T + j;
            if (b < d) out[d + a * d + b] = acc[i][j];
        }
    }
    if (threadIdx.x == 0) out[E - 1] = static_cast<float>(cnt);
}

// Fixed-order fp64 reduction of the partials (deterministic).
__global__ void __launch_bounds__(128)
k_pca_reduce(const float* __restrict__ part, int E, double* __restrict__ sum,
             int32_t* __restrict__ bins0, int32_t* __restrict__ bins1, int nparts) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    // the counting sorts' bin counts and fill cursors (2 x 4096 per side)
    for (int b = e; b < 2 * (1 << (2 * kMortonBits)); b += gridDim.x * blockDim.x) {
        if (bins0) bins0[b] = 0;
        if (bins1) bins1[b] = 0;
    }
    if (e >= E) return;
    // every partial's load in flight at once, then the fixed-order sum
    float v[kPcaBlocks];
#pragma unroll
    for (int b = 0; b < kPcaBlocks; b++) v[b] = b < nparts ? part[static_cast<size_t>(b) * E + e] : 0.0f;
    double acc = 0.0;
#pragma unroll
    for (int b = 0; b < kPcaBlocks; b++) acc += static_cast<double>(v[b]);
    sum[e] = acc;
}

// The counting sorts' bin counts and fill cursors, when the directions were
// computed ahead (k_pca_reduce zeroes them otherwise).
__global__ void k_zero_bins(int32_t* __restrict__ bins0, int32_t* __restrict__ bins1) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < 2 * (1 << (2 * kMortonBits))) {
        if (bins0) bins0[b] = 0;
        if (bins1) bins1[b] = 0;
    }
}

// One block: the covariance (fp32, symmetric, read by columns so lanes hit
// distinct banks), kPcaIters subspace iterations on two vectors with
// Gram-Schmidt (a few suffice: any plane near the leading one prunes about
// as well), then the key quantisation and the bound's scale s of the fp32
// directions (fp64).
__global__ void __launch_bounds__(256)
k_pca_eig(const double* __restrict__ sum, int d, const float* __restrict__ mu,
          BandInfo* __restrict__ info) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    extern __shared__ float Cs[];  // [d][d]
    __shared__ float v[2][kPcaMaxD];
    __shared__ float wpart[2][8][kPcaMaxD];
    __shared__ double mean[kPcaMaxD];
    __shared__ float fred[3][8];
    __shared__ double dred[5][8];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    const double m = sum[d + d * d];
    const double im = m > 0 ? 1.0 / m : 0.0;
    for (int c = t; c < d; c += blockDim.x) mean[c] = sum[c] * im;
    for (int c = t; c < kPcaMaxD; c += blockDim.x) {
        v[0][c] = c < d ? 1.0f + 0.001f * c : 0.0f;
        v[1][c] = c < d ? ((c & 1) ? 1.0f : -1.0f) * (1.0f + 0.002f * c) : 0.0f;
    }
    __syncthreads();
    // all of a thread's loads of the sums in flight before their use (the
    // dependent load-per-element loop was two thirds of this kernel's time)
    for (int e0 = 0; e0 < d * d; e0 += 16 * static_cast<int>(blockDim.x)) {
        double sv[16];
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const int e = e0 + t + i * static_cast<int>(blockDim.x);
            sv[i] = e < d * d ? sum[d + e] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 16; i++) {
            const int e = e0 + t + i * static_cast<int>(blockDim.x);
            if (e < d * d) {
                const int a = e / d, b = e - a * d;
                Cs[e] = static_cast<float>(m > 0 ? sv[i] * im - mean[a] * mean[b] : (a == b ? 1.0 : 0.0));
            }
        }
    }
    __syncthreads();
    const int np = min(8, max(1, static_cast<int>(blockDim.x) / d));  // column groups
    const int a = t % d, pg = t / d;
    const int bw = (d + np - 1) / np;
    const int b0 = pg * bw, b1 = min(d, b0 + bw);
    float l0 = 0.0f, l1 = 0.0f;
    for (int it = 0; it < kPcaIters; it++) {
        if (pg < np) {
            float w0 = 0.0f, w1 = 0.0f;
            for (int b = b0; b < b1; b++) {
                const float c = Cs[b * d + a];  // = C[a][b]
                w0 = fmaf(c, v[0][b], w0);
                w1 = fmaf(c, v[1][b], w1);
            }
            wpart[0][pg][a] = w0;
            wpart[1][pg][a] = w1;
        }
        __syncthreads();
        float w0 = 0.0f, w1 = 0.0f, q0 = 0.0f, q1 = 0.0f, q2 = 0.0f;
        if (t < d) {
            for (int g = 0; g < np; g++) {
                w0 += wpart[0][g][t];
                w1 += wpart[1][g][t];
            }
            q0 = w0 * w0;
            q1 = w0 * w1;
            q2 = w1 * w1;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            q0 += __shfl_xor_sync(0xffffffffu, q0, o);
            q1 += __shfl_xor_sync(0xffffffffu, q1, o);
            q2 += __shfl_xor_sync(0xffffffffu, q2, o);
        }
        if (lane == 0) {
            fred[0][wid] = q0;
            fred[1][wid] = q1;
            fred[2][wid] = q2;
        }
        __syncthreads();
        q0 = q1 = q2 = 0.0f;
        for (int w = 0; w < 8; w++) {
            q0 += fred[0][w];
            q1 += fred[1][w];
            q2 += fred[2][w];
        }
        // v0 = w0 / |w0|; v1 = (w1 - (w0.w1 / |w0|^2) w0) / |..|
        const float r0 = q0 > 0.0f ? rsqrtf(q0) : 0.0f;
        const float c01 = q0 > 0.0f ? q1 * r0 * r0 : 0.0f;
        const float e2 = q2 - c01 * q1;
        const float r1 = e2 > 0.0f ? rsqrtf(e2) : 0.0f;
        l0 = q0 * r0;
        l1 = e2 * r1;
        if (t < d) {
            v[0][t] = r0 > 0.0f ? w0 * r0 : (t == 0 ? 1.0f : 0.0f);
            v[1][t] = r1 > 0.0f ? (w1 - c01 * w0) * r1 : (t == 1 ? 1.0f : 0.0f);
        }
        __syncthreads();
    }
    for (int c = t; c < kPcaMaxD; c += blockDim.x) {
        info->u[0][c] = c < d ? v[0][c] : 0.0f;
        info->u[1][c] = c < d ? v[1][c] : 0.0f;
    }
    double g[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // u0.u0, u1.u1, u0.u1, u0.centre, u1.centre
    if (t < d) {
        const double x0 = v[0][t], x1 = v[1][t];
        const double centre = mean[t];  // projections are of x - mu
        g[0] = x0 * x0;
        g[1] = x1 * x1;
        g[2] = x0 * x1;
        g[3] = x0 * centre;
        g[4] = x1 * centre;
    }
#pragma unroll
    for (int q = 0; q < 5; q++) {
        for (int o = 16; o > 0; o >>= 1) g[q] += __shfl_xor_sync(0xffffffffu, g[q], o);
        if (lane == 0) dred[q][wid] = g[q];
    }
    __syncthreads();
    if (t == 0) {
        for (int q = 0; q < 5; q++) {
            g[q] = 0.0;
            for (int w = 0; w < 8; w++) g[q] += dred[q][w];
        }
        const double h = 0.5 * (g[0] + g[1]), q = 0.5 * (g[0] - g[1]);
        info->s = sqrt(h + sqrt(q * q + g[2] * g[2])) * (1.0 + 1e-12);
        const double cen[2] = {g[3], g[4]}, lam[2] = {l0, l1};
        for (int k = 0; k < 2; k++) {
            const double sd = sqrt(fmax(lam[k], 0.0));
            info->lo[k] = cen[k] - 3.0 * sd;
            info->inv[k] = sd > 0 ? static_cast<double>(1 << kMortonBits) / (6.0 * sd) : 0.0;
        }
        info->bmax = 0ull;
        info->xmax = 0u;
    }
}

__device__ __forceinline__ uint32_t spread_bits(uint32_t x) {  // low 8 bits -> even positions
    x &= 0xffu;
    x = (x | (x << 4)) & 0x0f0fu;
    x = (x | (x << 2)) & 0x3333u;
    x = (x | (x << 1)) & 0x5555u;
    return x;
}

// Eight lanes per row, four rows per warp step: lane sub = lane % 8 owns
// columns 32 i + 4 sub + j (i < NV, j < 4), so each group reads its row in
// coalesced 128-byte float4 runs.  Projections of the centred row x - mu in
// fp32 FMA chains with the error scale b = sum_k |u_k| |x_k - mu_k|: the
// computed projection is within (d + 2) 2^-24 b of the exact one (the
// centring cancels in every difference of two rows).  Outputs: the
// projections, the Morton sort key, and b max-reduced per block (one
// atomicMax per block), and (single-GPU joins) the counting sort's bin
// counts, zeroed by k_pca_reduce.
template <int NV>
__global__ void __launch_bounds__(256, 2)
k_band_keys(const float* __restrict__ X, int64_t n, int d, const float* __restrict__ mu,
            BandInfo* __restrict__ info, float2* __restrict__ proj, uint32_t* __restrict__ key,
            int32_t* __restrict__ val, int32_t* __restrict__ bin_count) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ float bred[8], xred[8];
    __shared__ float4 us[3][32 * NV / 4];  // u0, u1, mu
    for (int c = threadIdx.x; c < 32 * NV / 4; c += blockDim.x) {
        us[0][c] = reinterpret_cast<const float4*>(info->u[0])[c];
        us[1][c] = reinterpret_cast<const float4*>(info->u[1])[c];
        float4 m;
        m.x = 4 * c < d ? mu[4 * c] : 0.0f;
        m.y = 4 * c + 1 < d ? mu[4 * c + 1] : 0.0f;
        m.z = 4 * c + 2 < d ? mu[4 * c + 2] : 0.0f;
        m.w = 4 * c + 3 < d ? mu[4 * c + 3] : 0.0f;
        us[2][c] = m;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int grp = lane >> 3, sub = lane & 7;
    const float lo0 = static_cast<float>(info->lo[0]), lo1 = static_cast<float>(info->lo[1]);
    const float inv0 = static_cast<float>(info->inv[0]), inv1 = static_cast<float>(info->inv[1]);
    const bool vec = d == 32 * NV && (reinterpret_cast<uintptr_t>(X) % 16 == 0);
    // 8 or 16 rows per warp step (RPG per lane group), all loads issued first
    constexpr int RPG = NV >= 3 ? 2 : 4;  // rows per lane group in flight
    const int64_t step = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5) * 4 * RPG;
    float bm = 0.0f, xm = 0.0f;
    for (int64_t r0 = (static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + wib) * 4 * RPG; r0 < n;
         r0 += step) {
        float x[RPG][NV][4];
#pragma unroll
        for (int h = 0; h < RPG; h++) {
            const int64_t row = r0 + 4 * h + grp;
            const bool on = row < n;
            const float* xr = X + (on ? row : 0) * d;
#pragma unroll
            for (int i = 0; i < NV; i++) {
                const int c0 = 32 * i + 4 * sub;
                if (vec) {
                    const float4 q = on ? __ldg(reinterpret_cast<const float4*>(xr + c0)) : make_float4(0, 0, 0, 0);
                    x[h][i][0] = q.x;
                    x[h][i][1] = q.y;
                    x[h][i][2] = q.z;
                    x[h][i][3] = q.w;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; j++) x[h][i][j] = (on && c0 + j < d) ? __ldg(xr + c0 + j) : 0.0f;
                }
            }
        }
#pragma unroll
        for (int h = 0; h < RPG; h++) {
            const int64_t row = r0 + 4 * h + grp;
            const bool on = row < n;
            float p0 = 0.0f, p1 = 0.0f, b = 0.0f;
#pragma unroll
            for (int i = 0; i < NV; i++) {
                const float4 w0 = us[0][8 * i + sub], w1 = us[1][8 * i + sub], mm = us[2][8 * i + sub];
                const float ua[4] = {w0.x, w0.y, w0.z, w0.w}, ub[4] = {w1.x, w1.y, w1.z, w1.w};
                const float mc[4] = {mm.x, mm.y, mm.z, mm.w};
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    const float xc = x[h][i][j] - mc[j];
                    if (fabsf(xc) <= kBigLimit) xm = fmaxf(xm, fabsf(xc));  // (NaN, inf: no)
                    p0 = fmaf(ua[j], xc, p0);
                    p1 = fmaf(ub[j], xc, p1);
                    b = fmaf(fabsf(ua[j]) + fabsf(ub[j]), fabsf(xc), b);
                }
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                p0 += __shfl_xor_sync(0xffffffffu, p0, o);
                p1 += __shfl_xor_sync(0xffffffffu, p1, o);
                b += __shfl_xor_sync(0xffffffffu, b, o);
            }
            if (on && sub == 0) {
                uint32_t kk = (1u << (2 * kMortonBits)) - 1;  // non-finite rows sort last
                if (isfinite(p0) && isfinite(p1) && isfinite(b)) {
                    const float lim = static_cast<float>((1 << kMortonBits) - 1);
                    const uint32_t q0 = static_cast<uint32_t>(fminf(fmaxf((p0 - lo0) * inv0, 0.0f), lim));
                    const uint32_t q1 = static_cast<uint32_t>(fminf(fmaxf((p1 - lo1) * inv1, 0.0f), lim));
                    kk = spread_bits(q0) | (spread_bits(q1) << 1);
                    bm = fmaxf(bm, b);
                } else {
                    // rows whose projections overflow fp32 are left in every box's
                    // way (NaN boxes keep every tile); truly non-finite rows match nothing
                    p0 = p1 = __int_as_float(0x7fc00000);
                }
                proj[row] = make_float2(p0, p1);
                key[row] = kk;
                val[row] = static_cast<int32_t>(row);
                if (bin_count) atomicAdd(bin_count + kk, 1);
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        bm = fmaxf(bm, __shfl_xor_sync(0xffffffffu, bm, o));
        xm = fmaxf(xm, __shfl_xor_sync(0xffffffffu, xm, o));
    }
    if (lane == 0) {
        bred[wib] = bm;
        xred[wib] = xm;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.0f, mx = 0.0f;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); w++) {
            m = fmaxf(m, bred[w]);
            mx = fmaxf(mx, xred[w]);
        }
        if (m > 0) atomicMax(&info->bmax, static_cast<unsigned long long>(__double_as_longlong(static_cast<double>(m))));
        if (mx > 0) atomicMax(&info->xmax, __float_as_uint(mx));
    }
}

// Counting sort of the 12-bit keys for single-GPU joins: k_band_keys counts
// the bins, each scatter block scans them and reserves its slots per bin
// with one atomic (the order inside a bin is arbitrary -- harmless, since
// the tile test is exact for any order).
// Sharded joins need every rank to build the same order and use the
// deterministic stable counting sort below (k_rank_*) instead.
constexpr int kBins = 1 << (2 * kMortonBits);

constexpr int kScatterRows = 4;  // rows per thread (4096 per 1024-thread block)
template <int RPT>
__global__ void __launch_bounds__(1024)
k_bin_scatter(const uint32_t* __restrict__ key, int64_t n, const int32_t* __restrict__ count,
              int32_t* __restrict__ fill, int32_t* __restrict__ perm) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ int32_t cnt[kBins], base[kBins];
    __shared__ int32_t wsum[32];
    // every block scans the 4096 bin counts itself (16 KB from L2): the bin
    // offsets need no kernel of their own
    constexpr int per = kBins / 1024;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    // this block's keys load while the counts are scanned
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * blockDim.x * RPT;
    uint32_t k[RPT];
#pragma unroll
    for (int i = 0; i < RPT; i++) {
        const int64_t r = r0 + i * blockDim.x + threadIdx.x;
        k[i] = r < n ? __ldg(key + r) : 0xffffffffu;
    }
    int32_t v[per], lsum = 0;
#pragma unroll
    for (int i = 0; i < per; i++) {
        v[i] = __ldcg(count + t * per + i);
        lsum += v[i];
        cnt[t * per + i] = 0;
    }
    int32_t incl = lsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int32_t x = wsum[lane], xi = x;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t y = __shfl_up_sync(0xffffffffu, xi, o);
            if (lane >= o) xi += y;
        }
        wsum[lane] = xi - x;
    }
    __syncthreads();
    int32_t run = wsum[wid] + incl - lsum;
#pragma unroll
    for (int i = 0; i < per; i++) {
        base[t * per + i] = run;
        run += v[i];
    }
    __syncthreads();
    int32_t local[RPT];
#pragma unroll
    for (int i = 0; i < RPT; i++) {
        const int64_t r = r0 + i * blockDim.x + threadIdx.x;
        local[i] = r < n ? atomicAdd(&cnt[k[i]], 1) : 0;
    }
    __syncthreads();
    // one global reservation per (block, bin)
    for (int b = threadIdx.x; b < kBins; b += blockDim.x)
        if (cnt[b]) base[b] += atomicAdd(fill + b, cnt[b]);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RPT; i++) {
        const int64_t r = r0 + i * blockDim.x + threadIdx.x;
        if (r < n) {
            PDB_DCHECK(k[i] < static_cast<uint32_t>(kBins) && base[k[i]] + local[i] < n);
            perm[base[k[i]] + local[i]] = static_cast<int32_t>(r);
        }
    }
}

// Deterministic stable counting sort of the 12-bit keys (sharded joins:
// every rank must build the same order).  k_rank_local: per block of
// kRankRows consecutive rows, each row's rank among the block's earlier rows
// with the same key -- the block's warps take turns (row order), each warp
// ranking its 32 rows with __match_any_sync against a shared running count
// per bin -- and the block's per-bin totals.
constexpr int kRankRows = 4096;
__global__ void __launch_bounds__(1024)
k_rank_local(const uint32_t* __restrict__ key, int64_t n, int32_t* __restrict__ rank,
             int32_t* __restrict__ bcnt) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ int32_t running[kBins];
    for (int b = threadIdx.x; b < kBins; b += blockDim.x) running[b] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kRankRows;
    for (int pass = 0; pass < kRankRows / 1024; pass++) {
        const int64_t row = base + pass * 1024 + threadIdx.x;
        const uint32_t k = row < n ? __ldg(key + row) : 0xffffffffu;  // sentinel past the end
        const uint32_t same = __match_any_sync(0xffffffffu, k);
        const int below = __popc(same & ((1u << lane) - 1u));
        const bool last = (same >> lane) == 1u;  // highest lane of its key group
        for (int turn = 0; turn < 32; turn++) {
            if (turn == w && row < n) {
                const int32_t b0 = running[k];
                rank[row] = b0 + below;
                __syncwarp(__activemask());
                if (last) running[k] = b0 + __popc(same);
            }
            __syncthreads();
        }
    }
    for (int b = threadIdx.x; b < kBins; b += blockDim.x)
        bcnt[static_cast<int64_t>(blockIdx.x) * kBins + b] = running[b];
}

// In place: bcnt[blk][bin] -> the sorted position of the block's first row
// of that bin: the bin's start (exclusive scan of the global counts) plus the
// earlier blocks' counts of the bin.  One thread per bin.
__global__ void __launch_bounds__(256)
k_rank_offsets(const int32_t* __restrict__ count, int32_t* __restrict__ bcnt, int64_t nblk) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ int32_t wsum[8];
    __shared__ int32_t start_of_block;
    const int bin = blockIdx.x * blockDim.x + threadIdx.x;
    // this block's bins start after every lower bin: sum of count[0 .. first)
    int32_t part = 0;
    for (int b = threadIdx.x; b < blockIdx.x * blockDim.x; b += blockDim.x) part += count[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t t = 0;
        for (int q = 0; q < 8; q++) t += wsum[q];
        start_of_block = t;
    }
    __syncthreads();
    // exclusive scan of count over this block's 256 bins
    const int32_t c = count[bin];
    int32_t incl = c;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    __syncthreads();
    if (lane == 31) wsum[wid] = incl;
    __syncthreads();
    int32_t wpre = 0;
    for (int q = 0; q < wid; q++) wpre += wsum[q];
    int32_t run = start_of_block + wpre + incl - c;
    // then down the blocks (independent loads issued ahead of the running sum)
    for (int64_t b0 = 0; b0 < nblk; b0 += 8) {
        int32_t v[8];
#pragma unroll
        for (int q = 0; q < 8; q++) v[q] = b0 + q < nblk ? bcnt[(b0 + q) * kBins + bin] : 0;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            if (b0 + q < nblk) bcnt[(b0 + q) * kBins + bin] = run;
            run += v[q];
        }
    }
}

__global__ void __launch_bounds__(1024)
k_rank_scatter(const uint32_t* __restrict__ key, int64_t n, const int32_t* __restrict__ rank,
               const int32_t* __restrict__ boff, int32_t* __restrict__ perm) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kRankRows;
    for (int i = threadIdx.x; i < kRankRows; i += blockDim.x) {
        const int64_t row = base + i;
        if (row >= n) break;
        const uint32_t k = __ldg(key + row);
        const int64_t pos = static_cast<int64_t>(__ldg(boff + static_cast<int64_t>(blockIdx.x) * kBins + k)) +
                            __ldg(rank + row);
        PDB_DCHECK(k < static_cast<uint32_t>(kBins) && pos >= 0 && pos < n);
        perm[pos] = static_cast<int32_t>(row);
    }
}

// One warp per block of `blk` sorted rows: the projected bounding box
// (min0, max0, min1, max1).  A row without finite projections (non-finite
// data, or fp32 overflow of a huge row) makes its block's box the whole
// plane, so no tile of that block is ever pruned.
__global__ void __launch_bounds__(256)
k_band_boxes(const float2* __restrict__ proj, const int32_t* __restrict__ perm, int64_t n, int blk,
             int64_t n_blk, double4* __restrict__ box) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int64_t b = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (b >= n_blk) return;
    const float inf = __int_as_float(0x7f800000);
    float lo0 = inf, hi0 = -inf, lo1 = inf, hi1 = -inf;
    bool wild = false;
    const int64_t r1 = min(n, (b + 1) * blk);
    for (int64_t r = b * blk + lane; r < r1; r += 32) {
        const float2 q = proj[__ldg(perm + r)];
        if (!(isfinite(q.x) && isfinite(q.y))) wild = true;
        lo0 = fminf(lo0, q.x);
        hi0 = fmaxf(hi0, q.x);
        lo1 = fminf(lo1, q.y);
        hi1 = fmaxf(hi1, q.y);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo0 = fminf(lo0, __shfl_xor_sync(0xffffffffu, lo0, o));
        hi0 = fmaxf(hi0, __shfl_xor_sync(0xffffffffu, hi0, o));
        lo1 = fminf(lo1, __shfl_xor_sync(0xffffffffu, lo1, o));
        hi1 = fmaxf(hi1, __shfl_xor_sync(0xffffffffu, hi1, o));
    }
    wild = __any_sync(0xffffffffu, wild);
    if (lane == 0) {
        const double dinf = __longlong_as_double(0x7ff0000000000000ll);
        box[b] = wild ? make_double4(-dinf, dinf, -dinf, dinf) : make_double4(lo0, hi0, lo1, hi1);
    }
}

struct BandPlan {
    const double4* boxL;
    const double4* boxR;  // nullptr for a self-join: tile J = row blocks 2J, 2J + 1
    const double4* sup;   // union box of each group of 32 consecutive tiles
    const BandInfo* info;
    double tau;
    int d, nt, self, P, shard, n_slots, nbl;
};

__device__ __forceinline__ double4 box_r(const BandPlan& q, int J) {
    if (q.boxR) return q.boxR[J];
    const double4 a = q.boxL[2 * J];
    if (2 * J + 1 >= q.nbl) return a;
    const double4 b = q.boxL[2 * J + 1];
    return make_double4(fmin(a.x, b.x), fmax(a.y, b.y), fmin(a.z, b.z), fmax(a.w, b.w));
}

// Squared threshold of the box test: (s tau + projection error)^2, widened.
__device__ __forceinline__ double band_thr2(const BandPlan& q) {
    const double bmax = __longlong_as_double(static_cast<long long>(q.info->bmax));
    const double err = 4.0 * (q.d + 8) * 5.9604644775390625e-08 * bmax;  // 4 (d+8) 2^-24 bmax
    const double t = (q.tau * q.info->s + err) * (1.0 + 1e-9);
    return t * t;
}

// One warp per group of 32 consecutive column tiles: their union box (the
// tiles are Morton-ordered, so a group is compact and most groups fail the
// test as a whole).
__global__ void __launch_bounds__(256)
k_band_groups(const BandPlan q, double4* __restrict__ sup) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int g = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (g >= (q.nt + 31) / 32) return;
    const double inf = __longlong_as_double(0x7ff0000000000000ll);
    double4 u = make_double4(inf, -inf, inf, -inf);
    const int J = g * 32 + lane;
    if (J < q.nt) u = box_r(q, J);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        u.x = fmin(u.x, __shfl_xor_sync(0xffffffffu, u.x, o));
        u.y = fmax(u.y, __shfl_xor_sync(0xffffffffu, u.y, o));
        u.z = fmin(u.z, __shfl_xor_sync(0xffffffffu, u.z, o));
        u.w = fmax(u.w, __shfl_xor_sync(0xffffffffu, u.w, o));
    }
    if (lane == 0) sup[g] = u;
}

__device__ __forceinline__ bool band_keep(const double4& a, const double4& b, double thr2) {
    const double g0 = fmax(0.0, fmax(b.x - a.y, a.x - b.y));
    const double g1 = fmax(0.0, fmax(b.z - a.w, a.z - b.w));
    return !(g0 * g0 + g1 * g1 > thr2);  // NaN-safe: keeps the tile
}

__device__ __forceinline__ int slot_rb(const BandPlan& q, int k) {
    const int pos = (k & 1) ? q.P - 1 - q.shard : q.shard;
    return k * q.P + pos;
}

// Walks row slot `a`'s candidate column tiles J >= j0 in ascending order:
// one load per lane tests 32 groups' union boxes at once, then the tile
// boxes of up to four surviving groups are loaded together, so a slot costs
// a few dependent load latencies instead of one per group.  f(J, keep) is
// called by the whole warp (J differs per lane) once per surviving group.
template <class F>
__device__ __forceinline__ void band_walk(const BandPlan& q, const double4& a, double thr2, int j0,
                                          int lane, F&& f) {
    const int g_end = (q.nt + 31) >> 5;
    for (int gb = j0 >> 5; gb < g_end; gb += 32) {
        const int g = gb + lane;
        uint32_t gm = __ballot_sync(0xffffffffu, g < g_end && band_keep(a, q.sup[g], thr2));
        while (gm) {
            int gs[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                gs[i] = gm ? gb + __ffs(gm) - 1 : -1;
                gm &= gm - 1;
            }
            double4 bx[4];
#pragma unroll
            for (int i = 0; i < 4; i++) {
                const int J = gs[i] * 32 + lane;
                bx[i] = (gs[i] >= 0 && J >= j0 && J < q.nt) ? box_r(q, J) : make_double4(0, 0, 0, 0);
            }
#pragma unroll
            for (int i = 0; i < 4; i++) {
                if (gs[i] < 0) break;  // warp-uniform
                const int J = gs[i] * 32 + lane;
                f(J, J >= j0 && J < q.nt && band_keep(a, bx[i], thr2));
            }
        }
    }
}

// One warp per row slot of this shard: surviving column tiles.
__global__ void __launch_bounds__(256)
k_band_count(const BandPlan q, int32_t* __restrict__ cnt) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int k = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= q.n_slots) return;
    const int rb = slot_rb(q, k);
    const double thr2 = band_thr2(q);
    const double4 a = q.boxL[rb];
    int c = 0;
    band_walk(q, a, thr2, q.self ? rb >> 1 : 0, lane, [&](int, bool keep) { c += keep; });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[k] = c;
}

// One block: list offsets, tiles per unit, unit offsets; zeroes the screen /
// re-check counters (the first kernel they follow).
__global__ void __launch_bounds__(1024)
k_band_scan(const int32_t* __restrict__ cnt, int n_slots, int units_target, int64_t* __restrict__ list_off,
            int64_t* __restrict__ unit_off, int64_t* __restrict__ n_units, int32_t* __restrict__ dev_ch,
            unsigned long long* __restrict__ counters, unsigned long long* host_units) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    __shared__ int64_t part[32];
    __shared__ int ch_s;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
    if (t < 5) counters[t] = 0;
    const int per = (n_slots + 1023) / 1024;
    const int k0 = min(t * per, n_slots), k1 = min((t + 1) * per, n_slots);
    auto scan = [&](int64_t local) -> int64_t {  // exclusive prefix of this thread's range
        int64_t incl = local;  // warp shuffles, then one warp over the 32 warp totals
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) part[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            const int64_t x = part[lane];
            int64_t xi = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t v = __shfl_up_sync(0xffffffffu, xi, o);
                if (lane >= o) xi += v;
            }
            part[lane] = xi - x;
        }
        __syncthreads();
        const int64_t r = part[wid] + incl - local;
        __syncthreads();
        return r;
    };
    int64_t local = 0;
    for (int k = k0; k < k1; k++) local += cnt[k];
    int64_t run = scan(local);
    if (t == 1023) {
        const int64_t total = run + local;
        int64_t c = total / units_target;
        c = c < 1 ? 1 : (c > 64 ? 64 : c);
        ch_s = static_cast<int>(c);
        *dev_ch = ch_s;
    }
    if (t == 0) list_off[0] = 0;
    for (int k = k0; k < k1; k++) {
        run += cnt[k];
        list_off[k + 1] = run;
    }
    __syncthreads();
    const int ch = ch_s;
    local = 0;
    for (int k = k0; k < k1; k++) local += (cnt[k] + ch - 1) / ch;
    run = scan(local);
    if (t == 0) unit_off[0] = 0;
    for (int k = k0; k < k1; k++) {
        run += (cnt[k] + ch - 1) / ch;
        unit_off[k + 1] = run;
    }
    if (t == 1023) {
        *n_units = run;
        if (host_units) {  // mapped pinned slot: the host reads it after an event
            *reinterpret_cast<volatile unsigned long long*>(host_units) = static_cast<unsigned long long>(run);
            __threadfence_system();
        }
    }
}

// One warp per row slot: the surviving tiles in ascending order and the
// slot's norm maxima over them (the screen's margin for the whole slot).
__global__ void __launch_bounds__(256)
k_band_write(const BandPlan q, const int64_t* __restrict__ list_off, int32_t* __restrict__ list,
             const float* __restrict__ tmaxS, const float* __restrict__ tmaxN,
             float* __restrict__ smaxS, float* __restrict__ smaxN,
             const int64_t* __restrict__ unit_off, const int32_t* __restrict__ dev_ch,
             int4* __restrict__ unit_info, const float* __restrict__ hnL,
             const float* __restrict__ snL, int64_t nL, double tau_p, double uu, double gam,
             float* __restrict__ hrow, const unsigned* __restrict__ f16xmax) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    {  // fp16 copies measure distances in units of 2^-s (fp16_scale)
        const float sc = fp16_scale(f16xmax, q.tau, q.d);
        if (sc > 0.0f) tau_p *= static_cast<double>(sc);
    }
    const int k = static_cast<int>((static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (k >= q.n_slots) return;
    const int rb = slot_rb(q, k);
    // the slot's row norms, loaded during the walk (the row thresholds below)
    const int64_t i_end = min(nL, static_cast<int64_t>(rb + 1) * BM);
    float hnv[BM / 32], snv[BM / 32];
#pragma unroll
    for (int q = 0; q < BM / 32; q++) {
        const int64_t i = static_cast<int64_t>(rb) * BM + lane + 32 * q;
        hnv[q] = i < i_end ? hnL[i] : 0.0f;
        snv[q] = i < i_end ? snL[i] : 0.0f;
    }
    const double thr2 = band_thr2(q);
    const double4 a = q.boxL[rb];
    int64_t w = list_off[k];
    float ms = 0.0f, mn = 0.0f;
    band_walk(q, a, thr2, q.self ? rb >> 1 : 0, lane, [&](int J, bool keep) {
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) {
            list[w + __popc(bal & ((1u << lane) - 1u))] = J;
            ms = fmaxf(ms, tmaxS[J]);
            mn = fmaxf(mn, tmaxN[J]);
        }
        w += __popc(bal);
    });
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ms = fmaxf(ms, __shfl_xor_sync(0xffffffffu, ms, o));
        mn = fmaxf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    }
    if (lane == 0) {
        smaxS[k] = ms;
        smaxN[k] = mn;
    }
    // each row's screen threshold, exactly as k_screen's epilogue would
    // compute it from the slot maxima (one load per unit there instead)
#pragma unroll
    for (int q = 0; q < BM / 32; q++) {
        const int64_t i = static_cast<int64_t>(rb) * BM + lane + 32 * q;
        if (i >= i_end) continue;  // (not break: the arrays stay in registers)
        const float hn = hnv[q], sn = snv[q];
        float h;
        if (sn == kFlagNonFinite) {
            h = __int_as_float(0x7f800000);
        } else if (sn == kFlagBig) {
            h = -__int_as_float(0x7f800000);
        } else {
            const double r = tau_p + uu * (static_cast<double>(sn) + ms) + 1e-30;
            const double T = r * r + gam * (static_cast<double>(hn) + mn);
            h = __double2float_rd((static_cast<double>(hn) - T) * 0.5);
        }
        hrow[i] = h;
    }
    // the slot's work units, decoded once for the screen
    const int ch = *dev_ch;
    const int64_t l0 = list_off[k], l1 = list_off[k + 1], u0 = unit_off[k], u1 = unit_off[k + 1];
    for (int64_t u = u0 + lane; u < u1; u += 32) {
        const int64_t o0 = l0 + (u - u0) * ch;
        unit_info[u] = make_int4(rb, static_cast<int>(o0), static_cast<int>(min(o0 + ch, l1)), k);
    }
}

// Grouped copy of R for dense re-checks: XT[(g * ldt + p) * 8 + c] =
// R[perm[p]][8 g + c] (zero past d), p the column position.  Consecutive
// threads take consecutive positions of one group, so the writes coalesce.
__global__ void __launch_bounds__(256)
k_group_copy(const float* __restrict__ R, int64_t n, int d, const int32_t* __restrict__ perm,
             float* __restrict__ XT) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int G = (d + 7) / 8;
    const int64_t total = n * G;
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(t / n);
        const int64_t p = t - static_cast<int64_t>(g) * n;
        const int64_t src = perm ? __ldg(perm + p) : p;
        const float* r = R + src * d + 8 * g;
        float v[8];
#pragma unroll
        for (int c = 0; c < 8; c++) v[c] = 8 * g + c < d ? __ldg(r + c) : 0.0f;
        float4* o = reinterpret_cast<float4*>(XT + (static_cast<int64_t>(g) * n + p) * 8);
        o[0] = make_float4(v[0], v[1], v[2], v[3]);
        o[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
}

// ---------------------------------------------------------------------------
// K3: exact re-check.  The fp64 chain is written with explicit _rn
// intrinsics so it can never be contracted into FMAs: diff = a - b,
// acc = acc + diff * diff, sequential in k, then sqrt -- src/index.cpp:69-76.
// A warp loads 32 candidate records (row i, first column j0, 32-bit mask)
// and flattens their set bits into one queue: the c-th candidate belongs to
// the lane whose exclusive popcount prefix covers c, and is that lane's
// (c - prefix)-th set bit.  Every batch of 32 candidates keeps all lanes
// busy whatever the masks' skew (records of tight clusters carry ~30 bits,
// scattered ones 1-2), and lanes of one record share their row of L.
// Survivors are compacted with a ballot and one atomic per batch.
// G: 0 rows of L and R row-major; 1 R from the grouped copy XT (column
// order); 2 (self-joins) both sides from XT, L by its row position.
template <int G>
__global__ void __launch_bounds__(256)
k_recheck(const int4* __restrict__ rec, const unsigned long long* __restrict__ n_rec,
          unsigned long long cap, const float* __restrict__ L, const float* __restrict__ R,
          int d, double tau, int32_t* __restrict__ out_l, int32_t* __restrict__ out_r,
          float* __restrict__ out_d, unsigned long long out_cap,
          unsigned long long* __restrict__ out_count, const int32_t* __restrict__ permL,
          const int32_t* __restrict__ permR, int self_join, const float* __restrict__ XT,
          int64_t ldt) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const unsigned long long n = min(*n_rec, cap);
    const int lane = threadIdx.x & 31;
    const bool vec8 =
        (d % 8 == 0) && ((reinterpret_cast<uintptr_t>(L) | reinterpret_cast<uintptr_t>(R)) % 32 == 0);
    // k records per warp step: 32, or fewer when the records are too few to
    // give every warp a step of 32, and no more than ~32 candidates per step
    // (n_rec[3] counts them).  Dense records of a sorted small join carry
    // ~30 candidates each: 32 consecutive ones on one warp left most warps
    // idle (config 1 with the band plan's order: re-check 0.124 -> 0.097 ms);
    // sparse buffers -- mostly the zeroed tails of reserved slots -- keep one
    // step per warp, and buffers long enough for >= 4 full steps per warp
    // keep 32.
    const unsigned long long ncand = n_rec[3];
    // blocks that take part: all of them for candidate-heavy buffers, a
    // quarter (one resident wave) when the candidates are few -- a sparse
    // buffer is mostly zeroed slot tails, and the extra blocks' start-up
    // then outweighs their share (r02h: config 1 re-check 0.087 -> 0.082 ms
    // with 16 blocks per SM, configs 2 / 3 0.014 -> 0.011 / 0.025 -> 0.017 ms
    // with 4)
    unsigned active = gridDim.x;
    if (ncand < static_cast<unsigned long long>(gridDim.x) * 256)
        active = max(gridDim.x / 4, static_cast<unsigned>((ncand + 255) / 256));
    if (blockIdx.x >= active) return;
    const unsigned long long warps = static_cast<unsigned long long>(active) * (blockDim.x >> 5);
    unsigned long long kk = min(32ull, (n + warps - 1) / warps);
    if (n < 128 * warps) {  // (long buffers: 32, config 5 re-check 77 vs 102 ms at ~6)
        if (ncand > 32 * n) kk = 1;
        else if (ncand > 0) kk = min(kk, 32 * n / ncand);
    }
    const unsigned k = static_cast<unsigned>(max(1ull, kk));
    const unsigned long long stride = warps * k;
    for (unsigned long long base = (static_cast<unsigned long long>(blockIdx.x) * (blockDim.x >> 5) +
                                    (threadIdx.x >> 5)) * k;
         base < n; base += stride) {
        const unsigned long long idx = base + lane;
        int4 rc = make_int4(0, 0, 0, 0);
        if (static_cast<unsigned>(lane) < k && idx < n) rc = __ldcs(rec + idx);  // (read once: evict first)
        const uint32_t mask = static_cast<uint32_t>(rc.z);
        // banded plans screen row-sorted copies: map back to input rows
        const int my_i = (permL && mask) ? __ldg(permL + rc.x) : rc.x;
        // exclusive prefix of the popcounts over the warp
        const int cnt = __popc(mask);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int excl = incl - cnt;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int c0 = 0; c0 < total; c0 += 32) {
            const int c = c0 + lane;
            // source lane: the last lane whose exclusive prefix is <= c
            int src = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int e = __shfl_sync(0xffffffffu, excl, src + step);
                if (e <= c) src += step;
            }
            const int s_excl = __shfl_sync(0xffffffffu, excl, src);
            const uint32_t s_mask = __shfl_sync(0xffffffffu, mask, src);
            const int s_j0 = __shfl_sync(0xffffffffu, rc.y, src);
            int a = __shfl_sync(0xffffffffu, my_i, src);
            const int a_pos = G == 2 ? __shfl_sync(0xffffffffu, rc.x, src) : 0;
            bool ok = false;
            double dist = 0.0;
            int j = 0;
            if (c < total) {
                const int k = __fns(s_mask, 0, c - s_excl + 1);  // that lane's (c - excl)-th set bit
                j = s_j0 + k;
                const int jp = j;  // column position (sorted under a band plan)
                PDB_DCHECK(k >= 0 && k < 32 && jp >= 0 && jp < ldt);
                if (permR) j = __ldg(permR + j);
                PDB_DCHECK(j >= 0 && j < ldt && a >= 0);
                // euclidean(L_i, R_j); bitwise symmetric, so a self-join pair
                // can be reported as (min, max)
                dist = G == 2 ? exact_dist_grouped2(XT + static_cast<int64_t>(a_pos) * 8,
                                                    XT + static_cast<int64_t>(jp) * 8, ldt * 8, d)
                     : G == 1 ? exact_dist_grouped(L + static_cast<int64_t>(a) * d,
                                                   XT + static_cast<int64_t>(jp) * 8, ldt * 8, d, vec8)
                              : exact_dist(L + static_cast<int64_t>(a) * d, R + static_cast<int64_t>(j) * d, d, vec8);
                ok = dist <= tau;
                if (self_join && a > j) {
                    const int t = a;
                    a = j;
                    j = t;
                }
            }
            const uint32_t ball = __ballot_sync(0xffffffffu, ok);
            if (!ball) continue;
            unsigned long long w = 0;
            if (lane == 0) w = atomicAdd(out_count, static_cast<unsigned long long>(__popc(ball)));
            w = __shfl_sync(0xffffffffu, w, 0);
            if (ok) {
                const unsigned long long pos = w + __popc(ball & ((1u << lane) - 1u));
                if (pos < out_cap) {
                    // streaming stores: the pairs must not evict the rows
                    // the re-check is still reading from L2
                    __stcs(out_l + pos, a);
                    __stcs(out_r + pos, j);
                    __stcs(out_d + pos, static_cast<float>(dist));
                }
            }
        }
    }
}

// K3 for candidate-heavy joins (the grouped copy XT of R; G = 1: L
// row-major with d % 8 == 0 and 32-byte rows, G = 2: self-join, L from XT
// by row position).  Two stages per warp: every candidate of the flattened
// queue (as in k_recheck) first gets the fp32 pre-filter (filter_dist2,
// FMA pipe); the survivors go to a per-warp shared-memory queue, and each
// full batch of 32 survivors runs the reference's fp64 chain, so every
// lane of the exact stage is busy.  The chain's float -> double
// conversions run on the XU pipe at a quarter of the fp64 rate and bounded
// the one-stage kernel (ncu, config 5: XU 75 % busy, 2.85e9 candidates for
// 1.04e9 pairs); the filter skips them for candidates that cannot be
// pairs.  Every emitted pair and distance still comes from the exact chain.
template <int G>
__global__ void __launch_bounds__(256)
k_recheck_filtered(const int4* __restrict__ rec, const unsigned long long* __restrict__ n_rec,
                   unsigned long long cap, const float* __restrict__ L, int d, double tau,
                   float thr, int32_t* __restrict__ out_l, int32_t* __restrict__ out_r,
                   float* __restrict__ out_d, unsigned long long out_cap,
                   unsigned long long* __restrict__ out_count, const int32_t* __restrict__ permL,
                   const int32_t* __restrict__ permR, int self_join, const float* __restrict__ XT,
                   int64_t ldt) {
    static_assert(G == 1 || G == 2, "grouped modes only");
    __shared__ int2 queue[8][64];
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const unsigned long long n = min(*n_rec, cap);
    const int lane = threadIdx.x & 31;
    int2* q = queue[threadIdx.x >> 5];
    int nq = 0;  // warp-uniform
    const int64_t gs = ldt * 8;
    // lanes < m re-check q[lane] exactly and emit the pairs
    auto exact_batch = [&](int m) {
        bool ok = false;
        double dist = 0.0;
        int a = 0, j = 0;
        if (lane < m) {
            const int2 e = q[lane];
            a = permL ? __ldg(permL + e.x) : e.x;
            j = permR ? __ldg(permR + e.y) : e.y;
            PDB_DCHECK(a >= 0 && j >= 0 && j < ldt);
            dist = G == 2 ? exact_dist_grouped2(XT + static_cast<int64_t>(e.x) * 8,
                                                XT + static_cast<int64_t>(e.y) * 8, gs, d)
                          : exact_dist_grouped(L + static_cast<int64_t>(a) * d,
                                               XT + static_cast<int64_t>(e.y) * 8, gs, d, true);
            ok = dist <= tau;
            if (self_join && a > j) {
                const int t = a;
                a = j;
                j = t;
            }
        }
        const uint32_t ball = __ballot_sync(0xffffffffu, ok);
        if (!ball) return;
        unsigned long long w = 0;
        if (lane == 0) w = atomicAdd(out_count, static_cast<unsigned long long>(__popc(ball)));
        w = __shfl_sync(0xffffffffu, w, 0);
        if (ok) {
            const unsigned long long pos = w + __popc(ball & ((1u << lane) - 1u));
            if (pos < out_cap) {
                __stcs(out_l + pos, a);
                __stcs(out_r + pos, j);
                __stcs(out_d + pos, static_cast<float>(dist));
            }
        }
    };
    // k records per warp step: 32, or fewer when the records are too few to
    // give every warp a step of 32, and no more than ~32 candidates per step
    // (n_rec[3] counts them).  Dense records of a sorted small join carry
    // ~30 candidates each: 32 consecutive ones on one warp left most warps
    // idle (config 1 with the band plan's order: re-check 0.124 -> 0.097 ms);
    // sparse buffers -- mostly the zeroed tails of reserved slots -- keep one
    // step per warp, and buffers long enough for >= 4 full steps per warp
    // keep 32.
    const unsigned long long warps = static_cast<unsigned long long>(gridDim.x) * (blockDim.x >> 5);
    const unsigned long long ncand = n_rec[3];
    unsigned long long kk = min(32ull, (n + warps - 1) / warps);
    if (n < 128 * warps) {  // (long buffers: 32, config 5 re-check 77 vs 102 ms at ~6)
        if (ncand > 32 * n) kk = 1;
        else if (ncand > 0) kk = min(kk, 32 * n / ncand);
    }
    const unsigned k = static_cast<unsigned>(max(1ull, kk));
    const unsigned long long stride = warps * k;
    for (unsigned long long base = (static_cast<unsigned long long>(blockIdx.x) * (blockDim.x >> 5) +
                                    (threadIdx.x >> 5)) * k;
         base < n; base += stride) {
        const unsigned long long idx = base + lane;
        int4 rc = make_int4(0, 0, 0, 0);
        if (static_cast<unsigned>(lane) < k && idx < n) rc = __ldcs(rec + idx);  // (read once: evict first)
        const uint32_t mask = static_cast<uint32_t>(rc.z);
        const int cnt = __popc(mask);
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        const int excl = incl - cnt;
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        for (int c0 = 0; c0 < total; c0 += 32) {
            const int c = c0 + lane;
            int src = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const int e = __shfl_sync(0xffffffffu, excl, src + step);
                if (e <= c) src += step;
            }
            const int s_excl = __shfl_sync(0xffffffffu, excl, src);
            const uint32_t s_mask = __shfl_sync(0xffffffffu, mask, src);
            const int s_j0 = __shfl_sync(0xffffffffu, rc.y, src);
            const int pa = __shfl_sync(0xffffffffu, rc.x, src);
            bool pass = false;
            int jp = 0;
            if (c < total) {
                jp = s_j0 + __fns(s_mask, 0, c - s_excl + 1);
                PDB_DCHECK(jp >= 0 && jp < ldt && pa >= 0);
                const float* ap;
                int64_t as;
                if (G == 2) {
                    ap = XT + static_cast<int64_t>(pa) * 8;
                    as = gs;
                } else {
                    ap = L + static_cast<int64_t>(permL ? __ldg(permL + pa) : pa) * d;
                    as = 8;
                }
                pass = filter_dist2(ap, as, XT + static_cast<int64_t>(jp) * 8, gs, d) <= thr;
            }
            const uint32_t ball = __ballot_sync(0xffffffffu, pass);
            if (pass) q[nq + __popc(ball & ((1u << lane) - 1u))] = make_int2(pa, jp);
            nq += __popc(ball);
            __syncwarp();
            if (nq >= 32) {
                exact_batch(32);
                nq -= 32;
                __syncwarp();
                int2 t = make_int2(0, 0);
                if (lane < nq) t = q[32 + lane];
                __syncwarp();
                if (lane < nq) q[lane] = t;
                __syncwarp();
            }
        }
    }
    if (nq > 0) exact_batch(nq);
}

__global__ void k_pack_keys(const int32_t* __restrict__ l, const int32_t* __restrict__ r,
                            int64_t n, unsigned long long* __restrict__ keys) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        keys[k] = (static_cast<unsigned long long>(static_cast<uint32_t>(l[k])) << 32) |
                  static_cast<uint32_t>(r[k]);
}

__global__ void k_unpack_keys(const unsigned long long* __restrict__ keys, int64_t n,
                              int32_t* __restrict__ l, int32_t* __restrict__ r) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        l[k] = static_cast<int32_t>(keys[k] >> 32);
        r[k] = static_cast<int32_t>(keys[k] & 0xffffffffu);
    }
}

// ---------------------------------------------------------------------------
// Cosine join over bf16 rows (BASELINE config 4; restated, not in the
// reference).  Contract: cos = dot / (sqrt(na) * sqrt(nb)) >= min_cos with
// dot, na, nb accumulated sequentially in fp64 over k = 0..d-1 from the
// exact bf16 values (oracle/pdb_oracle.c orc_cosine_join_bf16).

__device__ __forceinline__ float bf16_to_f32(uint16_t b) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

__global__ void k_pad_bf16(const uint16_t* __restrict__ X, int64_t n, int d, int DP,
                           uint16_t* __restrict__ Xp) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (row >= n) return;
    for (int k = lane; k < DP; k += 32) Xp[row * DP + k] = k < d ? X[row * d + k] : 0;
}

// One warp per row.  L mode (h != null): h_i = rd(cmarg * ||x_i||), +inf
// for zero / non-finite rows, -inf when cmarg <= 0.  R mode (g != null,
// rows up to npad): g_j = ru(1 / ||y_j||), 0 for zero / non-finite rows and
// padding.
__global__ void k_prep_cos(const uint16_t* __restrict__ X, int64_t n, int d, double cmarg,
                           float* __restrict__ h, float* __restrict__ g, int64_t npad) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    const int64_t rows = h ? n : npad;
    if (row >= rows) return;
    double acc = 0.0;
    bool finite = true;
    if (row < n) {
        for (int k = lane; k < d; k += 32) {
            const float v = bf16_to_f32(X[row * d + k]);
            if (!isfinite(v)) finite = false;
            acc += static_cast<double>(v) * static_cast<double>(v);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    finite = __all_sync(0xffffffffu, finite);
    if (lane) return;
    const bool valid = row < n && finite && acc > 0.0 && isfinite(acc);
    const float inf = __int_as_float(0x7f800000);
    if (h) {
        if (!valid) h[row] = inf;
        else if (cmarg <= 0.0) h[row] = -inf;
        else h[row] = __double2float_rd(cmarg * sqrt(acc));
    } else {
        g[row] = valid ? __double2float_ru(1.0 / sqrt(acc)) : 0.0f;
    }
}

// Same contract as orc_cosine_join_bf16: dot, |a|^2, |b|^2 accumulated in
// k order in fp64 from the exact bf16 values; rows are read 8 columns per
// 16-byte load, 64 columns per batch of loads.
__device__ __forceinline__ double exact_cos(const uint16_t* __restrict__ a,
                                            const uint16_t* __restrict__ b, int d) {
    double dot = 0.0, na = 0.0, nb = 0.0;
    auto step = [&](uint32_t xa, uint32_t yb) {  // two bf16 columns per word
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const double x = __uint_as_float(h ? (xa & 0xFFFF0000u) : (xa << 16));
            const double y = __uint_as_float(h ? (yb & 0xFFFF0000u) : (yb << 16));
            dot = __dadd_rn(dot, __dmul_rn(x, y));
            na = __dadd_rn(na, __dmul_rn(x, x));
            nb = __dadd_rn(nb, __dmul_rn(y, y));
        }
    };
    int k = 0;
    if (((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0) {
        const uint4* a8 = reinterpret_cast<const uint4*>(a);
        const uint4* b8 = reinterpret_cast<const uint4*>(b);
        for (; k + 64 <= d; k += 64) {
            uint4 x[8], y[8];
#pragma unroll
            for (int q = 0; q < 8; q++) {
                x[q] = __ldg(a8 + k / 8 + q);
                y[q] = __ldg(b8 + k / 8 + q);
            }
#pragma unroll
            for (int q = 0; q < 8; q++) {
                step(x[q].x, y[q].x);
                step(x[q].y, y[q].y);
                step(x[q].z, y[q].z);
                step(x[q].w, y[q].w);
            }
        }
    }
    for (; k < d; k++) {
        const double x = bf16_to_f32(__ldg(a + k)), y = bf16_to_f32(__ldg(b + k));
        dot = __dadd_rn(dot, __dmul_rn(x, y));
        na = __dadd_rn(na, __dmul_rn(x, x));
        nb = __dadd_rn(nb, __dmul_rn(y, y));
    }
    return __ddiv_rn(dot, __dmul_rn(__dsqrt_rn(na), __dsqrt_rn(nb)));
}

__global__ void __launch_bounds__(256)
k_recheck_cos(const int4* __restrict__ rec, const unsigned long long* __restrict__ n_rec,
              unsigned long long cap, const uint16_t* __restrict__ L,
              const uint16_t* __restrict__ R, int d, double min_cos, int32_t* __restrict__ out_l,
              int32_t* __restrict__ out_r, float* __restrict__ out_d, unsigned long long out_cap,
              unsigned long long* __restrict__ out_count) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const unsigned long long n = min(*n_rec, cap);
    const int lane = threadIdx.x & 31;
    const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
    for (unsigned long long base = static_cast<unsigned long long>(blockIdx.x) * blockDim.x +
                                   (threadIdx.x & ~31u);
         base < n; base += stride) {
        const unsigned long long idx = base + lane;
        int4 rc = make_int4(0, 0, 0, 0);
        if (idx < n) rc = rec[idx];
        uint32_t mask = static_cast<uint32_t>(rc.z);
        while (__any_sync(0xffffffffu, mask != 0)) {
            bool ok = false;
            double cs = 0.0;
            int j = 0;
            if (mask) {
                const int k = __ffs(mask) - 1;
                mask &= mask - 1;
                j = rc.y + k;
                cs = exact_cos(L + static_cast<int64_t>(rc.x) * d, R + static_cast<int64_t>(j) * d, d);
                ok = cs >= min_cos;
            }
            const uint32_t ball = __ballot_sync(0xffffffffu, ok);
            if (!ball) continue;
            unsigned long long w = 0;
            if (lane == 0) w = atomicAdd(out_count, static_cast<unsigned long long>(__popc(ball)));
            w = __shfl_sync(0xffffffffu, w, 0);
            if (ok) {
                const unsigned long long pos = w + __popc(ball & ((1u << lane) - 1u));
                if (pos < out_cap) {
                    out_l[pos] = rc.x;
                    out_r[pos] = j;
                    out_d[pos] = static_cast<float>(cs);
                }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Host side.
CUtensorMap make_tmap(const DeviceCtx& ctx, const void* base, int64_t rows, int DP, int box_rows,
                      bool bf16) {
    CUtensorMap m;
    const int es = bf16 ? 2 : 4;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(DP), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(DP) * es};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / es), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ctx.encode_tiled);
    const CUresult r = enc(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                           2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(PDB_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

// The folded-g rows: [n, kGCols] bf16, one 32-byte K=16 slice per row,
// loaded 256 rows at a time in the 32B-swizzled layout of sdesc_k_sw32.
CUtensorMap make_tmap_g(const DeviceCtx& ctx, const void* base, int64_t rows, int box_rows) {
    CUtensorMap m;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(kGCols), static_cast<cuuint64_t>(rows)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(kGCols) * 2};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(kGCols), static_cast<cuuint32_t>(box_rows)};
    const cuuint32_t estr[2] = {1, 1};
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ctx.encode_tiled);
    const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) fail(PDB_ERR_CUDA, "cuTensorMapEncodeTiled (g) failed (" + std::to_string(r) + ")");
    return m;
}

template <int DP, bool A_RES, int STAGES, int MODE>
void launch_screen(const DeviceCtx& ctx, const CUtensorMap& tA, const CUtensorMap& tB,
                   const CUtensorMap& tG, const ScreenParams& p, cudaStream_t s) {
    constexpr size_t smem = ScreenSmem<DP, A_RES, STAGES, MODE>::kBytes;
    static_assert(smem <= 232448, "shared memory budget");
    auto k = k_screen<DP, A_RES, STAGES, MODE>;
    set_max_smem(reinterpret_cast<const void*>(k), static_cast<int>(smem));
    const int64_t grid = std::min<int64_t>(ctx.sm_count, std::max<int64_t>(p.n_units, 1));
    launch_pdl(k, dim3(static_cast<unsigned>(grid)), dim3(Epi<DP>::kThreads), smem, s, tA, tB, tG, p);
    PDB_CUDA(cudaGetLastError());
}

template <int DP>
void launch_screen_pair(const DeviceCtx& ctx, const CUtensorMap& tA, const CUtensorMap& tB,
                        const CUtensorMap& tG, const ScreenParams& p, cudaStream_t s) {
    constexpr size_t smem = PairSmem<DP>::kBytes;
    static_assert(smem <= 232448, "shared memory budget");
    auto k = k_screen_pair<DP>;
    set_max_smem(reinterpret_cast<const void*>(k), static_cast<int>(smem));
    const int64_t clusters = std::min<int64_t>(ctx.sm_count / 2, std::max<int64_t>(p.n_units, 1));
    launch_pdl(k, dim3(static_cast<unsigned>(2 * clusters)), dim3(kThreads), smem, s, tA, tB, tG, p);
    PDB_CUDA(cudaGetLastError());
}

void dispatch_screen(int DP, int mode, const DeviceCtx& ctx, const CUtensorMap& tA,
                     const CUtensorMap& tB, const CUtensorMap& tG, const ScreenParams& p,
                     cudaStream_t s) {
    if (mode == kModeL2Bf16Pair) {
        switch (DP) {
            case 64: launch_screen_pair<64>(ctx, tA, tB, tG, p, s); return;
            case 128: launch_screen_pair<128>(ctx, tA, tB, tG, p, s); return;
        }
        fail(PDB_ERR_CONFIG, "join: unsupported padded dimension for the paired screen");
    }
    if (mode == kModeL2Bf16Aug) {
        switch (DP) {
            case 64: launch_screen<64, true, 4, kModeL2Bf16Aug>(ctx, tA, tB, tG, p, s); return;
            case 128: launch_screen<128, true, 4, kModeL2Bf16Aug>(ctx, tA, tB, tG, p, s); return;
        }
        fail(PDB_ERR_CONFIG, "join: unsupported padded dimension for the folded-g screen");
    }
    if (mode == kModeL2Bf16 || mode == kModeCosBf16) {
#define PDB_BF16_CASES(M)                                                                 \
        switch (DP) {                                                                     \
            case 64: launch_screen<64, true, 5, M>(ctx, tA, tB, tG, p, s); return;        \
            case 128: launch_screen<128, true, 4, M>(ctx, tA, tB, tG, p, s); return;      \
            case 256: launch_screen<256, false, 4, M>(ctx, tA, tB, tG, p, s); return;     \
            case 512: launch_screen<512, false, 4, M>(ctx, tA, tB, tG, p, s); return;     \
            case 1024: launch_screen<1024, false, 4, M>(ctx, tA, tB, tG, p, s); return;   \
            case 2048: launch_screen<2048, false, 4, M>(ctx, tA, tB, tG, p, s); return;   \
            case 4096: launch_screen<4096, false, 4, M>(ctx, tA, tB, tG, p, s); return;   \
        }
        if (mode == kModeL2Bf16) {
            PDB_BF16_CASES(kModeL2Bf16)
        } else {
            PDB_BF16_CASES(kModeCosBf16)
        }
#undef PDB_BF16_CASES
        fail(PDB_ERR_CONFIG, "join: unsupported padded dimension");
    }
    switch (DP) {
        case 32: launch_screen<32, true, 6, kModeL2Tf32>(ctx, tA, tB, tG, p, s); return;
        case 64: launch_screen<64, true, 5, kModeL2Tf32>(ctx, tA, tB, tG, p, s); return;
        case 96: launch_screen<96, true, 4, kModeL2Tf32>(ctx, tA, tB, tG, p, s); return;
        case 128: launch_screen<128, true, 4, kModeL2Tf32>(ctx, tA, tB, tG, p, s); return;
        case 256: launch_screen<256, false, 4, kModeL2Tf32>(ctx, tA, tB, tG, p, s); return;
        case 512: launch_screen<512, false, 4, kModeL2Tf32>(ctx, tA, tB, tG, p, s); return;
        case 1024: launch_screen<1024, false, 4, kModeL2Tf32>(ctx, tA, tB, tG, p, s); return;
        case 2048: launch_screen<2048, false, 4, kModeL2Tf32>(ctx, tA, tB, tG, p, s); return;
    }
    fail(PDB_ERR_CONFIG, "similarity join: unsupported padded dimension");
}

// Resident-A variants for d <= 128; beyond that A streams with B and the
// padded width is the next power of two (zero columns change no dot).
int padded_dim(int d) {
    if (d <= 32) return 32;
    if (d <= 64) return 64;
    if (d <= 96) return 96;
    if (d <= 128) return 128;
    int DP = 256;
    while (DP < d) DP *= 2;
    return DP;
}

// bf16: K-blocks of 64 elements; resident A up to 128, then powers of two.
int padded_dim_bf16(int d) {
    if (d <= 64) return 64;
    if (d <= 128) return 128;
    int DP = 256;
    while (DP < d) DP *= 2;
    return DP;
}

// Optional CUDA-event timing of the phases of one call.
struct PhaseTimer {
    bool on = false;
    cudaStream_t s = nullptr;
    cudaEvent_t* ev = nullptr;
    PhaseTimer(bool enable, cudaStream_t st) : on(enable), s(st) {
        if (!on) return;
        // events are created once per host thread and device, then reused
        thread_local cudaEvent_t cache[64][6];
        thread_local bool made[64] = {};
        int dev = 0;
        PDB_CUDA(cudaGetDevice(&dev));
        if (!made[dev]) {
            for (auto& e : cache[dev]) PDB_CUDA(cudaEventCreate(&e));
            made[dev] = true;
        }
        ev = cache[dev];
    }
    void mark(int k) {
        if (on) PDB_CUDA(cudaEventRecord(ev[k], s));
    }
    float ms(int a, int b) {
        if (!on) return 0.0f;
        // only read after the call's stream synchronisation: both events
        // have completed
        float t = 0.0f;
        PDB_CUDA(cudaEventElapsedTime(&t, ev[a], ev[b]));
        return t;
    }
};

// Work units (column chunk c, row block rb), chunk-major, for this shard.
struct UnitPlan {
    int64_t* off = nullptr;  // device [n_chunks + 1], caller-provided (<= nt + 1 entries)
    int ch = 1, nt = 0, n_chunks = 0;
    int rpt = 2;             // row blocks per column tile (2: 128-row blocks, 1: pairs)
    int64_t n_rb = 0;
    int64_t n_units = 0;
};

// pair: units over 256-row block pairs (k_screen_pair; one shard only).
void plan_units(const DeviceCtx& ctx, int64_t nL, int64_t nR, bool self, int P, int shard,
                bool pair, UnitPlan& u) {
    u.nt = static_cast<int>(ceil_div(nR, BN));
    u.rpt = pair ? 1 : 2;
    u.n_rb = ceil_div(nL, pair ? 2 * BM : BM);
    const int64_t n_rb = u.n_rb;
    double total_tiles = 0;
    for (int64_t rb = 0; rb < n_rb; rb++)
        total_tiles += self ? static_cast<double>(u.nt - (pair ? rb : rb >> 1)) : static_cast<double>(u.nt);
    if (pair) total_tiles *= 2;  // 128x256 tiles
    total_tiles /= P;
    static const double div = [] {
        const char* e = getenv("PDB_UNIT_DIV");
        return e ? atof(e) : 16.0;
    }();
    u.ch = static_cast<int>(std::clamp<double>(total_tiles / (div * ctx.sm_count), 1.0, 64.0));
    u.n_chunks = static_cast<int>(ceil_div(u.nt, u.ch));
    // the same unit count k_chunk_plan scans on the device
    int64_t n_units = 0;
    for (int c = 0; c < u.n_chunks; c++) {
        int64_t lim = n_rb;  // row blocks rb < lim are valid in chunk c
        if (self) lim = std::min<int64_t>(n_rb, u.rpt * (static_cast<int64_t>(c) + 1) * u.ch);
        const int64_t full = lim / P, rem = lim % P;
        const int64_t pos_last = (full & 1) ? P - 1 - shard : shard;
        n_units += full + (pos_last < rem ? 1 : 0);
    }
    u.n_units = n_units;
}

// A per-thread mapped pinned slot of 8 words: [0, 4) the counter read-back,
// [4] the band plan's unit count.  Null when mapped memory is unavailable.
struct PinSlot {
    unsigned long long* h = nullptr;
    unsigned long long* d = nullptr;
};
PinSlot pinned_slot() {
    thread_local unsigned long long* h_pin = [] {
        void* q = nullptr;
        if (cudaHostAlloc(&q, 64, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            cudaGetLastError();
            q = nullptr;
        }
        return static_cast<unsigned long long*>(q);
    }();
    PinSlot r;
    if (h_pin && cudaHostGetDevicePointer(reinterpret_cast<void**>(&r.d), h_pin, 0) == cudaSuccess)
        r.h = h_pin;
    else
        cudaGetLastError(), r.d = nullptr;
    return r;
}

// Second stream of the band plan (per thread and device): the box / count /
// scan chain runs on it beside the bf16 preparation, and its scan's unit
// count reaches the host while the main stream still writes the tile lists.
struct PlanAux {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, scan = nullptr, kfork = nullptr, kjoin = nullptr;
};
// (PDB_PLAN_AUX=0: one PDL-chained stream)
bool use_plan_aux() {
    static const bool on = [] {
        const char* e = std::getenv("PDB_PLAN_AUX");
        return !(e && e[0] == '0');
    }();
    return on;
}

PlanAux* plan_aux() {
    thread_local PlanAux cache[64];
    thread_local bool made[64] = {};
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    PlanAux& a = cache[dev & 63];
    if (!made[dev & 63]) {
        if (cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.scan, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.kfork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&a.kjoin, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        made[dev & 63] = true;
    }
    return &a;
}

// Where the host can read a band plan's unit count early (null ev: read
// p.dev_n_units on the main stream).
struct UnitsReady {
    cudaEvent_t ev = nullptr;
    const unsigned long long* h = nullptr;
};
constexpr unsigned long long kUnitsUnset = ~0ull;

// Candidate records live in a per-thread, per-device buffer that only grows
// (plain cudaMalloc: usable from any stream): a multi-GB record buffer is
// mapped once, not on every call.  Freed at thread exit or by
// pdb_release_caches().
struct RecCache {
    int4* p = nullptr;
    unsigned long long cap = 0;
    void release() {
        if (p) cudaFree(p);  // (errors ignored: may run during process teardown)
        p = nullptr;
        cap = 0;
    }
};
struct RecCaches {
    RecCache c[64];
    ~RecCaches() {
        for (auto& r : c) r.release();
    }
};
RecCaches& rec_caches() {
    thread_local RecCaches caches;
    return caches;
}

// PDB_K3_GROUPED, read on every call: 0 never re-check from the grouped copy
// of R, 1 (default) when the sampled output is candidate-heavy, 2 always.
int grouped_mode() {
    const char* e = std::getenv("PDB_K3_GROUPED");
    if (!e || !e[0]) return 1;
    return std::clamp(atoi(e), 0, 2);
}

// PDB_SCREEN_FP16, read on every call: fp16 screen copies for band-plan
// joins (fp16_scale) 0 never, 1 (default) when the sampled screen shows a
// candidate-heavy output, 2 always.  (Measured: fp16 MMAs ran the screen
// 2-5 % slower than bf16 on configs 3 and 5, so joins whose candidates are
// already ~ their pairs keep bf16.)
int screen_fp16_mode() {
    const char* e = std::getenv("PDB_SCREEN_FP16");
    if (!e || !e[0]) return 1;
    return std::clamp(atoi(e), 0, 2);
}

// Threshold of K3's fp32 pre-filter (filter_dist2): a reference pair has
// exact squared distance S <= tau^2 (1 + 1e-9) (the fp64 chain errs far
// below that), and the filter's sum is at most S (1 + 2^-24)^(d + 2) +
// d 2^-149; the float threshold is rounded up.  +inf (no filtering) when
// that bound is not far below FLT_MAX, or with PDB_K3_FILTER=0 (read on
// every call).
float recheck_filter_threshold(double tau, int d) {
    const char* e = std::getenv("PDB_K3_FILTER");
    if (e && e[0] && atoi(e) == 0) return INFINITY;
    const double t2 = tau * tau * (1.0 + 1e-9) * (1.0 + (d + 3) * std::ldexp(1.0, -24) * 1.01) +
                      d * std::ldexp(1.0, -149);
    if (!(t2 < 1e37)) return INFINITY;
    float f = static_cast<float>(t2);
    if (static_cast<double>(f) < t2) f = std::nextafter(f, INFINITY);
    return f;
}

// The shared back half of both joins: screen (with a sampled output-size
// estimate for large problems), exact re-check, one counter read-back,
// overflow handling, optional sort, stats.  `recheck(recs, cap, out)`
// enqueues the mode's re-check kernel.
template <class Recheck, class OnHeavy>
void screen_and_recheck(const DeviceCtx& ctx, cudaStream_t s, int DP, int mode,
                        const CUtensorMap& tA, const CUtensorMap& tB, const CUtensorMap& tG,
                        ScreenParams p,
                        int64_t nL, int64_t nR, const pdb_join_opts& o, pdb_dev_pairs* out,
                        pdb_join_stats* stats, PhaseTimer& tm, int launches,
                        unsigned long long* counters_p, UnitsReady ready, Recheck&& recheck,
                        OnHeavy&& on_heavy) {
    struct {
        unsigned long long* p;
    } counters{counters_p};  // [records, tiles, pairs, candidates, next unit]
    unsigned long long cap = static_cast<unsigned long long>(
        std::max<int64_t>(1 << 21, 4 * (nL + nR)));  // candidate records
    unsigned long long out_need = static_cast<unsigned long long>(
        std::max<int64_t>(1 << 20, 4 * (nL + nR)));
    // pinned per-thread read-back slot (a pageable destination would add a
    // staging copy to the one synchronisation of the call)
    // (mapped: a one-warp kernel stores the counters straight into it, no
    // copy-engine round trip)
    const PinSlot pin = pinned_slot();
    unsigned long long* h_pin = pin.h;
    unsigned long long* d_pin = pin.d;
    unsigned long long h_cnt[4] = {0, 0, 0, 0};
    int dev_id = 0;
    PDB_CUDA(cudaGetDevice(&dev_id));
    RecCache& rcache = rec_caches().c[dev_id & 63];
    struct {
        int4* p = nullptr;
    } recs;
    auto recs_reset = [&](unsigned long long need) {
        if (rcache.cap < need) {
            PDB_CUDA(cudaStreamSynchronize(s));
            if (rcache.p) PDB_CUDA(cudaFree(rcache.p));
            rcache.p = nullptr;
            rcache.cap = 0;
            // a quarter of headroom: the sampled estimate wobbles between
            // calls, and each growth re-maps a multi-GB buffer
            void* q = nullptr;
            unsigned long long got = need + need / 4;
            if (cudaMalloc(&q, static_cast<size_t>(got) * sizeof(int4)) != cudaSuccess) {
                cudaGetLastError();
                got = need;
                if (cudaMalloc(&q, static_cast<size_t>(got) * sizeof(int4)) != cudaSuccess) {
                    cudaGetLastError();
                    fail(PDB_ERR_OUT_OF_MEMORY, "cannot allocate the candidate record buffer");
                }
            }
            rcache.p = static_cast<int4*>(q);
            rcache.cap = got;
        }
        recs.p = rcache.p;
    };
    int passes = 0;
    auto ensure_out = [&](unsigned long long need) {
        if (static_cast<unsigned long long>(out->capacity) >= need && out->left) return;
        if (out->left) pdb_dev_pairs_free(out);
        // headroom for large outputs, as for the records (the pool keeps
        // the blocks, so only growth maps new memory)
        const int64_t c = static_cast<int64_t>(need > (1ull << 24) ? need + need / 4 : need);
        out->left = static_cast<int32_t*>(dev_alloc(c * sizeof(int32_t), s));
        out->right = static_cast<int32_t*>(dev_alloc(c * sizeof(int32_t), s));
        out->dist = static_cast<float*>(dev_alloc(c * sizeof(float), s));
        out->capacity = c;
    };
    auto read_counters = [&] {
        if (d_pin) {
            launch_pdl(k_export_counters, dim3(1), dim3(32), 0, s,
                       static_cast<const unsigned long long*>(counters.p), d_pin);
            PDB_CUDA(cudaGetLastError());
            PDB_CUDA(cudaStreamSynchronize(s));
            std::copy(h_pin, h_pin + 4, h_cnt);
        } else {
            PDB_CUDA(cudaMemcpyAsync(h_cnt, counters.p, 4 * sizeof(unsigned long long),
                                     cudaMemcpyDeviceToHost, s));
            PDB_CUDA(cudaStreamSynchronize(s));
        }
    };
    bool zeroed = true;  // k_chunk_plan zeroed the counters
    auto arm = [&] {
        p.rec = recs.p;
        p.cap = cap;
        p.counter = counters.p;
        p.tiles = counters.p + 1;
        p.ncand = counters.p + 3;
        p.next_unit = counters.p + 4;
        if (!zeroed) PDB_CUDA(cudaMemsetAsync(counters.p, 0, 5 * sizeof(unsigned long long), s));
        zeroed = false;
    };
    p.unit_step = 1;
    // Large problems: screen every 64th work unit first and size the record
    // and output buffers from that sample, so a heavy output (config 5:
    // ~1.4e9 candidates) does not cost a second full screen pass.
    constexpr int64_t kSampleStep = 64;
    int64_t units = p.n_units;  // dense estimate; a band plan's real count is on the device
    if (p.tile_list && units >= kSampleStep * ctx.sm_count) {
        const volatile unsigned long long* hv = ready.h;
        if (hv && ready.ev) {
            PDB_CUDA(cudaEventSynchronize(ready.ev));
        } else if (hv) {
            // spin on the mapped slot: the host learns the count as soon as
            // k_band_scan stores it, while the stream still writes the tile lists
            while (*hv == kUnitsUnset) {
                const cudaError_t q = cudaStreamQuery(s);
                if (q == cudaErrorNotReady) continue;
                PDB_CUDA(q);
                break;
            }
        }
        if (hv && *hv != kUnitsUnset) {
            units = static_cast<int64_t>(*hv);
        } else {
            PDB_CUDA(cudaMemcpyAsync(&units, p.dev_n_units, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            PDB_CUDA(cudaStreamSynchronize(s));
        }
    }
    // Short joins chain the re-check to the screen with programmatic
    // dependent launch; for long ones (config 5: 0.16 s screen) the early-
    // resident re-check CTAs measured ~20 % slower than a plain launch.
    const bool small = units < kSampleStep * ctx.sm_count;
    if (!small) {
        recs_reset(cap);
        arm();
        p.unit_step = kSampleStep;
        dispatch_screen(DP, mode, ctx, tA, tB, tG, p, s);
        launches++;
        read_counters();
        p.unit_step = 1;
        // Generous margins: the per-unit output of clustered data is heavily
        // skewed, so the 1/64 sample is a noisy estimate, and a miss costs a
        // second full screen (records) or re-check (pairs).
        // Sizes snap to a 2^(1/4) grid so that repeated calls with slightly
        // different estimates reuse the stream-ordered pool's blocks instead
        // of mapping new multi-GB ones.
        auto snap = [](double x) {
            double v = 1 << 20;
            while (v < x) v *= 1.189207115002721;  // 2^(1/4)
            return static_cast<unsigned long long>(v);
        };
        // (records: 3x the sample -- at 2x a 262k-row config-5 join still
        // overflowed once its clusters fell between the sampled units, and
        // a miss costs a whole second screen; 16 B per record)
        cap = std::max(cap, snap(h_cnt[0] * kSampleStep * 3.0));
        out_need = std::max(out_need, snap(h_cnt[3] * kSampleStep * 1.5));
    }
    // Re-check over a grouped copy of R when the sampled output is
    // candidate-heavy: >= 4 candidates per column row (config 5).  Sparse
    // records (config 1) gain nothing from it.  PDB_K3_GROUPED: see
    // grouped_mode().  The recheck callback may still fall back to the
    // row-major gather when the copy cannot be allocated.
    const bool heavy = !small && h_cnt[3] * kSampleStep >= 4ull * static_cast<unsigned long long>(nR);
    const int gmode = grouped_mode();
    bool grouped = gmode == 2 || (gmode == 1 && heavy);
    // a candidate-heavy join may re-make its screen copies in a finer format
    // (L2: fp16, see fp16_scale); the callback returns the format's switch
    if (heavy) {
        if (const unsigned* f = on_heavy()) p.f16xmax = f;
    }
    // Test hooks: PDB_TEST_REC_CAP / PDB_TEST_OUT_CAP cap the first pass's
    // record and pair buffers, forcing the overflow paths below.
    if (const char* e = std::getenv("PDB_TEST_REC_CAP"))
        cap = std::max<unsigned long long>(1, std::strtoull(e, nullptr, 10));
    if (const char* e = std::getenv("PDB_TEST_OUT_CAP"))
        out_need = std::max<unsigned long long>(1, std::strtoull(e, nullptr, 10));
    // (the sampled pass, when taken, counts as preparation in the phase times)
    tm.mark(1);
    // Screen and re-check run back to back and the host reads the counters
    // once.  A record overflow re-runs the screen with the exact record
    // count; an output overflow re-runs only the re-check.
    bool switched = false;
    for (int attempt = 0; attempt < 3; attempt++) {
        recs_reset(cap);
        ensure_out(out_need);
        arm();
        if (p.n_units > 0) {
            dispatch_screen(DP, mode, ctx, tA, tB, tG, p, s);
            launches++;
        }
        tm.mark(2);
        recheck(recs.p, counters.p, cap, out, small, grouped);
        launches++;
        tm.mark(3);
        passes++;
        read_counters();
        if (h_cnt[0] <= cap) break;
        cap = h_cnt[0] + h_cnt[0] / 8 + 1024;
        out_need = std::max(out_need, h_cnt[3]);
        // a short join (no sampled pass) that turns out candidate-heavy: the
        // re-screen runs on the finer copies (their records are fewer; a
        // third pass, with the exact count, covers the rare exception)
        if (small && !switched && h_cnt[3] >= 4ull * static_cast<unsigned long long>(nR)) {
            switched = true;
            if (const unsigned* f = on_heavy()) p.f16xmax = f;
        }
    }
    if (h_cnt[2] > static_cast<unsigned long long>(out->capacity)) {
        ensure_out(h_cnt[2]);
        PDB_CUDA(cudaMemsetAsync(counters.p + 2, 0, sizeof(unsigned long long), s));
        recheck(recs.p, counters.p, cap, out, small, grouped);
        launches++;
        tm.mark(3);
        read_counters();
    }
    const unsigned long long n_cand = h_cnt[3];
    const unsigned long long n_pairs = h_cnt[2];
    out->count = static_cast<int64_t>(n_pairs);

    if ((o.flags & PDB_JOIN_SORTED) && n_pairs > 1) {
        const int64_t n = static_cast<int64_t>(n_pairs);
        DevBuf<unsigned long long> k_in(n, s), k_out(n, s);
        DevBuf<float> v_out(n, s);
        k_pack_keys<<<592, 256, 0, s>>>(out->left, out->right, n, k_in.p);
        size_t tmp_bytes = 0;
        PDB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, k_in.p, k_out.p, out->dist,
                                                 v_out.p, n, 0, 64, s));
        DevBuf<uint8_t> tmp(tmp_bytes, s);
        PDB_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, k_in.p, k_out.p, out->dist,
                                                 v_out.p, n, 0, 64, s));
        k_unpack_keys<<<592, 256, 0, s>>>(k_out.p, n, out->left, out->right);
        PDB_CUDA(cudaMemcpyAsync(out->dist, v_out.p, n * sizeof(float), cudaMemcpyDeviceToDevice, s));
        PDB_CUDA(cudaGetLastError());
        launches += 4;  // pack, 2 cub passes (upper bound), unpack
    }
    tm.mark(4);
    if (stats) {
        stats->candidates = static_cast<int64_t>(n_cand);
        stats->pairs = static_cast<int64_t>(n_pairs);
        stats->tiles = static_cast<int64_t>(h_cnt[1]);
        stats->candidate_capacity = static_cast<int64_t>(cap) * 32;
        stats->launches = launches;
        stats->screen_passes = passes;
        stats->prep_ms = tm.ms(0, 1);
        stats->screen_ms = tm.ms(1, 2);
        stats->recheck_ms = tm.ms(2, 3);
        if (tm.on && (o.flags & PDB_JOIN_SORTED)) PDB_CUDA(cudaEventSynchronize(tm.ev[4]));
        stats->sort_ms = (o.flags & PDB_JOIN_SORTED) ? tm.ms(3, 4) : 0.0f;
        stats->screen_format = mode == kModeCosBf16 ? 3 : mode == kModeL2Tf32 ? 0 : (p.f16xmax ? 2 : 1);
        stats->reserved1 = 0;
    }
}

}  // namespace

void release_join_caches() {
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    PDB_CUDA(cudaDeviceSynchronize());
    rec_caches().c[dev & 63].release();
}

void run_sim_join_dev(const float* d_L, int64_t nL, const float* d_R, int64_t nR, int32_t d,
                      double tau, const pdb_join_opts& o, pdb_dev_pairs* out,
                      pdb_join_stats* stats, const JoinPre* pre) {
    const DeviceCtx& ctx = device_ctx();
    cudaStream_t s = static_cast<cudaStream_t>(o.stream);
    const bool self = (o.flags & PDB_JOIN_SELF) != 0;
    if (self) {
        d_R = d_L;
        nR = nL;
    }
    const int P = o.shard_count > 1 ? o.shard_count : 1;
    const int shard = o.shard_count > 1 ? o.shard_index : 0;
    if (stats) *stats = pdb_join_stats{};
    out->count = 0;
    // (a NaN tau, which the reference accepts, matches nothing: every
    // `euclidean <= tau` is false)
    if (nL == 0 || nR == 0 || tau != tau) return;
    PhaseTimer tm(stats != nullptr && (o.flags & PDB_JOIN_PHASE_TIMES) != 0, s);
    int launches = 0;
    tm.mark(0);

    // bf16 screen copies by default (twice the MMA rate of tf32 on this
    // SMEM-operand-bound screen); PDB_JOIN_TF32 asks for the tighter tf32 band.
    // For DP <= 128 the -||y||^2/2 term is folded into the accumulator by one
    // extra MMA (the screen is epilogue-bound there); PDB_NO_FOLD=1 disables.
    const bool tf32 = (o.flags & PDB_JOIN_TF32) != 0;
    const int DP = tf32 ? padded_dim(d) : padded_dim_bf16(d);
    static const bool no_fold = [] {
        const char* e = getenv("PDB_NO_FOLD");
        return e && e[0] == '1';
    }();
    const bool fold = !tf32 && DP <= 128 && !no_fold;
    const int mode = tf32 ? kModeL2Tf32 : (fold ? kModeL2Bf16Aug : kModeL2Bf16);
    if (DP > (tf32 ? 2048 : 4096))
        fail(PDB_ERR_CONFIG, "similarity join: d is larger than this build supports");
    const size_t es = tf32 ? 4 : 2;

    // CTA pairs for the folded-g screen (opt-in, PDB_SCREEN_PAIR=1, one GPU):
    // measured no faster than the 1-SM screen -- both run the tensor pipe at
    // ~62-64 % active, ~0.9 of the measured cuBLAS bf16 rate for the MMA
    // work they issue -- so the 1-SM kernel stays the default.
    const char* pe = getenv("PDB_SCREEN_PAIR");
    const bool pair = fold && P == 1 && pe && pe[0] == '1';
    // The band plan (exact tile pruning, see k_pca_partial) for resident-A
    // L2 joins of at least kBandMinRows rows per side; PDB_JOIN_DENSE or
    // PDB_JOIN_BAND=0 turn it off, PDB_JOIN_BAND=1 forces it.
    const char* be = getenv("PDB_JOIN_BAND");
    const int band_env = be ? atoi(be) : -1;
    bool band = !pair && DP <= 128 && d <= kPcaMaxD && (o.flags & PDB_JOIN_DENSE) == 0 &&
                band_env != 0 && (band_env == 1 || (nL >= kBandMinRows && nR >= kBandMinRows));

    // ---- scratch: one pool allocation for every small buffer ---------------
    const int64_t nt_ = ceil_div(nR, BN);
    const int64_t nbl = ceil_div(nL, BM);
    int n_slots = 0;
    int64_t list_cap = 0;
    size_t sort_tmp = 0;
    const int E = d + d * d + 1;
    const char* bd = getenv("PDB_BAND_DIV");
    const int units_target = (bd ? std::max(1, atoi(bd)) : 8) * ctx.sm_count;
    int64_t units_cap = 0;
    if (band) {
        const int64_t full = nbl / P, rem = nbl % P;
        const int64_t pos_last = (full & 1) ? P - 1 - shard : shard;
        n_slots = static_cast<int>(full + (pos_last < rem ? 1 : 0));
        for (int k = 0; k < n_slots; k++) {
            const int64_t rb = static_cast<int64_t>(k) * P + ((k & 1) ? P - 1 - shard : shard);
            list_cap += nt_ - (self ? rb >> 1 : 0);
        }
        // units <= total / ch + n_slots with ch = clamp(total / units_target, 1, 64)
        units_cap = 2 * static_cast<int64_t>(units_target) + list_cap / 64 + n_slots + 1;
        // too little screen to save (sharded joins also pay the stable sort)
        if (band_env != 1 && list_cap < (P > 1 ? kBandMinTilesSharded : kBandMinTiles)) band = false;
        // tile-list positions travel as int32 (unit_info, Unit): beyond 2^31
        // dense tiles per shard (> ~11.8 M rows self-joined on one GPU) the
        // join keeps the dense plan
        if (list_cap >= (int64_t{1} << 31)) band = false;
    }
    if (band) {
        sort_tmp = static_cast<size_t>(2 * kBins * 4);  // bin counts and fill cursors
        if (P > 1) {
            // ranks (n) + per-block bin counts / offsets of the stable sort
            const int64_t nmax = std::max(nL, nR);
            sort_tmp += Arena::need(nmax, 4) + Arena::need(ceil_div(nmax, kRankRows) * kBins, 4) + 512;
        }
    }
    const size_t band_bytes =
        !band ? 0
              : Arena::need(static_cast<size_t>(kPcaBlocks) * E, 4) + Arena::need(E, 8) +
                    Arena::need(1, sizeof(BandInfo)) +
                    Arena::need(nL, 16) + 4 * Arena::need(nL, 4) + Arena::need(sort_tmp, 1) +
                    (self ? 0 : Arena::need(nR, 16) + 4 * Arena::need(nR, 4) + Arena::need(sort_tmp, 1)) +
                    Arena::need(nbl, 32) + Arena::need(nt_, 32) + Arena::need(ceil_div(nt_, 32), 32) +
                    Arena::need(n_slots, 4) + 2 * Arena::need(n_slots + 1, 8) + Arena::need(2, 8) +
                    Arena::need(std::max<int64_t>(list_cap, 1), 4) + 2 * Arena::need(n_slots, 4) +
                    Arena::need(units_cap, 16) + Arena::need(nL, 4);
    Arena ar;
    ar.reserve(Arena::need(DP, 4) + Arena::need(static_cast<size_t>(nL) * DP, es) +
                   2 * Arena::need(nL, 4) +
                   (self ? 0 : Arena::need(static_cast<size_t>(nR) * DP, es) + 2 * Arena::need(nR, 4)) +
                   Arena::need(static_cast<size_t>(nt_) * BN, 4) + 4 * Arena::need(nt_ + 1, 4) +
                   Arena::need(nt_ + 2, 8) + Arena::need(5, 8) +
                   (fold ? Arena::need(static_cast<size_t>(nR) * kGCols, 2) : 0) + band_bytes,
               s);
    float* mu = ar.take<float>(DP);
    // a precomputed centre and directions (run_featurize_join_dev): the join's
    // first kernels (tile-statistic zeroing, bin zeroing) start right after
    // K1, and the stream waits for the PCA only before the first kernel that
    // reads them
    bool pre_waited = false;
    auto wait_pre = [&]() -> bool {
        if (!pre || pre_waited) return false;
        pre_waited = true;
        if (pre->ready) PDB_CUDA(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(pre->ready), 0));
        return pre->ready != nullptr;
    };
    if (pre) mu = const_cast<float*>(pre->mu);
    uint16_t* gx = fold ? ar.take<uint16_t>(static_cast<size_t>(nR) * kGCols) : nullptr;
    // R tile statistics: written by k_prep (DP <= 128, zeroed by k_col_mean)
    // or k_tile_stats (wider rows)
    const int nt_tiles = static_cast<int>(nt_);
    float* gR = ar.take<float>(static_cast<size_t>(nt_) * BN);
    float* tmaxS = ar.take<float>(nt_);
    float* tmaxN = ar.take<float>(nt_);
    const bool fused_stats = DP <= 128;

    // ---- preparation ----------------------------------------------------
    launch_pdl(k_col_mean, dim3(static_cast<unsigned>(ceil_div(DP, 32))), dim3(32, 32), 0, s, d_L,
               nL, d, DP, pre ? static_cast<float*>(nullptr) : mu, fused_stats ? tmaxS : nullptr,
               fused_stats ? tmaxN : nullptr, nt_tiles, gR, nR, static_cast<const float*>(nullptr));
    PDB_CUDA(cudaGetLastError());
    launches++;
    auto prep = [&](const float* X, int64_t n, uint8_t* Xp, float* hn, float* sn, uint16_t* g_out,
                    const int32_t* perm, const unsigned* f16x, bool r_side, cudaStream_t sp = nullptr,
                    bool pdl = true) {
        if (!sp) sp = s;
        if (DP <= 128) {  // g_out (the folded block) only exists for DP <= 128
            const unsigned g = static_cast<unsigned>(ceil_div(ceil_div(n, kRowsPerWarp) * 32, 256));
            auto pick = [&](auto k32, auto k64, auto k96, auto k128) {
                const int nv = DP / 32;
                auto k = nv == 1 ? k32 : nv == 2 ? k64 : nv == 3 ? k96 : k128;
                launch_pdl_if(pdl, k, dim3(g), dim3(256), 0, sp, X, n, d, DP, static_cast<const float*>(mu),
                           static_cast<void*>(Xp), hn, sn, g_out, perm, f16x, tau,
                           r_side ? gR : nullptr, r_side ? tmaxS : nullptr, r_side ? tmaxN : nullptr);
            };
            if (tf32) pick(k_prep<false, 1>, k_prep<false, 2>, k_prep<false, 3>, k_prep<false, 4>);
            else pick(k_prep<true, 1>, k_prep<true, 2>, k_prep<true, 3>, k_prep<true, 4>);
        } else {
            const unsigned g = static_cast<unsigned>(ceil_div(n * 32, 256));
            launch_pdl_if(pdl, tf32 ? k_prep_wide<false> : k_prep_wide<true>, dim3(g), dim3(256), 0, sp, X,
                       n, d, DP, static_cast<const float*>(mu), static_cast<void*>(Xp), hn, sn);
        }
        PDB_CUDA(cudaGetLastError());
        launches++;
    };
    // ---- band plan, part 1: directions, sort keys, row permutations ------
    int32_t* permL = nullptr;
    int32_t* permR = nullptr;
    BandInfo* info = nullptr;
    // fp16 screen copies (fp16_scale): band plans with DP <= 128 and bf16
    // copies; PDB_SCREEN_FP16=2 from the start, 1 (default) when the sampled
    // screen shows a candidate-heavy output, 0 never
    const unsigned* f16x = nullptr;  // the copies' switch (nullptr: bf16)
    const unsigned* f16_avail = nullptr;
    float2 *projL = nullptr, *projR = nullptr;
    if (band) {
        float* part = ar.take<float>(static_cast<size_t>(kPcaBlocks) * E);
        double* sum = ar.take<double>(E);
        info = pre && P == 1 ? static_cast<BandInfo*>(const_cast<void*>(pre->info)) : ar.take<BandInfo>(1);
        if (DP <= 128 && !tf32 && screen_fp16_mode() > 0) f16_avail = &info->xmax;
        if (screen_fp16_mode() == 2) f16x = f16_avail;
        uint8_t* tmpL = ar.take<uint8_t>(sort_tmp);
        uint8_t* tmpR = self ? nullptr : ar.take<uint8_t>(sort_tmp);
        if (pre && P == 1) {
            // directions computed ahead on a prefix sample (run_featurize_join_dev):
            // only the counting sorts' bins need zeroing (k_pca_reduce's job)
            k_zero_bins<<<2 * kBins / 256, 256, 0, s>>>(reinterpret_cast<int32_t*>(tmpL),
                                                         reinterpret_cast<int32_t*>(tmpR));
            launches++;
        } else {
            auto kp = d <= 16 ? k_pca_partial<1> : d <= 32 ? k_pca_partial<2> : d <= 64 ? k_pca_partial<4>
                                                                                      : k_pca_partial<8>;
            launch_pdl(kp, dim3(kPcaBlocks), dim3(256), 0, s, d_L, nL, d, static_cast<const float*>(mu),
                       part);
            launch_pdl(k_pca_reduce, dim3(static_cast<unsigned>(ceil_div(E, 128))), dim3(128), 0, s,
                       static_cast<const float*>(part), E, sum, reinterpret_cast<int32_t*>(tmpL),
                       reinterpret_cast<int32_t*>(tmpR), kPcaBlocks);
            const int eig_smem = d * d * 4;
            // (set_max_smem caches per function and device)
            set_max_smem(reinterpret_cast<const void*>(k_pca_eig), kPcaMaxD * kPcaMaxD * 4);
            launch_pdl(k_pca_eig, dim3(1), dim3(256), eig_smem, s, static_cast<const double*>(sum), d,
                       static_cast<const float*>(mu), info);
            launches += 3;
        }
        auto keys_and_sort = [&](const float* X, int64_t n, float2*& proj, int32_t*& perm,
                                 uint8_t* tmp, cudaStream_t ks, bool pdl_first) {
            proj = ar.take<float2>(n);
            uint32_t* k_in = ar.take<uint32_t>(n);
            int32_t* v_in = ar.take<int32_t>(n);
            perm = ar.take<int32_t>(n);
            const int nv = (d + 31) / 32;
            auto kk = nv == 1 ? k_band_keys<1> : nv == 2 ? k_band_keys<2> : nv == 3 ? k_band_keys<3>
                                                                                      : k_band_keys<4>;
            const unsigned gk = static_cast<unsigned>(
                // (8 warps x 4 lane groups x RPG rows per block step)
                std::min<int64_t>(ceil_div(n, d > 64 ? 64 : 128), int64_t{ctx.sm_count} * 16));
            int32_t* count = reinterpret_cast<int32_t*>(tmp);  // bin counts, zeroed by k_pca_reduce
            launch_pdl_if(pdl_first, kk, dim3(gk), dim3(256), 0, ks, X, n, d, static_cast<const float*>(mu),
                          info, proj, k_in, v_in, count);
            if (P > 1) {
                // every rank must build the same order: a deterministic stable
                // counting sort (block-local ranks in row order, per-bin block
                // offsets, scatter) -- the single-GPU scatter below orders
                // rows inside a bin by atomics
                const int64_t nblk = ceil_div(n, kRankRows);
                // (carved from this side's sort scratch, after the bin counts)
                int32_t* rank = reinterpret_cast<int32_t*>(tmp + 2 * kBins * 4 + 256);
                int32_t* bcnt = rank + ((n + 63) / 64) * 64;
                launch_pdl(k_rank_local, dim3(static_cast<unsigned>(nblk)), dim3(1024), 0, ks,
                           static_cast<const uint32_t*>(k_in), n, rank, bcnt);
                launch_pdl(k_rank_offsets, dim3(kBins / 256), dim3(256), 0, ks,
                           static_cast<const int32_t*>(count), bcnt, nblk);
                launch_pdl(k_rank_scatter, dim3(static_cast<unsigned>(nblk)), dim3(1024), 0, ks,
                           static_cast<const uint32_t*>(k_in), n, static_cast<const int32_t*>(rank),
                           static_cast<const int32_t*>(bcnt), perm);
                launches += 4;
            } else {
                // 4 rows per thread, or 1 when that leaves SMs idle (config 2:
                // 16 blocks of 4,096 rows vs 63 of 1,024)
                const int rpt = ceil_div(n, int64_t{1024} * kScatterRows) < ctx.sm_count ? 1 : kScatterRows;
                launch_pdl(rpt == 1 ? k_bin_scatter<1> : k_bin_scatter<kScatterRows>,
                           dim3(static_cast<unsigned>(ceil_div(n, int64_t{1024} * rpt))),
                           dim3(1024), 0, ks, static_cast<const uint32_t*>(k_in), n,
                           static_cast<const int32_t*>(count), count + kBins, perm);
                launches += 2;
            }
        };
        // a cross join's two sides are independent: R's keys and sort run on
        // the aux stream beside L's (each alone keeps HBM ~45 % busy)
        // (after a cross-stream wait on the precomputed directions: no PDL)
        const bool waited = wait_pre();
        PlanAux* kaux = !self && use_plan_aux() ? plan_aux() : nullptr;
        if (kaux) {
            PDB_CUDA(cudaEventRecord(kaux->kfork, s));
            PDB_CUDA(cudaStreamWaitEvent(kaux->s, kaux->kfork, 0));
        }
        keys_and_sort(d_L, nL, projL, permL, tmpL, s, !waited);
        if (self) {
            permR = permL;
            projR = projL;
        } else if (kaux) {
            // (the first kernel after a cross-stream wait launches without PDL)
            keys_and_sort(d_R, nR, projR, permR, tmpR, kaux->s, false);
            PDB_CUDA(cudaEventRecord(kaux->kjoin, kaux->s));
            PDB_CUDA(cudaStreamWaitEvent(s, kaux->kjoin, 0));
        } else {
            keys_and_sort(d_R, nR, projR, permR, tmpR, s, true);
        }
    }

    UnitPlan plan;
    plan.off = ar.take<int64_t>(nt_ + 2);
    plan_units(ctx, nL, nR, self, P, shard, pair, plan);
    const int nt = plan.nt;
    unsigned long long* counters = ar.take<unsigned long long>(5);
    // ---- band plan, part 2: boxes, surviving tiles, units -----------------
    // Boxes, groups, counts and the scan need only the projections and the
    // permutation: they run on the aux stream beside the bf16 preparation.
    int32_t* list = nullptr;
    int4* unit_info = nullptr;
    float* hrow = nullptr;
    int64_t *list_off = nullptr, *unit_off = nullptr, *dev_n_units = nullptr;
    int32_t* dev_ch = nullptr;
    float *cmaxS = nullptr, *cmaxN = nullptr;
    BandPlan bp{};
    UnitsReady ready;
    // (PDB_PLAN_AUX=0: one PDL-chained stream, the host spinning on the
    // mapped unit count instead -- ~2 us slower on config 2)
    PlanAux* aux = band && use_plan_aux() ? plan_aux() : nullptr;
    // The screen copies go to the aux stream (band plans): the tile walk
    // below (boxes, groups, counts, scan) is the longer chain and stays on
    // the PDL-chained main stream, so the cross-stream start-up gap (~6 us)
    // lands off the critical path (config-2 join: see DESIGN.md).
    // (a dense plan with a precomputed centre waits for it here)
    const bool waited_dense = wait_pre();
    cudaStream_t sp = s;
    if (aux) {
        PDB_CUDA(cudaEventRecord(aux->fork, s));
        PDB_CUDA(cudaStreamWaitEvent(aux->s, aux->fork, 0));
        sp = aux->s;
    }
    uint8_t* XpL = ar.take<uint8_t>(static_cast<size_t>(nL) * DP * es);
    float* hnL = ar.take<float>(nL);
    float* snL = ar.take<float>(nL);
    // (the first kernel after a cross-stream wait launches without PDL)
    prep(d_L, nL, XpL, hnL, snL, self ? gx : nullptr, permL, f16x, self, sp, !aux && !waited_dense);
    const uint8_t* XpR = XpL;
    const float *hnR = hnL, *snR = snL;
    if (!self) {
        uint8_t* xr = ar.take<uint8_t>(static_cast<size_t>(nR) * DP * es);
        float* hr = ar.take<float>(nR);
        float* sr = ar.take<float>(nR);
        prep(d_R, nR, xr, hr, sr, gx, permR, f16x, true, sp, true);
        XpR = xr;
        hnR = hr;
        snR = sr;
    }
    if (aux && !fused_stats)
        launch_pdl(k_tile_stats, dim3(nt), dim3(BN), 0, sp, hnR, snR, nR, gR, tmaxS, tmaxN);
    if (aux) PDB_CUDA(cudaEventRecord(aux->join, sp));
    if (band) {
        double4* boxL = ar.take<double4>(nbl);
        double4* boxR = ar.take<double4>(nt);
        int32_t* cnt = ar.take<int32_t>(n_slots);
        list_off = ar.take<int64_t>(n_slots + 1);
        unit_off = ar.take<int64_t>(n_slots + 1);
        dev_n_units = ar.take<int64_t>(1);
        dev_ch = ar.take<int32_t>(1);
        list = ar.take<int32_t>(std::max<int64_t>(list_cap, 1));
        unit_info = ar.take<int4>(units_cap);
        hrow = ar.take<float>(nL);
        cmaxS = ar.take<float>(n_slots);
        cmaxN = ar.take<float>(n_slots);
        double4* sup = ar.take<double4>(ceil_div(int64_t{nt}, 32));
        cudaStream_t sa = s;
        const PinSlot pin = pinned_slot();
        if (pin.h) *reinterpret_cast<volatile unsigned long long*>(pin.h + 4) = kUnitsUnset;
        launch_pdl(k_band_boxes, dim3(static_cast<unsigned>(ceil_div(nbl * 32, 256))),
                      dim3(256), 0, sa, static_cast<const float2*>(projL),
                      static_cast<const int32_t*>(permL), nL, BM, nbl, boxL);
        if (!self)
            launch_pdl(k_band_boxes, dim3(static_cast<unsigned>(ceil_div(int64_t{nt} * 32, 256))),
                       dim3(256), 0, sa, static_cast<const float2*>(projR),
                       static_cast<const int32_t*>(permR), nR, BN, static_cast<int64_t>(nt), boxR);
        bp = BandPlan{boxL, self ? nullptr : boxR, sup, info, tau, d, nt, static_cast<int>(self), P,
                      shard, n_slots, static_cast<int>(nbl)};
        launch_pdl(k_band_groups, dim3(static_cast<unsigned>(ceil_div(ceil_div(int64_t{nt}, 32) * 32, 256))),
                   dim3(256), 0, sa, bp, sup);
        const unsigned gs = static_cast<unsigned>(ceil_div(int64_t{n_slots} * 32, 256));
        if (n_slots > 0) launch_pdl(k_band_count, dim3(gs), dim3(256), 0, sa, bp, cnt);
        launch_pdl(k_band_scan, dim3(1), dim3(1024), 0, sa, static_cast<const int32_t*>(cnt), n_slots,
                   units_target, list_off, unit_off, dev_n_units, dev_ch, counters,
                   pin.d ? pin.d + 4 : nullptr);
        launches += 4 + (self ? 0 : 1);
        if (aux) PDB_CUDA(cudaEventRecord(aux->scan, sa));
        if (pin.h) ready = UnitsReady{aux ? aux->scan : nullptr, pin.h + 4};
    }

    // tile statistics (wide rows; k_prep wrote them otherwise) and (band
    // plan) each slot's tiles, maxima and row thresholds; re-run when the
    // copies are re-made in fp16
    auto tile_write = [&](bool first) {
        if (!fused_stats && !(first && aux))
            launch_pdl(k_tile_stats, dim3(nt), dim3(BN), 0, s, hnR, snR, nR, gR, tmaxS, tmaxN);
        if (first && aux) PDB_CUDA(cudaStreamWaitEvent(s, aux->join, 0));
        if (band && n_slots > 0)
            launch_pdl_if(!(first && aux), k_band_write, dim3(static_cast<unsigned>(ceil_div(int64_t{n_slots} * 32, 256))),
                          dim3(256), 0, s, bp,
                          static_cast<const int64_t*>(list_off), list, static_cast<const float*>(tmaxS),
                          static_cast<const float*>(tmaxN), cmaxS, cmaxN,
                          static_cast<const int64_t*>(unit_off), static_cast<const int32_t*>(dev_ch),
                          unit_info, static_cast<const float*>(hnL), static_cast<const float*>(snL), nL,
                          tau * (1.0 + 1e-9), 1.0,
                          (DP + (fold ? 64 : 0)) * std::ldexp(1.0, -23) + std::ldexp(1.0, -19), hrow,
                          f16x);
        launches += (fused_stats ? 0 : 1) + (band && n_slots > 0 ? 1 : 0);
    };
    // (the copies on the aux stream are joined above; a dense plan has no aux)
    tile_write(true);
    if (!band) {
        cmaxS = ar.take<float>(nt + 1);
        cmaxN = ar.take<float>(nt + 1);
        launch_pdl(k_chunk_plan, dim3(1), dim3(1024), 0, s, static_cast<const float*>(tmaxS),
                   static_cast<const float*>(tmaxN), nt, plan.ch, plan.n_chunks, plan.n_rb, plan.rpt,
                   static_cast<int>(self), P, shard, cmaxS, cmaxN, plan.off, counters);
        launches++;
    }
    PDB_CUDA(cudaGetLastError());
    launches++;
    uint8_t* XpR_w = self ? XpL : const_cast<uint8_t*>(XpR);
    float* hnR_w = const_cast<float*>(hnR);
    float* snR_w = const_cast<float*>(snR);

    const CUtensorMap tA = make_tmap(ctx, XpL, nL, DP, BM, !tf32);
    const CUtensorMap tB = make_tmap(ctx, XpR, nR, DP, pair ? BN / 2 : BN, !tf32);
    const CUtensorMap tG = fold ? make_tmap_g(ctx, gx, nR, pair ? BN / 2 : BN) : tB;
    ScreenParams p{};
    p.nL = nL;
    p.nR = nR;
    p.self_join = self;
    p.shard_index = shard;
    p.shard_count = P;
    p.ch = plan.ch;
    p.nt = nt;
    p.n_chunks = plan.n_chunks;
    p.n_units = plan.n_units;
    p.chunk_off = plan.off;
    p.hnL = hnL;
    p.snL = snL;
    p.gR = gR;
    p.tmaxS = tmaxS;
    p.tmaxN = tmaxN;
    p.cmaxS = cmaxS;
    p.cmaxN = cmaxN;
    p.tau_p = tau * (1.0 + 1e-9);
    p.u = 1.0;  // the error norms are stored directly (err_norm)
    p.gam = (DP + (fold ? 64 : 0)) * std::ldexp(1.0, -23) + std::ldexp(1.0, -19);
    p.f16xmax = f16x;
    p.f16tau = tau;
    p.f16d = d;
    if (band) {
        p.hrow = hrow;
        p.unit_info = unit_info;
        p.tile_list = list;
        p.slot_list_off = list_off;
        p.slot_unit_off = unit_off;
        p.dev_n_units = dev_n_units;
        p.dev_ch = dev_ch;
        p.n_slots = n_slots;
    }
    DevBuf<float> XT;  // grouped copy of R for candidate-heavy re-checks
    bool xt_filled = false;
    // (the pre-filter pays off only against bf16's wide candidate band:
    // config 5 re-check 141 -> 128 ms with bf16 copies, but 78 -> 86 ms
    // with fp16 copies, whose candidates are 1.27x the pairs)
    const float filter_thr_bf16 = recheck_filter_threshold(tau, d);
    screen_and_recheck(ctx, s, DP, pair ? kModeL2Bf16Pair : mode, tA, tB, tG, p, nL, nR, o, out, stats, tm, launches, counters, ready,
                       [&](const int4* recs, unsigned long long* counters,
                           unsigned long long cap, pdb_dev_pairs* o2, bool pdl, bool& grouped) {
                           if (grouped && !XT.p) {
                               // only a speed-up: without room for the copy
                               // the re-check gathers R row-major
                               XT.p = static_cast<float*>(dev_try_alloc(
                                   static_cast<size_t>(nR) * ((d + 7) / 8) * 8 * sizeof(float), s));
                               XT.s = s;
                           }
                           if (grouped && !XT.p) grouped = false;
                           if (grouped && !xt_filled) {
                               xt_filled = true;
                               // (PDL like the re-check: early-resident CTAs slow a long screen)
                               launch_pdl_if(pdl, k_group_copy, dim3(ctx.sm_count * 8), dim3(256), 0, s, d_R,
                                             nR, d, static_cast<const int32_t*>(permR), XT.p);
                               PDB_CUDA(cudaGetLastError());
                           }
                           // (separate instantiations: the grouped path's registers
                           // would otherwise spill in the row-major one)
                           // a self-join reads both sides from the one grouped copy
                           // (rows by position): c5 re-check 145 -> 139 ms
                           const bool both = grouped && self;
                           // the fp32 pre-filter (grouped copies only; L read
                           // 32 bytes at a time in the cross-join variant)
                           const bool vec8L = d % 8 == 0 && reinterpret_cast<uintptr_t>(d_L) % 32 == 0;
                           const float filter_thr = f16x ? INFINITY : filter_thr_bf16;
                           if (grouped && filter_thr < INFINITY && (both || vec8L)) {
                               launch_pdl_if(pdl, both ? k_recheck_filtered<2> : k_recheck_filtered<1>,
                                   dim3(ctx.sm_count * 8), dim3(256), 0, s,
                                   recs, counters, cap, d_L, d, tau, filter_thr, o2->left, o2->right,
                                   o2->dist, static_cast<unsigned long long>(o2->capacity),
                                   counters + 2, static_cast<const int32_t*>(permL),
                                   static_cast<const int32_t*>(permR), static_cast<int>(self),
                                   static_cast<const float*>(XT.p), nR);
                               PDB_CUDA(cudaGetLastError());
                               return;
                           }
                           // (16 blocks per SM; the kernel keeps a quarter of
                           // them when the candidates are few)
                           launch_pdl_if(pdl, both ? k_recheck<2> : grouped ? k_recheck<1> : k_recheck<0>,
                               dim3(ctx.sm_count * 16), dim3(256), 0, s,
                               recs, counters, cap, d_L, d_R, d, tau, o2->left, o2->right,
                               o2->dist, static_cast<unsigned long long>(o2->capacity),
                               counters + 2, static_cast<const int32_t*>(permL),
                               static_cast<const int32_t*>(permR), static_cast<int>(self),
                               static_cast<const float*>(grouped ? XT.p : nullptr), nR);
                           PDB_CUDA(cudaGetLastError());
                       },
                       [&]() -> const unsigned* {
                           // candidate-heavy: re-make the copies in fp16
                           // (the sampled pass screened bf16 copies)
                           if (!f16_avail || f16x) return nullptr;
                           f16x = f16_avail;
                           if (fused_stats) {  // re-zeroed: k_prep max-reduces into them
                               PDB_CUDA(cudaMemsetAsync(tmaxS, 0, nt_ * sizeof(float), s));
                               PDB_CUDA(cudaMemsetAsync(tmaxN, 0, nt_ * sizeof(float), s));
                           }
                           prep(d_L, nL, XpL, hnL, snL, self ? gx : nullptr, permL, f16x, self);
                           if (!self) prep(d_R, nR, XpR_w, hnR_w, snR_w, gx, permR, f16x, true);
                           tile_write(false);
                           return f16x;
                       });
}

void run_cos_join_dev(const uint16_t* d_L, int64_t nL, const uint16_t* d_R, int64_t nR,
                      int32_t d, double min_cos, const pdb_join_opts& o, pdb_dev_pairs* out,
                      pdb_join_stats* stats) {
    const DeviceCtx& ctx = device_ctx();
    cudaStream_t s = static_cast<cudaStream_t>(o.stream);
    const bool self = (o.flags & PDB_JOIN_SELF) != 0;
    if (self) {
        d_R = d_L;
        nR = nL;
    }
    const int P = o.shard_count > 1 ? o.shard_count : 1;
    const int shard = o.shard_count > 1 ? o.shard_index : 0;
    if (stats) *stats = pdb_join_stats{};
    out->count = 0;
    if (nL == 0 || nR == 0) return;
    PhaseTimer tm(stats != nullptr && (o.flags & PDB_JOIN_PHASE_TIMES) != 0, s);
    int launches = 0;
    tm.mark(0);
    const int DP = padded_dim_bf16(d);
    if (DP > 4096) fail(PDB_ERR_CONFIG, "cosine join: d > 4096 is not supported by this build");
    // Screen threshold on the cosine: c' - margin with c' = c - 1e-9 (the
    // fp64 reference's rounding) and margin = DP 2^-23 (fp32 accumulation of
    // exact bf16 products, relative to ||x|| ||y||) + 2^-20 (epilogue
    // roundings).  A threshold at or below 0 makes every pair a candidate.
    const double cmarg = min_cos - 1e-9 - (DP * std::ldexp(1.0, -23) + std::ldexp(1.0, -20));
    // The MMA reads the original rows when they already are a whole number
    // of 64-element K-blocks; otherwise through a zero-padded copy.
    const bool direct = d == DP && reinterpret_cast<uintptr_t>(d_L) % 16 == 0 &&
                        reinterpret_cast<uintptr_t>(d_R) % 16 == 0;
    DevBuf<uint16_t> padL, padR;
    const uint16_t *XL = d_L, *XR = d_R;
    if (!direct) {
        padL.reset(static_cast<size_t>(nL) * DP, s);
        launch_pdl(k_pad_bf16, dim3(static_cast<unsigned>(ceil_div(nL * 32, 256))), dim3(256), 0, s, d_L, nL, d, DP, padL.p);
        launches++;
        XL = padL.p;
        if (!self) {
            padR.reset(static_cast<size_t>(nR) * DP, s);
            launch_pdl(k_pad_bf16, dim3(static_cast<unsigned>(ceil_div(nR * 32, 256))), dim3(256), 0, s, d_R, nR, d, DP, padR.p);
            launches++;
            XR = padR.p;
        } else {
            XR = XL;
        }
        PDB_CUDA(cudaGetLastError());
    }
    const int64_t nt_ = ceil_div(nR, BN);
    Arena ar;
    ar.reserve(Arena::need(nL, 4) + Arena::need(static_cast<size_t>(nt_) * BN, 4) +
                   Arena::need(nt_ + 2, 8) + Arena::need(5, 8),
               s);
    UnitPlan plan;
    plan.off = ar.take<int64_t>(nt_ + 2);
    plan_units(ctx, nL, nR, self, P, shard, false, plan);
    const int nt = plan.nt;
    float* hL = ar.take<float>(nL);
    float* gR = ar.take<float>(static_cast<size_t>(nt) * BN);
    unsigned long long* counters = ar.take<unsigned long long>(5);
    launch_pdl(k_chunk_plan, dim3(1), dim3(1024), 0, s, static_cast<const float*>(nullptr),
               static_cast<const float*>(nullptr), nt, plan.ch, plan.n_chunks, plan.n_rb, plan.rpt,
               static_cast<int>(self), P, shard, static_cast<float*>(nullptr),
               static_cast<float*>(nullptr), plan.off, counters);
    launches++;
    launch_pdl(k_prep_cos, dim3(static_cast<unsigned>(ceil_div(nL * 32, 256))), dim3(256), 0, s, d_L, nL, d, cmarg, hL,
                                                                            nullptr, 0);
    launch_pdl(k_prep_cos, dim3(static_cast<unsigned>(ceil_div(static_cast<int64_t>(nt) * BN * 32, 256))), dim3(256), 0, s, 
        d_R, nR, d, cmarg, nullptr, gR, static_cast<int64_t>(nt) * BN);
    PDB_CUDA(cudaGetLastError());
    launches += 2;
    const CUtensorMap tA = make_tmap(ctx, XL, nL, DP, BM, true);
    const CUtensorMap tB = make_tmap(ctx, XR, nR, DP, BN, true);
    ScreenParams p{};
    p.nL = nL;
    p.nR = nR;
    p.self_join = self;
    p.shard_index = shard;
    p.shard_count = P;
    p.ch = plan.ch;
    p.nt = nt;
    p.n_chunks = plan.n_chunks;
    p.n_units = plan.n_units;
    p.chunk_off = plan.off;
    p.hnL = hL;
    p.gR = gR;
    screen_and_recheck(ctx, s, DP, kModeCosBf16, tA, tB, tB, p, nL, nR, o, out, stats, tm, launches,
                       counters, UnitsReady{},
                       [&](const int4* recs, unsigned long long* counters,
                           unsigned long long cap, pdb_dev_pairs* o2, bool pdl, bool&) {
                           launch_pdl_if(pdl, k_recheck_cos, dim3(ctx.sm_count * 16), dim3(256), 0, s, 
                               recs, counters, cap, d_L, d_R, d, min_cos, o2->left, o2->right,
                               o2->dist, static_cast<unsigned long long>(o2->capacity),
                               counters + 2);
                           PDB_CUDA(cudaGetLastError());
                       },
                       []() -> const unsigned* { return nullptr; });
}


// Spins until the first K1 round has stored its tiles (FeatOuts::done).
// Bounded: a count that never arrives (K1 gone wrong) traps after ~10 s
// instead of hanging the stream.
__global__ void k_wait_count(const unsigned* __restrict__ done, unsigned target) {
    if (threadIdx.x == 0) {
        const long long t0 = clock64();
        unsigned v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
            if (v >= target) break;
            __nanosleep(256);
            if (clock64() - t0 > (1ll << 34)) __trap();
        }
        __threadfence();
    }
    __syncthreads();
}

// Featurize then self-join in one call, with the band plan's centre and
// directions computed while K1 is still running.  K1 (persistent, rows in
// grid-stride order) leaves a few SMs' worth of CTA slots free and counts
// the tiles of its first round as their features are stored; on a
// high-priority stream a one-thread kernel waits for that count, then
// k_col_mean and the PCA (partials over the first round's tiles, reduce,
// eig) run beside the rest of K1, and the join starts from them (JoinPre).
// Any plane prunes correctly, so the prefix sample only changes which tiles
// are screened, never the pairs.  Falls back to featurize + join when the
// join would not use a band plan.
void run_featurize_join_dev(const uint8_t* d_frames, int64_t n, int32_t H, int32_t W, int32_t th,
                            int32_t tw, int32_t bins, int32_t mode, float* d_feats, double tau,
                            const pdb_join_opts& o0, pdb_dev_pairs* out, pdb_join_stats* stats) {
    device_ctx();
    pdb_join_opts o = o0;
    o.flags |= PDB_JOIN_SELF;
    cudaStream_t s = static_cast<cudaStream_t>(o.stream);
    const int64_t tpf = static_cast<int64_t>(W / tw) * (H / th);
    const int64_t nt = n * tpf;
    const int D = hist_dim(bins, mode);
    const bool tf32 = (o.flags & PDB_JOIN_TF32) != 0;
    const int DP = tf32 ? padded_dim(D) : padded_dim_bf16(D);
    const char* be = getenv("PDB_JOIN_BAND");
    const int band_env = be ? atoi(be) : -1;
    const char* pe = getenv("PDB_SCREEN_PAIR");
    const char* fe = getenv("PDB_FUSED_PCA");  // 0: plain featurize + join (A/B)
    const bool band = DP <= 128 && D <= kPcaMaxD && (o.flags & PDB_JOIN_DENSE) == 0 && band_env != 0 &&
                      o.shard_count <= 1 && (band_env == 1 || nt >= kBandMinRows) &&
                      !(pe && pe[0] == '1') && !(fe && fe[0] == '0');
    if (!band || tau != tau || nt == 0) {
        launch_featurize_tiles(d_frames, n, H, W, th, tw, bins, mode, d_feats, s);
        run_sim_join_dev(d_feats, nt, d_feats, nt, D, tau, o, out, stats);
        return;
    }
    struct Aux {
        cudaStream_t s = nullptr;
        cudaEvent_t pre = nullptr, k1 = nullptr, pca = nullptr;
    };
    thread_local Aux auxs[64];
    int dev = 0;
    PDB_CUDA(cudaGetDevice(&dev));
    Aux& a = auxs[dev & 63];
    if (!a.s) {
        int lo = 0, hi = 0;
        PDB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        PDB_CUDA(cudaStreamCreateWithPriority(&a.s, cudaStreamNonBlocking, hi));
        PDB_CUDA(cudaEventCreateWithFlags(&a.pre, cudaEventDisableTiming));
        PDB_CUDA(cudaEventCreateWithFlags(&a.k1, cudaEventDisableTiming));
        PDB_CUDA(cudaEventCreateWithFlags(&a.pca, cudaEventDisableTiming));
    }
    const int E = D + D * D + 1;
    DevBuf<float> mu(static_cast<size_t>(DP), s);
    DevBuf<float> part(static_cast<size_t>(kPcaBlocks) * E, s);
    DevBuf<double> sum(static_cast<size_t>(E), s);
    DevBuf<BandInfo> info(1, s);
    DevBuf<unsigned> done(1, s);
    PDB_CUDA(cudaMemsetAsync(done.p, 0, sizeof(unsigned), s));
    PDB_CUDA(cudaEventRecord(a.pre, s));
    // (SMs' worth of K1 CTA slots left to the PCA: config-2 step 0.350 ms
    // unfused; fused 0.345 / 0.344 / 0.349 ms with 0 / 1 / 2 reserved)
    static const int reserve = [] {
        const char* e = getenv("PDB_FJ_RESERVE");
        return e ? atoi(e) : 1;
    }();
    FeatOuts fo{};
    fo.p[0] = d_feats;
    fo.n = 1;
    fo.done = done.p;
    int64_t first = -1;
    launch_featurize_tiles_multi(d_frames, n, H, W, th, tw, bins, mode, fo, s, reserve, &first);
    int64_t n_rows = first;
    if (first > 0) {  // K1 signals its first round: the PCA starts beside it
        PDB_CUDA(cudaStreamWaitEvent(a.s, a.pre, 0));
        k_wait_count<<<1, 32, 0, a.s>>>(done.p, static_cast<unsigned>(first));
    } else {  // (other K1 variants: after K1, on its whole output)
        PDB_CUDA(cudaEventRecord(a.k1, s));
        PDB_CUDA(cudaStreamWaitEvent(a.s, a.k1, 0));
        n_rows = nt;
    }
    n_rows = std::min<int64_t>(n_rows, nt);
    k_col_mean<<<static_cast<unsigned>(ceil_div(DP, 32)), dim3(32, 8), 0, a.s>>>(
        d_feats, n_rows, D, DP, mu.p, nullptr, nullptr, 0, nullptr, 0, nullptr);
    auto kp = D <= 16 ? k_pca_partial<1> : D <= 32 ? k_pca_partial<2> : D <= 64 ? k_pca_partial<4>
                                                                              : k_pca_partial<8>;
    // (PDB_FJ_PCA_BLOCKS: a smaller sample finishes sooner beside K1 but
    // prunes worse -- 16 blocks: 19,990 tiles vs 19,460 and a 3 us slower
    // step -- so the full 4,096-row sample stays)
    static const int pca_blocks = [] {
        const char* e = getenv("PDB_FJ_PCA_BLOCKS");
        return std::clamp(e ? atoi(e) : kPcaBlocks, 1, kPcaBlocks);
    }();
    launch_pdl(kp, dim3(pca_blocks), dim3(256), 0, a.s, static_cast<const float*>(d_feats), n_rows, D,
               static_cast<const float*>(mu.p), part.p);
    launch_pdl(k_pca_reduce, dim3(static_cast<unsigned>(ceil_div(E, 128))), dim3(128), 0, a.s,
               static_cast<const float*>(part.p), E, sum.p, static_cast<int32_t*>(nullptr),
               static_cast<int32_t*>(nullptr), pca_blocks);
    set_max_smem(reinterpret_cast<const void*>(k_pca_eig), kPcaMaxD * kPcaMaxD * 4);
    launch_pdl(k_pca_eig, dim3(1), dim3(256), D * D * 4, a.s, static_cast<const double*>(sum.p), D,
               static_cast<const float*>(mu.p), info.p);
    PDB_CUDA(cudaGetLastError());
    PDB_CUDA(cudaEventRecord(a.pca, a.s));  // (the join waits for it, JoinPre::ready)
    const JoinPre pre{mu.p, info.p, a.pca};
    run_sim_join_dev(d_feats, nt, d_feats, nt, D, tau, o, out, stats, &pre);
    if (stats) stats->launches += 6;  // K1, the wait, col_mean, the PCA's three
}

}  // namespace pdb
