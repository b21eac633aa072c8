// histogram.cu -- K1: fused generate(tiles) -> color_histogram over uint8
// frames, plus the float-patch apply_transformer path.
//
// Reference semantics (proj/):
//   tile grid, emission order      src/etl.cpp:264-298
//   uint8 -> float crop            src/core.cpp:88-93   (fused away: the
//                                  float value of a byte is exact)
//   binning + normalisation        src/etl.cpp:336-348
// For a byte v and B < 65793, the reference's float expression
// (uint32)(v * B / 256.0f) is exactly (v*B) >> 8: v*B < 2^24 is an exact
// float, /256 is exact and the cast truncates.  Counts are integers; the
// reference accumulates them with `+= 1.0f`, which is exact below 2^24 and
// sticks at 2^24 above it, so count -> min(count, 2^24) reproduces it.  The
// normalisation is one IEEE round-to-nearest float division by
// (float)(h*w), done with __fdiv_rn (the library is built without
// fast-math).
//
// B200 mapping: one warp per tile, 4 tiles per 128-thread CTA.  Frames are
// read with 16-byte non-allocating loads, three per lane per task so each
// lane owns 16 whole RGB pixels (48 B); a 60x80 tile row is 5 such tasks.
// Counts live in shared memory as lane-private columns cnt[bin][lane]
// (bank = lane, so updates never conflict and need no atomics) and are
// reduced with one REDUX per bin at the end of the tile.  Bin counts too
// large for lane-private columns use per-warp shared-memory atomics.

#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>
#include <vector>

#include "pdb_internal.cuh"
#include "tc_ptx.cuh"

namespace pdb {

namespace {

constexpr int kWarpsPerCta = 4;

__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Reference float binning for arbitrary float values / large B.
__device__ __forceinline__ uint32_t bin_float(float v, uint32_t B) {
    float t = __fdiv_rn(__fmul_rn(v, __uint2float_rn(B)), 256.0f);
    uint32_t b = __float2uint_rz(t);  // NaN / negative -> 0, saturates high
    return b >= B ? B - 1 : b;
}

__device__ __forceinline__ float normalise(uint32_t cnt, float npix) {
    float c = cnt >= (1u << 24) ? 16777216.0f : __uint2float_rn(cnt);
    return __fdiv_rn(c, npix);
}

__device__ __forceinline__ uint32_t byte_at(const uint32_t (&w)[12], int k) {
    return (w[k >> 2] >> (8 * (k & 3))) & 0xFFu;
}

// ---------------------------------------------------------------------------
// Lane-private counter kernel: D = number of bins <= NB <= 64.
// BT > 0 fixes B at compile time (B=4 -> shifts), BT == 0 reads it at run time.
template <int NB, bool JOINT, int BT, bool VEC>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
k_hist_tiles_lane(const uint8_t* __restrict__ frames, int64_t n_tiles, int H, int W, int th,
                  int tw, int ntx, int tiles_per_frame, int B_rt, int D, float npix,
                  float* __restrict__ out) {
    extern __shared__ uint32_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + warp;
    if (tile >= n_tiles) return;  // warp-uniform; the CTA never synchronises
    const uint32_t B = BT > 0 ? static_cast<uint32_t>(BT) : static_cast<uint32_t>(B_rt);
    uint32_t* cnt = smem + warp * NB * 32 + lane;

#pragma unroll
    for (int b = 0; b < NB; b++) cnt[b * 32] = 0;

    const int64_t f = tile / tiles_per_frame;
    const int t = static_cast<int>(tile - f * tiles_per_frame);
    const int ty = t / ntx, tx = t - (t / ntx) * ntx;
    const uint8_t* base =
        frames + (static_cast<size_t>(f) * H * W + static_cast<size_t>(ty) * th * W +
                  static_cast<size_t>(tx) * tw) * 3;

    auto count_pixel = [&](uint32_t r, uint32_t g, uint32_t b) {
        const uint32_t br = (r * B) >> 8, bg = (g * B) >> 8, bb = (b * B) >> 8;
        if (JOINT) {
            cnt[((br * B + bg) * B + bb) * 32] += 1;
        } else {
            cnt[br * 32] += 1;
            cnt[(B + bg) * 32] += 1;
            cnt[(2 * B + bb) * 32] += 1;
        }
    };

    if (VEC) {
        // 16-pixel tasks: rows of the tile split in tw/16 segments of 48 B.
        const int segs = tw >> 4;
        const int ntask = th * segs;
        for (int task = lane; task < ntask; task += 32) {
            const int r = task / segs, s = task - r * segs;
            const uint8_t* p = base + (static_cast<size_t>(r) * W + s * 16) * 3;
            const uint4 a = ldg_stream(p), b = ldg_stream(p + 16), c = ldg_stream(p + 32);
            const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
            for (int px = 0; px < 16; px++)
                count_pixel(byte_at(w, 3 * px), byte_at(w, 3 * px + 1), byte_at(w, 3 * px + 2));
        }
    } else {
        const int npx = th * tw;
        for (int i = lane; i < npx; i += 32) {
            const int r = i / tw, x = i - r * tw;
            const uint8_t* p = base + (static_cast<size_t>(r) * W + x) * 3;
            count_pixel(p[0], p[1], p[2]);
        }
    }
    __syncwarp();

    // One REDUX per bin; lane (b % 32) keeps bin b, then coalesced stores.
    uint32_t mine[(NB + 31) / 32];
#pragma unroll
    for (int b = 0; b < NB; b++) {
        if (b < D) {
            const uint32_t tot = __reduce_add_sync(0xffffffffu, cnt[b * 32]);
            if ((b & 31) == lane) mine[b >> 5] = tot;
        }
    }
    float* o = out + tile * D;
#pragma unroll
    for (int j = 0; j < (NB + 31) / 32; j++) {
        const int b = j * 32 + lane;
        if (b < D) o[b] = normalise(mine[j], npix);
    }
}

// ---------------------------------------------------------------------------
// Joint histogram with B = 2^LB (LB = 1, 2 -> 8 or 64 bins): the config-2
// hot kernel, one warp per tile.
//
// Loads: a tile row is rc = 3*tw/16 16-byte chunks; a batch of RB =
// floor(96/rc) rows (6 for 80-px tiles) is fetched with three coalesced
// 16-byte loads per lane (consecutive lanes -> consecutive chunks, so each
// load instruction reads whole 240-byte row segments), staged in a 1.4 KB
// per-warp shared buffer, and re-read as one 48-byte group (16 whole RGB
// pixels) per lane.  The next batch's loads are issued before the current
// batch is binned.  (Measured on B200: letting each lane load its own 48 B
// straight from global capped the kernel at ~2 TB/s even with no counting.)
// Binning is SIMD-within-a-register: four pixels (three words) are
// quantised with one shift+mask per word, regrouped with byte permutes and
// combined into four packed joint indices with two multiply-adds.
// Counts live in lane-private shared words cnt[bin][lane] (CW = 32) or in
// 16-bit halves cnt[bin/2][lane] (CW = 16); bank = lane, so updates never
// conflict.  They are bumped with a plain read-modify-write: on B200 shared
// atomics (red.shared) measured ~2 lanes/clk/SM here and match.any warp
// aggregation was slower still.  CW = 16 requires fewer than 65536 pixels
// per lane per tile.
template <int LB, int WPC, int DEPTH, int CW>
__global__ void __launch_bounds__(WPC * 32)
k_hist_joint_pow2(const uint8_t* __restrict__ frames, int64_t n_tiles, int H, int W, int th,
                  int tw, int ntx, int tiles_per_frame, float npix, float* __restrict__ out) {
    constexpr int NB = 1 << (3 * LB);
    constexpr int NW = CW == 16 ? NB / 2 : NB;       // counter words per lane
    constexpr int kStageBytes = 96 * 16;             // 32 lanes x 3 chunks
    constexpr uint32_t kMask = ((1u << LB) - 1u) * 0x01010101u;
    extern __shared__ __align__(16) uint32_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile = static_cast<int64_t>(blockIdx.x) * WPC + warp;
    if (tile >= n_tiles) return;
    uint32_t* cnt = smem + warp * (NW * 32 + kStageBytes / 4) + lane;
    uint8_t* stage = reinterpret_cast<uint8_t*>(smem + warp * (NW * 32 + kStageBytes / 4) + NW * 32);
#pragma unroll
    for (int b = 0; b < NW; b++) cnt[b * 32] = 0;

    const int64_t f = tile / tiles_per_frame;
    const int t = static_cast<int>(tile - f * tiles_per_frame);
    const int ty = t / ntx, tx = t - (t / ntx) * ntx;
    const uint8_t* base =
        frames + (static_cast<size_t>(f) * H * W + static_cast<size_t>(ty) * th * W +
                  static_cast<size_t>(tx) * tw) * 3;
    const uint32_t row_bytes = static_cast<uint32_t>(W) * 3;
    const int segs = tw >> 4;          // 48-byte groups per tile row
    const int rc = 3 * segs;           // 16-byte chunks per tile row
    const int RB = 96 / rc;            // rows per batch
    const int nb = (th + RB - 1) / RB;
    // this lane's three chunks of a batch: chunk c = 32*j + lane
    uint32_t goff[3];
#pragma unroll
    for (int j = 0; j < 3; j++) {
        const int c = 32 * j + lane;
        goff[j] = static_cast<uint32_t>(c / rc) * row_bytes + static_cast<uint32_t>(c % rc) * 16u;
    }
    auto load = [&](int bt, uint4 (&v)[3]) {
        const int nrows = min(RB, th - bt * RB);
        const uint8_t* p = base + static_cast<size_t>(bt) * RB * row_bytes;
#pragma unroll
        for (int j = 0; j < 3; j++)
            if (32 * j + lane < nrows * rc) v[j] = ldg_stream(p + goff[j]);
    };
    uint4 cur[3], nxt[3];
    load(0, cur);
    if (DEPTH > 1 && nb > 1) load(1, nxt);
    for (int bt = 0; bt < nb; bt++) {
        const int ngroups = min(RB, th - bt * RB) * segs;
#pragma unroll
        for (int j = 0; j < 3; j++)
            reinterpret_cast<uint4*>(stage)[32 * j + lane] = cur[j];
        __syncwarp();
        uint4 a = make_uint4(0, 0, 0, 0), b = a, c = a;
        if (lane < ngroups) {
            const uint4* g = reinterpret_cast<const uint4*>(stage + lane * 48);
            a = g[0];
            b = g[1];
            c = g[2];
        }
        __syncwarp();
        if (DEPTH > 1) {
#pragma unroll
            for (int j = 0; j < 3; j++) cur[j] = nxt[j];
            if (bt + 2 < nb) load(bt + 2, nxt);
        } else if (bt + 1 < nb) {
            load(bt + 1, cur);
        }
        if (lane < ngroups) {
            const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
#pragma unroll
            for (int g = 0; g < 4; g++) {
                // q0 = [r0 g0 b0 r1], q1 = [g1 b1 r2 g2], q2 = [b2 r3 g3 b3] (byte 0 first)
                const uint32_t q0 = (w[3 * g] >> (8 - LB)) & kMask;
                const uint32_t q1 = (w[3 * g + 1] >> (8 - LB)) & kMask;
                const uint32_t q2 = (w[3 * g + 2] >> (8 - LB)) & kMask;
                const uint32_t R = __byte_perm(__byte_perm(q0, q1, 0x0630), q2, 0x5210);
                const uint32_t G = __byte_perm(__byte_perm(q0, q1, 0x0741), q2, 0x6210);
                const uint32_t Bv = __byte_perm(__byte_perm(q0, q1, 0x0052), q2, 0x7410);
                const uint32_t idx4 = R * (1u << (2 * LB)) + G * (1u << LB) + Bv;  // no carries
                if (CW == 32) {
#pragma unroll
                    for (int k = 0; k < 4; k++) cnt[__byte_perm(idx4, 0, 0x4440 | k) * 32] += 1u;
                } else {
                    const uint32_t word4 = (idx4 >> 1) & 0x7F7F7F7Fu;  // bin / 2
                    const uint32_t bit4 = idx4 & 0x01010101u;          // which half
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        cnt[__byte_perm(word4, 0, 0x4440 | k) * 32] +=
                            __byte_perm(bit4, 0, 0x4440 | k) * 0xFFFFu + 1u;
                }
            }
        }
    }
    __syncwarp();
    uint32_t mine[(NB + 31) / 32];
#pragma unroll
    for (int wd = 0; wd < NW; wd++) {
        const uint32_t v = cnt[wd * 32];
        if (CW == 32) {
            const uint32_t tot = __reduce_add_sync(0xffffffffu, v);
            if ((wd & 31) == lane) mine[wd >> 5] = tot;
        } else {
            const uint32_t lo = __reduce_add_sync(0xffffffffu, v & 0xFFFFu);
            const uint32_t hi = __reduce_add_sync(0xffffffffu, v >> 16);
            if (((2 * wd) & 31) == lane) mine[(2 * wd) >> 5] = lo;
            if (((2 * wd + 1) & 31) == lane) mine[(2 * wd + 1) >> 5] = hi;
        }
    }
    float* o = out + tile * NB;
#pragma unroll
    for (int j = 0; j < (NB + 31) / 32; j++) {
        const int bb = j * 32 + lane;
        if (bb < NB) o[bb] = normalise(mine[j], npix);
    }
}

// ---------------------------------------------------------------------------
// Same TMA ring as k_hist_joint_rows, with 8-bit lane-private counters so
// that 3-5 CTAs (24-40 counting warps) fit per SM and the load -> add ->
// store chains of the counting warps hide each other's shared-memory
// latency (the 32-bit version measured 27 % warp occupancy, latency-bound),
// and with the per-pixel arithmetic cut to two instructions (the 32-bit
// version was bound by the integer ALU pipe: ~126 ALU ops per 16 pixels).
//
// Pixel -> counter address: mask every byte to its top LB bits (the
// reference bin of byte v is v >> (8-LB), src/etl.cpp:343-344), so a word
// holding a pixel's R, G, B in bytes 0-2 is r<<(8-LB) | g<<(16-LB) |
// b<<(24-LB) | junk<<(32-LB).  One multiply-high by a 3-term constant
// gathers r, g, b into an 11-bit offset (an exhaustive search over all
// (r, g, b, junk) picked the constant; tests re-check the map is a
// bijection onto distinct counters), whose bits 2-6 are zero so the lane
// (bits 2-6) is OR-ed in: offset = (umulhi(p, M) & Q) | 4*lane | warp base.
// A counter is the byte at `offset`: bank = lane, so updates never
// conflict, and a warp needs 2 KB (B = 4).  Pixels 1-3 of each 12-byte
// group are aligned into a word with funnel shifts.
//
// A lane counts at most nb*16 <= 255 pixels per tile (checked by the
// launcher), so bytes never overflow; they are zeroed per tile and summed
// over lanes two bytes at a time in 16-bit halves with REDUX.
template <int LB>
struct PixMap;
template <>
struct PixMap<2> {  // 64 bins, offsets <= 1923
    static constexpr uint32_t kM = (1u << 16) | (1u << 20) | (1u << 26);
    static constexpr uint32_t kQ = 0x783u;
    static constexpr int kWords = 16;
};
template <>
struct PixMap<1> {  // 8 bins, offsets <= 259
    static constexpr uint32_t kM = (1u << 10) | (1u << 11) | (1u << 25);
    static constexpr uint32_t kQ = 0x183u;
    static constexpr int kWords = 3;
};

template <int LB>
__device__ __forceinline__ uint32_t pix_offset(uint32_t p) {
    return __umulhi(p, PixMap<LB>::kM) & PixMap<LB>::kQ;
}

template <int LB, int G, bool BULK>
__global__ void __launch_bounds__(17 * 32, 1)
k_hist_joint_rows8(const __grid_constant__ CUtensorMap tmap, const uint8_t* __restrict__ frames,
                   int n_rows, int nty, int H, int W3, int th, int tw, int ntx,
                   uint32_t stage_bytes, int S, int pf, int skip_epi, float npix,
                   const __grid_constant__ FeatOuts outs) {
    constexpr int NB = 1 << (3 * LB);
    constexpr int B = 1 << LB;
    constexpr int NWD = PixMap<LB>::kWords;        // counter words per lane
    constexpr uint32_t kTop = (((1u << LB) - 1u) << (8 - LB)) * 0x01010101u;
    extern __shared__ __align__(1024) uint8_t smem_r8[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // counter blocks: 2 KB-aligned shared-window address per warp
    const uint32_t s0 = ptx::smem_u32(smem_r8);
    const uint32_t cpad = (2048u - (s0 & 2047u)) & 2047u;
    uint8_t* stages = smem_r8 + cpad + ntx * 2048;  // 128-B aligned TMA destinations
    uint64_t* full = reinterpret_cast<uint64_t*>(stages + S * stage_bytes);
    uint64_t* empty = full + S;
    // per-warp park area for the epilogue's lane sums (32 words)
    uint32_t* park = reinterpret_cast<uint32_t*>(empty + S) + warp * 32;
    const int segs = tw >> 4;
    const int RB = 96 / (3 * segs);
    const int nb = (th + RB - 1) / RB;
    const int tile_bytes = RB * 3 * tw;

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; s++) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], ntx);
        }
        ptx::fence_mbar_init();
    }
    __syncthreads();

    if (warp == ntx) {  // producer
        if (lane == 0) {
            ptx::tma_prefetch_desc(&tmap);
            uint32_t it = 0;
            // L2 prefetch cursor, pf bands ahead of the loads: the bands in
            // flight to L2 need no shared memory, so the CTA keeps far more
            // bytes in flight than its S stages hold
            int p_tr = blockIdx.x, p_bt = 0;
            auto prefetch_next = [&] {
                if (p_tr >= n_rows) return;
                const int pf_f = p_tr / nty, pf_ty = p_tr - pf_f * nty;
                const int rows = min(RB, th - p_bt * RB);
                ptx::bulk_prefetch_l2(frames + (static_cast<size_t>(pf_f) * H + pf_ty * th + p_bt * RB) * W3,
                                      static_cast<uint32_t>(rows) * W3);
                if (++p_bt == nb) {
                    p_bt = 0;
                    p_tr += gridDim.x;
                }
            };
            for (int k = 0; k < pf; k++) prefetch_next();
            for (int tr = blockIdx.x; tr < n_rows; tr += gridDim.x) {
                const int f = tr / nty, ty = tr - f * nty;
                const int row0 = f * H + ty * th;
                for (int bt = 0; bt < nb; bt++, it++) {
                    if (pf > 0) prefetch_next();
                    const uint32_t s = it % S;
                    if (it >= static_cast<uint32_t>(S)) ptx::mbar_wait_sleep(&empty[s], ((it / S) - 1) & 1);
                    if (BULK) {
                        // RB whole frame rows are one contiguous run of bytes
                        const int rows = min(RB, th - bt * RB);
                        const uint32_t bytes = static_cast<uint32_t>(rows) * W3;
                        ptx::mbar_arrive_expect_tx(&full[s], bytes);
                        ptx::bulk_load(stages + s * stage_bytes,
                                       frames + (static_cast<size_t>(row0) + bt * RB) * W3, bytes,
                                       &full[s]);
                    } else {
                        ptx::mbar_arrive_expect_tx(&full[s], stage_bytes);
                        ptx::tma_load_3d(stages + s * stage_bytes, &tmap, &full[s], 0, row0 + bt * RB, 0);
                    }
                }
            }
        }
        return;
    }

    uint8_t* wcnt = smem_r8 + cpad + warp * 2048;
    uint32_t* wcnt32 = reinterpret_cast<uint32_t*>(wcnt);
    const uint32_t lbase = s0 + cpad + warp * 2048 + lane * 4;  // bits 0-1, 7-10 clear
    // where the counters of this lane's output bins (lane, lane + 32) live
    auto bin_word = [&](int bin) {
        const uint32_t r = bin / (B * B), g = (bin / B) % B, b = bin % B;
        return pix_offset<LB>((r << (8 - LB)) | (g << (16 - LB)) | (b << (24 - LB)));
    };
    const uint32_t o0 = bin_word(lane & (NB - 1)), o1 = bin_word((lane + 32) & (NB - 1));
    // stage ring position, carried across tile rows (the producer's order);
    // the full-band and last-band group counts are fixed per launch
    uint32_t s = 0, ph = 0;
    const int ng_full = RB * segs, ng_last = (th - (nb - 1) * RB) * segs;
    // a stage is tile-major (3-D tensor box) or RB whole frame rows (bulk)
    const uint8_t* my_stage = BULK ? stages + (lane / segs) * W3 + warp * 3 * tw + (lane % segs) * 48
                                   : stages + warp * tile_bytes + lane * 48;
    for (int tr = blockIdx.x; tr < n_rows; tr += gridDim.x) {
        // zero the warp's counters with 16-byte stores (any lane may clear
        // any word: the block belongs to the warp)
#pragma unroll
        for (int k = lane; k < NWD * 8; k += 32) reinterpret_cast<uint4*>(wcnt32)[k] = make_uint4(0, 0, 0, 0);
        __syncwarp();
        for (int bt = 0; bt < nb; bt++) {
            ptx::mbar_wait_sleep(&full[s], ph);
            const int ngroups = bt == nb - 1 ? ng_last : ng_full;
            uint32_t w[12];
            if (lane < ngroups) {
                const uint4* g = reinterpret_cast<const uint4*>(my_stage + s * stage_bytes);
                const uint4 a = g[0], b = g[1], c = g[2];
                w[0] = a.x & kTop;
                w[1] = a.y & kTop;
                w[2] = a.z & kTop;
                w[3] = a.w & kTop;
                w[4] = b.x & kTop;
                w[5] = b.y & kTop;
                w[6] = b.z & kTop;
                w[7] = b.w & kTop;
                w[8] = c.x & kTop;
                w[9] = c.y & kTop;
                w[10] = c.z & kTop;
                w[11] = c.w & kTop;
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&empty[s]);
            if (++s == static_cast<uint32_t>(S)) {
                s = 0;
                ph ^= 1;
            }
            if (lane < ngroups) {
                uint32_t ad[16];
#pragma unroll
                for (int g = 0; g < 4; g++) {
                    // pixels 4g..4g+3: [r0 g0 b0 r1][g1 b1 r2 g2][b2 r3 g3 b3]
                    const uint32_t w0 = w[3 * g], w1 = w[3 * g + 1], w2 = w[3 * g + 2];
                    ad[4 * g] = pix_offset<LB>(w0) | lbase;
                    ad[4 * g + 1] = pix_offset<LB>(__funnelshift_r(w0, w1, 24)) | lbase;
                    ad[4 * g + 2] = pix_offset<LB>(__funnelshift_r(w1, w2, 16)) | lbase;
                    ad[4 * g + 3] = pix_offset<LB>(w2 >> 8) | lbase;
                }
#ifdef PDB_CHECKED
                // every counter address inside this warp's 2 KB block and
                // this lane's byte column; the stage read inside the ring
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const uint32_t rel = ad[k] - (s0 + cpad + warp * 2048u);
                    PDB_DCHECK(rel < 2048u && ((rel >> 2) & 31u) == static_cast<uint32_t>(lane));
                }
                PDB_DCHECK(my_stage + s * stage_bytes + 48 <= stages + S * stage_bytes);
#endif
                if (G == 0) {
                    // (measurement only: the pipeline without the counting)
                    uint32_t x = 0;
#pragma unroll
                    for (int k = 0; k < 16; k++) x ^= ad[k];
                    if (x == 0xFFFFFFFFu) asm volatile("st.shared.u8 [%0], %1;" ::"r"(lbase), "r"(x) : "memory");
                } else if (G == 1) {
                    // one dependent read-modify-write per pixel
#pragma unroll
                    for (int k = 0; k < 16; k++) {
                        uint32_t v;
                        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(ad[k]) : "memory");
                        asm volatile("st.shared.u8 [%0], %1;" ::"r"(ad[k]), "r"(v + 1u) : "memory");
                    }
                } else {
                    // G pixels at a time: equal counters are merged in
                    // registers (the first occurrence carries the group's
                    // count), so the G reads are independent and issue back
                    // to back -- one shared-memory latency per G pixels
                    // instead of per pixel -- and merged pixels cost no
                    // access at all.
#pragma unroll
                    for (int k0 = 0; k0 < 16; k0 += G) {
                        constexpr int GG = G > 0 ? G : 1;
                        uint32_t keep[GG], inc[GG], v[GG];
#pragma unroll
                        for (int a = 0; a < G; a++) {
                            keep[a] = 1u;
                            inc[a] = 1u;
                        }
#pragma unroll
                        for (int a = 0; a < G; a++)
#pragma unroll
                            for (int b = a + 1; b < G; b++) {
                                const uint32_t e = ad[k0 + a] == ad[k0 + b];
                                inc[a] += e & keep[a];  // counted once, at its first occurrence
                                keep[b] &= e ^ 1u;
                            }
#pragma unroll
                        for (int a = 0; a < G; a++) {
                            v[a] = 0u;
                            asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0;\n\t"
                                         "@p ld.shared.u8 %0, [%1]; }"
                                         : "+r"(v[a]) : "r"(ad[k0 + a]), "r"(keep[a]) : "memory");
                        }
#pragma unroll
                        for (int a = 0; a < G; a++)
                            asm volatile("{ .reg .pred p; setp.ne.u32 p, %2, 0;\n\t"
                                         "@p st.shared.u8 [%0], %1; }"
                                         ::"r"(ad[k0 + a]), "r"(v[a] + inc[a]), "r"(keep[a])
                                         : "memory");
                    }
                }
            }
        }
        __syncwarp();
        // (measurement only: 1 skips the epilogue, 2 skips the lane reduction,
        // 3 skips the feature stores)
        if (skip_epi == 1) {
            if (outs.done && tr == static_cast<int>(blockIdx.x) && lane == 0) atomicAdd(outs.done, 1u);
            continue;
        }
        // sum bytes 0,2 and 1,3 of every counter word over lanes in 16-bit
        // halves; lane l keeps the totals of bins l and l+32.
        // Lane 0 parks the two half-sums of word wd in the warp's park area
        // (words 2wd, 2wd+1), then each lane fetches its two bins.  (Parking
        // inside the counter block chained every word's read behind the
        // previous store.)  Measured alternatives, all slower on config 2: a
        // compare-select pick of the warp-uniform sums (serial on the REDUX
        // results, +30 us), and a shuffle reduce-scatter (register pressure
        // costs the counting loop more than it saves).
#pragma unroll
        for (int w0 = 0; w0 < (skip_epi == 2 ? 0 : NWD); w0 += 4) {
            uint32_t cw[4];
#pragma unroll
            for (int k = 0; k < 4; k++) cw[k] = w0 + k < NWD ? wcnt32[(w0 + k) * 32 + lane] : 0u;
#pragma unroll
            for (int k = 0; k < 4; k++) {
                if (w0 + k >= NWD) break;
                const uint32_t s02 = __reduce_add_sync(0xffffffffu, cw[k] & 0x00FF00FFu);
                const uint32_t s13 = __reduce_add_sync(0xffffffffu, (cw[k] >> 8) & 0x00FF00FFu);
                if (lane == 0) {
                    park[2 * (w0 + k)] = s02;
                    park[2 * (w0 + k) + 1] = s13;
                }
            }
        }
        __syncwarp();
        auto fetch = [&](uint32_t o) {
            const uint32_t v2 = park[2 * (o >> 7) + (o & 1)];
            return (o & 2) ? v2 >> 16 : v2 & 0xFFFFu;
        };
        const uint32_t mine0 = fetch(o0), mine1 = NB > 32 ? fetch(o1) : 0u;
        __syncwarp();
        const int f = tr / nty, ty = tr - f * nty;
        const int64_t ofs = ((static_cast<int64_t>(f) * nty + ty) * ntx + warp) * NB;
        PDB_DCHECK(mine0 <= static_cast<uint32_t>(th * tw) && mine1 <= static_cast<uint32_t>(th * tw));
        PDB_DCHECK(ofs + NB <= static_cast<int64_t>(n_rows) * ntx * NB);
        const float v0 = normalise(mine0, npix), v1 = normalise(mine1, npix);
        // every output: the local features and, for a sharded step, each
        // peer's copy over NVLink (P2P stores overlapping the counting)
        // (outs is a __grid_constant__ parameter: the pointers are read from
        // the constant bank, not from a local-memory copy of the struct)
        for (int k = 0; k < (skip_epi == 3 ? 0 : outs.n); k++) {
            float* o = outs.p[k] + ofs;
            if (lane < NB) __stcs(o + lane, v0);
            if (NB > 32) __stcs(o + lane + 32, v1);
        }
        if (outs.done && tr == static_cast<int>(blockIdx.x)) {
            // this tile's features are stored: publish (a consumer on another
            // stream spins on the count, then reads the first round's tiles)
            __threadfence();
            __syncwarp();
            if (lane == 0) atomicAdd(outs.done, 1u);
        }
    }
    // peer stores become visible before anything the host orders after us
    if (outs.n > 1) __threadfence_system();
}

// ---------------------------------------------------------------------------
// Per-warp shared-memory atomic counters for larger bin counts.
// JOINT: B^3 <= 4096 bins.  Per-channel: raw byte-value counts [3][256],
// mapped to bins at the end (bin(v) is monotone in v), which handles any B.
template <bool JOINT>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
k_hist_tiles_atomic(const uint8_t* __restrict__ frames, int64_t n_tiles, int H, int W, int th,
                    int tw, int ntx, int tiles_per_frame, int B_rt, int64_t D, int slots,
                    float npix, float* __restrict__ out) {
    extern __shared__ uint32_t smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t tile = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + warp;
    if (tile >= n_tiles) return;
    const uint32_t B = static_cast<uint32_t>(B_rt);
    uint32_t* cnt = smem + static_cast<size_t>(warp) * slots;
    for (int k = lane; k < slots; k += 32) cnt[k] = 0;
    __syncwarp();

    const int64_t f = tile / tiles_per_frame;
    const int t = static_cast<int>(tile - f * tiles_per_frame);
    const int ty = t / ntx, tx = t - (t / ntx) * ntx;
    const uint8_t* base =
        frames + (static_cast<size_t>(f) * H * W + static_cast<size_t>(ty) * th * W +
                  static_cast<size_t>(tx) * tw) * 3;
    const int npx = th * tw;
    for (int i = lane; i < npx; i += 32) {
        const int r = i / tw, x = i - r * tw;
        const uint8_t* p = base + (static_cast<size_t>(r) * W + x) * 3;
        const uint32_t cr = p[0], cg = p[1], cb = p[2];
        if (JOINT) {
            const uint32_t idx = (((cr * B) >> 8) * B + ((cg * B) >> 8)) * B + ((cb * B) >> 8);
            atomicAdd(&cnt[idx], 1u);
        } else {
            atomicAdd(&cnt[cr], 1u);
            atomicAdd(&cnt[256 + cg], 1u);
            atomicAdd(&cnt[512 + cb], 1u);
        }
    }
    __syncwarp();
    float* o = out + tile * D;
    if (JOINT) {
        for (int k = lane; k < D; k += 32) o[k] = normalise(cnt[k], npix);
        return;
    }
    for (int64_t k = lane; k < D; k += 32) o[k] = 0.0f;
    __syncwarp();
    for (int c = 0; c < 3; c++) {
        const uint32_t* cc = cnt + 256 * c;
        for (int v = lane; v < 256; v += 32) {
            const uint32_t bv = bin_float(static_cast<float>(v), B);
            if (v > 0 && bin_float(static_cast<float>(v - 1), B) == bv) continue;
            uint32_t sum = 0;
            for (int u = v; u < 256 && bin_float(static_cast<float>(u), B) == bv; u++) sum += cc[u];
            o[static_cast<int64_t>(c) * B + bv] = normalise(sum, npix);
        }
    }
}

// ---------------------------------------------------------------------------
// apply_transformer over float pixel patches [n, h, w, 3]: one CTA per
// patch, shared-memory atomic counters (D <= kF32SmemBins) or global u32
// counters for very large D.
constexpr int kF32SmemBins = 12288;

__device__ __forceinline__ uint32_t f32_slot(const float* p, uint32_t B, bool joint, int c) {
    if (joint)
        return (bin_float(p[0], B) * B + bin_float(p[1], B)) * B + bin_float(p[2], B);
    return static_cast<uint32_t>(c) * B + bin_float(p[c], B);
}

__global__ void __launch_bounds__(256)
k_hist_f32_smem(const float* __restrict__ px, int64_t n, int64_t npx, int B_rt, int joint,
                int D, float npix, float* __restrict__ out) {
    extern __shared__ uint32_t smem[];
    const int64_t patch = blockIdx.x;
    const uint32_t B = static_cast<uint32_t>(B_rt);
    for (int k = threadIdx.x; k < D; k += blockDim.x) smem[k] = 0;
    __syncthreads();
    const float* base = px + patch * npx * 3;
    for (int64_t i = threadIdx.x; i < npx; i += blockDim.x) {
        const float* p = base + i * 3;
        if (joint) {
            atomicAdd(&smem[f32_slot(p, B, true, 0)], 1u);
        } else {
            for (int c = 0; c < 3; c++) atomicAdd(&smem[f32_slot(p, B, false, c)], 1u);
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < D; k += blockDim.x)
        out[patch * D + k] = normalise(smem[k], npix);
}

__global__ void k_hist_f32_global(const float* __restrict__ px, int64_t n, int64_t npx,
                                  int B_rt, int joint, int64_t D, uint32_t* __restrict__ cnt) {
    const int64_t patch = blockIdx.y;
    const uint32_t B = static_cast<uint32_t>(B_rt);
    const float* base = px + patch * npx * 3;
    uint32_t* cc = cnt + patch * D;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < npx;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const float* p = base + i * 3;
        if (joint) {
            atomicAdd(&cc[f32_slot(p, B, true, 0)], 1u);
        } else {
            for (int c = 0; c < 3; c++) atomicAdd(&cc[f32_slot(p, B, false, c)], 1u);
        }
    }
}

__global__ void k_normalise(const uint32_t* __restrict__ cnt, int64_t total, float npix,
                            float* __restrict__ out) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[k] = normalise(cnt[k], npix);
}

template <int NB, bool JOINT, int BT>
void launch_lane(bool vec, dim3 grid, size_t smem, cudaStream_t s, const uint8_t* frames,
                 int64_t n_tiles, int H, int W, int th, int tw, int ntx, int tpf, int B, int D,
                 float npix, float* out) {
    if (vec) {
        auto k = k_hist_tiles_lane<NB, JOINT, BT, true>;
        set_max_smem(reinterpret_cast<const void*>(k), static_cast<int>(smem));
        k<<<grid, kWarpsPerCta * 32, smem, s>>>(frames, n_tiles, H, W, th, tw, ntx, tpf, B, D,
                                                npix, out);
    } else {
        auto k = k_hist_tiles_lane<NB, JOINT, BT, false>;
        set_max_smem(reinterpret_cast<const void*>(k), static_cast<int>(smem));
        k<<<grid, kWarpsPerCta * 32, smem, s>>>(frames, n_tiles, H, W, th, tw, ntx, tpf, B, D,
                                                npix, out);
    }
}

}  // namespace

int hist_dim(int32_t bins, int32_t mode) {
    if (bins < 2) return -1;
    if (mode == PDB_HIST_PER_CHANNEL) {
        if (bins > (INT32_MAX / 3)) return -1;
        return 3 * bins;
    }
    if (mode == PDB_HIST_JOINT) return bins <= 16 ? bins * bins * bins : -1;
    return -1;
}

void launch_featurize_tiles(const uint8_t* d_frames, int64_t n_frames, int32_t H, int32_t W,
                            int32_t th, int32_t tw, int32_t bins, int32_t mode, float* d_out,
                            cudaStream_t s, int sm_reserve) {
    FeatOuts one{};
    one.p[0] = d_out;
    one.n = 1;
    one.done = nullptr;
    launch_featurize_tiles_multi(d_frames, n_frames, H, W, th, tw, bins, mode, one, s, sm_reserve);
}

void launch_featurize_tiles_multi(const uint8_t* d_frames, int64_t n_frames, int32_t H, int32_t W,
                                  int32_t th, int32_t tw, int32_t bins, int32_t mode,
                                  const FeatOuts& outs, cudaStream_t s, int sm_reserve,
                                  int64_t* first_round) {
    if (first_round) *first_round = -1;
    float* d_out = outs.p[0];
    const int D = hist_dim(bins, mode);
    const int ntx = W / tw, nty = H / th;
    const int tpf = ntx * nty;
    const int64_t n_tiles = n_frames * tpf;
    if (n_tiles == 0) return;
    const float npix_h = static_cast<float>(static_cast<uint64_t>(th) * static_cast<uint64_t>(tw));
    const bool vec = (W % 16 == 0) && (tw % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(d_frames) % 16 == 0);
    const dim3 grid(static_cast<unsigned>(ceil_div(n_tiles, kWarpsPerCta)));
    const bool joint = mode == PDB_HIST_JOINT;
    const int64_t lane_px = ceil_div(static_cast<int64_t>(th) * (tw / 16), 32) * 16;
    // PDB_K1_LEGACY=1 forces the LDG-staged kernel (A/B measurements only).
    static const bool k1_legacy = [] {
        const char* e = getenv("PDB_K1_LEGACY");
        return e && atoi(e) != 0;
    }();
    const int64_t n_rows = n_frames * nty;  // tile rows (frame, ty)
    const int rows_rb = (vec && tw >= 16) ? 96 / (3 * (tw / 16)) : 0;
    const int64_t row_smem = rows_rb > 0 ? static_cast<int64_t>(ntx) * rows_rb * 3 * tw : 0;
    const int nb_rows = rows_rb > 0 ? (th + rows_rb - 1) / rows_rb : 0;
    if (joint && (bins == 4 || bins == 2) && vec && 3 * tw <= 256 && ntx <= 16 &&
        nb_rows * 16 <= 255 && n_frames * H < (int64_t{1} << 31) && row_smem % 128 == 0 &&
        !k1_legacy) {
        const int lb = bins == 4 ? 2 : 1;
        const DeviceCtx& ctx = device_ctx();
        // 3-D view of the frames: {byte within a tile row, frame row, tile
        // column}, strides {W*3, 3*tw}; the box {3*tw, RB, ntx} lands a
        // stage tile-major.
        CUtensorMap m;
        const cuuint64_t dims[3] = {static_cast<cuuint64_t>(3 * tw),
                                    static_cast<cuuint64_t>(n_frames) * H,
                                    static_cast<cuuint64_t>(ntx)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(W) * 3,
                                       static_cast<cuuint64_t>(3 * tw)};
        const cuuint32_t box[3] = {static_cast<cuuint32_t>(3 * tw),
                                   static_cast<cuuint32_t>(rows_rb), static_cast<cuuint32_t>(ntx)};
        const cuuint32_t estr[3] = {1, 1, 1};
        auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ctx.encode_tiled);
        const CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(d_frames),
                               dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS)
            fail(PDB_ERR_CUDA, "cuTensorMapEncodeTiled (frames) failed (" + std::to_string(r) + ")");
        // 3 stages: with 2 KB of counters per warp this fits 4 CTAs (32
        // counting warps) per SM; measured 212 us on config 2 vs 218-248 us
        // for 4-6 stages.
        constexpr int kStages = 3;
        // A/B measurement knobs, read once: PDB_K1_GROUP (pixels per merged
        // read-modify-write group), PDB_K1_PF (L2 prefetch distance in bands;
        // whole frame rows, so only when the tile grid covers the width),
        // PDB_K1_BULK=1 (stages by 1-D bulk copies of whole frame rows),
        // PDB_K1_STAGES, PDB_K1_EPI=0, PDB_K1_CTAS (CTAs per SM).
        struct Knobs {
            int grp = 1, pf = 0, bulk = 0, stages = kStages, skip_epi = 0, ctas = 0;
        };
        static const Knobs kn = [] {
            Knobs k;
            auto rd = [](const char* n, int d) {
                const char* e = getenv(n);
                return e ? atoi(e) : d;
            };
            k.grp = rd("PDB_K1_GROUP", 1);
            k.pf = rd("PDB_K1_PF", 0);
            k.bulk = rd("PDB_K1_BULK", 0);
            k.stages = std::max(1, rd("PDB_K1_STAGES", kStages));
            const int e = rd("PDB_K1_EPI", 1);
            k.skip_epi = e == 0 ? 1 : e == 2 ? 2 : e == 3 ? 3 : 0;
            k.ctas = rd("PDB_K1_CTAS", 0);
            return k;
        }();
        const int grp = kn.grp;
        const int pf = (W % tw == 0 && (W * 3) % 16 == 0) ? kn.pf : 0;
        const bool bulk = kn.bulk != 0 && (W * 3) % 16 == 0;
        auto pick = [&](auto g0, auto g1, auto g2, auto g4) {
            return grp == 4 ? g4 : grp == 2 ? g2 : grp == 0 ? g0 : g1;
        };
#ifdef PDB_K1_VARIANTS
        // (the A/B build: every measured variant; `make K1_VARIANTS=1`)
        auto kern = bulk ? (lb == 1 ? pick(k_hist_joint_rows8<1, 0, true>, k_hist_joint_rows8<1, 1, true>,
                                           k_hist_joint_rows8<1, 2, true>, k_hist_joint_rows8<1, 4, true>)
                                    : pick(k_hist_joint_rows8<2, 0, true>, k_hist_joint_rows8<2, 1, true>,
                                           k_hist_joint_rows8<2, 2, true>, k_hist_joint_rows8<2, 4, true>))
                         : (lb == 1 ? pick(k_hist_joint_rows8<1, 0, false>, k_hist_joint_rows8<1, 1, false>,
                                           k_hist_joint_rows8<1, 2, false>, k_hist_joint_rows8<1, 4, false>)
                                    : pick(k_hist_joint_rows8<2, 0, false>, k_hist_joint_rows8<2, 1, false>,
                                           k_hist_joint_rows8<2, 2, false>, k_hist_joint_rows8<2, 4, false>));
#else
        // the product build carries only the chosen variant (module load time
        // grows with every instantiation)
        (void)pick;
        (void)bulk;
        auto kern = lb == 1 ? k_hist_joint_rows8<1, 1, false> : k_hist_joint_rows8<2, 1, false>;
#endif
        const int n_stages = kn.stages;
        const int skip_epi = kn.skip_epi;
        // (a bulk stage holds RB whole frame rows, edge columns included)
        const int64_t stage_b = bulk ? (static_cast<int64_t>(rows_rb) * W * 3 + 127) / 128 * 128 : row_smem;
        const size_t smem = 2048 + static_cast<size_t>(ntx) * 2048 +
                            static_cast<size_t>(n_stages) * stage_b + n_stages * 16 + ntx * 128;
        set_max_smem(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
        const int threads = (ntx + 1) * 32;
        // resident CTAs per SM, cached per (kernel, block, smem, device): the
        // query costs microseconds of host time per call otherwise
        int per_sm = 0;
        {
            struct Occ {
                const void* k;
                int threads, dev;
                size_t smem;
                int per_sm;
            };
            static std::mutex mu;
            static std::vector<Occ> cache;
            std::lock_guard<std::mutex> lk(mu);
            for (const Occ& o : cache)
                if (o.k == reinterpret_cast<const void*>(kern) && o.threads == threads &&
                    o.smem == smem && o.dev == ctx.device)
                    per_sm = o.per_sm;
            if (per_sm == 0) {
                PDB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
                cache.push_back({reinterpret_cast<const void*>(kern), threads, ctx.device, smem, per_sm});
            }
        }
        if (kn.ctas > 0) per_sm = std::min(per_sm, kn.ctas);
        // (sm_reserve: SMs' worth of CTAs left free for concurrent work)
        const int64_t cap = static_cast<int64_t>(std::max(per_sm, 1)) *
                            std::max(1, ctx.sm_count - std::max(0, sm_reserve));
        const dim3 g(static_cast<unsigned>(std::min(n_rows, cap)));
        if (first_round) *first_round = static_cast<int64_t>(g.x) * ntx;
        kern<<<g, threads, smem, s>>>(m, d_frames, static_cast<int>(n_rows), nty, H, W * 3, th, tw,
                                      ntx, static_cast<uint32_t>(stage_b), n_stages, pf, skip_epi,
                                      npix_h, outs);
        PDB_CUDA(cudaGetLastError());
        return;  // every output written by the kernel
    } else if (joint && (bins == 4 || bins == 2) && vec && tw <= 512 && lane_px < 65536) {
        const int lb = bins == 4 ? 2 : 1;
        // 32-bit lane-private counters, 4 warps per CTA, one batch of
        // prefetch: the fastest of the measured (counter width x CTA size x
        // prefetch depth) variants on B200 (273.6 us for config 2 vs
        // 289-317 us for the others).
        constexpr int kWpc = 4;
        const size_t smem = static_cast<size_t>(kWpc) * ((1 << (3 * lb)) * 32 * 4 + 96 * 16);
        auto k = lb == 1 ? k_hist_joint_pow2<1, kWpc, 1, 32> : k_hist_joint_pow2<2, kWpc, 1, 32>;
        set_max_smem(reinterpret_cast<const void*>(k), static_cast<int>(smem));
        const dim3 g2(static_cast<unsigned>(ceil_div(n_tiles, kWpc)));
        k<<<g2, kWpc * 32, smem, s>>>(d_frames, n_tiles, H, W, th, tw, ntx, tpf, npix_h, d_out);
    } else if (D <= 64) {
        const size_t smem = static_cast<size_t>(kWarpsPerCta) * 64 * 32 * 4;
        if (joint && bins == 4)
            launch_lane<64, true, 4>(vec, grid, smem, s, d_frames, n_tiles, H, W, th, tw, ntx,
                                     tpf, bins, D, npix_h, d_out);
        else if (joint)
            launch_lane<64, true, 0>(vec, grid, smem, s, d_frames, n_tiles, H, W, th, tw, ntx,
                                     tpf, bins, D, npix_h, d_out);
        else if (bins == 4)
            launch_lane<12, false, 4>(vec, grid, static_cast<size_t>(kWarpsPerCta) * 12 * 32 * 4,
                                      s, d_frames, n_tiles, H, W, th, tw, ntx, tpf, bins, D,
                                      npix_h, d_out);
        else if (bins == 8)
            launch_lane<24, false, 8>(vec, grid, static_cast<size_t>(kWarpsPerCta) * 24 * 32 * 4,
                                      s, d_frames, n_tiles, H, W, th, tw, ntx, tpf, bins, D,
                                      npix_h, d_out);
        else
            launch_lane<64, false, 0>(vec, grid, smem, s, d_frames, n_tiles, H, W, th, tw, ntx,
                                      tpf, bins, D, npix_h, d_out);
    } else {
        const int slots = joint ? D : 768;
        const size_t smem = static_cast<size_t>(kWarpsPerCta) * slots * 4;
        if (joint) {
            set_max_smem(reinterpret_cast<const void*>(k_hist_tiles_atomic<true>), static_cast<int>(smem));
            k_hist_tiles_atomic<true><<<grid, kWarpsPerCta * 32, smem, s>>>(
                d_frames, n_tiles, H, W, th, tw, ntx, tpf, bins, D, slots, npix_h, d_out);
        } else {
            set_max_smem(reinterpret_cast<const void*>(k_hist_tiles_atomic<false>), static_cast<int>(smem));
            k_hist_tiles_atomic<false><<<grid, kWarpsPerCta * 32, smem, s>>>(
                d_frames, n_tiles, H, W, th, tw, ntx, tpf, bins, D, slots, npix_h, d_out);
        }
    }
    PDB_CUDA(cudaGetLastError());
    // kernels without multi-output stores: copy the local features to the
    // peers (copy engines over NVLink)
    for (int k = 1; k < outs.n; k++)
        PDB_CUDA(cudaMemcpyAsync(outs.p[k], d_out, static_cast<size_t>(n_tiles) * D * sizeof(float),
                                 cudaMemcpyDeviceToDevice, s));
}

void launch_hist_f32(const float* d_px, int64_t n, int32_t h, int32_t w, int32_t bins,
                     int32_t mode, float* d_out, cudaStream_t s) {
    const int64_t D = hist_dim(bins, mode);
    const int64_t npx = static_cast<int64_t>(h) * w;
    if (n == 0) return;
    const float npix = static_cast<float>(static_cast<uint64_t>(npx));
    const int joint = mode == PDB_HIST_JOINT;
    if (D <= kF32SmemBins) {
        const size_t smem = static_cast<size_t>(D) * 4;
        set_max_smem(reinterpret_cast<const void*>(k_hist_f32_smem), static_cast<int>(smem));
        k_hist_f32_smem<<<static_cast<unsigned>(n), 256, smem, s>>>(d_px, n, npx, bins, joint,
                                                                    static_cast<int>(D), npix,
                                                                    d_out);
    } else {
        DevBuf<uint32_t> cnt(static_cast<size_t>(n * D), s);
        PDB_CUDA(cudaMemsetAsync(cnt.p, 0, static_cast<size_t>(n * D) * 4, s));
        dim3 g(static_cast<unsigned>(std::min<int64_t>(ceil_div(npx, 256), 64)),
               static_cast<unsigned>(n));
        k_hist_f32_global<<<g, 256, 0, s>>>(d_px, n, npx, bins, joint, D, cnt.p);
        k_normalise<<<592, 256, 0, s>>>(cnt.p, n * D, npix, d_out);
    }
    PDB_CUDA(cudaGetLastError());
}

}  // namespace pdb
