// gen.cpp -- seeded synthetic workloads for the hot path (BASELINE.json
// configs 1-5).  Host C++, multi-threaded, counter-based: every row / frame
// draws from its own SplitMix64 stream keyed by (seed, salt, index), so the
// bytes do not depend on the thread count.  The generator algorithm is the
// reference's own portable one (SplitMix64, mix_seed, Box-Muller gaussian:
// include/patchdb/rng.hpp:11-52), restated here; the reference substitutes
// seeded synthetic scenes for its datasets the same way.
//
// Exported as plain C (libpdb_gen.so) so bench.py, the tests and the C++
// shim can share one definition of every workload.

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#define GEN_API extern "C" __attribute__((visibility("default")))

namespace {

struct Rng {  // SplitMix64, rng.hpp:11-43
    uint64_t s;
    explicit Rng(uint64_t seed) : s(seed) {}
    uint64_t next() {
        s += 0x9E3779B97F4A7C15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
    double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    uint64_t below(uint64_t n) {
        return static_cast<uint64_t>((static_cast<unsigned __int128>(next()) * n) >> 64);
    }
    double gaussian() {
        double u1 = uniform();
        double u2 = uniform();
        while (u1 <= 0.0) u1 = uniform();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

uint64_t mix_seed(uint64_t a, uint64_t b) {  // rng.hpp:49-52
    Rng m(a ^ (b + 0x9E3779B97F4A7C15ull + (a << 6) + (a >> 2)));
    return m.next();
}

constexpr uint64_t kSaltCentre = 0xC3A7E5ull;
constexpr uint64_t kSaltRow = 0x20B5ull;
constexpr uint64_t kSaltPlant = 0x91A7ull;
constexpr uint64_t kSaltBlock = 0xB10Cull;
constexpr uint64_t kSaltNoise = 0x7015Eull;
constexpr uint64_t kSaltCopy = 0xC0B1ull;

template <class F>
void parallel_for(int64_t n, int threads, F&& body) {
    if (threads <= 1 || n < 1024) {
        body(int64_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; t++) {
        int64_t a = n * t / threads, b = n * (t + 1) / threads;
        if (b > a) pool.emplace_back([&, a, b] { body(a, b); });
    }
    for (auto& th : pool) th.join();
}

int default_threads(int t) {
    if (t > 0) return t;
    unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(std::min(h, 64u)) : 1;
}

}  // namespace

// Gaussian mixture (configs 1 and 3): `centres` centres drawn U[0,1]^d
// from `seed`, row r = centre[below(centres)] + sigma * N(0,1) per
// coordinate from the stream (row_seed, r), then optionally L1-normalised
// (x /= sum|x| in fp64, then cast) -- config 1.  Two relations over the
// same centres use one `seed` and different `row_seed`s.
GEN_API int pdb_gen_clusters(float* out, int64_t n, int32_t d, int32_t centres,
                             double sigma, int32_t l1_normalise, uint64_t seed,
                             uint64_t row_seed, int32_t threads) {
    if (n < 0 || d < 1 || centres < 1) return 1;
    std::vector<double> C(static_cast<size_t>(centres) * d);
    for (int32_t c = 0; c < centres; c++) {
        Rng g(mix_seed(mix_seed(seed, kSaltCentre), static_cast<uint64_t>(c)));
        for (int32_t k = 0; k < d; k++) C[static_cast<size_t>(c) * d + k] = g.uniform();
    }
    parallel_for(n, default_threads(threads), [&](int64_t a, int64_t b) {
        std::vector<double> x(static_cast<size_t>(d));
        for (int64_t r = a; r < b; r++) {
            Rng g(mix_seed(mix_seed(row_seed, kSaltRow), static_cast<uint64_t>(r)));
            uint64_t c = g.below(static_cast<uint64_t>(centres));
            double s = 0.0;
            for (int32_t k = 0; k < d; k++) {
                x[k] = C[c * d + k] + sigma * g.gaussian();
                s += std::fabs(x[k]);
            }
            float* o = out + r * d;
            for (int32_t k = 0; k < d; k++)
                o[k] = static_cast<float>(l1_normalise && s > 0.0 ? x[k] / s : x[k]);
        }
    });
    return 0;
}

// Config 3 planting: each row of L is replaced, with probability `frac`
// (decided by its own stream), by R[below(nR)] + sigma_p * N(0,1).  Writes
// the planted (left, right) index pairs to `plant_l/plant_r` (capacity
// `cap`) in ascending left order and returns how many were planted.
GEN_API int64_t pdb_gen_plant(float* L, int64_t nL, const float* R, int64_t nR, int32_t d,
                              double frac, double sigma_p, uint64_t seed, int32_t* plant_l,
                              int32_t* plant_r, int64_t cap) {
    int64_t n = 0;
    for (int64_t r = 0; r < nL; r++) {
        Rng g(mix_seed(mix_seed(seed, kSaltPlant), static_cast<uint64_t>(r)));
        if (g.uniform() >= frac) continue;
        uint64_t src = g.below(static_cast<uint64_t>(nR));
        for (int32_t k = 0; k < d; k++)
            L[r * d + k] = static_cast<float>(static_cast<double>(R[src * d + k]) +
                                              sigma_p * g.gaussian());
        if (n < cap) {
            plant_l[n] = static_cast<int32_t>(r);
            plant_r[n] = static_cast<int32_t>(src);
        }
        n++;
    }
    return n;
}

// Config 5: points on the probability simplex.  A fraction `clustered` of
// rows fall in `centres` tight clusters (centre = Dirichlet(1) point, row =
// centre + sigma * N(0,1), clipped at 0 and renormalised to L1 = 1); the rest
// are Dirichlet(1) (normalised Exp(1) draws), i.e. uniform on the simplex.
GEN_API int pdb_gen_simplex(float* out, int64_t n, int32_t d, int32_t centres,
                            double clustered, double sigma, uint64_t seed, int32_t threads) {
    if (n < 0 || d < 1 || centres < 1) return 1;
    std::vector<double> C(static_cast<size_t>(centres) * d);
    for (int32_t c = 0; c < centres; c++) {
        Rng g(mix_seed(mix_seed(seed, kSaltCentre), static_cast<uint64_t>(c)));
        double s = 0;
        for (int32_t k = 0; k < d; k++) {
            double u = g.uniform();
            C[static_cast<size_t>(c) * d + k] = -std::log(1.0 - u);
            s += C[static_cast<size_t>(c) * d + k];
        }
        for (int32_t k = 0; k < d; k++) C[static_cast<size_t>(c) * d + k] /= s;
    }
    parallel_for(n, default_threads(threads), [&](int64_t a, int64_t b) {
        std::vector<double> x(static_cast<size_t>(d));
        for (int64_t r = a; r < b; r++) {
            Rng g(mix_seed(mix_seed(seed, kSaltRow), static_cast<uint64_t>(r)));
            double s = 0;
            if (g.uniform() < clustered) {
                uint64_t c = g.below(static_cast<uint64_t>(centres));
                for (int32_t k = 0; k < d; k++) {
                    x[k] = std::max(0.0, C[c * d + k] + sigma * g.gaussian());
                    s += x[k];
                }
            } else {
                for (int32_t k = 0; k < d; k++) {
                    x[k] = -std::log(1.0 - g.uniform());
                    s += x[k];
                }
            }
            float* o = out + r * d;
            for (int32_t k = 0; k < d; k++) o[k] = static_cast<float>(s > 0 ? x[k] / s : 0.0);
        }
    });
    return 0;
}

// Uniform U[0,1)^d rows (the reference's simjoin_scaling probe,
// src/bench.cpp:1145-1175, draws the same distribution).
GEN_API int pdb_gen_uniform(float* out, int64_t n, int32_t d, uint64_t seed,
                            int32_t threads) {
    parallel_for(n, default_threads(threads), [&](int64_t a, int64_t b) {
        for (int64_t r = a; r < b; r++) {
            Rng g(mix_seed(mix_seed(seed, kSaltRow), static_cast<uint64_t>(r)));
            for (int32_t k = 0; k < d; k++) out[r * d + k] = static_cast<float>(g.uniform());
        }
    });
    return 0;
}

// Config 2 frames [count,H,W,3] uint8: frames f0 .. f0+count-1 of the
// video (any range can be generated independently, so ranks generate only
// their own shard).  Background: piecewise-constant colour blocks of
// block x block pixels, one uniform RGB colour per block per frame.  Noise:
// per pixel and channel, uniform integer in [-noise, noise], clamped to
// [0,255].  Every frame f with f % period == period-1 is a near-copy: it
// reuses the block colours of an earlier original frame
// (f - 1 - (mix % min(f, 10)), followed back to an original) and is
// re-noised with `copy_noise` (period 20 -> exactly 5% of frames).
// src_of[k] receives the source frame of frame f0+k (or -1) when non-null.
namespace {
int64_t frame_source(int64_t f, int32_t period, uint64_t seed) {
    while (f >= 1 && f % period == period - 1) {
        uint64_t m = mix_seed(mix_seed(seed, kSaltCopy), static_cast<uint64_t>(f));
        int64_t span = std::min<int64_t>(f, 10);
        f = f - 1 - static_cast<int64_t>(m % static_cast<uint64_t>(span));
    }
    return f;
}
}  // namespace

GEN_API int pdb_gen_frames(uint8_t* out, int64_t f0, int64_t count, int32_t H, int32_t W,
                           int32_t block, int32_t noise, int32_t copy_noise, int32_t period,
                           uint64_t seed, int64_t* src_of, int32_t threads) {
    if (f0 < 0 || count < 0 || H < 1 || W < 1 || block < 1 || period < 1) return 1;
    std::vector<int64_t> src(static_cast<size_t>(count), -1);
    for (int64_t k = 0; k < count; k++) {
        const int64_t f = f0 + k;
        const int64_t s = frame_source(f, period, seed);
        if (s != f) src[k] = s;
    }
    if (src_of) std::memcpy(src_of, src.data(), src.size() * sizeof(int64_t));
    const int32_t bx = (W + block - 1) / block, by = (H + block - 1) / block;
    parallel_for(count, default_threads(threads), [&](int64_t a, int64_t b) {
        std::vector<uint8_t> col(static_cast<size_t>(bx) * by * 3);
        for (int64_t k = a; k < b; k++) {
            const int64_t f = f0 + k;
            const int64_t cf = src[k] >= 0 ? src[k] : f;
            for (int64_t q = 0; q < static_cast<int64_t>(bx) * by; q++) {
                Rng g(mix_seed(mix_seed(mix_seed(seed, kSaltBlock), static_cast<uint64_t>(cf)),
                               static_cast<uint64_t>(q)));
                uint64_t v = g.next();
                col[q * 3 + 0] = static_cast<uint8_t>(v);
                col[q * 3 + 1] = static_cast<uint8_t>(v >> 8);
                col[q * 3 + 2] = static_cast<uint8_t>(v >> 16);
            }
            const int32_t amp = src[k] >= 0 ? copy_noise : noise;
            const uint64_t span = static_cast<uint64_t>(2 * amp + 1);
            uint64_t fseed = mix_seed(mix_seed(seed, kSaltNoise), static_cast<uint64_t>(f));
            uint8_t* fr = out + k * static_cast<int64_t>(H) * W * 3;
            for (int32_t y = 0; y < H; y++) {
                Rng g(mix_seed(fseed, static_cast<uint64_t>(y)));
                const uint8_t* crow = col.data() + static_cast<size_t>(y / block) * bx * 3;
                for (int32_t x = 0; x < W; x++) {
                    uint64_t v = g.next();
                    const uint8_t* c = crow + static_cast<size_t>(x / block) * 3;
                    for (int ch = 0; ch < 3; ch++) {
                        int n = amp == 0 ? 0
                                         : static_cast<int>(((v >> (16 * ch)) & 0xFFFF) * span >> 16) -
                                               amp;
                        int p = static_cast<int>(c[ch]) + n;
                        fr[(static_cast<size_t>(y) * W + x) * 3 + ch] =
                            static_cast<uint8_t>(p < 0 ? 0 : (p > 255 ? 255 : p));
                    }
                }
            }
        }
    });
    return 0;
}
