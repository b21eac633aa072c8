// pdb_patchdb.hpp -- header-only C++ adapter that lets code written against
// the reference patchdb operator API call the B200 kernels with its own
// types.  It is the drop-in a reference maintainer would use inside
// proj/src: same argument meaning, same output order,
// same exception types.
//
//   sim_join_pairs(left, right, tau, side, &probes)
//       == patchdb::sim_join_pairs (include/patchdb/query.hpp:209-211,
//          src/query.cpp:485-528 + 1094-1104): pairs in probe order, then
//          ascending build-side patch id; probes = probe-side rows.
//   color_histogram(patch, bins)
//       == the data vector of patchdb::apply_transformer(color_histogram)
//          (src/etl.cpp:330-354); the caller wraps it with derive_patch.
//   featurize_tiles(frames, tile_w, tile_h, bins)
//       == the data vectors of transform(generate(frames, tiles),
//          color_histogram) in emission order (src/etl.cpp:264-373).
//
// PatchT needs `uint64_t patch_id`, `std::vector<float> data`,
// `std::vector<uint32_t> shape`; FrameT needs `width`, `height`, `pixels`.
// Errors: define PDB_PATCHDB_REFERENCE_ERRORS before including this header
// (with the reference's patchdb/core.hpp visible) to throw the reference's
// own exception classes; otherwise the same-named classes below are thrown.
#pragma once

#include <algorithm>
#include <cstdint>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <utility>
#include <vector>

#include "pdb_cuda.h"

namespace pdb {
namespace patchdb {

#ifdef PDB_PATCHDB_REFERENCE_ERRORS
using ::patchdb::ConfigError;
using ::patchdb::DimensionMismatchError;
using ::patchdb::DuplicatePatchIdError;
using ::patchdb::Error;
using ::patchdb::MixedDimensionError;
using ::patchdb::ShapeError;
#else
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : Error {
    using Error::Error;
};
struct ShapeError : Error {
    using Error::Error;
};
struct MixedDimensionError : Error {
    using Error::Error;
};
struct DimensionMismatchError : Error {
    using Error::Error;
};
struct DuplicatePatchIdError : Error {
    using Error::Error;
};
#endif

// Mirrors patchdb::BuildSide (query.hpp:84).
enum class BuildSide : uint8_t { automatic, left, right };

struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(int st) {
    if (st == PDB_OK) return;
    const std::string msg = pdb_last_error();
    switch (st) {
        case PDB_ERR_CONFIG: throw ConfigError(msg);
        case PDB_ERR_SHAPE: throw ShapeError(msg);
        case PDB_ERR_MIXED_DIMENSION: throw MixedDimensionError(msg);
        case PDB_ERR_DIMENSION_MISMATCH: throw DimensionMismatchError(msg);
        case PDB_ERR_DUPLICATE_ID: throw DuplicatePatchIdError(msg);
        case PDB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        default: throw DeviceError(std::string(pdb_status_name(st)) + ": " + msg);
    }
}

namespace detail {
// src/query.cpp:467-477
template <class PatchT>
size_t checked_dim(const std::vector<PatchT>& items) {
    size_t d = items.empty() ? 0 : items[0].data.size();
    if (!items.empty() && d == 0)
        throw ShapeError("similarity join needs non-empty patch data");
    for (const PatchT& p : items)
        if (p.data.size() != d)
            throw MixedDimensionError("similarity join saw " + std::to_string(d) + " and " +
                                      std::to_string(p.data.size()) + " dimensional patches");
    return d;
}

template <class PatchT>
std::vector<float> pack(const std::vector<PatchT>& items, size_t d) {
    std::vector<float> m(items.size() * d);
    for (size_t i = 0; i < items.size(); i++)
        std::copy(items[i].data.begin(), items[i].data.end(), m.begin() + i * d);
    return m;
}
}  // namespace detail

// Position pairs (left index, right index) in the reference's emission
// order -- run_sim_join's core (src/query.cpp:485-528) on the B200.
template <class PatchT>
std::vector<std::pair<size_t, size_t>> sim_join_positions(const std::vector<PatchT>& left,
                                                          const std::vector<PatchT>& right,
                                                          double tau,
                                                          BuildSide side = BuildSide::automatic,
                                                          uint64_t* index_probes = nullptr) {
    if (tau < 0.0) throw ConfigError("similarity join needs tau >= 0");
    const BuildSide chosen = side != BuildSide::automatic
                                 ? side
                                 : (left.size() <= right.size() ? BuildSide::left : BuildSide::right);
    const size_t dl = detail::checked_dim(left), dr = detail::checked_dim(right);
    if (!left.empty() && !right.empty() && dl != dr)
        throw DimensionMismatchError("similarity join over " + std::to_string(dl) + " and " +
                                     std::to_string(dr) + " dimensional sides");
    if (index_probes) *index_probes = 0;
    if (left.empty() || right.empty()) return {};
    const auto& build = chosen == BuildSide::left ? left : right;
    {
        std::unordered_set<uint64_t> seen;
        seen.reserve(build.size());
        for (const PatchT& p : build)
            if (!seen.insert(p.patch_id).second)
                throw DuplicatePatchIdError("patch id " + std::to_string(p.patch_id) +
                                            " appears twice on the build side");
    }
    // Emission order: probe order, then ascending build-side patch id
    // (balltree_within sorts ids).  When the build side's ids ascend with
    // its positions (the usual case) that is the device's sorted (probe,
    // build) order: the probe side goes in as L with PDB_JOIN_SORTED and no
    // host sort is needed.  Otherwise the pairs are sorted here.
    const auto& probe = chosen == BuildSide::left ? right : left;
    bool ids_ascend = true;
    for (size_t i = 1; i < build.size() && ids_ascend; i++)
        ids_ascend = build[i - 1].patch_id < build[i].patch_id;
    const std::vector<float> P = detail::pack(probe, dl), B = detail::pack(build, dl);
    pdb_join_opts o{};
    o.flags = ids_ascend ? PDB_JOIN_SORTED : 0u;
    pdb_pairs pr{};
    check(pdb_sim_join(P.data(), static_cast<int64_t>(probe.size()), B.data(),
                       static_cast<int64_t>(build.size()), static_cast<int32_t>(dl), tau, &o, &pr));
    std::vector<std::pair<size_t, size_t>> out(static_cast<size_t>(pr.count));
    const bool swap = chosen == BuildSide::left;  // pairs are (left pos, right pos)
    for (int64_t k = 0; k < pr.count; k++) {
        const size_t pi = static_cast<size_t>(pr.left[k]), bi = static_cast<size_t>(pr.right[k]);
        out[static_cast<size_t>(k)] = swap ? std::pair<size_t, size_t>{bi, pi}
                                           : std::pair<size_t, size_t>{pi, bi};
    }
    pdb_pairs_free(&pr);
    if (!ids_ascend) {
        if (chosen == BuildSide::left) {
            std::sort(out.begin(), out.end(), [&](const auto& a, const auto& b) {
                if (a.second != b.second) return a.second < b.second;
                return left[a.first].patch_id < left[b.first].patch_id;
            });
        } else {
            std::sort(out.begin(), out.end(), [&](const auto& a, const auto& b) {
                if (a.first != b.first) return a.first < b.first;
                return right[a.second].patch_id < right[b.second].patch_id;
            });
        }
    }
    if (index_probes) *index_probes = chosen == BuildSide::left ? right.size() : left.size();
    return out;
}

// compile_nl_join with a pure within predicate over single-patch tuples
// (src/query.cpp:142-151, 705-744): (left index, right index) of every pair
// with euclidean <= radius, in nested-loop order -- the B200 cross join,
// sorted.  A dimension mismatch throws as the predicate's first evaluation
// does; empty sides give nothing.
template <class PatchT>
std::vector<std::pair<size_t, size_t>> nl_within_positions(const std::vector<PatchT>& left,
                                                           const std::vector<PatchT>& right,
                                                           double radius) {
    if (left.empty() || right.empty()) return {};
    const size_t d = left[0].data.size();
    for (const auto* side : {&left, &right})
        for (const PatchT& p : *side)
            if (p.data.size() != d)
                throw DimensionMismatchError("distance between " + std::to_string(d) + " and " +
                                             std::to_string(p.data.size()) +
                                             " dimensional patches");
    std::vector<std::pair<size_t, size_t>> out;
    if (!(radius >= 0.0)) return out;
    if (d == 0) {  // zero-dimensional patches are all at distance 0
        for (size_t i = 0; i < left.size(); i++)
            for (size_t j = 0; j < right.size(); j++) out.emplace_back(i, j);
        return out;
    }
    const std::vector<float> L = detail::pack(left, d), R = detail::pack(right, d);
    pdb_join_opts o{};
    o.flags = PDB_JOIN_SORTED;
    pdb_pairs pr{};
    check(pdb_sim_join(L.data(), static_cast<int64_t>(left.size()), R.data(),
                       static_cast<int64_t>(right.size()), static_cast<int32_t>(d), radius, &o,
                       &pr));
    out.resize(static_cast<size_t>(pr.count));
    for (int64_t k = 0; k < pr.count; k++)
        out[static_cast<size_t>(k)] = {static_cast<size_t>(pr.left[k]),
                                       static_cast<size_t>(pr.right[k])};
    pdb_pairs_free(&pr);
    return out;
}

// run_dedup's grouping (src/query.cpp:535-566) on the B200: representatives
// in kept order and, per representative, its members in arrival order.
struct DedupGroups {
    std::vector<size_t> reps;
    std::vector<std::vector<size_t>> members;
};

template <class PatchT>
DedupGroups dedup_groups(const std::vector<PatchT>& items, double tau) {
    if (tau < 0.0) throw ConfigError("dedup needs tau >= 0");
    DedupGroups g;
    if (items.empty()) return g;
    const size_t d = items[0].data.size();
    if (d == 0) throw ShapeError("dedup needs non-empty patch data");
    for (const PatchT& p : items)
        if (p.data.size() != d)
            throw MixedDimensionError("dedup saw " + std::to_string(d) + " and " +
                                      std::to_string(p.data.size()) + " dimensional patches");
    const std::vector<float> X = detail::pack(items, d);
    std::vector<int64_t> rep_of(items.size());
    int64_t n_reps = 0;
    check(pdb_dedup(X.data(), static_cast<int64_t>(items.size()), static_cast<int32_t>(d), tau,
                    nullptr, rep_of.data(), &n_reps));
    std::vector<size_t> slot(items.size());
    for (size_t i = 0; i < items.size(); i++) {
        if (rep_of[i] == static_cast<int64_t>(i)) {
            slot[i] = g.reps.size();
            g.reps.push_back(i);
            g.members.push_back({});
        }
        g.members[slot[static_cast<size_t>(rep_of[i])]].push_back(i);
    }
    return g;
}

// patchdb::sim_join_pairs (query.hpp:209-211).
template <class PatchT>
std::vector<std::pair<PatchT, PatchT>> sim_join_pairs(const std::vector<PatchT>& left,
                                                      const std::vector<PatchT>& right, double tau,
                                                      BuildSide side = BuildSide::automatic,
                                                      uint64_t* index_probes = nullptr) {
    const auto pos = sim_join_positions(left, right, tau, side, index_probes);
    std::vector<std::pair<PatchT, PatchT>> out;
    out.reserve(pos.size());
    for (const auto& [li, ri] : pos) out.emplace_back(left[li], right[ri]);
    return out;
}

// Histogram data of apply_transformer(color_histogram{bins}) for a pixel
// patch [h, w, 3] (src/etl.cpp:330-354).
template <class PatchT>
std::vector<float> color_histogram(const PatchT& p, uint32_t bins) {
    if (bins < 2) throw ConfigError("color_histogram needs at least 2 bins per channel");
    if (!(p.shape.size() == 3 && p.shape[2] == 3))
        throw ShapeError("transformer input must be pixel shaped [h,w,3], patch " +
                         std::to_string(p.patch_id) + " is not");
    std::vector<float> out(3u * bins);
    check(pdb_color_histogram_f32(p.data.data(), 1, static_cast<int32_t>(p.shape[0]),
                                  static_cast<int32_t>(p.shape[1]), static_cast<int32_t>(bins),
                                  PDB_HIST_PER_CHANNEL, out.data()));
    return out;
}

// Histogram data vectors of transform(generate(frames, tiles), color_histogram)
// in emission order (frames of one size).
template <class FrameT>
std::vector<std::vector<float>> featurize_tiles(const std::vector<FrameT>& frames,
                                                uint32_t tile_w, uint32_t tile_h, uint32_t bins) {
    if (bins < 2) throw ConfigError("color_histogram needs at least 2 bins per channel");
    if (tile_w < 1 || tile_h < 1) throw ConfigError("tiles generator needs tile_w and tile_h >= 1");
    if (frames.empty()) return {};
    const uint32_t W = frames[0].width, H = frames[0].height;
    std::vector<uint8_t> buf;
    buf.reserve(frames.size() * W * H * 3);
    for (const FrameT& f : frames) {
        if (f.width != W || f.height != H)
            throw ShapeError("featurize_tiles needs frames of one size");
        buf.insert(buf.end(), f.pixels.begin(), f.pixels.end());
    }
    const size_t per = static_cast<size_t>(W / tile_w) * (H / tile_h), D = 3u * bins;
    std::vector<float> flat(frames.size() * per * D);
    check(pdb_featurize_tiles(buf.data(), static_cast<int64_t>(frames.size()),
                              static_cast<int32_t>(H), static_cast<int32_t>(W),
                              static_cast<int32_t>(tile_h), static_cast<int32_t>(tile_w),
                              static_cast<int32_t>(bins), PDB_HIST_PER_CHANNEL, flat.data()));
    std::vector<std::vector<float>> out(frames.size() * per);
    for (size_t k = 0; k < out.size(); k++)
        out[k].assign(flat.begin() + k * D, flat.begin() + (k + 1) * D);
    return out;
}

}  // namespace patchdb
}  // namespace pdb
