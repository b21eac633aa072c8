// Drop-in parity: the reference's own public operators (compiled from
// /root/reference/proj) against include/pdb_patchdb.hpp over the B200
// kernels, on the reference's own types and test-data builders
// (proj/tests/oracles.hpp).  Built by `make -C oracle dropin` into
// oracle/_ref/dropin_parity (test infrastructure); run on the GPU box by
// tests/test_dropin_gpu.py.  Prints "DROPIN OK <checks>" and exits 0.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "oracles.hpp"  // proj/tests/oracles.hpp (reference test fixtures)
#include "patchdb/core.hpp"
#include "patchdb/etl.hpp"
#include "patchdb/index.hpp"
#include "patchdb/query.hpp"

#define PDB_PATCHDB_REFERENCE_ERRORS
#include "pdb_patchdb.hpp"

using namespace patchdb;

static int checks = 0;
#define EXPECT(c)                                                           \
    do {                                                                    \
        if (!(c)) {                                                         \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            std::exit(1);                                                   \
        }                                                                   \
        checks++;                                                           \
    } while (0)

template <class E, class F>
static bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static void join_case(const std::vector<Patch>& L, const std::vector<Patch>& R, double tau) {
    const BuildSide sides[] = {BuildSide::automatic, BuildSide::left, BuildSide::right};
    for (int s = 0; s < 3; s++) {
        uint64_t pr_ref = 0, pr_b200 = 0;
        auto want = sim_join_pairs(L, R, tau, sides[s], &pr_ref);
        auto got = pdb::patchdb::sim_join_pairs(L, R, tau,
                                                static_cast<pdb::patchdb::BuildSide>(s), &pr_b200);
        EXPECT(want.size() == got.size());
        for (size_t k = 0; k < want.size(); k++) {
            EXPECT(want[k].first.patch_id == got[k].first.patch_id);
            EXPECT(want[k].second.patch_id == got[k].second.patch_id);
        }
        EXPECT(pr_ref == pr_b200);
    }
}

int main() {
    // test_query.cpp:268-300 workload: 60 x 40 random 6-d points, tau 0.45
    auto lp = oracle::to_patches(oracle::random_points(80, 60, 6));
    std::vector<Patch> rp;
    for (const auto& [p, id] : oracle::random_points(81, 40, 6)) rp.push_back(oracle::vec_patch(1000 + id, p));
    join_case(lp, rp, 0.45);
    // build-side ids not ascending with position: the adapter's host sort
    auto rev_l = lp;
    std::reverse(rev_l.begin(), rev_l.end());
    auto rev_r = rp;
    std::reverse(rev_r.begin(), rev_r.end());
    join_case(rev_l, rp, 0.45);
    join_case(lp, rev_r, 0.45);
    join_case(rev_l, rev_r, 0.6);
    // acceptance.cpp:140-198 shape (scaled): clustered 24-d, sigma 0.005, tau 0.1
    auto all = oracle::clustered_points(4242, 100, 40, 24, 0.005);
    std::vector<Patch> L2, R2;
    for (size_t c = 0; c < 100; c++)
        for (size_t j = 0; j < 40; j++) {
            const auto& [p, id] = all[c * 40 + j];
            (j < 20 ? L2 : R2).push_back(oracle::vec_patch(j < 20 ? id : 1000000 + id, p));
        }
    join_case(L2, R2, 0.1);
    // self-join: sim_join_pairs(X, X) -> ordered pairs incl. the diagonal
    auto x = oracle::to_patches(oracle::clustered_points(7, 30, 25, 16, 0.01));
    join_case(x, x, 0.05);
    // inclusive radius (test_index.cpp:330-342)
    std::vector<Patch> dup;
    for (uint64_t i = 1; i <= 5; i++) dup.push_back(oracle::vec_patch(i, {1.0f, 1.0f}));
    dup.push_back(oracle::vec_patch(6, {2.0f, 1.0f}));
    std::vector<Patch> q{oracle::vec_patch(100, {1.0f, 1.0f})};
    join_case(dup, q, 1.0);
    join_case(dup, q, 0.999);
    // NaN tau: the reference rejects only tau < 0.0 (src/query.cpp:488), so a
    // NaN passes and matches nothing; the adapter must agree, not throw
    join_case(lp, rp, std::nan(""));
    join_case(x, x, std::nan(""));
    // errors
    EXPECT((throws_as<ConfigError>([&] { pdb::patchdb::sim_join_pairs(lp, rp, -1.0); })));
    auto bad = lp;
    bad.push_back(oracle::vec_patch(9999, {1.0f}));
    EXPECT((throws_as<MixedDimensionError>([&] { pdb::patchdb::sim_join_pairs(bad, rp, 0.45); })));
    EXPECT((throws_as<DimensionMismatchError>(
        [&] { pdb::patchdb::sim_join_pairs(lp, std::vector<Patch>{oracle::vec_patch(1, {1.0f})}, 0.45); })));
    EXPECT(pdb::patchdb::sim_join_pairs(std::vector<Patch>{}, rp, 0.45).empty());

    // apply_transformer(color_histogram) on the reference's textured frames
    for (uint32_t bins : {2u, 4u, 8u, 13u, 64u, 300u}) {
        Frame f = oracle::textured_frame("v", 3, 40, 30);
        Patch p = make_patch(f, {5, 3, 37, 29}, {});
        TransformerSpec t;
        t.kind = TransformerKind::color_histogram;
        t.bins = bins;
        Patch want = apply_transformer(p, t);
        auto got = pdb::patchdb::color_histogram(p, bins);
        EXPECT(want.data == got);
    }
    // transform(generate(frames, tiles), color_histogram)
    std::vector<Frame> frames;
    for (uint64_t i = 0; i < 4; i++) frames.push_back(oracle::textured_frame("v", i, 64, 48));
    for (uint32_t bins : {4u, 8u}) {
        GeneratorSpec g;
        g.kind = GeneratorKind::tiles;
        g.tile_w = 16;
        g.tile_h = 12;
        TransformerSpec t;
        t.kind = TransformerKind::color_histogram;
        t.bins = bins;
        auto want = drain(*transform(generate(std::make_unique<VectorStream<Frame>>(frames), g), t));
        auto got = pdb::patchdb::featurize_tiles(frames, 16, 12, bins);
        EXPECT(want.size() == got.size());
        for (size_t k = 0; k < want.size(); k++) EXPECT(want[k].data == got[k]);
    }
    // nl_join with a pure within predicate (src/query.cpp:142-151, 705-744)
    for (double r : {0.3, 0.45, 5.0}) {
        std::vector<Tuple> lt, rt;
        for (const auto& p : lp) lt.push_back(Tuple{p});
        for (const auto& p : rp) rt.push_back(Tuple{p});
        ExecContext ctx;
        auto res = execute(*PlanNode::nl_join(PlanNode::memory(lt), PlanNode::memory(rt),
                                              Predicate::within_of(0, 1, r)),
                           ctx);
        auto got = pdb::patchdb::nl_within_positions(lp, rp, r);
        EXPECT(res.tuples.size() == got.size());
        for (size_t k = 0; k < got.size(); k++) {
            EXPECT(res.tuples[k][0].patch_id == lp[got[k].first].patch_id);
            EXPECT(res.tuples[k][1].patch_id == rp[got[k].second].patch_id);
        }
    }
    EXPECT((throws_as<DimensionMismatchError>([&] {
        pdb::patchdb::nl_within_positions(lp, std::vector<Patch>{oracle::vec_patch(1, {1.0f})}, 1.0);
    })));
    // dedup (src/query.cpp:535-582): group sizes and lineage parents of
    // PlanNode::dedup, kept set of dedup_stream
    for (double tau : {0.05, 0.2, 0.6, std::nan("")}) {
        auto items = oracle::to_patches(oracle::clustered_points(11, 40, 12, 8, 0.02));
        std::vector<Tuple> tt;
        for (const auto& p : items) tt.push_back(Tuple{p});
        ExecContext ctx;
        auto res = execute(*PlanNode::dedup(PlanNode::memory(tt), tau), ctx);
        auto g = pdb::patchdb::dedup_groups(items, tau);
        EXPECT(res.tuples.size() == g.reps.size());
        for (size_t r = 0; r < g.reps.size(); r++) {
            EXPECT(res.tuples[r][0].lineage[0].parent_id() == items[g.reps[r]].patch_id);
            EXPECT(res.tuples[r][0].meta_int("group_size") ==
                   static_cast<int64_t>(g.members[r].size()));
        }
        auto kept = drain(*dedup_stream(std::make_unique<VectorStream<Patch>>(items), tau));
        EXPECT(kept.size() == g.reps.size());
        for (size_t r = 0; r < kept.size(); r++) EXPECT(kept[r].patch_id == items[g.reps[r]].patch_id);
    }
    EXPECT((throws_as<ConfigError>([&] { pdb::patchdb::dedup_groups(lp, -0.5); })));
    std::printf("DROPIN OK %d\n", checks);
    return 0;
}
