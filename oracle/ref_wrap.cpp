// ref_wrap.cpp -- extern "C" entry points over the UNMODIFIED reference
// sources, compiled where they lie under $PATCHDB_REF (default
// /root/reference/proj) by oracle/Makefile into oracle/_ref/libpdb_ref.so.
//
// TEST / BASELINE INFRASTRUCTURE ONLY: used by tests (to pin the C
// restatement and to mint tests/golden fixtures) and by bench.py's
// cpu_baseline / --impl reference legs.  Never linked by the product.
//
// The reference functions are called through their public API exactly as
// a reference user would:
//   transform(generate(VectorStream<Frame>, tiles), color_histogram)
//       include/patchdb/etl.hpp:66-69, src/etl.cpp:252-373
//   apply_transformer                       src/etl.cpp:330-354
//   sim_join_pairs                          src/query.cpp:1094-1104
//   build_balltree + balltree_within        src/index.cpp:700-842
//   euclidean                               src/index.cpp:69-76
// The library is built with -fvisibility=hidden so the reference's
// `patchdb` symbols never clash with anything else in the process.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <thread>
#include <unordered_map>
#include <vector>

#include "patchdb/core.hpp"
#include "patchdb/etl.hpp"
#include "patchdb/index.hpp"
#include "patchdb/query.hpp"
#include "patchdb/storage.hpp"
#include "patchdb/planfile.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace patchdb;

namespace {

thread_local std::string g_err;

// Error codes mirror include/pdb_cuda.h so tests compare behaviour 1:1.
int code_of(const std::exception& e) {
    if (dynamic_cast<const ConfigError*>(&e)) return 1;
    if (dynamic_cast<const ShapeError*>(&e)) return 2;
    if (dynamic_cast<const MixedDimensionError*>(&e)) return 3;
    if (dynamic_cast<const DimensionMismatchError*>(&e)) return 4;
    if (dynamic_cast<const DuplicatePatchIdError*>(&e)) return 5;
    return 99;
}

std::vector<Frame> make_frames(const uint8_t* frames, int64_t n, int32_t H, int32_t W,
                               int64_t first_no) {
    std::vector<Frame> out(static_cast<size_t>(n));
    size_t fb = static_cast<size_t>(H) * W * 3;
    for (int64_t f = 0; f < n; f++) {
        Frame& fr = out[static_cast<size_t>(f)];
        fr.video_id = "v";
        fr.frame_no = static_cast<uint64_t>(first_no + f);
        fr.width = static_cast<uint32_t>(W);
        fr.height = static_cast<uint32_t>(H);
        fr.channels = 3;
        fr.pixels.assign(frames + f * fb, frames + (f + 1) * fb);
    }
    return out;
}

std::vector<Patch> make_vecs(const float* X, int64_t n, int32_t d, uint64_t first_id) {
    std::vector<Patch> out(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; i++) {
        Patch& p = out[static_cast<size_t>(i)];
        p.patch_id = first_id + static_cast<uint64_t>(i);
        p.data.assign(X + i * d, X + (i + 1) * d);
        p.shape = {static_cast<uint32_t>(d)};
    }
    return out;
}

// Featurize a frame range through the reference stream stages.
int64_t featurize_range(const uint8_t* frames, int64_t f0, int64_t f1, int32_t H,
                        int32_t W, int32_t th, int32_t tw, int32_t bins, float* out,
                        int64_t out_row0) {
    GeneratorSpec g;
    g.kind = GeneratorKind::tiles;
    g.tile_w = static_cast<uint32_t>(tw);
    g.tile_h = static_cast<uint32_t>(th);
    TransformerSpec t;
    t.kind = TransformerKind::color_histogram;
    t.bins = static_cast<uint32_t>(bins);
    size_t fb = static_cast<size_t>(H) * W * 3;
    auto stream = transform(
        generate(std::make_unique<VectorStream<Frame>>(
                     make_frames(frames + f0 * fb, f1 - f0, H, W, f0)),
                 g),
        t);
    int64_t row = out_row0;
    const size_t D = 3u * static_cast<size_t>(bins);
    while (auto p = stream->next()) {
        std::memcpy(out + row * D, p->data.data(), D * sizeof(float));
        row++;
    }
    return row - out_row0;
}

}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// Per-channel colour histograms of the tiles of uint8 frames [F,H,W,3].
// Frames are sharded across `threads` host threads (each shard is an
// independent reference stream; the reference itself is single-threaded).
REF_API int ref_featurize_tiles(const uint8_t* frames, int64_t n, int32_t H, int32_t W,
                                int32_t th, int32_t tw, int32_t bins, float* out,
                                int32_t threads) {
    try {
        if (threads <= 1 || n < 2) {
            featurize_range(frames, 0, n, H, W, th, tw, bins, out, 0);
            return 0;
        }
        int64_t per_frame = static_cast<int64_t>(W / tw) * (H / th);
        std::vector<std::thread> pool;
        std::atomic<int> rc{0};
        for (int32_t k = 0; k < threads; k++) {
            int64_t f0 = n * k / threads, f1 = n * (k + 1) / threads;
            if (f1 <= f0) continue;
            pool.emplace_back([&, f0, f1] {
                try {
                    featurize_range(frames, f0, f1, H, W, th, tw, bins, out, f0 * per_frame);
                } catch (const std::exception& e) {
                    rc = code_of(e);
                }
            });
        }
        for (auto& t : pool) t.join();
        return rc;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// apply_transformer(color_histogram) on float pixel patches [n,h,w,3].
REF_API int ref_color_histogram_f32(const float* px, int64_t n, int32_t h, int32_t w,
                                    int32_t bins, float* out) {
    try {
        TransformerSpec t;
        t.kind = TransformerKind::color_histogram;
        t.bins = static_cast<uint32_t>(bins);
        size_t pix = static_cast<size_t>(h) * w * 3;
        for (int64_t i = 0; i < n; i++) {
            Patch p;
            p.patch_id = static_cast<uint64_t>(i + 1);
            p.shape = {static_cast<uint32_t>(h), static_cast<uint32_t>(w), 3u};
            p.data.assign(px + i * pix, px + (i + 1) * pix);
            Patch q = apply_transformer(p, t);
            std::memcpy(out + i * q.data.size(), q.data.data(), q.data.size() * sizeof(float));
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

REF_API double ref_euclidean(const float* a, const float* b, int64_t d) {
    return euclidean(a, b, static_cast<size_t>(d));
}

// sim_join_pairs(left, right, tau, side): left ids 1..nL, right ids
// 2^32+1..; returns positions (left index, right index) in the reference's
// emission order.  Caller frees with ref_free.  side: 0 automatic, 1 left,
// 2 right (query.hpp:84).
REF_API int ref_sim_join(const float* L, int64_t nL, const float* R, int64_t nR, int32_t d,
                         double tau, int32_t side, int64_t* out_count, int32_t** out_left,
                         int32_t** out_right, uint64_t* out_probes) {
    try {
        auto left = make_vecs(L, nL, d, 1);
        auto right = make_vecs(R, nR, d, (1ull << 32) + 1);
        uint64_t probes = 0;
        auto pairs = sim_join_pairs(left, right, tau, static_cast<BuildSide>(side), &probes);
        int64_t n = static_cast<int64_t>(pairs.size());
        int32_t* a = static_cast<int32_t*>(std::malloc(std::max<int64_t>(n, 1) * sizeof(int32_t)));
        int32_t* b = static_cast<int32_t*>(std::malloc(std::max<int64_t>(n, 1) * sizeof(int32_t)));
        for (int64_t k = 0; k < n; k++) {
            a[k] = static_cast<int32_t>(pairs[k].first.patch_id - 1);
            b[k] = static_cast<int32_t>(pairs[k].second.patch_id - ((1ull << 32) + 1));
        }
        *out_count = n;
        *out_left = a;
        *out_right = b;
        if (out_probes) *out_probes = probes;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

REF_API void ref_free(void* p) { std::free(p); }

// Timed CPU baseline of the reference join: the reference's own build
// (build_balltree over the build side) and probe (balltree_within) with the
// probe loop of src/query.cpp:516-526 spread over `threads` host threads
// (BallTreeIndex is immutable after build).  Probes rows
// [p0, p1) of L against all of R.  self_join counts only j > i.  Returns
// the number of matched pairs; *build_s / *probe_s receive wall seconds.
REF_API int64_t ref_join_probe_timed(const float* L, int64_t nL, const float* R,
                                     int64_t nR, int32_t d, double tau, int32_t self_join,
                                     int64_t p0, int64_t p1, int32_t threads,
                                     double* build_s, double* probe_s) {
    try {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::pair<std::vector<float>, uint64_t>> pts;
        pts.reserve(static_cast<size_t>(nR));
        for (int64_t j = 0; j < nR; j++)
            pts.emplace_back(std::vector<float>(R + j * d, R + (j + 1) * d),
                             static_cast<uint64_t>(j));
        BallTreeIndex tree = build_balltree(pts);
        auto t1 = std::chrono::steady_clock::now();
        if (p1 > nL) p1 = nL;
        std::atomic<int64_t> total{0};
        std::atomic<int64_t> next{p0};
        std::vector<std::thread> pool;
        for (int32_t k = 0; k < std::max(threads, 1); k++)
            pool.emplace_back([&] {
                int64_t local = 0;
                for (;;) {
                    int64_t i0 = next.fetch_add(64);
                    if (i0 >= p1) break;
                    int64_t i1 = std::min(i0 + 64, p1);
                    for (int64_t i = i0; i < i1; i++) {
                        std::vector<float> q(L + i * d, L + (i + 1) * d);
                        auto ids = balltree_within(tree, q, tau);
                        if (self_join) {
                            for (uint64_t id : ids)
                                if (static_cast<int64_t>(id) > i) local++;
                        } else {
                            local += static_cast<int64_t>(ids.size());
                        }
                    }
                }
                total += local;
            });
        for (auto& t : pool) t.join();
        auto t2 = std::chrono::steady_clock::now();
        if (build_s) *build_s = std::chrono::duration<double>(t1 - t0).count();
        if (probe_s) *probe_s = std::chrono::duration<double>(t2 - t1).count();
        return total;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// The same build + probe as ref_join_probe_timed, returning the pairs:
// probe rows [0, nL) of L against all of R, per probe row the ids
// balltree_within returns (ascending), probe rows in order.  *out_l / *out_r
// are malloc'd (ref_free).  Returns the pair count or -1.
REF_API int64_t ref_join_probe_pairs(const float* L, int64_t nL, const float* R, int64_t nR,
                                     int32_t d, double tau, int32_t threads, int32_t** out_l,
                                     int32_t** out_r, double* build_s, double* probe_s) {
    try {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::pair<std::vector<float>, uint64_t>> pts;
        pts.reserve(static_cast<size_t>(nR));
        for (int64_t j = 0; j < nR; j++)
            pts.emplace_back(std::vector<float>(R + j * d, R + (j + 1) * d),
                             static_cast<uint64_t>(j));
        BallTreeIndex tree = build_balltree(pts);
        auto t1 = std::chrono::steady_clock::now();
        std::vector<std::vector<uint64_t>> hits(static_cast<size_t>(nL));
        std::atomic<int64_t> next{0};
        std::vector<std::thread> pool;
        for (int32_t k = 0; k < std::max(threads, 1); k++)
            pool.emplace_back([&] {
                for (;;) {
                    int64_t i0 = next.fetch_add(16);
                    if (i0 >= nL) break;
                    int64_t i1 = std::min<int64_t>(i0 + 16, nL);
                    for (int64_t i = i0; i < i1; i++) {
                        std::vector<float> q(L + i * d, L + (i + 1) * d);
                        hits[static_cast<size_t>(i)] = balltree_within(tree, q, tau);
                    }
                }
            });
        for (auto& t : pool) t.join();
        auto t2 = std::chrono::steady_clock::now();
        int64_t n = 0;
        for (const auto& h : hits) n += static_cast<int64_t>(h.size());
        *out_l = static_cast<int32_t*>(std::malloc(static_cast<size_t>(std::max<int64_t>(n, 1)) * 4));
        *out_r = static_cast<int32_t*>(std::malloc(static_cast<size_t>(std::max<int64_t>(n, 1)) * 4));
        int64_t o = 0;
        for (int64_t i = 0; i < nL; i++)
            for (uint64_t id : hits[static_cast<size_t>(i)]) {
                (*out_l)[o] = static_cast<int32_t>(i);
                (*out_r)[o] = static_cast<int32_t>(id);
                o++;
            }
        if (build_s) *build_s = std::chrono::duration<double>(t1 - t0).count();
        if (probe_s) *probe_s = std::chrono::duration<double>(t2 - t1).count();
        return n;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// PlanNode::dedup over memory tuples (src/query.cpp:535-582, executed by
// compile_dedup): item i carries the unique label "i", so each output
// group's group_labels lists its members and its lineage parent is the
// representative.  rep_of[i] = index of item i's representative.
REF_API int ref_dedup(const float* X, int64_t n, int32_t d, double tau, int64_t* rep_of,
                      int64_t* n_reps) {
    try {
        auto items = make_vecs(X, n, d, 1);
        std::vector<Tuple> tuples;
        tuples.reserve(items.size());
        for (int64_t i = 0; i < n; i++) {
            Patch& p = items[static_cast<size_t>(i)];
            p.meta.emplace("label", MetaValue{std::to_string(i)});
            LineageStep step;
            step.op_name = "make_patch";
            step.source = FrameId{"synthetic", 0};
            p.lineage.push_back(std::move(step));
            tuples.push_back(Tuple{p});
        }
        ExecContext ctx;
        auto plan = PlanNode::dedup(PlanNode::memory(std::move(tuples)), tau);
        auto res = execute(*plan, ctx);
        for (int64_t i = 0; i < n; i++) rep_of[i] = -1;
        for (const auto& t : res.tuples) {
            const int64_t rep = static_cast<int64_t>(t[0].lineage[0].parent_id()) - 1;
            for (const auto& lab : t[0].meta_str_list("group_labels"))
                rep_of[std::stoll(lab)] = rep;
        }
        *n_reps = static_cast<int64_t>(res.tuples.size());
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// dedup_stream (src/query.cpp:1063-1092): indices of the kept patches, in
// order.  Returns the count; kept must hold n entries.
REF_API int64_t ref_dedup_stream(const float* X, int64_t n, int32_t d, double tau,
                                 int64_t* kept) {
    try {
        auto items = make_vecs(X, n, d, 1);
        auto s = dedup_stream(std::make_unique<VectorStream<Patch>>(std::move(items)), tau);
        int64_t m = 0;
        while (auto p = s->next()) kept[m++] = static_cast<int64_t>(p->patch_id) - 1;
        return m;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

namespace {
std::vector<Tuple> tuples_of(const std::vector<Patch>& ps) {
    std::vector<Tuple> out;
    out.reserve(ps.size());
    for (const auto& p : ps) out.push_back(Tuple{p});
    return out;
}
}  // namespace

// PlanNode::nl_join(memory(L), memory(R), within_of(0, 1, radius))
// (src/query.cpp:142-151, 705-744): (left index, right index) in the
// nested-loop emission order.  Caller frees with ref_free.
REF_API int ref_nl_within(const float* L, int64_t nL, const float* R, int64_t nR, int32_t d,
                          double radius, int64_t* out_count, int32_t** out_left,
                          int32_t** out_right) {
    try {
        auto left = make_vecs(L, nL, d, 1);
        auto right = make_vecs(R, nR, d, (1ull << 32) + 1);
        ExecContext ctx;
        auto plan = PlanNode::nl_join(PlanNode::memory(tuples_of(left)),
                                      PlanNode::memory(tuples_of(right)),
                                      Predicate::within_of(0, 1, radius));
        auto res = execute(*plan, ctx);
        int64_t n = static_cast<int64_t>(res.tuples.size());
        int32_t* a = static_cast<int32_t*>(std::malloc(std::max<int64_t>(n, 1) * sizeof(int32_t)));
        int32_t* b = static_cast<int32_t*>(std::malloc(std::max<int64_t>(n, 1) * sizeof(int32_t)));
        for (int64_t k = 0; k < n; k++) {
            a[k] = static_cast<int32_t>(res.tuples[k][0].patch_id - 1);
            b[k] = static_cast<int32_t>(res.tuples[k][1].patch_id - ((1ull << 32) + 1));
        }
        *out_count = n;
        *out_left = a;
        *out_right = b;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// The q1 near-duplicate-frame query (src/bench.cpp:695-730) on in-memory
// frames: whole-image colour histograms (generate whole_image +
// color_histogram, B bins), then select(sim_join(h, h, tau), frameno != frameno).
// Returns (frame a, frame b) per result tuple in emission order; free with ref_free.
REF_API int ref_q1(const uint8_t* frames, int64_t n, int32_t H, int32_t W, int32_t bins,
                   double tau, int64_t* out_count, int32_t** out_a, int32_t** out_b) {
    try {
        GeneratorSpec g;
        g.kind = GeneratorKind::whole_image;
        TransformerSpec t;
        t.kind = TransformerKind::color_histogram;
        t.bins = static_cast<uint32_t>(bins);
        auto stream = transform(
            generate(std::make_unique<VectorStream<Frame>>(make_frames(frames, n, H, W, 0)), g),
            t);
        std::vector<Patch> hist;
        while (auto p = stream->next()) hist.push_back(std::move(*p));
        ExecContext ctx;
        auto plan = PlanNode::select(
            PlanNode::sim_join(PlanNode::memory(tuples_of(hist)),
                               PlanNode::memory(tuples_of(hist)), tau),
            Predicate::cmp_of(CmpOp::ne, Operand::meta(0, "frameno"),
                              Operand::meta(1, "frameno")));
        auto res = execute(*plan, ctx);
        int64_t m = static_cast<int64_t>(res.tuples.size());
        int32_t* a = static_cast<int32_t*>(std::malloc(std::max<int64_t>(m, 1) * sizeof(int32_t)));
        int32_t* b = static_cast<int32_t*>(std::malloc(std::max<int64_t>(m, 1) * sizeof(int32_t)));
        for (int64_t k = 0; k < m; k++) {
            a[k] = static_cast<int32_t>(res.tuples[k][0].meta_int("frameno"));
            b[k] = static_cast<int32_t>(res.tuples[k][1].meta_int("frameno"));
        }
        *out_count = m;
        *out_a = a;
        *out_b = b;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// VideoStore::ingest (src/storage.cpp:311-378): writes frames 0..n-1 of
// video `vid` into a store at `path` (layout 0 frame_file, 1 encoded_file,
// 2 segmented_file; quant_step 0 = lossless, else lossy with that step).
REF_API int ref_store_write(const uint8_t* frames, int64_t n, int32_t H, int32_t W, int32_t layout,
                            int32_t quant_step, int32_t clip_len, const char* path) {
    try {
        auto fs = make_frames(frames, n, H, W, 0);
        StoreDescriptor desc;
        desc.layout = static_cast<Layout>(layout);
        desc.codec = quant_step ? CodecConfig::lossy(static_cast<uint8_t>(quant_step))
                                : CodecConfig::lossless();
        desc.clip_len = static_cast<uint32_t>(clip_len);
        desc.path = path;
        VectorStream<Frame> s(std::move(fs));
        VideoStore::ingest(s, desc);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return code_of(e);
    }
}

// VideoStore::open + scan([lo, hi)) (src/storage.cpp:380-501): the decoded
// frames into out [hi-lo, H, W, 3]; returns the frame count (or -code).
REF_API int64_t ref_store_scan(const char* path, int64_t lo, int64_t hi, uint8_t* out) {
    try {
        auto vs = VideoStore::open(path);
        IoCounters io;
        std::optional<std::pair<uint64_t, uint64_t>> range;
        if (lo >= 0) range = std::make_pair(static_cast<uint64_t>(lo), static_cast<uint64_t>(hi));
        auto s = vs.scan(range, io);
        int64_t k = 0;
        while (auto f = s->next()) {
            std::memcpy(out + k * f->pixels.size(), f->pixels.data(), f->pixels.size());
            k++;
        }
        return k;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -code_of(e);
    }
}

#include "json.hpp"

namespace {
nlohmann::json patch_json(const Patch& p, bool with_data) {
    using nlohmann::json;
    json d;
    d["id"] = p.patch_id;
    d["shape"] = p.shape;
    json meta = json::object();
    for (const auto& [k, v] : p.meta) {
        if (const auto* i = std::get_if<int64_t>(&v)) meta[k] = *i;
        else if (const auto* f = std::get_if<double>(&v)) meta[k] = *f;
        else if (const auto* s = std::get_if<std::string>(&v)) meta[k] = *s;
        else if (const auto* b = std::get_if<BoundingBox>(&v)) meta[k] = {b->x1, b->y1, b->x2, b->y2};
        else meta[k] = std::get<std::vector<std::string>>(v);
    }
    d["meta"] = meta;
    json lin = json::array();
    for (const auto& s : p.lineage) {
        json st;
        st["op"] = s.op_name;
        if (s.kind() == SourceKind::base_frame) st["frame"] = {s.frame().video_id, s.frame().frame_no};
        else st["parent"] = s.parent_id();
        st["digest"] = s.params_digest;
        if (s.region) st["region"] = {s.region->x1, s.region->y1, s.region->x2, s.region->y2};
        lin.push_back(st);
    }
    d["lineage"] = lin;
    if (with_data) d["data"] = p.data;
    return d;
}
}  // namespace

// patchdb.run_query (bindings/py_module.cpp:168-213) on the reference: parse
// the plan file, materialize its ETL section (materialize_etl, py_module.cpp:
// 68-76), execute the plan.  Returns a malloc'd JSON document
// {"tuples": [[patch, ...], ...]} (patch: id, shape, meta, lineage, data),
// or NULL with ref_last_error set.  reset_ids: restart the patch-id counter.
REF_API char* ref_run_query(const char* plan_json, int32_t with_data, int64_t reset_ids) {
    try {
        if (reset_ids > 0) reset_patch_ids(static_cast<uint64_t>(reset_ids));
        PlanFile pf = PlanFile::parse(plan_json);
        if (!pf.plan) throw ValidationError("plan file has no plan section");
        auto stages = plan_stages(pf);
        if (!stages.empty()) {
            auto violations = validate_pipeline(stages);
            // check_stages (bindings/py_module.cpp:54-66): every violation
            std::string msg;
            for (const auto& v : violations) {
                if (!msg.empty()) msg += "; ";
                msg += "stage " + std::to_string(v.stage) + ": " + v.message;
            }
            if (!msg.empty()) throw ValidationError(msg);
        }
        std::map<std::string, PatchCollection> cols;
        if (pf.etl) {
            const EtlSection& etl = *pf.etl;
            auto it = pf.stores.find(etl.store);
            std::string store_path = it == pf.stores.end() ? etl.store : it->second;
            VideoStore vs = VideoStore::open(store_path);
            IoCounters io;
            auto stream = generate(vs.scan(std::nullopt, io), etl.generator);
            for (const auto& t : etl.transformers) stream = transform(std::move(stream), t);
            cols.emplace(etl.name, PatchCollection::materialize(*stream, etl.output));
        }
        for (const auto& [alias, path] : pf.collections)
            cols.emplace(alias, PatchCollection::open(path, false));
        std::map<std::string, VideoStore> stores;
        for (const auto& [alias, path] : pf.stores) stores.emplace(alias, VideoStore::open(path));
        ExecContext ctx;
        for (const auto& [alias, col] : cols) ctx.collections[alias] = &col;
        for (const auto& [alias, vs] : stores) ctx.videos[vs.video_id()] = &vs;
        ExecResult res = execute(*pf.plan, ctx);
        nlohmann::json out;
        out["tuples"] = nlohmann::json::array();
        for (const auto& t : res.tuples) {
            nlohmann::json slots = nlohmann::json::array();
            for (const auto& p : t) slots.push_back(patch_json(p, with_data != 0));
            out["tuples"].push_back(slots);
        }
        const std::string s = out.dump();
        char* buf = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(buf, s.c_str(), s.size() + 1);
        return buf;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}
