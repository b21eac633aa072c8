// videostore.cu -- the frame source: reads the reference's
// VideoStore files and feeds K1.
//
// Format (all integers big-endian, include/patchdb/bytes.hpp):
//   record store   src/record_store.cpp: "PDBS0001", values, then an index of
//                  (u32 key length, key, u64 offset, u64 length) and a footer
//                  (u64 index offset, u64 entry count, "PDBSIDX1")
//   descriptor     key 0xFF x 8 (src/storage.cpp:292-304, 380-393): u8 layout,
//                  u8 codec mode, u8 quant step, u32 clip_len, u32 width,
//                  u32 height, u64 frame count, str8 video id
//   frame_file     key u64 frame_no -> u32 w, u32 h, u8 channels, u8 0, pixels
//                  (parse_frame_record, src/storage.cpp:274-290)
//   encoded_file   key 0 -> one clip holding every frame
//   segmented_file key c*clip_len -> the clip of frames [c*clip_len, ...)
//   clip           u32 frames, u32 w, u32 h, u8 mode, u8 step, then one
//                  zlib stream: frame 0 intra, later frames as byte-wise
//                  wrapping deltas against the previous decoded frame
//                  (ClipEncoder / ClipDecoder, src/storage.cpp:170-261)
//
// Decoding is host work by nature (zlib): clips decode in parallel on host
// threads into pinned memory, each inflated clip undoes its deltas in place,
// and the frames go to the device in chunks that K1 consumes while the next
// chunk is decoded and copied.
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "pdb_internal.cuh"

namespace pdb {

namespace {

uint32_t be32(const uint8_t* p) {
    return (uint32_t{p[0]} << 24) | (uint32_t{p[1]} << 16) | (uint32_t{p[2]} << 8) | p[3];
}
uint64_t be64(const uint8_t* p) { return (uint64_t{be32(p)} << 32) | be32(p + 4); }

struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) std::fclose(f);
    }
};

}  // namespace

struct Store {
    std::string path;
    std::map<std::string, std::pair<uint64_t, uint64_t>> index;  // key -> (offset, length)
    uint8_t layout = 0, codec = 0, quant = 0;
    uint32_t clip_len = 0, width = 0, height = 0;
    uint64_t frames = 0;
    std::string video_id;
    // pinned staging of pdb_store_featurize, kept between calls
    mutable uint8_t* pin[2] = {nullptr, nullptr};
    mutable size_t pin_bytes = 0;
    ~Store() {
        if (pin[0]) cudaFreeHost(pin[0]);
        if (pin[1]) cudaFreeHost(pin[1]);
    }

    std::string read(uint64_t off, uint64_t len) const {
        File fh;
        fh.f = std::fopen(path.c_str(), "rb");
        if (!fh.f) fail(PDB_ERR_IO, "cannot open " + path);
        std::string v(len, '\0');
        if (std::fseek(fh.f, static_cast<long>(off), SEEK_SET) != 0 ||
            std::fread(v.data(), 1, len, fh.f) != len)
            fail(PDB_ERR_IO, "read failed on " + path);
        return v;
    }
    bool get(const std::string& key, std::string& out) const {
        auto it = index.find(key);
        if (it == index.end()) return false;
        out = read(it->second.first, it->second.second);
        return true;
    }
    static std::string key_u64(uint64_t v) {
        std::string k(8, '\0');
        for (int i = 0; i < 8; i++) k[i] = static_cast<char>(v >> (56 - 8 * i));
        return k;
    }
};

namespace {

std::unique_ptr<Store> open_store(const char* path) {
    auto st = std::make_unique<Store>();
    st->path = path;
    File fh;
    fh.f = std::fopen(path, "rb");
    if (!fh.f) fail(PDB_ERR_IO, std::string("cannot open record store at ") + path);
    std::fseek(fh.f, 0, SEEK_END);
    const long size = std::ftell(fh.f);
    constexpr long kMagic = 8, kFooter = 24;
    if (size < kMagic + kFooter) fail(PDB_ERR_IO, std::string("record store ") + path + " is truncated");
    uint8_t head[8], foot[24];
    std::fseek(fh.f, 0, SEEK_SET);
    if (std::fread(head, 1, 8, fh.f) != 8 || std::memcmp(head, "PDBS0001", 8) != 0)
        fail(PDB_ERR_IO, std::string("record store ") + path + " has a bad file magic");
    std::fseek(fh.f, size - kFooter, SEEK_SET);
    if (std::fread(foot, 1, 24, fh.f) != 24 || std::memcmp(foot + 16, "PDBSIDX1", 8) != 0)
        fail(PDB_ERR_IO, std::string("record store ") + path + " has a bad footer magic");
    const uint64_t index_off = be64(foot), n_entries = be64(foot + 8);
    if (index_off < static_cast<uint64_t>(kMagic) ||
        index_off > static_cast<uint64_t>(size - kFooter))
        fail(PDB_ERR_IO, std::string("record store ") + path + " has a corrupt index offset");
    std::vector<uint8_t> raw(static_cast<size_t>(size - kFooter) - index_off);
    std::fseek(fh.f, static_cast<long>(index_off), SEEK_SET);
    if (std::fread(raw.data(), 1, raw.size(), fh.f) != raw.size())
        fail(PDB_ERR_IO, std::string("record store ") + path + ": cannot read index");
    size_t p = 0;
    auto need = [&](size_t n) {
        if (p + n > raw.size()) fail(PDB_ERR_IO, "record store index is truncated");
    };
    for (uint64_t i = 0; i < n_entries; i++) {
        need(4);
        const uint32_t kl = be32(&raw[p]);
        p += 4;
        need(kl + 16);
        std::string key(reinterpret_cast<const char*>(&raw[p]), kl);
        p += kl;
        st->index[key] = {be64(&raw[p]), be64(&raw[p + 8])};
        p += 16;
    }
    std::string d;
    if (!st->get(std::string(8, '\xFF'), d)) fail(PDB_ERR_IO, std::string("store ") + path + " has no descriptor record");
    const uint8_t* q = reinterpret_cast<const uint8_t*>(d.data());
    if (d.size() < 24) fail(PDB_ERR_IO, "store descriptor is truncated");
    st->layout = q[0];
    st->codec = q[1];
    st->quant = q[2];
    st->clip_len = be32(q + 3);
    st->width = be32(q + 7);
    st->height = be32(q + 11);
    st->frames = be64(q + 15);
    const size_t idl = q[23];
    if (d.size() < 24 + idl) fail(PDB_ERR_IO, "store descriptor is truncated");
    st->video_id.assign(d.data() + 24, idl);
    if (st->layout > 2) fail(PDB_ERR_IO, "unknown storage layout");
    return st;
}

// Inflates a clip blob; frames [0, upto) land in out (frame-major), with the
// deltas undone.  Frames >= upto are not produced (the stream is read no
// further), like ClipDecoder::next stopping early.
void decode_clip(const std::string& blob, uint32_t W, uint32_t H, uint32_t upto, uint8_t* out) {
    if (blob.size() < 14) fail(PDB_ERR_IO, "clip blob truncated");
    const uint8_t* b = reinterpret_cast<const uint8_t*>(blob.data());
    const uint32_t nf = be32(b), w = be32(b + 4), h = be32(b + 8);
    if (w != W || h != H) fail(PDB_ERR_IO, "clip size does not match the store");
    upto = std::min(upto, nf);
    const size_t fb = static_cast<size_t>(W) * H * 3;
    z_stream zs{};
    if (inflateInit(&zs) != Z_OK) fail(PDB_ERR_IO, "inflateInit failed");
    zs.next_in = const_cast<Bytef*>(b + 14);
    zs.avail_in = static_cast<uInt>(blob.size() - 14);
    const size_t want = fb * upto;
    size_t done = 0;
    bool end = false;
    while (done < want) {
        if (end) {
            inflateEnd(&zs);
            fail(PDB_ERR_IO, "compressed stream ended early");
        }
        zs.next_out = out + done;
        const size_t chunk = std::min<size_t>(want - done, size_t{1} << 30);
        zs.avail_out = static_cast<uInt>(chunk);
        const int rc = inflate(&zs, Z_NO_FLUSH);
        done += chunk - zs.avail_out;
        if (rc == Z_STREAM_END) end = true;
        else if (rc != Z_OK) {
            inflateEnd(&zs);
            fail(PDB_ERR_IO, "inflate error " + std::to_string(rc));
        }
    }
    inflateEnd(&zs);
    // frame k = delta_k + frame k-1 (byte-wise, wrapping)
    for (uint32_t k = 1; k < upto; k++) {
        uint8_t* cur = out + k * fb;
        const uint8_t* prev = cur - fb;
        for (size_t i = 0; i < fb; i++) cur[i] = static_cast<uint8_t>(cur[i] + prev[i]);
    }
}

}  // namespace

// Decodes frames [lo, hi) into host memory out [hi-lo, H, W, 3] on
// `threads` host threads (segmented clips and frame records in parallel).
void store_read_host(const Store& st, uint64_t lo, uint64_t hi, uint8_t* out, int threads) {
    const size_t fb = static_cast<size_t>(st.width) * st.height * 3;
    if (lo >= hi) return;
    threads = std::max(1, threads);
    std::vector<std::thread> pool;
    std::atomic<uint64_t> next{0};
    std::string first_error;
    std::atomic<int> error_status{0};
    auto run = [&](auto&& body, uint64_t n_items) {
        next = 0;
        pool.clear();
        for (int t = 0; t < std::min<int64_t>(threads, static_cast<int64_t>(n_items)); t++)
            pool.emplace_back([&] {
                for (;;) {
                    const uint64_t k = next.fetch_add(1);
                    if (k >= n_items || error_status.load()) break;
                    try {
                        body(k);
                    } catch (const Failure& f) {
                        int z = 0;
                        if (error_status.compare_exchange_strong(z, f.status)) first_error = f.msg;
                    }
                }
            });
        for (auto& th : pool) th.join();
        if (error_status.load()) fail(error_status.load(), first_error);
    };
    if (st.layout == 0) {  // frame_file: one raw record per frame
        run([&](uint64_t k) {
            const uint64_t no = lo + k;
            std::string v;
            if (!st.get(Store::key_u64(no), v)) fail(PDB_ERR_IO, "missing frame record");
            const uint8_t* q = reinterpret_cast<const uint8_t*>(v.data());
            if (v.size() < 10 || q[9] != 0) fail(PDB_ERR_IO, "unknown frame record encoding byte");
            if (v.size() - 10 != fb) fail(PDB_ERR_IO, "frame record has wrong pixel count");
            std::memcpy(out + k * fb, q + 10, fb);
        }, hi - lo);
    } else if (st.layout == 1) {  // encoded_file: one sequential clip from frame 0
        std::string blob;
        if (!st.get(Store::key_u64(0), blob)) return;
        std::vector<uint8_t> all(fb * hi);
        decode_clip(blob, st.width, st.height, static_cast<uint32_t>(hi), all.data());
        std::memcpy(out, all.data() + lo * fb, (hi - lo) * fb);
    } else {  // segmented_file: independent clips of clip_len frames
        const uint64_t cl = st.clip_len;
        const uint64_t c0 = lo / cl, c1 = (hi + cl - 1) / cl;
        run([&](uint64_t k) {
            const uint64_t start = (c0 + k) * cl;
            std::string blob;
            if (!st.get(Store::key_u64(start), blob)) fail(PDB_ERR_IO, "missing clip record");
            const uint64_t upto = std::min(hi, start + cl) - start;
            if (start >= lo && start + upto <= hi) {
                decode_clip(blob, st.width, st.height, static_cast<uint32_t>(upto),
                            out + (start - lo) * fb);
            } else {  // a clip straddling lo: decode whole, keep the range
                std::vector<uint8_t> tmp(fb * upto);
                decode_clip(blob, st.width, st.height, static_cast<uint32_t>(upto), tmp.data());
                const uint64_t a = std::max(lo, start);
                std::memcpy(out + (a - lo) * fb, tmp.data() + (a - start) * fb,
                            (start + upto - a) * fb);
            }
        }, c1 - c0);
    }
}

}  // namespace pdb

#define PDB_API extern "C" __attribute__((visibility("default")))

using pdb::Store;

namespace {
// capi.cu's guard: Failure / allocation errors -> status codes.
template <class F>
int pdb_guarded(F&& body) {
    pdb::clear_error();
    try {
        body();
        return PDB_OK;
    } catch (const pdb::Failure& f) {
        pdb::set_error(f.msg);
        return f.status;
    } catch (const std::bad_alloc&) {
        pdb::set_error("host allocation failed");
        return PDB_ERR_OUT_OF_MEMORY;
    } catch (...) {
        pdb::set_error("unexpected exception");
        return PDB_ERR_CUDA;
    }
}
}  // namespace

PDB_API int pdb_store_open(const char* path, pdb_store** out) {
    if (out) *out = nullptr;
    return pdb_guarded([&] {
        if (!path || !out) pdb::fail(PDB_ERR_INVALID_ARGUMENT, "null argument");
        *out = reinterpret_cast<pdb_store*>(pdb::open_store(path).release());
    });
}

PDB_API void pdb_store_close(pdb_store* s) { delete reinterpret_cast<Store*>(s); }

PDB_API int pdb_store_describe(const pdb_store* s, pdb_store_info* info) {
    return pdb_guarded([&] {
        if (!s || !info) pdb::fail(PDB_ERR_INVALID_ARGUMENT, "null argument");
        const Store& st = *reinterpret_cast<const Store*>(s);
        info->frame_count = static_cast<int64_t>(st.frames);
        info->width = static_cast<int32_t>(st.width);
        info->height = static_cast<int32_t>(st.height);
        info->layout = st.layout;
        info->codec_mode = st.codec;
        info->quant_step = st.quant;
        info->clip_len = static_cast<int32_t>(st.clip_len);
        std::snprintf(info->video_id, sizeof(info->video_id), "%s", st.video_id.c_str());
    });
}

namespace {
// VideoStore::scan's range rule (src/storage.cpp:397-404): lo >= hi is a
// ConfigError; both ends clamp to the frame count.
void clamp_range(const Store& st, int64_t lo, int64_t hi, uint64_t& a, uint64_t& b) {
    if (lo < 0 || hi < 0) {
        a = 0;
        b = st.frames;
        return;
    }
    if (lo >= hi) pdb::fail(PDB_ERR_CONFIG, "scan range low bound must be below high bound");
    a = std::min<uint64_t>(static_cast<uint64_t>(lo), st.frames);
    b = std::min<uint64_t>(static_cast<uint64_t>(hi), st.frames);
}
}  // namespace

PDB_API int pdb_store_read(const pdb_store* s, int64_t lo, int64_t hi, uint8_t* frames,
                           int64_t* n_frames, int32_t threads) {
    if (n_frames) *n_frames = 0;
    return pdb_guarded([&] {
        if (!s || !n_frames) pdb::fail(PDB_ERR_INVALID_ARGUMENT, "null argument");
        const Store& st = *reinterpret_cast<const Store*>(s);
        uint64_t a, b;
        clamp_range(st, lo, hi, a, b);
        if (a < b && !frames) pdb::fail(PDB_ERR_INVALID_ARGUMENT, "null frame buffer");
        pdb::store_read_host(st, a, b, frames, threads);
        *n_frames = static_cast<int64_t>(b > a ? b - a : 0);
    });
}

PDB_API int pdb_store_featurize(const pdb_store* s, int64_t lo, int64_t hi, int32_t tile_h,
                                int32_t tile_w, int32_t bins, int32_t mode, float* d_features,
                                int64_t* n_frames, int32_t threads, void* stream) {
    if (n_frames) *n_frames = 0;
    return pdb_guarded([&] {
        if (!s || !n_frames) pdb::fail(PDB_ERR_INVALID_ARGUMENT, "null argument");
        const Store& st = *reinterpret_cast<const Store*>(s);
        uint64_t a, b;
        clamp_range(st, lo, hi, a, b);
        const int32_t H = static_cast<int32_t>(st.height), W = static_cast<int32_t>(st.width);
        if (pdb::hist_dim(bins, mode) < 0) pdb::fail(PDB_ERR_CONFIG, "bad histogram bins / mode");
        if (tile_w < 1 || tile_h < 1) pdb::fail(PDB_ERR_CONFIG, "tile size must be positive");
        pdb::device_ctx();
        const int64_t n = static_cast<int64_t>(b > a ? b - a : 0);
        *n_frames = n;
        if (n == 0) return;
        if (!d_features) pdb::fail(PDB_ERR_INVALID_ARGUMENT, "null feature buffer");
        cudaStream_t cs = stream ? static_cast<cudaStream_t>(stream) : cudaStreamPerThread;
        const size_t fb = static_cast<size_t>(H) * W * 3;
        const int64_t tpf = static_cast<int64_t>(W / tile_w) * (H / tile_h);
        const int D = pdb::hist_dim(bins, mode);
        // Decoding (zlib, host) is the bound: give it every thread.  Ranges up
        // to 2 GB decode in one parallel pass into cached pinned memory;
        // longer ones go in chunks of one clip per thread, chunk k+1
        // decoding while chunk k is copied and featurized.
        const int64_t cl = std::max<int64_t>(st.clip_len, 1);
        const int64_t per_thread = st.layout == 2 ? cl : 8;
        int64_t chunk = per_thread * std::max(threads, 1);
        if (static_cast<size_t>(n) * fb <= (size_t{2} << 30)) chunk = n;
        if (st.layout == 1) {  // sequential codec: decode once, then stream
            pdb::DevBuf<uint8_t> dF(static_cast<size_t>(n) * fb, cs);
            std::vector<uint8_t> host(static_cast<size_t>(n) * fb);
            pdb::store_read_host(st, a, b, host.data(), threads);
            PDB_CUDA(cudaMemcpyAsync(dF.p, host.data(), host.size(), cudaMemcpyHostToDevice, cs));
            pdb::launch_featurize_tiles(dF.p, n, H, W, tile_h, tile_w, bins, mode, d_features, cs);
            PDB_CUDA(cudaStreamSynchronize(cs));
            return;
        }
        const size_t need = static_cast<size_t>(chunk) * fb;
        if (st.pin_bytes < need) {
            for (auto& p : st.pin) {
                if (p) cudaFreeHost(p);
                p = nullptr;
            }
            st.pin_bytes = 0;
            for (auto& p : st.pin)
                if (cudaHostAlloc(reinterpret_cast<void**>(&p), need, cudaHostAllocDefault) !=
                    cudaSuccess) {
                    cudaGetLastError();
                    pdb::fail(PDB_ERR_OUT_OF_MEMORY, "pinned staging allocation failed");
                }
            st.pin_bytes = need;
        }
        uint8_t* const* pin = st.pin;
        pdb::DevBuf<uint8_t> dF(static_cast<size_t>(chunk) * fb * 2, cs);
        cudaEvent_t done[2];
        PDB_CUDA(cudaEventCreateWithFlags(&done[0], cudaEventDisableTiming));
        PDB_CUDA(cudaEventCreateWithFlags(&done[1], cudaEventDisableTiming));
        int k = 0;
        for (int64_t f0 = 0; f0 < n; f0 += chunk, k ^= 1) {
            const int64_t cnt = std::min(chunk, n - f0);
            PDB_CUDA(cudaEventSynchronize(done[k]));  // staging slot k free again
            pdb::store_read_host(st, a + f0, a + f0 + cnt, pin[k], threads);
            uint8_t* dst = dF.p + static_cast<size_t>(k) * chunk * fb;
            PDB_CUDA(cudaMemcpyAsync(dst, pin[k], static_cast<size_t>(cnt) * fb,
                                     cudaMemcpyHostToDevice, cs));
            PDB_CUDA(cudaEventRecord(done[k], cs));
            pdb::launch_featurize_tiles(dst, cnt, H, W, tile_h, tile_w, bins, mode,
                                        d_features + f0 * tpf * D, cs);
        }
        PDB_CUDA(cudaStreamSynchronize(cs));
        cudaEventDestroy(done[0]);
        cudaEventDestroy(done[1]);
    });
}
