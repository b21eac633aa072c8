// dedup.cu -- near-duplicate grouping on the tau-graph.
//
// Reference semantics: run_dedup (src/query.cpp:535-566) behind
// PlanNode::dedup, and dedup_stream (src/query.cpp:1063-1092).  Items are
// scanned in order; item i is kept as a representative iff no kept
// representative lies within tau (euclidean <= tau, src/index.cpp:69-76);
// otherwise it joins the nearest kept representative, the earliest on ties.
//
// B200 plan:
//   1. the tau-graph: every pair i < j with euclidean <= tau, from the
//      similarity self-join (K2 tensor-core screen + K3 exact re-check), so
//      the graph is exactly the reference's set of "within tau" relations;
//   2. CSR of each item's lower neighbours: keys (j << 32 | i) radix-sorted;
//   3. the greedy scan as rounds: an undecided item becomes a non-rep as soon
//      as one lower neighbour is a rep, and a rep once all lower neighbours
//      are decided non-reps.  Statuses only move from undecided to final and
//      each final value is the sequential scan's, so the rounds reproduce it
//      exactly; a round costs one pass over the undecided items' edges;
//   4. attach: a non-rep's representative is the rep neighbour with the
//      smallest distance -- recomputed with the reference's fp64 chain, since
//      ties between fp32-rounded distances need not be ties in fp64 -- the
//      lowest index on ties.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>

#include "exact.cuh"
#include "pdb_internal.cuh"
#include "tc_ptx.cuh"

namespace pdb {

namespace {

__global__ void k_graph_keys(const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                             int64_t n, unsigned long long* __restrict__ keys) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x)
        keys[k] = (static_cast<unsigned long long>(static_cast<uint32_t>(right[k])) << 32) |
                  static_cast<uint32_t>(left[k]);
}

// off[i] = first key with upper word >= i (keys sorted), i = 0..n; also
// clears the item statuses and the round / representative counters.
__global__ void k_csr_offsets(const unsigned long long* __restrict__ keys, int64_t m, int64_t n,
                              int64_t* __restrict__ off, uint8_t* __restrict__ status,
                              unsigned long long* __restrict__ cnt) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    if (blockIdx.x == 0 && threadIdx.x < 3) cnt[threadIdx.x] = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i <= n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (i < n) status[i] = 0;
        const unsigned long long t = static_cast<unsigned long long>(i) << 32;
        int64_t lo = 0, hi = m;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < t) lo = mid + 1;
            else hi = mid;
        }
        off[i] = lo;
    }
}

constexpr uint8_t kUndecided = 0, kRep = 1, kMember = 2;
// at most this many undecided items after a host check: the sequential tail
constexpr unsigned int kTailSwitch = 65536;

// One round of the greedy scan over the still undecided items.
// Round counters are double-buffered: a round counts into cnt[r & 1] and
// clears cnt[(r + 1) & 1] for the next one (the previous round, which used
// it, has completed), so rounds chain without host memsets.
__global__ void k_dedup_round(const unsigned long long* __restrict__ keys,
                              const int64_t* __restrict__ off, int64_t n,
                              uint8_t* status, unsigned long long* cnt, int r) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    unsigned int* undecided = reinterpret_cast<unsigned int*>(cnt + (r & 1));
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[(r + 1) & 1] = 0;
    unsigned int left = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (status[i] != kUndecided) continue;
        bool any_rep = false, all_done = true;
        PDB_DCHECK(off[i] <= off[i + 1]);
        for (int64_t e = off[i]; e < off[i + 1]; e++) {
            const int64_t j = static_cast<int64_t>(keys[e] & 0xffffffffull);
            PDB_DCHECK(j >= 0 && j < i && static_cast<int64_t>(keys[e] >> 32) == i);
            // volatile: statuses decided earlier in this round may be seen
            const uint8_t sj = *reinterpret_cast<volatile uint8_t*>(status + j);
            if (sj == kRep) {
                any_rep = true;
                break;
            }
            if (sj == kUndecided) all_done = false;
        }
        if (any_rep) status[i] = kMember;
        else if (all_done) status[i] = kRep;
        else left++;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) left += __shfl_xor_sync(0xffffffffu, left, o);
    if ((threadIdx.x & 31) == 0 && left) atomicAdd(undecided, left);
}

// The sequential tail of the greedy scan.  Once few items are undecided
// (dependency chains: a chain of k items needs k rounds), one block decides
// them in index order -- exactly the reference's sequential scan restricted
// to them, since every lower neighbour of an item is final when its turn
// comes.  The sorted undecided list is walked in chunks: the chunk's CSR
// edges are staged in shared memory with each lower neighbour encoded as its
// position in the chunk (>= 0) or its final status outside it (-1 rep, -2
// not), then one thread decides the chunk item by item from shared memory.
// An item with more edges than the stage holds is decided from global
// memory.
constexpr int kTailItems = 4096;

__global__ void __launch_bounds__(1024)
k_dedup_tail(const unsigned long long* __restrict__ keys, const int64_t* __restrict__ off,
             const int32_t* __restrict__ list, int64_t U, uint8_t* status, int edge_cap) {
    extern __shared__ int32_t tsm[];
    int32_t* s_item = tsm;                      // [kTailItems]
    int32_t* s_beg = s_item + kTailItems;       // [kTailItems + 1] edge offsets
    int32_t* s_edge = s_beg + kTailItems + 1;   // [edge_cap] codes
    uint8_t* s_stat = reinterpret_cast<uint8_t*>(s_edge + edge_cap);  // [kTailItems]
    __shared__ int32_t s_c;
    const int t = threadIdx.x;
    for (int64_t u0 = 0; u0 < U;) {
        // 1. the chunk: as many items as fit kTailItems and edge_cap edges
        const int64_t navail = min(static_cast<int64_t>(kTailItems), U - u0);
        for (int k = t; k < kTailItems; k += blockDim.x) {
            if (k < navail) {
                const int64_t i = list[u0 + k];
                s_item[k] = static_cast<int32_t>(i);
                s_beg[k + 1] = static_cast<int32_t>(min(off[i + 1] - off[i], static_cast<int64_t>(edge_cap) + 1));
            }
        }
        __syncthreads();
        if (t == 0) {
            // serial prefix (kTailItems values) and the cut
            int32_t acc = 0, c = 0;
            s_beg[0] = 0;
            for (int k = 0; k < navail; k++) {
                const int32_t dk = s_beg[k + 1];
                if (acc + dk > edge_cap && c > 0) break;
                acc += min(dk, edge_cap);
                s_beg[k + 1] = acc;
                c++;
                if (dk > edge_cap) break;  // a huge item goes alone (global path)
            }
            s_c = c;
        }
        __syncthreads();
        const int c = s_c;
        const bool global_path = c == 1 && (off[s_item[0] + 1] - off[s_item[0]]) > edge_cap;
        // 2. stage the edges' codes
        if (!global_path) {
            const int32_t ne = s_beg[c];
            for (int e = t; e < ne; e += blockDim.x) {
                int lo = 0, hi = c;  // item k with s_beg[k] <= e < s_beg[k + 1]
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (s_beg[mid] <= e) lo = mid;
                    else hi = mid;
                }
                const int64_t i = s_item[lo];
                const int64_t j = static_cast<int64_t>(keys[off[i] + (e - s_beg[lo])] & 0xffffffffull);
                PDB_DCHECK(j >= 0 && j < i);
                int32_t code;
                int a = 0, b = lo;  // is j an item of this chunk (before i)?
                while (a < b) {
                    const int mid = (a + b) >> 1;
                    if (s_item[mid] < j) a = mid + 1;
                    else b = mid;
                }
                if (a < lo && s_item[a] == j) code = a;
                else code = status[j] == kRep ? -1 : -2;  // final: outside the chunk
                s_edge[e] = code;
            }
        }
        __syncthreads();
        // 3. decide the chunk in order
        if (t == 0) {
            if (global_path) {
                const int64_t i = s_item[0];
                bool rep_nb = false;
                for (int64_t e = off[i]; e < off[i + 1] && !rep_nb; e++)
                    rep_nb = status[keys[e] & 0xffffffffull] == kRep;
                s_stat[0] = rep_nb ? kMember : kRep;
            } else {
                for (int k = 0; k < c; k++) {
                    bool rep_nb = false;
                    for (int32_t e = s_beg[k]; e < s_beg[k + 1]; e++) {
                        const int32_t code = s_edge[e];
                        if (code == -1 || (code >= 0 && s_stat[code] == kRep)) {
                            rep_nb = true;
                            break;
                        }
                    }
                    s_stat[k] = rep_nb ? kMember : kRep;
                }
            }
        }
        __syncthreads();
        // 4. publish the chunk's statuses (later chunks read them as final)
        for (int k = t; k < c; k += blockDim.x) status[s_item[k]] = s_stat[k];
        __threadfence_block();
        __syncthreads();
        u0 += c;
    }
}

struct IsUndecided {
    const uint8_t* status;
    __device__ bool operator()(int32_t i) const { return status[i] == kUndecided; }
};

// rep_of[i]: i for representatives, else the rep neighbour nearest in the
// reference's fp64 distance (lowest index on ties; neighbours ascend).
__global__ void k_dedup_attach(const unsigned long long* __restrict__ keys,
                               const int64_t* __restrict__ off, int64_t n,
                               const uint8_t* __restrict__ status, const float* __restrict__ X,
                               int d, int64_t* __restrict__ rep_of,
                               unsigned long long* __restrict__ n_reps) {
    ptx::pdl_wait();
    ptx::pdl_trigger();
    const bool vec8 = (d % 8 == 0) && (reinterpret_cast<uintptr_t>(X) % 32 == 0);
    unsigned int reps = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        if (status[i] == kRep) {
            rep_of[i] = i;
            reps++;
            continue;
        }
        int64_t best = -1;
        double best_dist = __longlong_as_double(0x7ff0000000000000ll);  // +inf
        for (int64_t e = off[i]; e < off[i + 1]; e++) {
            const int64_t j = static_cast<int64_t>(keys[e] & 0xffffffffull);
            PDB_DCHECK(j >= 0 && j < i);
            if (status[j] != kRep) continue;
            // euclidean(items[i], items[rep]) -- the reference's argument order
            const double dist = exact_dist(X + i * d, X + j * d, d, vec8);
            if (dist < best_dist) {
                best_dist = dist;
                best = j;
            }
        }
        PDB_DCHECK(best >= 0 && best < i);  // every member has a representative neighbour
        rep_of[i] = best;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) reps += __shfl_xor_sync(0xffffffffu, reps, o);
    if ((threadIdx.x & 31) == 0 && reps) atomicAdd(n_reps, static_cast<unsigned long long>(reps));
}

}  // namespace

void run_dedup_dev(const float* d_X, int64_t n, int32_t d, double tau, cudaStream_t s,
                   int64_t* d_rep_of, int64_t* n_reps) {
    *n_reps = 0;
    if (n == 0) return;
    const DeviceCtx& ctx = device_ctx();
    // 1. the tau-graph (i < j, exact euclidean <= tau)
    pdb_join_opts o{};
    o.flags = PDB_JOIN_SELF;
    o.stream = s;
    pdb_dev_pairs g{};
    struct PairsGuard {
        pdb_dev_pairs* p;
        ~PairsGuard() { pdb_dev_pairs_free(p); }
    } guard{&g};
    run_sim_join_dev(d_X, n, d_X, n, d, tau, o, &g, nullptr);
    const int64_t m = g.count;

    // 2. lower-neighbour CSR: keys (j << 32 | i) sorted ascending
    DevBuf<unsigned long long> k_in(static_cast<size_t>(std::max<int64_t>(m, 1)), s),
        keys(static_cast<size_t>(std::max<int64_t>(m, 1)), s);
    DevBuf<int64_t> off(static_cast<size_t>(n) + 1, s);
    const unsigned grid = static_cast<unsigned>(ctx.sm_count * 4);
    if (m > 0) {
        k_graph_keys<<<grid, 256, 0, s>>>(g.left, g.right, m, k_in.p);
        int bits = 1;
        while ((int64_t{1} << bits) < n) bits++;
        size_t tmp_bytes = 0;
        PDB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k_in.p, keys.p, m, 0, 32 + bits, s));
        DevBuf<uint8_t> tmp(tmp_bytes, s);
        PDB_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, k_in.p, keys.p, m, 0, 32 + bits, s));
    }
    // 3. greedy rounds until every item is decided
    DevBuf<uint8_t> status(static_cast<size_t>(n), s);
    DevBuf<unsigned long long> cnt(3, s);  // [0], [1] round counters, [2] representatives
    launch_pdl(k_csr_offsets, dim3(grid), dim3(256), 0, s, static_cast<const unsigned long long*>(keys.p),
               m, n, off.p, status.p, cnt.p);
    PDB_CUDA(cudaGetLastError());
    thread_local unsigned long long* h_cnt = [] {
        void* q = nullptr;
        if (cudaHostAlloc(&q, 16, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            q = nullptr;
        }
        return static_cast<unsigned long long*>(q);
    }();
    unsigned long long local[2];
    unsigned long long* hc = h_cnt ? h_cnt : local;
    int r = 0;
    for (int check = 0;; check++) {
        // a few rounds per host check: most items settle in the first two
        for (int k = 0; k < 4; k++, r++)
            launch_pdl(k_dedup_round, dim3(grid), dim3(256), 0, s,
                       static_cast<const unsigned long long*>(keys.p),
                       static_cast<const int64_t*>(off.p), n, status.p, cnt.p, r);
        // the last round's count (it cleared the other counter)
        PDB_CUDA(cudaMemcpyAsync(hc, cnt.p + ((r - 1) & 1), sizeof(unsigned long long),
                                 cudaMemcpyDeviceToHost, s));
        PDB_CUDA(cudaStreamSynchronize(s));
        const unsigned int und = static_cast<unsigned int>(hc[0]);
        if (und == 0) break;
        if (und <= kTailSwitch) {
            // few undecided items left (dependency chains): the sequential
            // tail in one block instead of one round per chain link
            DevBuf<int32_t> list(und, s);
            DevBuf<int> nsel(1, s);
            cub::CountingInputIterator<int32_t> idx(0);
            size_t tb = 0;
            PDB_CUDA(cub::DeviceSelect::If(nullptr, tb, idx, list.p, nsel.p, n,
                                           IsUndecided{status.p}, s));
            DevBuf<uint8_t> tmp(tb, s);
            PDB_CUDA(cub::DeviceSelect::If(tmp.p, tb, idx, list.p, nsel.p, n,
                                           IsUndecided{status.p}, s));
            const int edge_cap = 40000;
            const size_t smem = static_cast<size_t>(kTailItems) * 4 + (kTailItems + 1) * 4 +
                                static_cast<size_t>(edge_cap) * 4 + kTailItems;
            set_max_smem(reinterpret_cast<const void*>(k_dedup_tail), static_cast<int>(smem));
            k_dedup_tail<<<1, 1024, smem, s>>>(static_cast<const unsigned long long*>(keys.p),
                                                static_cast<const int64_t*>(off.p), list.p,
                                                static_cast<int64_t>(und), status.p, edge_cap);
            PDB_CUDA(cudaGetLastError());
            break;
        }
        if (check > n) fail(PDB_ERR_CUDA, "dedup rounds did not converge");  // unreachable
    }

    // 4. attach members to their nearest representative
    launch_pdl(k_dedup_attach, dim3(grid), dim3(256), 0, s, static_cast<const unsigned long long*>(keys.p),
               static_cast<const int64_t*>(off.p), n, static_cast<const uint8_t*>(status.p), d_X, d,
               d_rep_of, cnt.p + 2);
    PDB_CUDA(cudaGetLastError());
    PDB_CUDA(cudaMemcpyAsync(hc + 1, cnt.p + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    PDB_CUDA(cudaStreamSynchronize(s));
    *n_reps = static_cast<int64_t>(hc[1]);
}

}  // namespace pdb
