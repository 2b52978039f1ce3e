// sa_part.cu -- the partitioned index (not in the paper): for a reference whose
// index exceeds one GPU, part g of nparts holds only the suffixes whose route key -- their first
// route_bases (rb) bases, e_rb of sa_suffix_e -- lies in [K_g, K_{g+1}).  Those suffixes are a contiguous
// range of SA ranks [R_g, R_{g+1}) (the route-level table T_r gives R_g = T_r[K_g]), so a part's slice of
// the SA, of the k-mer bracket table and of the records answers every read whose route key it owns, with
// global ranks.  This file builds ONLY that slice (the whole text is replicated; the suffix array of the
// other parts is never formed), and provides the two kernels around the exchange:
//
//   route (sa_match_route, csrc/sa_match.cu): reads ordered by route key, reads shorter than rb last;
//   pack  (sa_part_pack): the send buffer, block g = the reads routed to part g + ALL short reads;
//   -- all-to-all of rows; sa_match_batch on the part; all-to-all of intervals back (the caller's NCCL) --
//   collect (sa_part_collect): a routed read's interval is its part's answer; a short read's interval
//            is the sum over parts of their clamped answers (below), written at the read's own index.
//
// Why short reads go to every part: a read P of m < rb bases spans route keys [x.4^(rb-m), (x+1).4^(rb-m)),
// possibly several parts.  Every part answers it clamped to its own ranks: the search brackets are cut
// to [R_g, R_{g+1}], so the binary search returns clamp(lo, R_g, R_{g+1}) (and the same for hi), and since
// the parts tile [0, n), lo = sum_g (clamp(lo, R_g, R_{g+1}) - R_g).  Reads of m >= rb lie inside their
// own part's ranks: R_g <= T_r[key] <= lo <= hi <= T_r[key + 1] <= R_{g+1}.
//
// The slice's suffix array is built by MSD refinement on the packed text (the rank array of prefix
// doubling would need the other parts' suffixes): sort the part's suffixes by their first 21 bases
// (3 bits per base, 0 past the end, so a suffix that ends inside the window is unique), then re-sort
// every group of still-tied suffixes by its next 21 bases, and so on.  Each round costs two stable
// radix sorts of the tied suffixes only; the number of rounds is the longest repeat inside the part / 21.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <vector>

#include "sa_internal.cuh"

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t n) {
    uint64_t b = (n + kThreads - 1) / kThreads;
    const uint64_t cap = 148ull * 64;
    if (b > cap) b = cap;
    if (b == 0) b = 1;
    return (unsigned)b;
}

#define GRID_STRIDE(i, n) \
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (uint64_t)gridDim.x * blockDim.x)

template <typename F>
sa_status cub_call(F f, cudaStream_t st, const char *what) {
    size_t bytes = 0;
    cudaError_t e = f(nullptr, bytes);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        sa_set_error("%s (size query): %s", what, cudaGetErrorString(e));
        return SA_ECUDA;
    }
    DevBuf<uint8_t> tmp;
    SA_TRY(tmp.alloc(bytes, st, what));
    e = f(tmp.p, bytes);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        sa_set_error("%s: %s", what, cudaGetErrorString(e));
        return SA_ECUDA;
    }
    return SA_OK;
}

// route-level histogram: hist[e_rb(i) + 1] for every suffix i (e in [-1, 4^rb - 1])
__global__ void k_route_hist(const uint64_t *__restrict__ text, uint64_t n, unsigned rb, uint32_t *__restrict__ hist) {
    GRID_STRIDE(i, n) { atomicAdd(hist + (sa_suffix_e(text, n, i, rb) + 1), 1u); }
}

struct InPart {  // suffix i belongs to the part: K0 <= e_rb(i) < K1
    const uint64_t *text;
    uint64_t n;
    unsigned rb;
    int64_t K0, K1;
    __device__ __forceinline__ bool operator()(uint32_t i) const {
        const int64_t e = sa_suffix_e(text, n, i, rb);
        return e >= K0 && e < K1;
    }
};

// the 21 bases of the text from base b at 3 bits each (1..4 = a..t, 0 past the end)
__device__ __forceinline__ uint64_t key21(const uint64_t *__restrict__ text, uint64_t n, uint64_t b) {
    if (b >= n) return 0;
    const uint64_t w = text_window(text, b);
    uint64_t key = 0;
#pragma unroll
    for (int j = 0; j < 21; ++j) {
        const uint64_t c = (b + j < n) ? ((w >> (62 - 2 * j)) & 3u) + 1u : 0u;
        key = (key << 3) | c;
    }
    return key;
}

__global__ void k_keys0(const uint32_t *__restrict__ pos, uint64_t cnt, const uint64_t *__restrict__ text, uint64_t n,
                        uint64_t *__restrict__ keys) {
    GRID_STRIDE(t, cnt) { keys[t] = key21(text, n, pos[t]); }
}

// round r: tied suffix A[t] (an index into the slice's order) gets key = its bases [off, off+21) and its
// permutation slot t
__global__ void k_msd_keys(const uint32_t *__restrict__ A, uint64_t cnt, const uint32_t *__restrict__ order,
                           const uint64_t *__restrict__ text, uint64_t n, uint64_t off,
                           uint64_t *__restrict__ keys, uint32_t *__restrict__ slot) {
    GRID_STRIDE(t, cnt) {
        const uint32_t i = A[t];
        keys[t] = key21(text, n, (uint64_t)order[i] + off);
        slot[t] = (uint32_t)t;
    }
}

__global__ void k_gather_group(const uint32_t *__restrict__ A, const uint32_t *__restrict__ ghead,
                               const uint32_t *__restrict__ perm, uint64_t cnt, uint32_t *__restrict__ grp) {
    GRID_STRIDE(t, cnt) { grp[t] = ghead[A[perm[t]]]; }
}

// after the two stable sorts (by key, then by group): slot t of the tied list takes suffix
// order[A[perm[t]]] with key keys_by_key[rank of perm[t] in the key sort] -- gathered here
__global__ void k_msd_apply(const uint32_t *__restrict__ A, const uint32_t *__restrict__ perm_final, uint64_t cnt,
                            const uint32_t *__restrict__ old_order, const uint64_t *__restrict__ key_of_slot,
                            uint32_t *__restrict__ new_pos, uint64_t *__restrict__ new_key) {
    GRID_STRIDE(t, cnt) {
        const uint32_t src = perm_final[t];  // original tied-list slot
        new_pos[t] = old_order[A[src]];
        new_key[t] = key_of_slot[src];
    }
}

__global__ void k_scatter_pos(const uint32_t *__restrict__ A, uint64_t cnt, const uint32_t *__restrict__ new_pos,
                              uint32_t *__restrict__ order) {
    GRID_STRIDE(t, cnt) { order[A[t]] = new_pos[t]; }
}

// run starts of (group, key) over the tied list: cand = A[t] at a start, else 0 (max-scan -> head)
__global__ void k_run_cand(const uint32_t *__restrict__ A, const uint32_t *__restrict__ grp, const uint64_t *__restrict__ key,
                           uint64_t cnt, uint32_t *__restrict__ cand, uint8_t *__restrict__ tied) {
    GRID_STRIDE(t, cnt) {
        const bool start = t == 0 || grp[t] != grp[t - 1] || key[t] != key[t - 1];
        const bool next_start = t + 1 == cnt || grp[t + 1] != grp[t] || key[t + 1] != key[t];
        cand[t] = start ? A[t] : 0u;
        tied[t] = (start && next_start) ? 0 : 1;
    }
}

__global__ void k_set_head(const uint32_t *__restrict__ A, const uint32_t *__restrict__ head, uint64_t cnt,
                           uint32_t *__restrict__ ghead) {
    GRID_STRIDE(t, cnt) { ghead[A[t]] = head[t]; }
}

// round 0 over the whole slice: group heads and tied flags of the sorted keys
__global__ void k_run_cand0(const uint64_t *__restrict__ key, uint64_t cnt, uint32_t *__restrict__ cand,
                            uint8_t *__restrict__ tied) {
    GRID_STRIDE(t, cnt) {
        const bool start = t == 0 || key[t] != key[t - 1];
        const bool next_start = t + 1 == cnt || key[t + 1] != key[t];
        cand[t] = start ? (uint32_t)t : 0u;
        tied[t] = (start && next_start) ? 0 : 1;
    }
}

struct MaxU32 {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

// T[x - x0] = r0 + #{slice suffixes with e_k < x} for x in [x0, x1]: the global table clamped to the
// slice's ranks (k_table of csrc/sa_build.cu restricted to the slice)
__global__ void k_table_slice(const uint64_t *__restrict__ text, uint64_t n, const uint32_t *__restrict__ sa, uint64_t cnt,
                              unsigned k, int64_t x0, int64_t x1, uint32_t r0, uint32_t *__restrict__ T) {
    GRID_STRIDE(r, cnt + 1) {
        int64_t lo = (r == 0) ? x0 : sa_suffix_e(text, n, sa[r - 1], k) + 1;
        int64_t hi = (r == cnt) ? x1 : sa_suffix_e(text, n, sa[r], k);
        if (lo < x0) lo = x0;
        if (hi > x1) hi = x1;
        for (int64_t x = lo; x <= hi; ++x) T[x - x0] = r0 + (uint32_t)r;
    }
}

// ---- the exchange kernels ---------------------------------------------------------------------
// block g of the send buffer starts at B_g = offs[g] + g * n_short and holds offs[g+1] - offs[g] routed
// reads followed by the n_short short reads (ordered rows [offs[nparts], Q))
__device__ __forceinline__ uint32_t block_of(const uint64_t *__restrict__ offs, uint32_t nparts, uint64_t n_short,
                                             uint64_t u) {
    uint32_t lo = 0, hi = nparts;  // last g with B_g <= u
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (offs[mid] + mid * n_short <= u) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void k_part_pack(const uint64_t *__restrict__ words, const uint32_t *__restrict__ lens, uint32_t stride,
                            const uint64_t *__restrict__ offs, uint32_t nparts, uint64_t Q, uint64_t total,
                            uint64_t *__restrict__ send_words, uint32_t *__restrict__ send_lens) {
    const uint64_t n_long = offs[nparts], n_short = Q - n_long;
    GRID_STRIDE(u, total) {
        const uint32_t g = block_of(offs, nparts, n_short, u);
        const uint64_t i = u - (offs[g] + g * n_short), routed = offs[g + 1] - offs[g];
        const uint64_t src = i < routed ? offs[g] + i : n_long + (i - routed);
        for (uint32_t j = 0; j < stride; ++j) send_words[u * stride + j] = words[src * stride + j];
        if (send_lens) send_lens[u] = lens[src];
    }
}

__global__ void k_part_collect(const uint2 *__restrict__ back, const uint64_t *__restrict__ offs, uint32_t nparts,
                               uint64_t Q, const uint64_t *__restrict__ part_ranks, const uint32_t *__restrict__ order,
                               uint2 *__restrict__ out) {
    const uint64_t n_long = offs[nparts], n_short = Q - n_long;
    GRID_STRIDE(t, Q) {
        uint2 v;
        if (t < n_long) {  // a routed read: its part's answer is global
            uint32_t lo = 0, hi = nparts;  // last g with offs[g] <= t
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (offs[mid] <= t) lo = mid; else hi = mid;
            }
            v = back[offs[lo] + lo * n_short + (t - offs[lo])];
        } else {  // a short read: sum over the parts of (clamped answer - the part's first rank)
            const uint64_t i = t - n_long;
            uint64_t slo = 0, shi = 0;
            for (uint32_t g = 0; g < nparts; ++g) {
                const uint2 p = back[offs[g + 1] + (uint64_t)(g + 1) * n_short - n_short + i];
                slo += p.x - part_ranks[g];
                shi += p.y - part_ranks[g];
            }
            v = make_uint2((uint32_t)slo, (uint32_t)shi);
        }
        out[order ? order[t] : t] = v;
    }
}

// The slice's suffix array (sorted positions of the part's suffixes), MSD refinement by 21 bases.
sa_status build_slice_sa(sa_index *idx, int64_t K0, int64_t K1, uint64_t cnt, cudaStream_t st) {
    const uint64_t n = idx->n;
    const unsigned rb = idx->route_bases;
    uint32_t *order = idx->sa;  // cnt entries
    if (cnt == 0) return SA_OK;
    {   // members of the part, in position order
        DevBuf<int64_t> num;
        SA_TRY(num.alloc(1, st, "slice count"));
        InPart pred{idx->text, n, rb, K0, K1};
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceSelect::If(tmp, bytes, thrust::counting_iterator<uint32_t>(0), order, num.p, (int64_t)n,
                                         pred, st);
        }, st, "slice select"));
        int64_t got = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&got, num.p, 8, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        if ((uint64_t)got != cnt) {
            sa_set_error("partition: %lld members selected, route table says %llu", (long long)got,
                         (unsigned long long)cnt);
            return SA_ECUDA;
        }
    }
    DevBuf<uint32_t> ghead, A;
    uint64_t nA = 0;
    {   // round 0: sort the members by their first 21 bases
        DevBuf<uint64_t> ka, kb;
        DevBuf<uint32_t> vb, cand;
        DevBuf<uint8_t> tied;
        SA_TRY(ka.alloc(cnt, st, "slice keys"));
        SA_TRY(kb.alloc(cnt, st, "slice keys (alt)"));
        SA_TRY(vb.alloc(cnt, st, "slice values (alt)"));
        k_keys0<<<grid_for(cnt), kThreads, 0, st>>>(order, cnt, idx->text, n, ka.p);
        SA_CUDA_TRY(cudaGetLastError());
        cub::DoubleBuffer<uint64_t> dk(ka.p, kb.p);
        cub::DoubleBuffer<uint32_t> dv(order, vb.p);
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceRadixSort::SortPairs(tmp, bytes, dk, dv, (int64_t)cnt, 0, 63, st);
        }, st, "slice sort"));
        if (dv.Current() != order)
            SA_CUDA_TRY(cudaMemcpyAsync(order, dv.Current(), cnt * 4, cudaMemcpyDeviceToDevice, st));
        SA_TRY(cand.alloc(cnt, st, "slice heads"));
        SA_TRY(tied.alloc(cnt, st, "slice tied flags"));
        k_run_cand0<<<grid_for(cnt), kThreads, 0, st>>>(dk.Current(), cnt, cand.p, tied.p);
        SA_CUDA_TRY(cudaGetLastError());
        SA_TRY(ghead.alloc(cnt, st, "slice group heads"));
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceScan::InclusiveScan(tmp, bytes, cand.p, ghead.p, MaxU32(), (int64_t)cnt, st);
        }, st, "slice head scan"));
        DevBuf<int64_t> num;
        SA_TRY(num.alloc(1, st, "tied count"));
        SA_TRY(A.alloc(cnt, st, "tied list"));
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceSelect::Flagged(tmp, bytes, thrust::counting_iterator<uint32_t>(0), tied.p, A.p, num.p,
                                              (int64_t)cnt, st);
        }, st, "tied compaction"));
        int64_t h = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&h, num.p, 8, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        nA = (uint64_t)h;
    }
    uint64_t off = 21;
    uint32_t rounds = 0;
    while (nA > 0) {
        if (off > n + 21) {
            sa_set_error("partition SA build did not converge (%llu tied suffixes)", (unsigned long long)nA);
            return SA_ECUDA;
        }
        DevBuf<uint64_t> key, key_sorted, key_final;
        DevBuf<uint32_t> slot, perm, grp, grp_sorted, perm_final, pos, cand, head;
        DevBuf<uint8_t> tied;
        SA_TRY(key.alloc(nA, st, "msd keys"));
        SA_TRY(key_sorted.alloc(nA, st, "msd keys sorted"));
        SA_TRY(slot.alloc(nA, st, "msd slots"));
        SA_TRY(perm.alloc(nA, st, "msd perm"));
        k_msd_keys<<<grid_for(nA), kThreads, 0, st>>>(A.p, nA, order, idx->text, n, off, key.p, slot.p);
        SA_CUDA_TRY(cudaGetLastError());
        // stable by key, then stable by group: groups keep their places, members ordered by key
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceRadixSort::SortPairs(tmp, bytes, key.p, key_sorted.p, slot.p, perm.p, (int64_t)nA, 0, 63, st);
        }, st, "msd key sort"));
        SA_TRY(grp.alloc(nA, st, "msd groups"));
        SA_TRY(grp_sorted.alloc(nA, st, "msd groups sorted"));
        SA_TRY(perm_final.alloc(nA, st, "msd perm final"));
        k_gather_group<<<grid_for(nA), kThreads, 0, st>>>(A.p, ghead.p, perm.p, nA, grp.p);
        SA_CUDA_TRY(cudaGetLastError());
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceRadixSort::SortPairs(tmp, bytes, grp.p, grp_sorted.p, perm.p, perm_final.p, (int64_t)nA, 0,
                                                   32, st);
        }, st, "msd group sort"));
        SA_TRY(pos.alloc(nA, st, "msd positions"));
        SA_TRY(key_final.alloc(nA, st, "msd keys final"));
        k_msd_apply<<<grid_for(nA), kThreads, 0, st>>>(A.p, perm_final.p, nA, order, key.p, pos.p, key_final.p);
        SA_CUDA_TRY(cudaGetLastError());
        k_scatter_pos<<<grid_for(nA), kThreads, 0, st>>>(A.p, nA, pos.p, order);
        SA_CUDA_TRY(cudaGetLastError());
        SA_TRY(cand.alloc(nA, st, "msd run starts"));
        SA_TRY(tied.alloc(nA, st, "msd tied flags"));
        k_run_cand<<<grid_for(nA), kThreads, 0, st>>>(A.p, grp_sorted.p, key_final.p, nA, cand.p, tied.p);
        SA_CUDA_TRY(cudaGetLastError());
        SA_TRY(head.alloc(nA, st, "msd heads"));
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceScan::InclusiveScan(tmp, bytes, cand.p, head.p, MaxU32(), (int64_t)nA, st);
        }, st, "msd head scan"));
        k_set_head<<<grid_for(nA), kThreads, 0, st>>>(A.p, head.p, nA, ghead.p);
        SA_CUDA_TRY(cudaGetLastError());
        DevBuf<uint32_t> A2;
        DevBuf<int64_t> num;
        SA_TRY(num.alloc(1, st, "tied count"));
        SA_TRY(A2.alloc(nA, st, "tied list"));
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceSelect::Flagged(tmp, bytes, A.p, tied.p, A2.p, num.p, (int64_t)nA, st);
        }, st, "tied compaction"));
        int64_t h = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&h, num.p, 8, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        A.reset();
        A.p = A2.release();
        A.count = (uint64_t)h;
        A.st = st;
        nA = (uint64_t)h;
        off += 21;
        ++rounds;
    }
    idx->build_rounds = rounds;
    return SA_OK;
}

sa_status build_part(sa_index *idx, const char *ref_ascii, cudaStream_t st) {
    const uint64_t n = idx->n;
    const unsigned rb = idx->route_bases, k = idx->k;
    SA_TRY(sa_pack_text(idx, ref_ascii, st));
    // ---- route-level table T_r (replicated in every part: it routes short reads and sets the bounds) ----
    const uint64_t nkeys = 1ull << (2 * rb);
    SA_CUDA_TRY(cudaMalloc(&idx->route_table, (nkeys + 1) * sizeof(uint32_t)));
    SA_CUDA_TRY(cudaMemsetAsync(idx->route_table, 0, (nkeys + 1) * sizeof(uint32_t), st));
    k_route_hist<<<grid_for(n), kThreads, 0, st>>>(idx->text, n, rb, idx->route_table);
    SA_CUDA_TRY(cudaGetLastError());
    SA_TRY(cub_call([&](void *tmp, size_t &bytes) {  // T_r[K] = #{e_rb < K} = sum_{j <= K} hist[j]
        return cub::DeviceScan::InclusiveSum(tmp, bytes, idx->route_table, idx->route_table, (int64_t)(nkeys + 1), st);
    }, st, "route table scan"));
    std::vector<uint32_t> Tr(nkeys + 1);
    SA_CUDA_TRY(cudaMemcpyAsync(Tr.data(), idx->route_table, (nkeys + 1) * 4, cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    // ---- boundaries: K_g = the smallest route key whose first suffix has rank >= g*n/nparts ----
    const uint32_t P = idx->nparts;
    idx->part_keys.assign(P + 1, 0);
    idx->part_ranks.assign(P + 1, 0);
    idx->part_keys[P] = (uint32_t)nkeys;
    for (uint32_t g = 1; g < P; ++g) {
        const uint64_t target = (uint64_t)g * n / P;
        const uint32_t *b = std::lower_bound(Tr.data() + idx->part_keys[g - 1], Tr.data() + nkeys,
                                             (uint32_t)target);  // (Tr is non-decreasing)
        idx->part_keys[g] = (uint32_t)(b - Tr.data());
    }
    // (part 0 also holds the suffixes whose e_rb is -1 -- shorter than rb and all 'a': they sort first)
    for (uint32_t g = 0; g <= P; ++g) idx->part_ranks[g] = g == 0 ? 0 : g == P ? n : Tr[idx->part_keys[g]];
    SA_CUDA_TRY(cudaMalloc(&idx->part_ranks_dev, (P + 1) * sizeof(uint64_t)));
    SA_CUDA_TRY(cudaMemcpyAsync(idx->part_ranks_dev, idx->part_ranks.data(), (P + 1) * 8, cudaMemcpyHostToDevice, st));
    const uint64_t K0 = idx->part_keys[idx->part], K1 = idx->part_keys[idx->part + 1];
    const uint64_t r0 = idx->part_ranks[idx->part], r1 = idx->part_ranks[idx->part + 1];
    const unsigned sh = 2 * (k - rb);
    const uint64_t x0 = K0 << sh, x1 = K1 << sh;
    idx->x_base = x0;
    idx->rank_base = r0;
    idx->rank_end = r1;
    // ---- the slice's suffix array ----
    const uint64_t cnt = r1 - r0;
    SA_CUDA_TRY(cudaMalloc(&idx->sa, (cnt ? cnt : 1) * sizeof(uint32_t)));
    SA_TRY(build_slice_sa(idx, idx->part == 0 ? -1 : (int64_t)K0, (int64_t)K1, cnt, st));
    // ---- the slice of the k-mer bracket table (entries x0 .. x1, clamped to the slice's ranks) ----
    idx->table_entries = x1 - x0 + 1;
    SA_CUDA_TRY(cudaMalloc(&idx->table, (idx->table_entries + 4) * sizeof(uint32_t)));
    k_table_slice<<<grid_for(cnt + 1), kThreads, 0, st>>>(idx->text, n, idx->sa, cnt, k, (int64_t)x0, (int64_t)x1,
                                                         (uint32_t)r0, idx->table);
    SA_CUDA_TRY(cudaGetLastError());
    // ---- records ----
    uint64_t sa_bytes = cnt * sizeof(uint32_t);
    if (idx->layout != 0) {
        SA_TRY(sa_build_records(idx, idx->sa, cnt, st));
        SA_CUDA_TRY(cudaFree(idx->sa));
        idx->sa = nullptr;
        sa_bytes = cnt * (idx->layout == 2 ? 2 : 1) * sizeof(uint4);
    }
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    idx->device_bytes = idx->n_words * 8 + sa_bytes + idx->table_entries * 4 + (nkeys + 1) * 4 + (P + 1) * 8;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, idx->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    return SA_OK;
}

}  // namespace

// ---- C ABI ------------------------------------------------------------------------------------
extern "C" sa_status sa_index_create_part(const char *ref_ascii, uint64_t n, const sa_index_opts *opts, uint32_t part,
                                          uint32_t nparts, uint32_t route_bases, sa_index **out) {
    sa_clear_error();
    if (!out) { sa_set_error("out is NULL"); return SA_EINVAL; }
    *out = nullptr;
    if (nparts < 2 || part >= nparts || route_bases == 0 || route_bases > 12) {
        sa_set_error("bad partition %u of %u (nparts >= 2) / route_bases %u (1..12)", part, nparts, route_bases);
        return SA_EINVAL;
    }
    if (n == 0) { sa_set_error("empty reference (n = 0)"); return SA_EEMPTY; }
    if (!ref_ascii) { sa_set_error("ref_ascii is NULL"); return SA_EINVAL; }
    if (n > 0xFFFFFFFFull) { sa_set_error("reference of %llu bases exceeds 2^32-1", (unsigned long long)n); return SA_ETOOLONG; }
    sa_index_opts o{-1, 0, 0, 0};
    if (opts) o = *opts;
    if ((o.flags & ~(SA_INDEX_PLAIN | SA_INDEX_REC32)) != 0 ||
        (o.flags & (SA_INDEX_PLAIN | SA_INDEX_REC32)) == (SA_INDEX_PLAIN | SA_INDEX_REC32) || o.reserved != 0) {
        sa_set_error("partition: opts.flags may only select the layout (no DC3 build, no sub-tables)");
        return SA_EINVAL;
    }
    if (o.kmer_k > 16) { sa_set_error("kmer_k %u out of range 1..16", o.kmer_k); return SA_EINVAL; }
    uint32_t k = o.kmer_k;
    if (k == 0) {
        k = 1;
        while (k < 16 && (1ull << (2 * k)) <= n) ++k;
    }
    if (route_bases >= k) {
        sa_set_error("route_bases %u must be < k %u", route_bases, k);
        return SA_EINVAL;
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        (void)cudaGetLastError();
        sa_set_error("no CUDA device available");
        return SA_ECUDA;
    }
    int dev = o.device;
    if (dev < 0) SA_CUDA_TRY(cudaGetDevice(&dev));
    if (dev >= ndev) { sa_set_error("device %d out of range (%d devices)", dev, ndev); return SA_EINVAL; }
    int prev = 0;
    SA_CUDA_TRY(cudaGetDevice(&prev));
    SA_CUDA_TRY(cudaSetDevice(dev));
    sa_index *idx = new (std::nothrow) sa_index();
    if (!idx) { cudaSetDevice(prev); sa_set_error("host allocation failed"); return SA_ENOMEM; }
    idx->device = dev;
    idx->n = n;
    idx->k = k;
    idx->layout = (o.flags & SA_INDEX_PLAIN) ? 0 : (o.flags & SA_INDEX_REC32) ? 2 : 1;
    idx->part = part;
    idx->nparts = nparts;
    idx->route_bases = route_bases;
    cudaStream_t st = nullptr;
    sa_status s = SA_OK;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
        (void)cudaGetLastError();
        sa_set_error("stream creation failed");
        s = SA_ECUDA;
    }
    if (s == SA_OK) s = build_part(idx, ref_ascii, st);
    if (st) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    if (s != SA_OK) {
        sa_free_index(idx);
        cudaSetDevice(prev);
        return s;
    }
    cudaSetDevice(prev);
    *out = idx;
    return SA_OK;
}

extern "C" sa_status sa_index_part_info(const sa_index *idx, uint32_t *part, uint32_t *nparts, uint32_t *route_bases,
                                        uint64_t *rank_lo, uint64_t *rank_hi, uint32_t *part_keys,
                                        uint64_t *part_ranks) {
    sa_clear_error();
    if (!idx) { sa_set_error("index is NULL"); return SA_EINVAL; }
    const bool split = idx->nparts > 1;
    if (part) *part = idx->part;
    if (nparts) *nparts = idx->nparts;
    if (route_bases) *route_bases = idx->route_bases;
    if (rank_lo) *rank_lo = split ? idx->rank_base : 0;
    if (rank_hi) *rank_hi = split ? idx->rank_end : idx->n;
    for (uint32_t g = 0; g <= idx->nparts; ++g) {
        if (part_keys) part_keys[g] = split ? idx->part_keys[g] : (g ? 0xFFFFFFFFu : 0u);
        if (part_ranks) part_ranks[g] = split ? idx->part_ranks[g] : (g ? idx->n : 0);
    }
    return SA_OK;
}

extern "C" sa_status sa_part_pack(const sa_index *idx, const uint64_t *ordered_words, const uint32_t *ordered_len,
                                  uint32_t stride_words, const uint64_t *dest_offsets, uint64_t Q, uint64_t send_rows,
                                  uint64_t *send_words, uint32_t *send_len, void *stream) {
    sa_clear_error();
    if (!idx || idx->nparts < 2) { sa_set_error("not a partitioned index"); return SA_EINVAL; }
    if (send_rows == 0) return SA_OK;
    if (!ordered_words || !dest_offsets || !send_words || stride_words == 0 || (ordered_len && !send_len)) {
        sa_set_error("sa_part_pack: NULL argument or dense layout");
        return SA_EINVAL;
    }
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    k_part_pack<<<grid_for(send_rows), kThreads, 0, (cudaStream_t)stream>>>(
        ordered_words, ordered_len, stride_words, dest_offsets, idx->nparts, Q, send_rows, send_words,
        ordered_len ? send_len : nullptr);
    SA_CUDA_TRY(cudaGetLastError());
    return SA_OK;
}

extern "C" sa_status sa_part_collect(const sa_index *idx, const uint32_t *back_lohi, const uint64_t *dest_offsets,
                                     uint64_t Q, const uint32_t *order, uint32_t *out_lohi, void *stream) {
    sa_clear_error();
    if (!idx || idx->nparts < 2) { sa_set_error("not a partitioned index"); return SA_EINVAL; }
    if (Q == 0) return SA_OK;
    if (!back_lohi || !dest_offsets || !out_lohi) { sa_set_error("sa_part_collect: NULL argument"); return SA_EINVAL; }
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    k_part_collect<<<grid_for(Q), kThreads, 0, (cudaStream_t)stream>>>(
        reinterpret_cast<const uint2 *>(back_lohi), dest_offsets, idx->nparts, Q, idx->part_ranks_dev, order,
        reinterpret_cast<uint2 *>(out_lohi));
    SA_CUDA_TRY(cudaGetLastError());
    return SA_OK;
}
