// sa_build.cu -- index build (off the timed path): validate + pack the reference, build the suffix
// array on the GPU, build the k-mer bracket table.
//
// The paper builds its suffix array on the CPU with DC3 (Sec. III).  Here the
// same object -- SA, all suffix starts in lexicographic order with a proper prefix first
// (Table I; reading A2) -- is built on the B200 by prefix doubling
// (DESIGN.md "Index build"):
//   round 0   key = the first 21 bases of each suffix at 3 bits/base (1..4 = a..t, 0 = past the
//             end, so a suffix that ends inside the window carries its own terminator) -> one CUB
//             radix sort of (key, position) over all n suffixes;
//   round r   h = 21 * 2^(r-1): only suffixes still tied with a neighbour are re-sorted by
//             (rank[s], rank[s+h]), rank = 1 + start of the suffix's group, rank[n] = 0.
// Tied suffixes always have >= h bases (a terminator inside the window would have split them),
// so s + h <= n and rank[] needs only one extra slot.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <cstring>
#include <vector>

#include "sa_internal.cuh"

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t n, int threads = kThreads) {
    uint64_t b = (n + threads - 1) / threads;
    const uint64_t cap = 148ull * 64;  // grid-stride beyond this
    if (b > cap) b = cap;
    if (b == 0) b = 1;
    return (unsigned)b;
}

#define GRID_STRIDE(i, n) \
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (uint64_t)gridDim.x * blockDim.x)

// ---- pack -------------------------------------------------------------------------------------
// One thread per output word: 32 ASCII bytes -> 2-bit codes, MSB-first.  A=0 C=1 G=2 T=3 via
// ((c>>1)&3) ^ ((c>>2)&1) (upper or lower case); anything else records its position.
__global__ void k_pack(const uint8_t *__restrict__ ascii, uint64_t len, uint64_t base_word, uint64_t *__restrict__ text,
                       unsigned long long *__restrict__ bad) {
    const uint64_t words = (len + 31) / 32;
    GRID_STRIDE(t, words) {
        const uint64_t b0 = t * 32;
        const unsigned cnt = (len - b0 < 32) ? (unsigned)(len - b0) : 32u;
        uint64_t w = 0;
        unsigned long long first_bad = ~0ull;
        for (unsigned j = 0; j < cnt; ++j) {
            const unsigned c = ascii[b0 + j];
            const unsigned lc = c | 0x20u;
            if (!(lc == 'a' || lc == 'c' || lc == 'g' || lc == 't')) {
                if (first_bad == ~0ull) first_bad = (base_word * 32 + b0 + j);
            }
            const uint64_t code = ((c >> 1) & 3u) ^ ((c >> 2) & 1u);
            w |= code << (62 - 2 * j);
        }
        text[base_word + t] = w;
        if (first_bad != ~0ull) atomicMin(bad, first_bad);
    }
}

// ---- suffix array: round 0 -------------------------------------------------------------------
__global__ void k_init_keys(const uint64_t *__restrict__ text, uint64_t n, uint64_t *__restrict__ keys,
                            uint32_t *__restrict__ vals) {
    GRID_STRIDE(i, n) {
        const uint64_t w = text_window(text, i);
        uint64_t key = 0;
#pragma unroll
        for (int j = 0; j < 21; ++j) {
            const uint64_t c = (i + j < n) ? ((w >> (62 - 2 * j)) & 3u) + 1u : 0u;
            key = (key << 3) | c;
        }
        keys[i] = key;
        vals[i] = (uint32_t)i;
    }
}

// head candidates: t where a new group starts (key differs from its left neighbour), else 0
__global__ void k_head_cand(const uint64_t *__restrict__ keys, uint64_t m, uint32_t *__restrict__ cand) {
    GRID_STRIDE(t, m) { cand[t] = (t == 0 || keys[t] != keys[t - 1]) ? (uint32_t)t : 0u; }
}

// active = member of a group of size > 1
__global__ void k_active(const uint64_t *__restrict__ keys, uint64_t m, uint8_t *__restrict__ flags) {
    GRID_STRIDE(t, m) {
        const bool head = (t == 0 || keys[t] != keys[t - 1]);
        const bool next_head = (t + 1 == m) || keys[t + 1] != keys[t];
        flags[t] = (head && next_head) ? 0 : 1;
    }
}

// round 0: rank[SA[r]] = head(r) + 1, rank[n] = 0
__global__ void k_rank0(const uint32_t *__restrict__ sa, const uint32_t *__restrict__ head, uint64_t n,
                        uint32_t *__restrict__ rank) {
    GRID_STRIDE(r, n) { rank[sa[r]] = head[r] + 1u; }
    if (blockIdx.x == 0 && threadIdx.x == 0) rank[n] = 0;
}

// ---- suffix array: doubling rounds -----------------------------------------------------------
__global__ void k_round_keys(const uint32_t *__restrict__ A, uint64_t nA, const uint32_t *__restrict__ sa,
                             const uint32_t *__restrict__ rank, uint64_t h, uint64_t *__restrict__ keys,
                             uint32_t *__restrict__ vals) {
    GRID_STRIDE(t, nA) {
        const uint32_t s = sa[A[t]];
        keys[t] = ((uint64_t)rank[s] << 32) | rank[(uint64_t)s + h];
        vals[t] = s;
    }
}

__global__ void k_round_scatter(const uint32_t *__restrict__ A, uint64_t nA, const uint32_t *__restrict__ vals,
                                const uint32_t *__restrict__ head, uint32_t *__restrict__ sa,
                                uint32_t *__restrict__ rank) {
    GRID_STRIDE(t, nA) {
        const uint32_t s = vals[t];
        sa[A[t]] = s;
        rank[s] = A[head[t]] + 1u;
    }
}

struct MaxU32 {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

// ---- k-mer bracket table ---------------------------------------------------------------------
// e(r) = (number of k-mers x with x <= suffix SA[r]) - 1: the k-mer code of a suffix with >= k bases,
// U-1 for a shorter suffix u whose a-padded k-mer is U (u > x  <=>  x < U).  e is non-decreasing
// along the SA, and T[x] = #{r : e(r) < x} = r for e(r-1) < x <= e(r).
__device__ __forceinline__ int64_t kmer_e(const uint64_t *__restrict__ text, uint64_t n, const uint32_t *__restrict__ sa,
                                          uint64_t r, unsigned k) {
    return sa_suffix_e(text, n, sa[r], k);
}

__global__ void k_table(const uint64_t *__restrict__ text, uint64_t n, const uint32_t *__restrict__ sa, unsigned k,
                        uint32_t *__restrict__ T) {
    const int64_t K = 1ll << (2 * k);
    GRID_STRIDE(r, n + 1) {
        const int64_t lo = (r == 0) ? 0 : kmer_e(text, n, sa, r - 1, k) + 1;
        const int64_t hi = (r == n) ? K : kmer_e(text, n, sa, r, k);
        for (int64_t x = lo; x <= hi; ++x) T[x] = (uint32_t)r;
    }
}

// ---- second-level tables for large buckets (SA_INDEX_SUBTABLE) ------------------------------------
// A bucket x with more than kBigBucket suffixes gets T2_x[y] = #{i : trunc_{k+4}(S_i) < x.y} for the
// 256 extensions y of x by 4 bases (+1 entry): the k+4 bracket table restricted to that bucket.
struct IsBigBucket {
    const uint32_t *T;
    __host__ __device__ int64_t operator()(uint32_t x) const { return T[(uint64_t)x + 1] - T[x] > kBigBucket ? 1 : 0; }
};

__device__ __forceinline__ uint64_t big_hash(uint32_t x, uint32_t bits) {
    return (uint64_t)((x * 0x9E3779B1u) >> (32 - bits));
}

// Slots are 64-bit {x << 32 | sub-table id}, published by ONE atomicCAS; the empty slot is ~0, which no
// entry can equal (ids are < 2^26), so every k-mer -- including the all-T bucket 0xFFFFFFFF at k = 16 --
// is a valid key.
__global__ void k_big_hash_insert(const uint32_t *__restrict__ big, uint64_t cnt, uint32_t bits,
                                  unsigned long long *__restrict__ H) {
    GRID_STRIDE(id, cnt) {
        const uint32_t x = big[id];
        const uint64_t mask = (1ull << bits) - 1;
        const unsigned long long e = ((unsigned long long)x << 32) | (uint32_t)id;
        for (uint64_t h = big_hash(x, bits);; h = (h + 1) & mask) {
            if (atomicCAS(&H[h], kBigEmpty, e) == kBigEmpty) break;
        }
    }
}

// one block per big bucket: T2[y] = r for e(r-1) < x.y <= e(r), r over the bucket's ranks
__global__ void k_big_subtables(const uint64_t *__restrict__ text, uint64_t n, const uint32_t *__restrict__ sa,
                                unsigned k, const uint32_t *__restrict__ T, const uint32_t *__restrict__ big,
                                uint32_t *__restrict__ sub) {
    const uint32_t x = big[blockIdx.x];
    uint32_t *T2 = sub + (uint64_t)blockIdx.x * 257;
    const uint64_t r0 = T[x], r1 = T[(uint64_t)x + 1];
    const int64_t base = (int64_t)x << 8;
    for (uint64_t r = r0 + threadIdx.x; r <= r1; r += blockDim.x) {
        const int64_t lo = (r == r0) ? 0 : kmer_e(text, n, sa, r - 1, k + 4) - base + 1;
        const int64_t hi = (r == r1) ? 256 : kmer_e(text, n, sa, r, k + 4) - base;
        const int64_t a = lo < 0 ? 0 : lo, b = hi > 256 ? 256 : hi;
        for (int64_t y = a; y <= b; ++y) T2[y] = (uint32_t)r;
    }
}

// ---- bucket trees (SA_INDEX_BUCKET_TREE) ------------------------------------------------------------
struct IsTreeBucket {
    const uint32_t *T;
    __host__ __device__ bool operator()(uint32_t x) const { return T[(uint64_t)x + 1] - T[x] >= kTreeMin; }
};
struct TreeLinesOf {  // lines of bucket x's tree: (4^E - 1) / 3
    const uint32_t *T;
    const uint32_t *xs;
    __host__ __device__ uint64_t operator()(uint64_t id) const {
        const uint32_t x = xs[id];
        const uint32_t e = tree_pairs(T[(uint64_t)x + 1] - T[x]);
        return ((1ull << (2 * e)) - 1) / 3;
    }
};

__global__ void k_tree_hash_insert(const uint32_t *__restrict__ xs, const uint64_t *__restrict__ line0, uint64_t cnt,
                                   uint32_t bits, unsigned long long *__restrict__ H) {
    GRID_STRIDE(id, cnt) {
        const uint32_t x = xs[id];
        const uint64_t mask = (1ull << bits) - 1;
        const unsigned long long e = ((unsigned long long)x << 32) | (uint32_t)line0[id];
        for (uint64_t h = (uint64_t)((x * 0x9E3779B1u) >> (32 - bits));; h = (h + 1) & mask)
            if (atomicCAS(&H[h], kBigEmpty, e) == kBigEmpty) break;
    }
}

// one block per tree bucket: node i (BFS, 1-based) of the bucket's binary search over (T[x]-1, T[x+1])
// at depth < 2E holds the record of its pivot -- the midpoints search_read takes -- at line
// tree_line(pair root) slot 0 (pair root = a node at even depth), 1 (its left child) or 2 (its right)
__global__ void k_tree_fill(const uint32_t *__restrict__ T, const uint32_t *__restrict__ xs, const uint64_t *__restrict__ line0,
                            uint64_t cnt, const uint4 *__restrict__ rec, uint4 *__restrict__ tree) {
    for (uint64_t id = blockIdx.x; id < cnt; id += gridDim.x) {
        const uint32_t x = xs[id];
        const uint32_t L0 = T[x], R0 = T[(uint64_t)x + 1];
        const uint32_t E = tree_pairs(R0 - L0);
        const uint32_t nodes = (1u << (2 * E)) - 1;
        for (uint32_t i = 1 + threadIdx.x; i <= nodes; i += blockDim.x) {
            uint32_t Lp1 = L0, R = R0;
            for (int b = ilog2_u32(i) - 1; b >= 0; --b) {
                const uint32_t p = (uint32_t)(((uint64_t)Lp1 - 1 + R) >> 1);
                if ((i >> b) & 1) Lp1 = p + 1; else R = p;
            }
            uint64_t p = ((uint64_t)Lp1 - 1 + R) >> 1;
            if (p < L0 || p >= R0) p = L0;  // an empty node: never probed
            const uint32_t r = (ilog2_u32(i) & 1) ? (i >> 1) : i;
            const uint32_t slot = i == r ? 0u : 1u + (i & 1u);
            const uint64_t at = (line0[id] + tree_line(r)) * 4 + slot;  // in records of 32 bytes
            tree[2 * at] = rec[2 * p];
            tree[2 * at + 1] = rec[2 * p + 1];
        }
    }
}

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

// head[t] = last group start <= t, for sorted keys[0..m)
sa_status group_heads(const uint64_t *keys, uint64_t m, uint32_t *head, cudaStream_t st) {
    k_head_cand<<<grid_for(m), kThreads, 0, st>>>(keys, m, head);
    SA_CUDA_TRY(cudaGetLastError());
    return cub_call(
        [&](void *tmp, size_t &bytes) {
            return cub::DeviceScan::InclusiveScan(tmp, bytes, head, head, MaxU32(), (int64_t)m, st);
        },
        st, "group head scan");
}

// out[j] = in[t] for flagged t (order kept); returns the count.  out is sized m (transient).
template <typename InIt>
sa_status compact(InIt in, const uint8_t *flags, uint64_t m, DevBuf<uint32_t> &out, uint64_t &count,
                  cudaStream_t st) {
    DevBuf<int64_t> d_num;
    SA_TRY(d_num.alloc(1, st, "compaction count"));
    SA_TRY(out.alloc(m, st, "active list"));
    SA_TRY(cub_call(
        [&](void *tmp, size_t &bytes) {
            return cub::DeviceSelect::Flagged(tmp, bytes, in, flags, out.p, d_num.p, (int64_t)m, st);
        },
        st, "compaction"));
    int64_t h_num = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&h_num, d_num.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    count = (uint64_t)h_num;
    return SA_OK;
}

sa_status sort_pairs(uint64_t *&keys, uint64_t *keys_alt, uint32_t *&vals, uint32_t *vals_alt, uint64_t m,
                     int end_bit, cudaStream_t st) {
    cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
    cub::DoubleBuffer<uint32_t> dv(vals, vals_alt);
    SA_TRY(cub_call(
        [&](void *tmp, size_t &bytes) {
            return cub::DeviceRadixSort::SortPairs(tmp, bytes, dk, dv, (int64_t)m, 0, end_bit, st);
        },
        st, "radix sort"));
    keys = dk.Current();
    vals = dv.Current();
    return SA_OK;
}

sa_status build_sa(sa_index *idx, cudaStream_t st) {
    const uint64_t n = idx->n;
    uint32_t *sa = idx->sa;
    DevBuf<uint32_t> rank, A;
    uint64_t nA = 0;
    {   // round 0
        DevBuf<uint64_t> ka, kb;
        DevBuf<uint32_t> vb;
        SA_TRY(ka.alloc(n, st, "round-0 keys"));
        SA_TRY(kb.alloc(n, st, "round-0 keys (alt)"));
        SA_TRY(vb.alloc(n, st, "round-0 values (alt)"));
        k_init_keys<<<grid_for(n), kThreads, 0, st>>>(idx->text, n, ka.p, sa);
        SA_CUDA_TRY(cudaGetLastError());
        uint64_t *keys = ka.p;
        uint32_t *vals = sa;
        SA_TRY(sort_pairs(keys, kb.p, vals, vb.p, n, 63, st));
        if (vals != sa) SA_CUDA_TRY(cudaMemcpyAsync(sa, vals, n * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        uint32_t *head = vb.p;  // reuse: vals now live in sa
        SA_TRY(group_heads(keys, n, head, st));
        SA_TRY(rank.alloc(n + 1, st, "rank"));
        k_rank0<<<grid_for(n), kThreads, 0, st>>>(sa, head, n, rank.p);
        SA_CUDA_TRY(cudaGetLastError());
        DevBuf<uint8_t> flags;
        SA_TRY(flags.alloc(n, st, "active flags"));
        k_active<<<grid_for(n), kThreads, 0, st>>>(keys, n, flags.p);
        SA_CUDA_TRY(cudaGetLastError());
        vb.reset();
        ka.reset();
        kb.reset();
        SA_TRY(compact(thrust::counting_iterator<uint32_t>(0), flags.p, n, A, nA, st));
    }
    uint64_t h = 21;
    uint32_t rounds = 0;
    while (nA > 0) {
        if (h >= n || rounds > 40) {
            sa_set_error("suffix array build did not converge (h=%llu, %llu tied suffixes)",
                         (unsigned long long)h, (unsigned long long)nA);
            return SA_ECUDA;
        }
        DevBuf<uint64_t> ka, kb;
        DevBuf<uint32_t> va, vb, head;
        SA_TRY(ka.alloc(nA, st, "round keys"));
        SA_TRY(kb.alloc(nA, st, "round keys (alt)"));
        SA_TRY(va.alloc(nA, st, "round values"));
        SA_TRY(vb.alloc(nA, st, "round values (alt)"));
        k_round_keys<<<grid_for(nA), kThreads, 0, st>>>(A.p, nA, sa, rank.p, h, ka.p, va.p);
        SA_CUDA_TRY(cudaGetLastError());
        uint64_t *keys = ka.p;
        uint32_t *vals = va.p;
        SA_TRY(sort_pairs(keys, kb.p, vals, vb.p, nA, 64, st));
        SA_TRY(head.alloc(nA, st, "round heads"));
        SA_TRY(group_heads(keys, nA, head.p, st));
        k_round_scatter<<<grid_for(nA), kThreads, 0, st>>>(A.p, nA, vals, head.p, sa, rank.p);
        SA_CUDA_TRY(cudaGetLastError());
        DevBuf<uint8_t> flags;
        SA_TRY(flags.alloc(nA, st, "active flags"));
        k_active<<<grid_for(nA), kThreads, 0, st>>>(keys, nA, flags.p);
        SA_CUDA_TRY(cudaGetLastError());
        head.reset();
        ka.reset();
        kb.reset();
        va.reset();
        vb.reset();
        DevBuf<uint32_t> A2;
        uint64_t nA2 = 0;
        SA_TRY(compact(A.p, flags.p, nA, A2, nA2, st));
        A.reset();
        A.p = A2.release();
        A.count = nA2;
        A.st = st;
        nA = nA2;
        h *= 2;
        ++rounds;
    }
    idx->build_rounds = rounds;
    return SA_OK;
}

// SA records (layouts in sa_search.cuh); bases past n read as 0 and are masked by length at search time.
//   L_REC16: {SA[r], bases k+32..k+47 (high half), bases k..k+31 (lo, hi)}
//   L_REC32: {SA[r], bases k+96..k+111 (high half), bases k..k+31 (lo, hi)}, {k+32..k+63, k+64..k+95}
__global__ void k_records(const uint64_t *__restrict__ text, uint64_t n, unsigned k, const uint32_t *__restrict__ sa,
                          uint4 *__restrict__ rec, int wide, uint64_t count) {
    GRID_STRIDE(r, count) {
        const uint64_t s = sa[r];
        const uint64_t c0 = text_window(text, s + k);
        if (!wide) {
            const uint64_t c1 = text_window(text, s + k + 32) >> 32;
            rec[r] = make_uint4((uint32_t)s, (uint32_t)c1, (uint32_t)c0, (uint32_t)(c0 >> 32));
        } else {
            const uint64_t c1 = text_window(text, s + k + 32);
            const uint64_t c2 = text_window(text, s + k + 64);
            const uint64_t c3 = text_window(text, s + k + 96) >> 32;
            rec[2 * r] = make_uint4((uint32_t)s, (uint32_t)c3, (uint32_t)c0, (uint32_t)(c0 >> 32));
            rec[2 * r + 1] = make_uint4((uint32_t)c1, (uint32_t)(c1 >> 32), (uint32_t)c2, (uint32_t)(c2 >> 32));
        }
    }
}

__global__ void k_extract_sa(const uint4 *__restrict__ rec, uint64_t count, unsigned per, uint32_t *__restrict__ out) {
    GRID_STRIDE(r, count) { out[r] = rec[r * per].x; }
}

}  // namespace

sa_status sa_extract_sa(const sa_index *idx, uint32_t *host_out) {
    const uint64_t n = idx->nparts > 1 ? idx->rank_end - idx->rank_base : idx->n;  // a partition: its slice
    if (idx->layout == 0) {
        SA_CUDA_TRY(cudaMemcpy(host_out, idx->sa, n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        return SA_OK;
    }
    const unsigned per = idx->layout == 2 ? 2 : 1;
    const uint64_t CH = 1ull << 28;
    DevBuf<uint32_t> tmp;
    SA_TRY(tmp.alloc(n < CH ? n : CH, nullptr, "SA export staging"));
    for (uint64_t off = 0; off < n; off += CH) {
        const uint64_t c = (n - off < CH) ? n - off : CH;
        k_extract_sa<<<grid_for(c), kThreads>>>(idx->rec + off * per, c, per, tmp.p);
        SA_CUDA_TRY(cudaGetLastError());
        SA_CUDA_TRY(cudaMemcpy(host_out + off, tmp.p, c * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    }
    return SA_OK;
}

// the trees of every bucket of >= kTreeMin suffixes (after the records; k-mers in chunks of 2^30)
sa_status build_bucket_trees(sa_index *idx, cudaStream_t st) {
    const uint64_t K = 1ull << (2 * idx->k);
    const uint64_t CH = 1ull << 30;
    thrust::counting_iterator<uint32_t> xs(0);
    DevBuf<int64_t> cnt;
    SA_TRY(cnt.alloc(1, st, "tree bucket count"));
    int64_t total = 0;
    for (uint64_t x0 = 0; x0 < K; x0 += CH) {
        const uint64_t len = (K - x0 < CH) ? K - x0 : CH;
        thrust::transform_iterator<IsTreeBucket, thrust::counting_iterator<uint32_t>, int64_t> flag(xs + x0,
                                                                                                 IsTreeBucket{idx->table});
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceReduce::Sum(tmp, bytes, flag, cnt.p, (int64_t)len, st);
        }, st, "tree bucket count"));
        int64_t c = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&c, cnt.p, 8, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        total += c;
    }
    if (total == 0) return SA_OK;
    DevBuf<uint32_t> big;
    SA_TRY(big.alloc((uint64_t)total, st, "tree buckets"));
    int64_t off = 0;
    for (uint64_t x0 = 0; x0 < K; x0 += CH) {
        const uint64_t len = (K - x0 < CH) ? K - x0 : CH;
        SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
            return cub::DeviceSelect::If(tmp, bytes, xs + x0, big.p + off, cnt.p, (int64_t)len, IsTreeBucket{idx->table},
                                         st);
        }, st, "tree bucket select"));
        int64_t c = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&c, cnt.p, 8, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        off += c;
    }
    // first line of every bucket's tree: exclusive scan of its line counts
    DevBuf<uint64_t> line0;
    SA_TRY(line0.alloc((uint64_t)total + 1, st, "tree offsets"));
    thrust::counting_iterator<uint64_t> ids(0);
    thrust::transform_iterator<TreeLinesOf, thrust::counting_iterator<uint64_t>, uint64_t> lines(ids,
                                                                                               TreeLinesOf{idx->table, big.p});
    SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, lines, line0.p, (int64_t)total, st);
    }, st, "tree offsets scan"));
    uint64_t last_off = 0, last_lines = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&last_off, line0.p + total - 1, 8, cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    {
        uint32_t x = 0, a = 0, b = 0;
        SA_CUDA_TRY(cudaMemcpy(&x, big.p + total - 1, 4, cudaMemcpyDeviceToHost));
        SA_CUDA_TRY(cudaMemcpy(&a, idx->table + x, 4, cudaMemcpyDeviceToHost));
        SA_CUDA_TRY(cudaMemcpy(&b, idx->table + (uint64_t)x + 1, 4, cudaMemcpyDeviceToHost));
        const uint32_t e = tree_pairs(b - a);
        last_lines = ((1ull << (2 * e)) - 1) / 3;
    }
    const uint64_t nlines = last_off + last_lines;
    if (nlines >= 0xFFFFFFFFull) { sa_set_error("bucket trees: too many lines"); return SA_ENOMEM; }
    uint32_t bits = 1;
    while ((1ull << bits) < 2ull * (uint64_t)total) ++bits;
    SA_CUDA_TRY(cudaMalloc(&idx->tree, nlines * 128));
    SA_CUDA_TRY(cudaMalloc(&idx->tree_hash, (1ull << bits) * sizeof(unsigned long long)));
    SA_CUDA_TRY(cudaMemsetAsync(idx->tree_hash, 0xFF, (1ull << bits) * sizeof(unsigned long long), st));
    k_tree_hash_insert<<<grid_for((uint64_t)total), kThreads, 0, st>>>(big.p, line0.p, (uint64_t)total, bits,
                                                                       idx->tree_hash);
    SA_CUDA_TRY(cudaGetLastError());
    k_tree_fill<<<148 * 32, 128, 0, st>>>(idx->table, big.p, line0.p, (uint64_t)total, idx->rec, idx->tree);
    SA_CUDA_TRY(cudaGetLastError());
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    idx->tree_count = (uint64_t)total;
    idx->tree_lines = nlines;
    idx->tree_bits = bits;
    return SA_OK;
}

// idx->rec = the records of the `count` suffixes sa[0..count) (layout 1 or 2); trims the memory pool
// first so the records can take the build's transient memory.
sa_status sa_build_records(sa_index *idx, const uint32_t *sa, uint64_t count, cudaStream_t st) {
    const uint64_t per = idx->layout == 2 ? 2 : 1;
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, idx->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    SA_CUDA_TRY(cudaMalloc(&idx->rec, (count ? count : 1) * per * sizeof(uint4)));
    if (count) {
        k_records<<<grid_for(count), kThreads, 0, st>>>(idx->text, idx->n, idx->k, sa, idx->rec, per == 2, count);
        SA_CUDA_TRY(cudaGetLastError());
    }
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    return SA_OK;
}

// Upload + validate + pack the reference (chunks of 256 MiB) into idx->text.
sa_status sa_pack_text(sa_index *idx, const char *ref_ascii, cudaStream_t st) {
    const uint64_t n = idx->n;
    idx->n_words = (n + 31) / 32 + kGuardWords;
    SA_CUDA_TRY(cudaMalloc(&idx->text, idx->n_words * sizeof(uint64_t)));
    SA_CUDA_TRY(cudaMemsetAsync(idx->text, 0, idx->n_words * sizeof(uint64_t), st));
    const uint64_t CH = 256ull << 20;
    DevBuf<uint8_t> dbuf;
    DevBuf<unsigned long long> bad;
    SA_TRY(dbuf.alloc(n < CH ? n : CH, st, "upload staging"));
    SA_TRY(bad.alloc(1, st, "validation flag"));
    SA_CUDA_TRY(cudaMemsetAsync(bad.p, 0xFF, sizeof(unsigned long long), st));
    for (uint64_t off = 0; off < n; off += CH) {
        const uint64_t len = (n - off < CH) ? n - off : CH;
        SA_CUDA_TRY(cudaMemcpyAsync(dbuf.p, ref_ascii + off, len, cudaMemcpyHostToDevice, st));
        k_pack<<<grid_for((len + 31) / 32), kThreads, 0, st>>>(dbuf.p, len, off / 32, idx->text, bad.p);
        SA_CUDA_TRY(cudaGetLastError());
    }
    unsigned long long h_bad = 0;
    SA_CUDA_TRY(cudaMemcpyAsync(&h_bad, bad.p, sizeof(h_bad), cudaMemcpyDeviceToHost, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    if (h_bad != ~0ull) {
        const unsigned char c = (unsigned char)ref_ascii[h_bad];
        sa_set_error("reference symbol 0x%02x ('%c') at position %llu is not A/C/G/T", c, (c >= 32 && c < 127) ? c : '?',
                     h_bad);
        return SA_ESYMBOL;
    }
    return SA_OK;
}

sa_status sa_build_index(sa_index *idx, const char *ref_ascii, cudaStream_t st) {
    const uint64_t n = idx->n;
    // ---- 1. upload + validate + pack ----
    SA_TRY(sa_pack_text(idx, ref_ascii, st));
    // ---- 2. suffix array ----
    SA_CUDA_TRY(cudaMalloc(&idx->sa, n * sizeof(uint32_t)));
    if (idx->build_dc3) SA_TRY(sa_build_sa_dc3(idx, st, nullptr, nullptr));  // the paper's DC3
    else SA_TRY(build_sa(idx, st));                                           // prefix doubling (default)
    // ---- 3. k-mer bracket table ----
    const uint64_t K = 1ull << (2 * idx->k);
    SA_CUDA_TRY(cudaMalloc(&idx->table, (K + 1) * sizeof(uint32_t)));
    idx->table_entries = K + 1;
    k_table<<<grid_for(n + 1), kThreads, 0, st>>>(idx->text, n, idx->sa, idx->k, idx->table);
    SA_CUDA_TRY(cudaGetLastError());
    // ---- 3b. second-level tables for the large buckets (SA_INDEX_SUBTABLE) ----
    if (idx->subtables && idx->k + 4 <= 32) {
        // count, then select, the large buckets (chunks of 2^30 k-mers)
        thrust::counting_iterator<uint32_t> xs(0);
        const uint64_t CH = 1ull << 30;
        DevBuf<int64_t> cnt;
        SA_TRY(cnt.alloc(1, st, "big bucket count"));
        thrust::transform_iterator<IsBigBucket, thrust::counting_iterator<uint32_t>, int64_t> flag(xs, IsBigBucket{idx->table});
        int64_t total = 0;
        for (uint64_t x0 = 0; x0 < K; x0 += CH) {
            const uint64_t len = (K - x0 < CH) ? K - x0 : CH;
            SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
                return cub::DeviceReduce::Sum(tmp, bytes, flag + x0, cnt.p, (int64_t)len, st);
            }, st, "big bucket count"));
            int64_t c = 0;
            SA_CUDA_TRY(cudaMemcpyAsync(&c, cnt.p, 8, cudaMemcpyDeviceToHost, st));
            SA_CUDA_TRY(cudaStreamSynchronize(st));
            total += c;
        }
        if (total > 0 && total < (1ll << 26)) {
            DevBuf<uint32_t> big;
            SA_TRY(big.alloc((uint64_t)total, st, "big buckets"));
            int64_t off = 0;
            for (uint64_t x0 = 0; x0 < K; x0 += CH) {
                const uint64_t len = (K - x0 < CH) ? K - x0 : CH;
                SA_TRY(cub_call([&](void *tmp, size_t &bytes) {
                    return cub::DeviceSelect::If(tmp, bytes, xs + x0, big.p + off, cnt.p, (int64_t)len,
                                                 IsBigBucket{idx->table}, st);
                }, st, "big bucket select"));
                int64_t c = 0;
                SA_CUDA_TRY(cudaMemcpyAsync(&c, cnt.p, 8, cudaMemcpyDeviceToHost, st));
                SA_CUDA_TRY(cudaStreamSynchronize(st));
                off += c;
            }
            uint32_t bits = 1;
            while ((1ull << bits) < 2ull * (uint64_t)total) ++bits;
            SA_CUDA_TRY(cudaMalloc(&idx->big_sub, (uint64_t)total * 257 * sizeof(uint32_t)));
            SA_CUDA_TRY(cudaMalloc(&idx->big_hash, (1ull << bits) * sizeof(unsigned long long)));
            SA_CUDA_TRY(cudaMemsetAsync(idx->big_hash, 0xFF, (1ull << bits) * sizeof(unsigned long long), st));
            k_big_hash_insert<<<grid_for((uint64_t)total), kThreads, 0, st>>>(big.p, (uint64_t)total, bits, idx->big_hash);
            SA_CUDA_TRY(cudaGetLastError());
            k_big_subtables<<<(unsigned)total, 128, 0, st>>>(idx->text, n, idx->sa, idx->k, idx->table, big.p,
                                                            idx->big_sub);
            SA_CUDA_TRY(cudaGetLastError());
            SA_CUDA_TRY(cudaStreamSynchronize(st));
            idx->big_count = (uint64_t)total;
            idx->big_bits = bits;
        }
    }
    // ---- 4. SA records (default layout) ----
    uint64_t sa_bytes = n * sizeof(uint32_t);
    if (idx->layout != 0) {
        SA_TRY(sa_build_records(idx, idx->sa, n, st));
        SA_CUDA_TRY(cudaFree(idx->sa));
        idx->sa = nullptr;
        sa_bytes = n * (idx->layout == 2 ? 2 : 1) * sizeof(uint4);
    }
    // ---- 5. bucket trees (SA_INDEX_BUCKET_TREE; rec32 records) ----
    if (idx->bucket_tree && idx->layout == 2) SA_TRY(build_bucket_trees(idx, st));
    SA_CUDA_TRY(cudaStreamSynchronize(st));
    idx->device_bytes = idx->n_words * 8 + sa_bytes + (K + 1) * 4 + idx->big_count * 257 * 4 +
                        (idx->big_count ? (1ull << idx->big_bits) * 8 : 0) + idx->tree_lines * 128 +
                        (idx->tree_count ? (1ull << idx->tree_bits) * 8 : 0);
    // hand the build's transient memory back to the driver
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, idx->device) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    return SA_OK;
}
