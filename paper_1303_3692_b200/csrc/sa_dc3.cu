// sa_dc3.cu -- the paper's suffix-array construction, DC3 / skew (Sec. III), on the
// GPU: SURVEY.md Sec. 8(f) row f2, selected with SA_INDEX_BUILD_DC3.  The default builder is prefix
// doubling (sa_build.cu); both must give the same, unique, suffix array.
//
// With B_k = {i in [0, n) : i mod 3 = k} and the sample set C = B_1 u B_2 (reading A17):
//   step 1: radix sort the sample positions by their triples (t_i, t_i+1, t_i+2), name the
//          triples by rank; if names repeat, recurse on R = R_1 . R_2 (the names in position order)
//          -> rank(S_i) for every sample suffix (Table II);
//   step 2: the non-sample suffixes in the order of the pairs (t_i, rank(S_i+1)): the
//          sample order restricted to B_1 shifted by one, then a stable sort by t_i;
//   step 3: merge, comparing S_i (i in C) with S_j (j in B_0) as
//          (t_i, rank(S_i+1)) vs (t_j, rank(S_j+1))                 if i in B_1,
//          (t_i, t_i+1, rank(S_i+2)) vs (t_j, t_j+1, rank(S_j+2))   if i in B_2.
// The symbol 0 marks "past the end" (the text uses 1..4 for a..t), so a suffix that is a proper
// prefix of another sorts first (reading A2).  As in the skew algorithm of Karkkainen and Sanders, a
// dummy sample position n is added when n mod 3 = 1 so that every B_0 suffix has a ranked neighbour.
// The merge is a GPU merge-path merge (thrust::merge) with that comparator.
#include <cub/cub.cuh>
#include <thrust/execution_policy.h>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <thrust/merge.h>

#include <vector>

#include "sa_internal.cuh"

namespace {

constexpr int kThreads = 256;

inline unsigned grid_for(uint64_t n) {
    uint64_t b = (n + kThreads - 1) / kThreads;
    if (b > 148ull * 64) b = 148ull * 64;
    return (unsigned)(b ? b : 1);
}

#define GRID_STRIDE(i, n) \
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (uint64_t)gridDim.x * blockDim.x)

inline int bits_for(uint64_t v) {  // bits needed to hold values 0..v
    int b = 1;
    while (b < 64 && (v >> b)) ++b;
    return b;
}

template <typename F>
sa_status cub_run(F f, cudaStream_t st, const char *what) {
    size_t bytes = 0;
    cudaError_t e = f(nullptr, bytes);
    if (e != cudaSuccess) { (void)cudaGetLastError(); sa_set_error("%s: %s", what, cudaGetErrorString(e)); return SA_ECUDA; }
    DevBuf<uint8_t> tmp;
    SA_TRY(tmp.alloc(bytes, st, what));
    e = f(tmp.p, bytes);
    if (e != cudaSuccess) { (void)cudaGetLastError(); sa_set_error("%s: %s", what, cudaGetErrorString(e)); return SA_ECUDA; }
    return SA_OK;
}

// ---- kernels ---------------------------------------------------------------------------------
// sample positions: 3j+1 for j < n0 (the last one is the dummy n when n mod 3 = 1), then 3j+2 for j < n2
__global__ void k_sample_positions(uint64_t n0, uint64_t n02, uint32_t *pos) {
    GRID_STRIDE(t, n02) { pos[t] = (uint32_t)(t < n0 ? 3 * t + 1 : 3 * (t - n0) + 2); }
}

// packed triple key (symbols < 2^b)
__global__ void k_triple_keys(const uint32_t *__restrict__ s, const uint32_t *__restrict__ pos, uint64_t m, int b,
                              uint64_t *__restrict__ key) {
    GRID_STRIDE(t, m) {
        const uint64_t i = pos[t];
        key[t] = ((uint64_t)s[i] << (2 * b)) | ((uint64_t)s[i + 1] << b) | s[i + 2];
    }
}

// one symbol as the key (for the three stable LSD passes when a triple does not fit 64 bits)
__global__ void k_symbol_keys(const uint32_t *__restrict__ s, const uint32_t *__restrict__ pos, uint64_t m, int off,
                              uint32_t *__restrict__ key) {
    GRID_STRIDE(t, m) { key[t] = s[(uint64_t)pos[t] + off]; }
}

// flag[t] = 1 if the triple at sorted slot t differs from slot t-1 (names = inclusive sum)
__global__ void k_new_name(const uint32_t *__restrict__ s, const uint32_t *__restrict__ sorted, uint64_t m,
                           uint32_t *__restrict__ flag) {
    GRID_STRIDE(t, m) {
        uint32_t f = 1;
        if (t > 0) {
            const uint64_t i = sorted[t], j = sorted[t - 1];
            f = (s[i] != s[j] || s[i + 1] != s[j + 1] || s[i + 2] != s[j + 2]) ? 1u : 0u;
        }
        flag[t] = f;
    }
}

// R = R_1 . R_2: the name of position i goes to i/3 (i mod 3 = 1) or n0 + i/3 (i mod 3 = 2)
__global__ void k_place_names(const uint32_t *__restrict__ sorted, const uint32_t *__restrict__ name, uint64_t m,
                              uint64_t n0, uint32_t *__restrict__ R) {
    GRID_STRIDE(t, m) {
        const uint64_t i = sorted[t];
        R[(i % 3 == 1) ? i / 3 : n0 + i / 3] = name[t];
    }
}

__global__ void k_rank_from_sa(const uint32_t *__restrict__ SA12, uint64_t m, uint32_t *__restrict__ R) {
    GRID_STRIDE(t, m) { R[SA12[t]] = (uint32_t)(t + 1); }
}

__global__ void k_sa_from_unique_names(const uint32_t *__restrict__ R, uint64_t m, uint32_t *__restrict__ SA12) {
    GRID_STRIDE(t, m) { SA12[R[t] - 1] = (uint32_t)t; }
}

// sample-array entry -> text position
struct SamplePos {
    uint64_t n0;
    __host__ __device__ uint32_t operator()(uint32_t v) const {
        return (uint32_t)(v < n0 ? 3ull * v + 1 : 3ull * (v - n0) + 2);
    }
};

struct IsB1 {  // SA12 entries that are B_1 positions (the dummy n included when n mod 3 = 1)
    uint64_t n0;
    __host__ __device__ bool operator()(uint32_t v) const { return v < n0; }
};

__global__ void k_b1_to_b0(const uint32_t *__restrict__ sel, uint64_t m, uint32_t *__restrict__ out) {
    GRID_STRIDE(t, m) { out[t] = 3 * sel[t]; }  // S_{i} with i+1 in B_1, in rank(S_{i+1}) order
}

__global__ void k_first_symbol(const uint32_t *__restrict__ s, const uint32_t *__restrict__ pos, uint64_t m,
                               uint32_t *__restrict__ key) {
    GRID_STRIDE(t, m) { key[t] = s[pos[t]]; }
}

// step 3 comparator on text positions (0 <= x, y < n)
struct SuffixLess {
    const uint32_t *s;  // text symbols, 3 zeros past the end
    const uint32_t *R;  // sample ranks: R[i/3] for i mod 3 = 1, R[n0 + i/3] for i mod 3 = 2; zeros past
    uint64_t n0;
    __device__ __forceinline__ uint32_t rank(uint64_t x) const { return x % 3 == 1 ? R[x / 3] : R[n0 + x / 3]; }
    __device__ bool operator()(uint32_t xa, uint32_t ya) const {
        const uint64_t x = xa, y = ya;
        const unsigned mx = (unsigned)(x % 3), my = (unsigned)(y % 3);
        if (mx != 0 && my != 0) return rank(x) < rank(y);
        // one or both in B_0: compare one symbol + the rank of a sample suffix when the shifted pair
        // is (B_1 or B_2 | B_2 or B_1 ...): (t, rank(+1)) works unless a B_2 meets a B_0 (then +1 lands
        // in B_0 for the B_2 side) -- use (t, t+1, rank(+2)) there
        if (mx == 2 || my == 2) {
            if (s[x] != s[y]) return s[x] < s[y];
            if (s[x + 1] != s[y + 1]) return s[x + 1] < s[y + 1];
            return rank(x + 2) < rank(y + 2);
        }
        if (s[x] != s[y]) return s[x] < s[y];
        return rank(x + 1) < rank(y + 1);
    }
};

// Sorts the sample positions `pos` (m of them) by triple, stably.
sa_status sort_triples(const uint32_t *s, uint64_t K, DevBuf<uint32_t> &pos, uint64_t m, cudaStream_t st) {
    const int b = bits_for(K);
    DevBuf<uint32_t> pos2;
    SA_TRY(pos2.alloc(m, st, "dc3 sort values"));
    if (3 * b <= 64) {
        DevBuf<uint64_t> k1, k2;
        SA_TRY(k1.alloc(m, st, "dc3 triple keys"));
        SA_TRY(k2.alloc(m, st, "dc3 triple keys (alt)"));
        k_triple_keys<<<grid_for(m), kThreads, 0, st>>>(s, pos.p, m, b, k1.p);
        SA_CUDA_TRY(cudaGetLastError());
        cub::DoubleBuffer<uint64_t> dk(k1.p, k2.p);
        cub::DoubleBuffer<uint32_t> dv(pos.p, pos2.p);
        SA_TRY(cub_run([&](void *t, size_t &bytes) {
            return cub::DeviceRadixSort::SortPairs(t, bytes, dk, dv, (int64_t)m, 0, 3 * b, st);
        }, st, "dc3 triple sort"));
        if (dv.Current() != pos.p) SA_CUDA_TRY(cudaMemcpyAsync(pos.p, dv.Current(), m * 4, cudaMemcpyDeviceToDevice, st));
        return SA_OK;
    }
    // three stable LSD passes, last symbol first
    DevBuf<uint32_t> k1, k2;
    SA_TRY(k1.alloc(m, st, "dc3 symbol keys"));
    SA_TRY(k2.alloc(m, st, "dc3 symbol keys (alt)"));
    for (int off = 2; off >= 0; --off) {
        k_symbol_keys<<<grid_for(m), kThreads, 0, st>>>(s, pos.p, m, off, k1.p);
        SA_CUDA_TRY(cudaGetLastError());
        cub::DoubleBuffer<uint32_t> dk(k1.p, k2.p);
        cub::DoubleBuffer<uint32_t> dv(pos.p, pos2.p);
        SA_TRY(cub_run([&](void *t, size_t &bytes) {
            return cub::DeviceRadixSort::SortPairs(t, bytes, dk, dv, (int64_t)m, 0, b, st);
        }, st, "dc3 symbol sort"));
        if (dv.Current() != pos.p) SA_CUDA_TRY(cudaMemcpyAsync(pos.p, dv.Current(), m * 4, cudaMemcpyDeviceToDevice, st));
    }
    return SA_OK;
}

struct Dc3Trace {
    uint32_t *sample_rank = nullptr;  // host, n entries (top level only)
    uint32_t *nonsample = nullptr;    // host, n0 entries (top level only)
};

// s: n + 3 symbols in [0, K] (s[n..n+2] = 0, real symbols >= 1).  SA: n entries.
sa_status dc3(const uint32_t *s, uint64_t n, uint64_t K, uint32_t *SA, cudaStream_t st, int depth, Dc3Trace *tr) {
    if (depth > 64) { sa_set_error("DC3 recursion too deep"); return SA_ECUDA; }
    if (n == 1) {
        const uint32_t z = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(SA, &z, 4, cudaMemcpyHostToDevice, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        return SA_OK;
    }
    const uint64_t n0 = (n + 2) / 3, n1 = (n + 1) / 3, n2 = n / 3, n02 = n0 + n2;
    (void)n1;  // n0 - n1 = 1 exactly when the dummy sample n exists (n mod 3 = 1)
    // ---- step 1: sort and name the sample triples ----
    DevBuf<uint32_t> pos, R, SA12;
    SA_TRY(pos.alloc(n02, st, "dc3 sample positions"));
    k_sample_positions<<<grid_for(n02), kThreads, 0, st>>>(n0, n02, pos.p);
    SA_CUDA_TRY(cudaGetLastError());
    SA_TRY(sort_triples(s, K, pos, n02, st));
    uint32_t max_name = 0;
    SA_TRY(R.alloc(n02 + 3, st, "dc3 reduced string"));
    SA_CUDA_TRY(cudaMemsetAsync(R.p, 0, (n02 + 3) * 4, st));
    {
        DevBuf<uint32_t> name;
        SA_TRY(name.alloc(n02, st, "dc3 names"));
        k_new_name<<<grid_for(n02), kThreads, 0, st>>>(s, pos.p, n02, name.p);
        SA_CUDA_TRY(cudaGetLastError());
        SA_TRY(cub_run([&](void *t, size_t &bytes) {
            return cub::DeviceScan::InclusiveSum(t, bytes, name.p, name.p, (int64_t)n02, st);
        }, st, "dc3 naming scan"));
        k_place_names<<<grid_for(n02), kThreads, 0, st>>>(pos.p, name.p, n02, n0, R.p);
        SA_CUDA_TRY(cudaGetLastError());
        SA_CUDA_TRY(cudaMemcpyAsync(&max_name, name.p + n02 - 1, 4, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
    }
    pos.reset();
    SA_TRY(SA12.alloc(n02, st, "dc3 sample SA"));
    if (max_name < n02) {  // names repeat: recurse on R
        SA_TRY(dc3(R.p, n02, max_name, SA12.p, st, depth + 1, nullptr));
        k_rank_from_sa<<<grid_for(n02), kThreads, 0, st>>>(SA12.p, n02, R.p);
    } else {
        k_sa_from_unique_names<<<grid_for(n02), kThreads, 0, st>>>(R.p, n02, SA12.p);
    }
    SA_CUDA_TRY(cudaGetLastError());
    // ---- step 2: the B_0 suffixes ordered by (t_i, rank(S_{i+1})) ----
    // the B_1 entries of the sample order, shifted left by one, are B_0 in rank(S_{i+1}) order (the
    // dummy n, smallest of all, brings n-1 first); a stable sort by t_i finishes it
    DevBuf<uint32_t> SA0, sel;
    SA_TRY(sel.alloc(n0, st, "dc3 B0 selection"));
    {
        DevBuf<int64_t> cnt;
        SA_TRY(cnt.alloc(1, st, "dc3 count"));
        SA_TRY(cub_run([&](void *t, size_t &bytes) {
            return cub::DeviceSelect::If(t, bytes, SA12.p, sel.p, cnt.p, (int64_t)n02, IsB1{n0}, st);
        }, st, "dc3 B1 select"));
        int64_t h = 0;
        SA_CUDA_TRY(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
        if ((uint64_t)h != n0) {
            sa_set_error("DC3: %lld B0 suffixes, expected %llu", (long long)h, (unsigned long long)n0);
            return SA_ECUDA;
        }
    }
    SA_TRY(SA0.alloc(n0, st, "dc3 SA0"));
    {
        DevBuf<uint32_t> b0, k1, k2;
        SA_TRY(b0.alloc(n0, st, "dc3 B0"));
        SA_TRY(k1.alloc(n0, st, "dc3 B0 keys"));
        SA_TRY(k2.alloc(n0, st, "dc3 B0 keys (alt)"));
        k_b1_to_b0<<<grid_for(n0), kThreads, 0, st>>>(sel.p, n0, b0.p);
        SA_CUDA_TRY(cudaGetLastError());
        k_first_symbol<<<grid_for(n0), kThreads, 0, st>>>(s, b0.p, n0, k1.p);
        SA_CUDA_TRY(cudaGetLastError());
        cub::DoubleBuffer<uint32_t> dk(k1.p, k2.p);
        cub::DoubleBuffer<uint32_t> dv(b0.p, SA0.p);
        SA_TRY(cub_run([&](void *t, size_t &bytes) {
            return cub::DeviceRadixSort::SortPairs(t, bytes, dk, dv, (int64_t)n0, 0, bits_for(K), st);
        }, st, "dc3 B0 sort"));
        if (dv.Current() != SA0.p) SA_CUDA_TRY(cudaMemcpyAsync(SA0.p, dv.Current(), n0 * 4, cudaMemcpyDeviceToDevice, st));
        SA_CUDA_TRY(cudaStreamSynchronize(st));
    }
    sel.reset();
    if (tr) {  // Table II (sample ranks, 1-based among the real samples) and the B_0 order
        std::vector<uint32_t> hR(n02), hSA12(n02);
        SA_CUDA_TRY(cudaMemcpy(hSA12.data(), SA12.p, n02 * 4, cudaMemcpyDeviceToHost));
        if (tr->sample_rank) {
            for (uint64_t i = 0; i < n; ++i) tr->sample_rank[i] = 0;
            uint32_t r = 0;
            for (uint64_t t = 0; t < n02; ++t) {
                const uint64_t p = hSA12[t] < n0 ? 3ull * hSA12[t] + 1 : 3ull * (hSA12[t] - n0) + 2;
                if (p < n) tr->sample_rank[p] = ++r;
            }
        }
        if (tr->nonsample) SA_CUDA_TRY(cudaMemcpy(tr->nonsample, SA0.p, n0 * 4, cudaMemcpyDeviceToHost));
    }
    // ---- step 3: merge ----
    {
        thrust::transform_iterator<SamplePos, const uint32_t *> a_first(SA12.p, SamplePos{n0});
        const uint64_t a_skip = (n % 3 == 1) ? 1 : 0;  // the dummy sample n sorts first: skip it
        SuffixLess less{s, R.p, n0};
        thrust::merge(thrust::cuda::par.on(st), a_first + a_skip, a_first + n02, SA0.p, SA0.p + n0, SA, less);
        SA_CUDA_TRY(cudaGetLastError());
        SA_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return SA_OK;
}

__global__ void k_text_symbols(const uint64_t *__restrict__ text, uint64_t n, uint32_t *__restrict__ s) {
    GRID_STRIDE(i, n + 3) { s[i] = i < n ? (uint32_t)((text[i >> 5] >> (62 - 2 * (i & 31))) & 3u) + 1u : 0u; }
}

}  // namespace

// The SA of the index's packed text by DC3 (into idx->sa, already allocated).
sa_status sa_build_sa_dc3(sa_index *idx, cudaStream_t st, uint32_t *trace_rank, uint32_t *trace_nonsample) {
    const uint64_t n = idx->n;
    DevBuf<uint32_t> s;
    SA_TRY(s.alloc(n + 3, st, "dc3 text symbols"));
    k_text_symbols<<<grid_for(n + 3), kThreads, 0, st>>>(idx->text, n, s.p);
    SA_CUDA_TRY(cudaGetLastError());
    Dc3Trace tr{trace_rank, trace_nonsample};
    return dc3(s.p, n, 4, idx->sa, st, 0, (trace_rank || trace_nonsample) ? &tr : nullptr);
}
