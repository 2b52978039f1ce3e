// sa_internal.cuh -- private types and device helpers of libsa (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <mutex>
#include <vector>

#include "sa.h"

// ---------------------------------------------------------------------------------------------
// errors
void sa_set_error(const char *fmt, ...);
void sa_clear_error();

#define SA_CUDA_TRY(call)                                                                              \
    do {                                                                                               \
        cudaError_t e_ = (call);                                                                       \
        if (e_ != cudaSuccess) {                                                                       \
            (void)cudaGetLastError();                                                                  \
            sa_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));          \
            return e_ == cudaErrorMemoryAllocation ? SA_ENOMEM : SA_ECUDA;                             \
        }                                                                                              \
    } while (0)

#define SA_TRY(call)                                                                                   \
    do {                                                                                               \
        sa_status s_ = (call);                                                                         \
        if (s_ != SA_OK) return s_;                                                                    \
    } while (0)

// RAII device buffer (stream-ordered allocator); freed on scope exit.
template <typename T>
struct DevBuf {
    T *p = nullptr;
    size_t count = 0;
    cudaStream_t st = nullptr;
    DevBuf() = default;
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    ~DevBuf() { reset(); }
    sa_status alloc(size_t n, cudaStream_t s, const char *what) {
        reset();
        st = s;
        if (n == 0) n = 1;
        cudaError_t e = cudaMallocAsync((void **)&p, n * sizeof(T), s);
        if (e != cudaSuccess) {
            (void)cudaGetLastError();
            p = nullptr;
            sa_set_error("device allocation of %zu bytes for %s failed: %s", n * sizeof(T), what,
                         cudaGetErrorString(e));
            return e == cudaErrorMemoryAllocation ? SA_ENOMEM : SA_ECUDA;
        }
        count = n;
        return SA_OK;
    }
    void reset() {
        if (p) cudaFreeAsync(p, st);
        p = nullptr;
        count = 0;
    }
    T *release() {
        T *r = p;
        p = nullptr;
        count = 0;
        return r;
    }
};

// ---------------------------------------------------------------------------------------------
// the index (immutable after create)
constexpr uint32_t kBigBucket = 32;  // SA_INDEX_SUBTABLE threshold (suffixes per k-mer bucket)
constexpr unsigned long long kBigEmpty = ~0ull;  // empty sub-table hash slot (no {x, id} entry equals it)
constexpr uint32_t kTreeMin = 32;  // SA_INDEX_BUCKET_TREE: buckets of at least this many suffixes get a tree

__host__ __device__ __forceinline__ int ilog2_u32(uint32_t v) {  // floor(log2 v), v > 0
#ifdef __CUDA_ARCH__
    return 31 - __clz(v);
#else
    return 31 - __builtin_clz(v);
#endif
}

// SA_INDEX_BUCKET_TREE: the pair levels stored for a bucket of B suffixes -- depths 0 .. 2E-1 of its
// binary search, E = max(1, (floor(log2 B) - 2) / 2): the deeper levels' intervals hold < ~8 suffixes,
// whose records already share lines in the flat array
__host__ __device__ __forceinline__ uint32_t tree_pairs(uint32_t B) {
    const int lg = ilog2_u32(B | 1);
    const int e = (lg - 2) / 2;
    return e < 1 ? 1u : (uint32_t)e;
}
// line of pair root r (at depth 2e) in a bucket's tree: lines are numbered level by level (4^e per level)
__host__ __device__ __forceinline__ uint64_t tree_line(uint32_t r) {
    const int d = ilog2_u32(r);  // even
    const uint64_t p4 = 1ull << d;        // 4^e
    return (p4 - 1) / 3 + (r - p4);
}
constexpr uint64_t kGuardWords = 6;  // zero words past the text: windows up to base n + 159 are readable

// SA values of the layout: base pointer + stride in uint32 units
struct SaView {
    const uint32_t *base;
    uint32_t stride;
};
struct sa_index {
    int device = 0;
    uint64_t n = 0;          // reference length
    uint32_t k = 0;          // k-mer bracket table
    uint64_t n_words = 0;    // packed text words incl. kGuardWords zero guard words
    uint64_t *text = nullptr;    // dev: 2-bit MSB-first, zero-padded past n (kGuardWords zero words)
    int layout = 1;              // sa_search::L_PLAIN (0), L_REC16 (1), L_REC32 (2)
    uint32_t *sa = nullptr;      // dev: n entries (L_PLAIN)
    uint4 *rec = nullptr;        // dev: n records of 1 (L_REC16) or 2 (L_REC32) uint4, see sa_search.cuh
    uint32_t *table = nullptr;   // dev: 4^k + 1 entries
    uint64_t device_bytes = 0;
    uint32_t build_rounds = 0;   // prefix-doubling rounds after the initial sort
    bool build_dc3 = false;      // SA_INDEX_BUILD_DC3: the SA by DC3 instead of prefix doubling
    // SA_INDEX_SUBTABLE: buckets of more than kBigBucket suffixes get a (k+4)-base sub-table
    bool subtables = false;
    uint64_t big_count = 0;      // large buckets
    uint32_t big_bits = 0;       // log2 of the hash table size
    unsigned long long *big_hash = nullptr;  // dev: open addressing, x << 32 | sub-table id, empty = kBigEmpty
    uint32_t *big_sub = nullptr; // dev: big_count x 257 global SA ranks
    // SA_INDEX_BUCKET_TREE: for every bucket of >= kTreeMin suffixes, the records of the top 2E levels of
    // its binary search, 3 per 128-byte line (a pivot and its two children: two levels per DRAM line)
    bool bucket_tree = false;
    uint64_t tree_count = 0, tree_lines = 0;
    uint32_t tree_bits = 0;
    unsigned long long *tree_hash = nullptr;  // dev: x << 32 | first line of the bucket's tree, empty = ~0
    uint4 *tree = nullptr;                    // dev: tree_lines x 128 bytes (4 record slots, 3 used)
    // partitioned index (sa_index_create_part, csrc/sa_part.cu): this index holds SA ranks
    // [rank_base, rank_end) and table entries [x_base, x_base + 4^(k-rb) * (keys in the part)] only:
    // the suffixes whose route key (first route_bases bases, sa_suffix_e) lies in
    // [part_keys[part], part_keys[part+1]); part_ranks[g] = first rank of part g (all parts);
    // route_table = the route-level bracket table T_r[K] = #{i : trunc_rb(S_i) < K}, K in [0, 4^rb]
    uint32_t part = 0, nparts = 1, route_bases = 0;
    uint64_t x_base = 0, rank_base = 0, rank_end = 0;
    std::vector<uint32_t> part_keys;
    std::vector<uint64_t> part_ranks;
    uint64_t table_entries = 0;          // entries of `table` (a partition: its slice)
    uint32_t *route_table = nullptr;     // dev
    uint64_t *part_ranks_dev = nullptr;  // dev copy of part_ranks
    // host-buffer pipeline (sa_match_batch_host); grown on demand, guarded by mu
    std::mutex mu;
    cudaStream_t pipe_stream[2] = {nullptr, nullptr};
    uint64_t *pipe_words[2] = {nullptr, nullptr};
    uint32_t *pipe_lens[2] = {nullptr, nullptr};
    uint32_t *pipe_out[2] = {nullptr, nullptr};
    uint32_t *pipe_order[2] = {nullptr, nullptr};  // per-chunk read ordering (a5)
    void *pipe_ws[2] = {nullptr, nullptr};         // its sort workspace
    size_t pipe_ws_bytes = 0;
    uint64_t pipe_chunk = 0;
    uint64_t pipe_words_cap = 0;
};

// ---------------------------------------------------------------------------------------------
// device helpers

// Loads of the search path.  SA_LD_MODE (compile time) selects the PTX cache operator for every
// random access of the match kernel: 0 = ld.global.nc (read-only path, default), 1 = ld.global.cg
// (L2 only), 2 = ld.global.nc.L1::no_allocate, 3 = ld.global.ca, 4 = ld.global.nc.L2::64B (64-byte
// L2 fetch: 2 DRAM sectors per random access instead of 4, profiles/r01-2b/gather_async.txt),
// 5 = 2 + 4.
#ifndef SA_LD_MODE
#define SA_LD_MODE 0
#endif
#if SA_LD_MODE == 1
#define SA_LD_OP "ld.global.cg"
#elif SA_LD_MODE == 2
#define SA_LD_OP "ld.global.nc.L1::no_allocate"
#elif SA_LD_MODE == 3
#define SA_LD_OP "ld.global.ca"
#elif SA_LD_MODE == 4
#define SA_LD_OP "ld.global.nc.L2::64B"
#elif SA_LD_MODE == 5
#define SA_LD_OP "ld.global.nc.L1::no_allocate.L2::64B"
#else
#define SA_LD_OP "ld.global.nc"
#endif
__device__ __forceinline__ uint32_t ld_u32(const uint32_t *p) {
    uint32_t v;
    asm(SA_LD_OP ".u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint64_t ld_u64(const uint64_t *p) {
    uint64_t v;
    asm(SA_LD_OP ".u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_v4u32(const void *p) {
    uint4 v;
    asm(SA_LD_OP ".v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ uint2 ld_v2u32(const void *p) {
    uint2 v;
    asm(SA_LD_OP ".v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ void ld_v2u64(const void *p, uint64_t &a, uint64_t &b) {
    asm(SA_LD_OP ".v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
// 256-bit load (sm_100): LDG.E.ENL2.256
__device__ __forceinline__ void ld_v4u64(const void *p, uint64_t &a, uint64_t &b, uint64_t &c, uint64_t &d) {
    asm(SA_LD_OP ".v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}

// Large batches (MatchArgs::wide, >= kWideQ reads): the read row (one random 32-byte row per read, used
// once) is loaded with L1::no_allocate + an L2::64B fetch (half the DRAM bytes of a 128-byte line), and
// the bracket-table pair with an L2::64B fetch.  Measured (profiles/r02/r02ae, r02af, r02aq): k_match 10.05 vs
// 10.45 ms per 100 M reads; at 12.5 M 1.49-1.50 vs 1.47 ms with 256-thread blocks, 1.351 vs 1.363 with the
// 64-thread blocks.  Batches below 2^20 reads (L2-sized indexes and batches) keep the plain loads.  A
// warp-uniform branch selects the instruction.
__device__ __forceinline__ void ld_row_v4u64(const void *p, bool wide, uint64_t &a, uint64_t &b, uint64_t &c,
                                             uint64_t &d) {
    if (wide) asm("ld.global.nc.L1::no_allocate.L2::64B.v4.u64 {%0, %1, %2, %3}, [%4];"
                  : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    else asm(SA_LD_OP ".v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
}
__device__ __forceinline__ void ld_row_v2u64(const void *p, bool wide, uint64_t &a, uint64_t &b) {
    if (wide) asm("ld.global.nc.L1::no_allocate.L2::64B.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
    else asm(SA_LD_OP ".v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
__device__ __forceinline__ uint64_t ld_row_u64(const uint64_t *p, bool wide) {
    uint64_t v;
    if (wide) asm("ld.global.nc.L1::no_allocate.L2::64B.u64 %0, [%1];" : "=l"(v) : "l"(p));
    else asm(SA_LD_OP ".u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ uint4 ld_tab_v4u32(const void *p, bool wide) {
    uint4 v;
    if (wide) asm("ld.global.nc.L2::64B.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    else asm(SA_LD_OP ".v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}
#ifndef SA_WIDE_Q_LOG2
#define SA_WIDE_Q_LOG2 20
#endif
constexpr uint64_t kWideQ = 1ull << SA_WIDE_Q_LOG2;  // reads per launch from which MatchArgs::wide is set (1 M)

// a load the compiler may not merge with an earlier load of the same address (re-reads a value instead
// of keeping it live in a register)
__device__ __forceinline__ uint32_t reload_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

// TMA bulk prefetch of global bytes [p, p + bytes) into L2 (cp.async.bulk.prefetch.L2: one instruction,
// no registers, no completion to wait for); the range is widened to 16-byte granules as the
// instruction requires.
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, uint64_t bytes) {
    const uint64_t a = reinterpret_cast<uint64_t>(p);
    const uint64_t lo = a & ~15ull, hi = (a + bytes + 15) & ~15ull;
    if (hi > lo)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(lo), "r"((uint32_t)(hi - lo)) : "memory");
}

// 32 bases of the packed text starting at base b (b < n + 32); bases past n read as 0 ('a').
__device__ __forceinline__ uint64_t text_window(const uint64_t *__restrict__ text, uint64_t b) {
    const uint64_t w = b >> 5;
    const unsigned sh = (unsigned)(b & 31u) << 1;
    const uint64_t x0 = ld_u64(text + w);
    const uint64_t x1 = ld_u64(text + w + 1);
    return sh ? (x0 << sh) | (x1 >> (64u - sh)) : x0;
}

// mask selecting the first L (0..32) bases of a packed word
__device__ __forceinline__ uint64_t prefix_mask(unsigned L) {
    return L >= 32 ? ~0ull : (L == 0 ? 0ull : ~(~0ull >> (2u * L)));
}

// e_j(s): the j-mer code of suffix s when it has >= j bases; U - 1 for a shorter suffix whose a-padded
// j-mer is U.  e is non-decreasing along the SA, and #{i : e_j(i) < x} = #{i : trunc_j(S_i) < x}: the
// bracket table T[x] counts the suffixes with e < x (k_table).
__device__ __forceinline__ int64_t sa_suffix_e(const uint64_t *__restrict__ text, uint64_t n, uint64_t s, unsigned j) {
    const uint64_t len = n - s;
    uint64_t w = text_window(text, s);
    if (len < j) w &= prefix_mask((unsigned)len);
    const int64_t code = (int64_t)(w >> (64 - 2 * j));
    return len >= j ? code : code - 1;
}

// (for a partition the base is shifted so that global SA ranks index it)
inline SaView sa_view(const sa_index *idx) {
    if (idx->layout == 0) return SaView{idx->sa - idx->rank_base, 1u};
    const uint32_t stride = idx->layout == 2 ? 8u : 4u;
    return SaView{reinterpret_cast<const uint32_t *>(idx->rec) - idx->rank_base * stride, stride};
}

// build / match entry points implemented in sa_build.cu / sa_match.cu
sa_status sa_build_index(sa_index *idx, const char *ref_ascii, cudaStream_t st);
sa_status sa_extract_sa(const sa_index *idx, uint32_t *host_out);
sa_status sa_pack_text(sa_index *idx, const char *ref_ascii, cudaStream_t st);
sa_status sa_build_sa_dc3(sa_index *idx, cudaStream_t st, uint32_t *trace_rank, uint32_t *trace_nonsample);
sa_status sa_build_records(sa_index *idx, const uint32_t *sa, uint64_t count, cudaStream_t st);
void sa_free_index(sa_index *idx);
