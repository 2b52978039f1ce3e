// sa_match.cu -- host side of the hot path: launch of the search kernel (sa_search.cuh), read
// ordering (sa_match_order), the host-buffer pipeline, locate, and their C ABI entry points.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstdlib>

#include "sa_internal.cuh"

#include "sa_search.cuh"
#include "sa_search_long.cuh"
#include "sa_search_dual.cuh"
#include "sa_search_staged.cuh"

// the hand-written read-ordering sort (csrc/sa_order.cu)
size_t sa_order_onesweep_bytes(uint64_t Q);
sa_status sa_order_onesweep(const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len, uint32_t stride,
                            uint64_t Q, uint32_t key_bases, uint8_t *ws, uint32_t *order, cudaStream_t st);

namespace {

using sa_search::MatchArgs;

template <int QW, int L, bool STATS>
cudaError_t launch_t(const MatchArgs &a, cudaStream_t st) {
    const int threads = SA_MATCH_THREADS;
    const unsigned blocks = (unsigned)((a.Q + threads - 1) / threads);
#ifdef SA_MATCH_DUAL  // A/B build: two reads per thread (sa_search_dual.cuh)
    if constexpr (QW > 0 && !STATS) {
        if (!a.tree_hash && !a.big_sub) {
            const uint64_t half = (a.Q + 1) / 2;
            sa_search::k_match_dual<QW, L><<<(unsigned)((half + 255) / 256), 256, 0, st>>>(a, half);
            return cudaGetLastError();
        }
    }
#endif
    if constexpr (L == sa_search::L_REC32) {
        if (a.tree_hash) {  // SA_INDEX_BUCKET_TREE
            sa_search::k_match<QW, L, STATS, true><<<blocks, threads, 0, st>>>(a);
            return cudaGetLastError();
        }
    }
    sa_search::k_match<QW, L, STATS><<<blocks, threads, 0, st>>>(a);
    return cudaGetLastError();
}

// long reads: G lanes per read (sa_search::k_match_group)
template <int G, int WPL, int L, bool STATS>
cudaError_t launch_g(const MatchArgs &a, cudaStream_t st) {
    const int threads = 256;
    const uint64_t blocks = (a.Q * G + threads - 1) / threads;
    if (blocks > 0x7FFFFFFFull) return cudaErrorInvalidConfiguration;
    sa_search::k_match_group<G, WPL, L, STATS><<<(unsigned)blocks, threads, 0, st>>>(a);
    return cudaGetLastError();
}

// long reads (more than 4 words): the warp-synchronous search with warp-cooperative text compares
template <int L, bool STATS>
cudaError_t launch_l(const MatchArgs &a, cudaStream_t st) {
    const int threads = 256;
    const unsigned blocks = (unsigned)((a.Q + threads - 1) / threads);
    sa_search::k_match_long<L, STATS><<<blocks, threads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_long(const MatchArgs &a, int layout, bool stats, cudaStream_t st) {
    using namespace sa_search;
    switch (layout) {
    case L_PLAIN: return stats ? launch_l<L_PLAIN, true>(a, st) : launch_l<L_PLAIN, false>(a, st);
    case L_REC32: return stats ? launch_l<L_REC32, true>(a, st) : launch_l<L_REC32, false>(a, st);
    default: return stats ? launch_l<L_REC16, true>(a, st) : launch_l<L_REC16, false>(a, st);
    }
}

// long reads with the phase-B verification staged in shared memory by TMA (sa_search_staged.cuh)
#ifndef SA_STAGE_WARP_BYTES
#define SA_STAGE_WARP_BYTES 6144  // staging bytes per warp (8 warps x 6 KB = 48 KB per block, 4 blocks per SM)
#endif
template <int L, bool STATS>
cudaError_t launch_s(const MatchArgs &a, uint32_t part_words, uint32_t slots, cudaStream_t st) {
    const int threads = 256;
    const unsigned blocks = (unsigned)((a.Q + threads - 1) / threads);
    const size_t smem = (size_t)8 * slots * (2 * part_words + 2) * 8;
    cudaError_t e = cudaFuncSetAttribute(sa_search::k_match_staged<L, STATS>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    sa_search::k_match_staged<L, STATS><<<blocks, threads, smem, st>>>(a, part_words, slots);
    return cudaGetLastError();
}

// the staging geometry for reads of at most m_max bases, or false when k_match<0> takes the launch.  The
// staged kernel is an A/B build (SA_MATCH_STAGED, variants/libsa_staged.so): bit-exact, but slower than
// k_match<0> at every read length (profiles/r02/r02u), so the default build never stages.
// (Also k_match<0>: the plain layout (no records), reads no longer than the record-decided prefix,
// windows too long for the budget, a read buffer that is not 16-byte aligned.)
bool staged_geometry(int layout, uint32_t k, uint32_t m_max, const void *words, uint32_t &part_words,
                     uint32_t &slots) {
#ifndef SA_MATCH_STAGED
    (void)layout; (void)k; (void)m_max; (void)words; (void)part_words; (void)slots;
    return false;
#else
    if (layout == sa_search::L_PLAIN || (reinterpret_cast<uintptr_t>(words) & 15)) return false;
    const uint32_t mt = k + (layout == sa_search::L_REC32 ? 112u : 48u);
    if (m_max <= mt) return false;
    const uint32_t lmax = m_max - mt;
    part_words = ((lmax + 31) / 32 + 4) & ~1u;
    slots = std::min<uint32_t>(32u, SA_STAGE_WARP_BYTES / (8u * (2u * part_words + 2u)));
    return slots >= 2;
#endif
}

cudaError_t launch_staged(const MatchArgs &a, int layout, bool stats, uint32_t part_words, uint32_t slots,
                          cudaStream_t st) {
    using namespace sa_search;
    if (layout == L_REC32)
        return stats ? launch_s<L_REC32, true>(a, part_words, slots, st) : launch_s<L_REC32, false>(a, part_words, slots, st);
    return stats ? launch_s<L_REC16, true>(a, part_words, slots, st) : launch_s<L_REC16, false>(a, part_words, slots, st);
}

template <int QW>
cudaError_t launch_tree(const MatchArgs &a, int layout, uint32_t levels, uint32_t key_bases, cudaStream_t st) {
    using namespace sa_search;
    const int threads = 256;
    const unsigned blocks = (unsigned)((a.Q + threads - 1) / threads);
    const size_t smem = (size_t)((1u << levels) - 1) * (layout == L_REC32 ? 32 : 16);
    if (layout == L_REC32) {
        cudaFuncSetAttribute(k_match_tree<QW, L_REC32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_match_tree<QW, L_REC32><<<blocks, threads, smem, st>>>(a, levels, key_bases);
    } else {
        cudaFuncSetAttribute(k_match_tree<QW, L_REC16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_match_tree<QW, L_REC16><<<blocks, threads, smem, st>>>(a, levels, key_bases);
    }
    return cudaGetLastError();
}

template <int G, int WPL>
cudaError_t launch_group(const MatchArgs &a, int layout, bool stats, cudaStream_t st) {
    using namespace sa_search;
    switch (layout) {
    case L_PLAIN: return stats ? launch_g<G, WPL, L_PLAIN, true>(a, st) : launch_g<G, WPL, L_PLAIN, false>(a, st);
    case L_REC32: return stats ? launch_g<G, WPL, L_REC32, true>(a, st) : launch_g<G, WPL, L_REC32, false>(a, st);
    default: return stats ? launch_g<G, WPL, L_REC16, true>(a, st) : launch_g<G, WPL, L_REC16, false>(a, st);
    }
}

// SA_MATCH_DEFER: the light pass over all slots, then the deferred reads (grid-stride, one wave)
template <int QW, int L>
cudaError_t launch_defer_t(const MatchArgs &a, uint32_t big, uint32_t *dq, uint2 *dbr, uint32_t *dcount,
                           cudaStream_t st) {
    const int threads = SA_MATCH_THREADS;
    const unsigned blocks = (unsigned)((a.Q + threads - 1) / threads);
    cudaError_t e = cudaMemsetAsync(dcount, 0, 4, st);
    if (e != cudaSuccess) return e;
    sa_search::k_match_light<QW, L><<<blocks, threads, 0, st>>>(a, big, dq, dbr, dcount);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned hb = (unsigned)std::min<uint64_t>(blocks, (uint64_t)sms * SA_MATCH_MINB);
    sa_search::k_match_heavy<QW, L><<<hb, threads, 0, st>>>(a, dq, dbr, dcount);
    return cudaGetLastError();
}

template <int QW>
cudaError_t launch_defer(const MatchArgs &a, int layout, uint32_t big, uint32_t *dq, uint2 *dbr, uint32_t *dcount,
                         cudaStream_t st) {
    using namespace sa_search;
    switch (layout) {
    case L_PLAIN: return launch_defer_t<QW, L_PLAIN>(a, big, dq, dbr, dcount, st);
    case L_REC32: return launch_defer_t<QW, L_REC32>(a, big, dq, dbr, dcount, st);
    default: return launch_defer_t<QW, L_REC16>(a, big, dq, dbr, dcount, st);
    }
}

template <int QW>
cudaError_t launch_qw(const MatchArgs &a, int layout, bool stats, cudaStream_t st) {
    using namespace sa_search;
    switch (layout) {
    case L_PLAIN: return stats ? launch_t<QW, L_PLAIN, true>(a, st) : launch_t<QW, L_PLAIN, false>(a, st);
    case L_REC32: return stats ? launch_t<QW, L_REC32, true>(a, st) : launch_t<QW, L_REC32, false>(a, st);
    default: return stats ? launch_t<QW, L_REC16, true>(a, st) : launch_t<QW, L_REC16, false>(a, st);
    }
}

// ---- presort (SA_MATCH_PRESORT) ---------------------------------------------------------------
// key = the read's first 16 bases (masked to its length), value = read index
// (short_last: a read shorter than key_bases gets the key 4^key_bases, after every full key -- the
// routing of a partitioned index sends those reads to every part)
__global__ void k_presort_keys(const uint64_t *__restrict__ words, const uint32_t *__restrict__ lens,
                               uint32_t fixed_len, uint32_t stride, uint64_t dense_words, uint64_t Q,
                               uint32_t key_bases, bool short_last, uint32_t *__restrict__ keys,
                               uint32_t *__restrict__ perm, uint64_t *__restrict__ k64) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Q; q += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t m;
        uint64_t w0;
        if (stride == 0) {  // dense layout: read q starts at bit 2*m*q of the stream
            m = fixed_len;
            const uint64_t bit = 2ull * m * q, i = bit >> 6;
            const unsigned sh = (unsigned)(bit & 63);
            const uint64_t lo = __ldg(reinterpret_cast<const unsigned long long *>(words) + i);
            const uint64_t hi = (sh && i + 1 < dense_words) ? __ldg(reinterpret_cast<const unsigned long long *>(words) + i + 1) : 0ull;
            w0 = sh ? (lo << sh) | (hi >> (64 - sh)) : lo;
        } else {
            m = min(lens ? __ldg(lens + q) : fixed_len, 32u * stride);
            w0 = __ldg(reinterpret_cast<const unsigned long long *>(words + q * stride));
        }
        const uint32_t pre = (uint32_t)((w0 & prefix_mask(min(m, key_bases))) >> (64 - 2 * key_bases));
        const uint32_t key = (short_last && m < key_bases) ? (1u << (2 * key_bases)) : pre;
        if (k64) {  // (SA_ORDER_PACKED)
            k64[q] = ((uint64_t)key << 27) | q;
        } else {
            keys[q] = key;
            perm[q] = (uint32_t)q;
        }
    }
}

// row t of the ordered copy = read order[t] (coalesced writes; the reads are gathered once here)
// (vec: one 256-bit copy per row; the caller sets it only for stride 4 with both buffers 32-byte aligned)
__global__ void k_gather_rows(const uint64_t *__restrict__ words, const uint32_t *__restrict__ lens, uint32_t stride,
                              bool vec, uint64_t Q, const uint32_t *__restrict__ order, uint64_t *__restrict__ out_words,
                              uint32_t *__restrict__ out_lens) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < Q; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = __ldg(order + t);
        if (out_words) {
            if (vec) {
                reinterpret_cast<ulonglong4 *>(out_words)[t] = reinterpret_cast<const ulonglong4 *>(words)[q];
            } else {
                for (uint32_t j = 0; j < stride; ++j) out_words[t * stride + j] = __ldg(words + q * stride + j);
            }
        }
        if (out_lens && lens) out_lens[t] = __ldg(lens + q);
    }
}

struct PresortLayout {
    size_t stats = 0, keys_in = 0, keys_out = 0, perm_in = 0, perm_out = 0, cub = 0, cub_bytes = 0, total = 0;
    size_t defer_q = 0, defer_br = 0, defer_cnt = 0;  // SA_MATCH_DEFER: list of reads, their brackets, count
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// workspace of sa_match_order (order_only: the permutation goes to the caller's buffer) and of
// sa_match_batch (stats first, then, with SA_MATCH_PRESORT, the same sort scratch + the permutation)
sa_status presort_layout(uint64_t Q, bool stats, bool presort, bool order_only, PresortLayout &L) {
    size_t off = 0;
    if (stats) { L.stats = off; off = align256(off + Q * 8); }
    if (presort) {
        if (Q >= (1ull << 32)) { sa_set_error("read ordering needs Q < 2^32"); return SA_EINVAL; }
#ifdef SA_ORDER_PACKED  // A/B build: (key << 27 | read) sorted as one 64-bit key (keys_in/keys_out hold 8 B each)
        L.keys_in = off; off = align256(off + Q * 8);
        L.keys_out = off; off = align256(off + Q * 8);
        L.perm_in = off; off = align256(off + Q * 4);
#else
        L.keys_in = off; off = align256(off + Q * 4);
        L.keys_out = off; off = align256(off + Q * 4);
        L.perm_in = off; off = align256(off + Q * 4);
#endif
        if (!order_only) { L.perm_out = off; off = align256(off + Q * 4); }
        size_t b = 0;
#ifdef SA_ORDER_PACKED
        cudaError_t e = cub::DeviceRadixSort::SortKeys(nullptr, b, (const uint64_t *)nullptr, (uint64_t *)nullptr,
                                                       (int64_t)Q, 27, 64);
#else
        cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                                        (const uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)Q, 0, 32);
#endif
        if (e != cudaSuccess) { sa_set_error("order size query: %s", cudaGetErrorString(e)); return SA_ECUDA; }
#ifdef SA_ORDER_ONESWEEP  // (A/B build) the hand-written sort (csrc/sa_order.cu) uses the same scratch region
        const size_t ob = sa_order_onesweep_bytes(Q);
        if (ob > b) b = ob;
#endif
        L.cub = off;
        L.cub_bytes = b;
        off = align256(off + b);
    }
    L.total = off;
    return SA_OK;
}

// the SA_MATCH_DEFER region after the rest of the workspace
void defer_layout(uint64_t Q, PresortLayout &L) {
    size_t off = L.total;
    L.defer_q = off; off = align256(off + Q * 4);
    L.defer_br = off; off = align256(off + Q * 8);
    L.defer_cnt = off; off = align256(off + 4);
    L.total = off;
}

constexpr uint32_t kDefaultKeyBases = 12;
constexpr uint32_t kMaxBucketBases = 13;  // SA_ORDER_BUCKETS: at most 4^13 counters (256 MB)

#ifdef SA_ORDER_PACKED
// the sorted packed keys (key << 27 | read index) -> the permutation
__global__ void k_unpack_order(const uint64_t *__restrict__ k64, uint64_t Q, uint32_t *__restrict__ order) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < Q; t += (uint64_t)gridDim.x * blockDim.x)
        order[t] = (uint32_t)(k64[t] & ((1u << 27) - 1));
}
#endif

sa_status order_reads(const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len, uint32_t stride, uint64_t Q,
                      uint32_t key_bases, uint8_t *ws, const PresortLayout &L, uint32_t *order, cudaStream_t st,
                      bool short_last = false) {
    uint32_t *keys_in = reinterpret_cast<uint32_t *>(ws + L.keys_in);
    uint32_t *keys_out = reinterpret_cast<uint32_t *>(ws + L.keys_out);
    uint32_t *perm_in = reinterpret_cast<uint32_t *>(ws + L.perm_in);
    uint64_t blocks = (Q + 255) / 256;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    const uint64_t dense_words = (Q * (uint64_t)fixed_len + 31) / 32;
    size_t b = L.cub_bytes;
    // key = the first key_bases bases: ceil(2*key_bases/8) radix passes.  Measured and dropped
    // (profiles/r01-3): 32-bit offsets (CUB's 23-items-per-thread tuning) +0.5 ms per 100 M reads; a
    // hand-written two-pass stable LSD counting sort with 10-12-bit digits +6.5-8.5 ms (its scattered
    // 4-byte stores are partial-sector DRAM read-modify-writes: 5.6 GB written, 5.2 GB read per pass
    // for 0.8 GB of payload; CUB's 8-bit digits keep each bin's run long enough to coalesce).
    const int end_bit = 2 * (int)key_bases + (short_last ? 1 : 0);
#ifdef SA_ORDER_ONESWEEP  // A/B build: the hand-written onesweep sort (csrc/sa_order.cu; measured slower)
    if (!short_last) return sa_order_onesweep(q_words, q_len, fixed_len, stride, Q, key_bases, ws + L.cub, order, st);
#endif
#ifdef SA_ORDER_PACKED
    if (!short_last && Q < (1ull << 27)) {
        // keys_in .. perm_in hold the packed 64-bit keys; keys_out .. (+8 B) the sorted ones
        uint64_t *k64 = reinterpret_cast<uint64_t *>(ws + L.keys_in);
        uint64_t *k64o = reinterpret_cast<uint64_t *>(ws + L.keys_out);
        k_presort_keys<<<(unsigned)blocks, 256, 0, st>>>(q_words, q_len, fixed_len, stride, dense_words, Q, key_bases,
                                                         short_last, nullptr, nullptr, k64);
        SA_CUDA_TRY(cudaGetLastError());
        SA_CUDA_TRY(cub::DeviceRadixSort::SortKeys(ws + L.cub, b, k64, k64o, (int64_t)Q, 27, 27 + end_bit, st));
        k_unpack_order<<<(unsigned)blocks, 256, 0, st>>>(k64o, Q, order);
        SA_CUDA_TRY(cudaGetLastError());
        return SA_OK;
    }
#endif
    k_presort_keys<<<(unsigned)blocks, 256, 0, st>>>(q_words, q_len, fixed_len, stride, dense_words, Q, key_bases,
                                                     short_last, keys_in, perm_in, nullptr);
    SA_CUDA_TRY(cudaGetLastError());
    SA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws + L.cub, b, keys_in, keys_out, perm_in, order, (int64_t)Q, 0,
                                                end_bit, st));
    return SA_OK;
}

// ---- bucket order (SA_ORDER_BUCKETS) ------------------------------------------------------------
// One placement pass instead of a radix sort: every read goes to the bucket of its first key_bases
// bases (4^key_bases buckets): count (k_bucket_count), exclusive scan of the counts (CUB), place
// (k_bucket_place: a slot claimed by an atomic on the bucket's offset).  The buckets come out in key
// order, as with the sort; inside a bucket the reads are in no fixed order (lanes of a warp with the same
// key claim their slots together, in lane order, after one __match_any_sync).  For batches whose
// permutation and counters stay in the 126 MB L2, so the scattered 4-byte slot writes and the counter
// atomics merge there instead of becoming partial-sector DRAM read-modify-writes (the reason the
// round-1 counting sorts lost at 100 M reads, order_reads).
__device__ __forceinline__ uint32_t read_key(const uint64_t *__restrict__ words, const uint32_t *__restrict__ lens,
                                             uint32_t fixed_len, uint32_t stride, uint64_t dense_words, uint64_t q,
                                             uint32_t key_bases) {
    uint32_t m;
    uint64_t w0;
    if (stride == 0) {
        m = fixed_len;
        const uint64_t bit = 2ull * m * q, i = bit >> 6;
        const unsigned sh = (unsigned)(bit & 63);
        const uint64_t lo = __ldg(reinterpret_cast<const unsigned long long *>(words) + i);
        const uint64_t hi = (sh && i + 1 < dense_words) ? __ldg(reinterpret_cast<const unsigned long long *>(words) + i + 1) : 0ull;
        w0 = sh ? (lo << sh) | (hi >> (64 - sh)) : lo;
    } else {
        m = min(lens ? __ldg(lens + q) : fixed_len, 32u * stride);
        w0 = __ldg(reinterpret_cast<const unsigned long long *>(words + q * stride));
    }
    return (uint32_t)((w0 & prefix_mask(min(m, key_bases))) >> (64 - 2 * key_bases));
}

__global__ void k_bucket_count(const uint64_t *__restrict__ words, const uint32_t *__restrict__ lens, uint32_t fixed_len,
                               uint32_t stride, uint64_t dense_words, uint64_t Q, uint32_t key_bases,
                               uint32_t *__restrict__ keys, uint32_t *__restrict__ cnt) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = q < Q;
    const uint32_t key = ok ? read_key(words, lens, fixed_len, stride, dense_words, q, key_bases) : 0xFFFFFFFFu;
    if (ok) keys[q] = key;
    const unsigned act = __ballot_sync(0xFFFFFFFFu, ok);
    if (!ok) return;
    const unsigned peers = __match_any_sync(act, key);  // (repeats: many reads share a key)
    if ((threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1)) atomicAdd(cnt + key, (uint32_t)__popc(peers));
}

__global__ void k_bucket_place(const uint32_t *__restrict__ keys, uint64_t Q, uint32_t *__restrict__ off,
                               uint32_t *__restrict__ order) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool ok = q < Q;
    const unsigned act = __ballot_sync(0xFFFFFFFFu, ok);
    if (!ok) return;
    const uint32_t key = keys[q];
    const unsigned peers = __match_any_sync(act, key);
    const unsigned lane = threadIdx.x & 31, leader = (unsigned)(__ffs(peers) - 1);
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(off + key, (uint32_t)__popc(peers));
    base = __shfl_sync(peers, base, (int)leader);
    order[base + __popc(peers & ((1u << lane) - 1u))] = (uint32_t)q;
}

struct BucketLayout {
    size_t keys = 0, cnt = 0, off = 0, scan = 0, scan_bytes = 0, total = 0;
};

sa_status bucket_layout(uint64_t Q, uint32_t key_bases, BucketLayout &B) {
    if (key_bases > kMaxBucketBases) {
        sa_set_error("SA_ORDER_BUCKETS: key_bases %u > %u", key_bases, kMaxBucketBases);
        return SA_EINVAL;
    }
    const uint64_t nb = 1ull << (2 * key_bases);
    size_t o = 0;
    B.keys = o; o = align256(o + Q * 4);
    B.cnt = o; o = align256(o + nb * 4);
    B.off = o; o = align256(o + nb * 4);
    size_t b = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)nb);
    if (e != cudaSuccess) { sa_set_error("scan size query: %s", cudaGetErrorString(e)); return SA_ECUDA; }
    B.scan = o; B.scan_bytes = b; o = align256(o + b);
    B.total = o;
    return SA_OK;
}

sa_status order_buckets(const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len, uint32_t stride, uint64_t Q,
                        uint32_t key_bases, uint8_t *ws, const BucketLayout &B, uint32_t *order, cudaStream_t st) {
    const uint64_t nb = 1ull << (2 * key_bases);
    uint32_t *keys = reinterpret_cast<uint32_t *>(ws + B.keys);
    uint32_t *cnt = reinterpret_cast<uint32_t *>(ws + B.cnt);
    uint32_t *off = reinterpret_cast<uint32_t *>(ws + B.off);
    const uint64_t dense_words = (Q * (uint64_t)fixed_len + 31) / 32;
    const uint64_t blocks = (Q + 255) / 256;
    if (blocks > 0x7FFFFFFFull) { sa_set_error("SA_ORDER_BUCKETS: Q too large"); return SA_EINVAL; }
    SA_CUDA_TRY(cudaMemsetAsync(cnt, 0, nb * 4, st));
    k_bucket_count<<<(unsigned)blocks, 256, 0, st>>>(q_words, q_len, fixed_len, stride, dense_words, Q, key_bases, keys, cnt);
    SA_CUDA_TRY(cudaGetLastError());
    size_t b = B.scan_bytes;
    SA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(ws + B.scan, b, cnt, off, (int64_t)nb, st));
    k_bucket_place<<<(unsigned)blocks, 256, 0, st>>>(keys, Q, off, order);
    SA_CUDA_TRY(cudaGetLastError());
    return SA_OK;
}

// ---- partitioned matching ----------------------------------------------
// offsets[g] = first slot of the sorted keys with key >= part_keys[g] (lower bound)
__global__ void k_route_offsets(const uint32_t *__restrict__ sorted_keys, uint64_t Q, const uint32_t *__restrict__ bounds,
                                uint32_t nb, uint64_t *__restrict__ offsets) {
    const uint32_t g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= nb) return;
    const uint64_t key = bounds[g];
    uint64_t lo = 0, hi = Q;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if ((uint64_t)sorted_keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    offsets[g] = lo;
}

__global__ void k_scatter_results(const uint32_t *__restrict__ order, const uint2 *__restrict__ in, uint64_t Q,
                                  uint2 *__restrict__ out) {
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < Q; t += (uint64_t)gridDim.x * blockDim.x)
        out[__ldg(order + t)] = in[t];
}

// ---- locate -----------------------------------------------------------------------------------
struct CountOp {
    const uint32_t *lohi;
    uint64_t Q;
    __host__ __device__ __forceinline__ uint64_t operator()(uint64_t q) const {
        return q < Q ? (uint64_t)(lohi[2 * q + 1] - lohi[2 * q]) : 0ull;
    }
};

// Locate, load-balanced in two parts.  Reads with at most kHeavy occurrences: one warp per read, lanes
// copy SA[lo .. hi) to positions[off ..] (contiguous, coalesced).  Heavier reads (repeats: up to 10^6
// occurrences) are cut into chunks of kHeavy positions and every chunk is copied by a whole block.
// SA values are read through the layout's view (stride 1 = plain SA, 4 / 8 = 16- / 32-byte records).
constexpr uint32_t kHeavy = 4096;

__global__ void k_locate(const uint32_t *__restrict__ sa, uint32_t sa_stride, const uint32_t *__restrict__ lohi,
                         const uint64_t *__restrict__ offsets, uint64_t Q, uint32_t *__restrict__ pos) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t q = warp; q < Q; q += nwarps) {
        const uint32_t lo = lohi[2 * q], hi = lohi[2 * q + 1];
        if (hi - lo > kHeavy) continue;  // the chunked kernel copies it
        const uint64_t off = offsets[q];
        for (uint64_t j = lane; j < (uint64_t)(hi - lo); j += 32) pos[off + j] = __ldg(sa + (lo + j) * sa_stride);
    }
}

struct ChunksOfRead {  // chunks of kHeavy positions of a heavy read (0 for the others)
    const uint32_t *lohi;
    __host__ __device__ uint64_t operator()(uint64_t q) const {
        const uint32_t c = lohi[2 * q + 1] - lohi[2 * q];
        return c > kHeavy ? (c + kHeavy - 1) / kHeavy : 0;
    }
};

// chunk_off[Q] = chunk_off[Q-1] + chunks of read Q-1 (the total)
__global__ void k_chunk_total(const uint32_t *__restrict__ lohi, uint64_t Q, uint64_t *__restrict__ chunk_off) {
    const uint32_t c = lohi[2 * (Q - 1) + 1] - lohi[2 * (Q - 1)];
    chunk_off[Q] = chunk_off[Q - 1] + (c > kHeavy ? (c + kHeavy - 1) / kHeavy : 0);
}

// block b copies chunk b (grid-stride): find its read by binary search over the chunk offsets
__global__ void k_locate_heavy(const uint32_t *__restrict__ sa, uint32_t sa_stride, const uint32_t *__restrict__ lohi,
                               const uint64_t *__restrict__ offsets, uint64_t Q, const uint64_t *__restrict__ chunk_off,
                               uint32_t *__restrict__ pos) {
    const uint64_t nchunks = chunk_off[Q];
    for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
        __shared__ uint64_t s_q;
        if (threadIdx.x == 0) {
            uint64_t a = 0, b = Q;  // last q with chunk_off[q] <= c
            while (b - a > 1) {
                const uint64_t mid = (a + b) >> 1;
                if (chunk_off[mid] <= c) a = mid; else b = mid;
            }
            s_q = a;
        }
        __syncthreads();
        const uint64_t q = s_q;
        __syncthreads();
        const uint32_t lo = lohi[2 * q], hi = lohi[2 * q + 1];
        const uint64_t j0 = (c - chunk_off[q]) * kHeavy;
        const uint64_t j1 = j0 + kHeavy < (uint64_t)(hi - lo) ? j0 + kHeavy : (uint64_t)(hi - lo);
        const uint64_t off = offsets[q];
        for (uint64_t j = j0 + threadIdx.x; j < j1; j += blockDim.x) pos[off + j] = __ldg(sa + (lo + j) * sa_stride);
    }
}

sa_status check_match_args(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                           uint32_t stride, uint64_t Q, const uint32_t *out) {
    if (!idx) { sa_set_error("index is NULL"); return SA_EINVAL; }
    if (Q == 0) return SA_OK;
    if (!q_words || !out) { sa_set_error("q_words/out NULL with Q=%llu", (unsigned long long)Q); return SA_EINVAL; }
    if (stride == 0) {  // dense layout
        if (q_len || fixed_len == 0) {
            sa_set_error("the dense layout (stride_words = 0) needs q_len = NULL and fixed_len > 0");
            return SA_EINVAL;
        }
    } else if (!q_len && fixed_len > 32u * stride) {
        sa_set_error("fixed_len %u exceeds 32*stride_words = %u", fixed_len, 32u * stride);
        return SA_EINVAL;
    }
    if (!q_len && fixed_len > 65535u) { sa_set_error("query length %u > 65535", fixed_len); return SA_EINVAL; }
    return SA_OK;
}

}  // namespace

// ---- C ABI ------------------------------------------------------------------------------------
extern "C" sa_status sa_match_workspace_size(const sa_index *idx, uint64_t Q, uint32_t stride_words, uint32_t flags,
                                             size_t *bytes) {
    sa_clear_error();
    if (!idx || !bytes) { sa_set_error("NULL argument"); return SA_EINVAL; }
    (void)stride_words;
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    PresortLayout L;
    SA_TRY(presort_layout(Q, flags & SA_MATCH_STATS, flags & SA_MATCH_PRESORT, false, L));
    if (flags & SA_MATCH_DEFER) defer_layout(Q, L);
    *bytes = L.total;
    return SA_OK;
}

extern "C" sa_status sa_match_order_workspace_size(uint64_t Q, size_t *bytes) {
    sa_clear_error();
    if (!bytes) { sa_set_error("NULL argument"); return SA_EINVAL; }
    PresortLayout L;
    SA_TRY(presort_layout(Q, false, true, true, L));
    *bytes = L.total;
    return SA_OK;
}

extern "C" sa_status sa_match_order_workspace_size_ex(uint64_t Q, uint32_t key_bases, size_t *bytes) {
    sa_clear_error();
    if (!bytes) { sa_set_error("NULL argument"); return SA_EINVAL; }
    if (!(key_bases & SA_ORDER_BUCKETS)) return sa_match_order_workspace_size(Q, bytes);
    uint32_t kb = key_bases & 0xFFu;
    if (kb == 0) kb = kDefaultKeyBases;
    BucketLayout B;
    SA_TRY(bucket_layout(Q, kb, B));
    *bytes = B.total;
    return SA_OK;
}

extern "C" sa_status sa_match_order(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len,
                                    uint32_t fixed_len, uint32_t stride_words, uint64_t Q, uint32_t key_bases,
                                    uint32_t *order, uint64_t *ordered_words, uint32_t *ordered_len,
                                    void *workspace, size_t ws_bytes, void *stream) {
    sa_clear_error();
    const bool buckets = (key_bases & SA_ORDER_BUCKETS) != 0;
    key_bases &= ~SA_ORDER_BUCKETS;
    if (key_bases > 16) { sa_set_error("key_bases %u > 16", key_bases); return SA_EINVAL; }
    if (key_bases == 0) key_bases = kDefaultKeyBases;
    SA_TRY(check_match_args(idx, q_words, q_len, fixed_len, stride_words, Q, order));
    if (Q == 0) return SA_OK;
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    if (buckets) {
        if (Q >= (1ull << 32)) { sa_set_error("read ordering needs Q < 2^32"); return SA_EINVAL; }
        BucketLayout B;
        SA_TRY(bucket_layout(Q, key_bases, B));
        if (!workspace || ws_bytes < B.total) {
            sa_set_error("workspace too small: %zu < %zu bytes", ws_bytes, B.total);
            return SA_EINVAL;
        }
        SA_TRY(order_buckets(q_words, q_len, fixed_len, stride_words, Q, key_bases, static_cast<uint8_t *>(workspace),
                             B, order, (cudaStream_t)stream));
    } else {
        PresortLayout L;
        SA_TRY(presort_layout(Q, false, true, true, L));
        if (!workspace || ws_bytes < L.total) {
            sa_set_error("workspace too small: %zu < %zu bytes", ws_bytes, L.total);
            return SA_EINVAL;
        }
        SA_TRY(order_reads(q_words, q_len, fixed_len, stride_words, Q, key_bases, static_cast<uint8_t *>(workspace), L,
                           order, (cudaStream_t)stream));
    }
    if ((ordered_words || ordered_len) && stride_words == 0) {
        sa_set_error("ordered rows are not available for the dense layout");
        return SA_EINVAL;
    }
    if (ordered_words || ordered_len) {
        const bool vec = stride_words == 4 && (reinterpret_cast<uintptr_t>(q_words) & 31) == 0 &&
                         (reinterpret_cast<uintptr_t>(ordered_words) & 31) == 0;
        uint64_t blocks = (Q + 255) / 256;
        if (blocks > 148ull * 16) blocks = 148ull * 16;
        k_gather_rows<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(q_words, q_len, stride_words, vec, Q, order,
                                                                          ordered_words, ordered_len);
        SA_CUDA_TRY(cudaGetLastError());
    }
    return SA_OK;
}

static sa_status match_launch(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                              uint32_t stride, uint64_t Q, uint32_t *out, uint32_t *stats, const uint32_t *order,
                              bool rows_ordered, cudaStream_t st, bool cooperative = false, uint32_t tree_flags = 0,
                              uint32_t defer_big = 0, uint32_t *dq = nullptr, uint2 *dbr = nullptr,
                              uint32_t *dcount = nullptr) {
    MatchArgs a;
    a.rows_ordered = rows_ordered;

    a.text = idx->text;
    a.sa = idx->sa;
    a.rec = idx->rec;
    a.table = idx->table;
    a.n = idx->n;
    a.text_words = idx->n_words;
    a.k = idx->k;
    a.words = q_words;
    a.lens = q_len;
    a.fixed_len = fixed_len;
    a.stride = stride;
    a.Q = Q;
    a.out = out;
    a.stats = stats;
    a.order = order;
    a.big_hash = idx->big_hash;
    a.big_sub = idx->big_sub;
    a.big_bits = idx->big_bits;
    a.tree_hash = idx->tree_hash;
    a.tree = idx->tree;
    a.tree_bits = idx->tree_bits;
    a.clo = 0;
    a.chi = (uint32_t)idx->n;
    a.route = nullptr;
    a.route_bases = 0;
#ifndef SA_NO_WIDE  // (A/B build: never wide)
    a.wide = Q >= kWideQ || (tree_flags & SA_MATCH_WIDE);
#else
    a.wide = false;
#endif
    if (idx->nparts > 1) {
        // a partition holds table entries [x_base, x_base + table_entries) and SA ranks [rank_base, rank_end):
        // address them with their global indices through shifted base pointers; every bracket is clamped
        // to the slice, so only in-slice indices are dereferenced (csrc/sa_part.cu)
        a.table = idx->table - idx->x_base;
        if (idx->layout == 0) a.sa = idx->sa - idx->rank_base;
        else a.rec = idx->rec - idx->rank_base * (idx->layout == 2 ? 2 : 1);
        a.clo = (uint32_t)idx->rank_base;
        a.chi = (uint32_t)idx->rank_end;
        a.route = idx->route_table;
        a.route_bases = idx->route_bases;
    }
    // one vector load per read row when the row is exactly QW words and suitably aligned
    const uintptr_t wp = reinterpret_cast<uintptr_t>(q_words);
    // (stride a multiple of 4 beyond 4 words: the long-read path's 4-word chunks are single loads)
    a.vec_rows = ((stride == 4 || (stride > 4 && stride % 4 == 0)) && (wp & 31) == 0) ||
                 (stride == 2 && (wp & 15) == 0);
    a.dense_words = stride == 0 ? (Q * (uint64_t)fixed_len + 31) / 32 : 0;
    const bool st_on = stats != nullptr;
    const uint32_t nw = stride ? stride : (fixed_len + 31) / 32;  // register words needed
    cudaError_t e;
    if (tree_flags & SA_MATCH_SMEM_TREE) {
        uint32_t levels = (tree_flags >> 8) & 15, kb = (tree_flags >> 12) & 31;
        if (levels == 0) levels = 8;
        if (kb == 0) kb = kDefaultKeyBases;
        if (idx->layout == 0 || nw > 4 || levels > 12 || kb > 16 || !order || idx->big_sub) {
            sa_set_error("SA_MATCH_SMEM_TREE: needs a record layout, reads of <= 128 bases, an order, levels <= 12, "
                         "key bases <= 16, no sub-tables");
            return SA_EINVAL;
        }
        if (nw <= 1) e = launch_tree<1>(a, idx->layout, levels, kb, st);
        else if (nw <= 2) e = launch_tree<2>(a, idx->layout, levels, kb, st);
        else e = launch_tree<4>(a, idx->layout, levels, kb, st);
        if (e != cudaSuccess) { sa_set_error("match launch: %s", cudaGetErrorString(e)); return SA_ECUDA; }
        return SA_OK;
    }
    if (dq && !st_on && nw <= 4) {  // SA_MATCH_DEFER: light pass + deferred heavy reads
        if (nw <= 1) e = launch_defer<1>(a, idx->layout, defer_big, dq, dbr, dcount, st);
        else if (nw <= 2) e = launch_defer<2>(a, idx->layout, defer_big, dq, dbr, dcount, st);
        else e = launch_defer<4>(a, idx->layout, defer_big, dq, dbr, dcount, st);
        if (e != cudaSuccess) { sa_set_error("match launch: %s", cudaGetErrorString(e)); return SA_ECUDA; }
        return SA_OK;
    }
    // reads of more than 4 words: one thread per read, words from global memory; with
    // SA_MATCH_COOPERATIVE G = 8 / 16 / 32 lanes per read (measured slower)
    if (nw <= 1) e = launch_qw<1>(a, idx->layout, st_on, st);
    else if (nw <= 2) e = launch_qw<2>(a, idx->layout, st_on, st);
    else if (nw <= 4) e = launch_qw<4>(a, idx->layout, st_on, st);
#ifndef SA_LONG_WARP  // one thread per read, two phases (k_match_staged, else k_match<0>); the A/B build
                      // SA_LONG_WARP takes k_match_long (warp-synchronous rounds, warp-cooperative compares)
    else if (!cooperative) {
        uint32_t part_words = 0, slots = 0;
        const uint32_t m_max = stride ? 32u * stride : fixed_len;
        if (staged_geometry(idx->layout, idx->k, m_max, q_words, part_words, slots))
            e = launch_staged(a, idx->layout, st_on, part_words, slots, st);
        else
            e = launch_qw<0>(a, idx->layout, st_on, st);
    }
#else
    else if (!cooperative) e = launch_long(a, idx->layout, st_on, st);
#endif
    else if (nw <= 8) e = launch_group<8, 1>(a, idx->layout, st_on, st);
    else if (nw <= 16) e = launch_group<16, 1>(a, idx->layout, st_on, st);
    else if (nw <= 32) e = launch_group<32, 1>(a, idx->layout, st_on, st);
    else if (nw <= 64) e = launch_group<32, 2>(a, idx->layout, st_on, st);
    else e = launch_group<32, 0>(a, idx->layout, st_on, st);
    if (e != cudaSuccess) { sa_set_error("match launch: %s", cudaGetErrorString(e)); return SA_ECUDA; }
    return SA_OK;
}

extern "C" sa_status sa_match_batch(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len,
                                    uint32_t fixed_len, uint32_t stride_words, uint64_t Q, const uint32_t *order,
                                    uint32_t *out_lohi, void *workspace, size_t ws_bytes, uint32_t flags,
                                    void *stream) {
    sa_clear_error();
    SA_TRY(check_match_args(idx, q_words, q_len, fixed_len, stride_words, Q, out_lohi));
    if (flags & ~(SA_MATCH_STATS | SA_MATCH_PRESORT | SA_MATCH_ROWS_ORDERED | SA_MATCH_COOPERATIVE | SA_MATCH_SMEM_TREE |
                  0x1FF00u | SA_MATCH_DEFER | SA_MATCH_DEFER_LOG2(15) | SA_MATCH_WIDE)) {
        sa_set_error("unknown flags 0x%x", flags);
        return SA_EINVAL;
    }
    const bool defer = (flags & SA_MATCH_DEFER) != 0;
    if (defer && (flags & (SA_MATCH_ROWS_ORDERED | SA_MATCH_STATS | SA_MATCH_SMEM_TREE))) {
        sa_set_error("SA_MATCH_DEFER does not combine with SA_MATCH_ROWS_ORDERED / SA_MATCH_STATS / SA_MATCH_SMEM_TREE");
        return SA_EINVAL;
    }
    if (Q == 0) return SA_OK;
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    const bool presort = (flags & SA_MATCH_PRESORT) && !order;
    PresortLayout L;
    SA_TRY(presort_layout(Q, flags & SA_MATCH_STATS, presort, false, L));
    if (defer) defer_layout(Q, L);
    if (L.total > 0 && (!workspace || ws_bytes < L.total)) {
        sa_set_error("workspace too small: %zu < %zu bytes", ws_bytes, L.total);
        return SA_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    uint32_t *stats = (flags & SA_MATCH_STATS) ? reinterpret_cast<uint32_t *>(ws + L.stats) : nullptr;
    if (presort) {
        uint32_t *perm = reinterpret_cast<uint32_t *>(ws + L.perm_out);
        SA_TRY(order_reads(q_words, q_len, fixed_len, stride_words, Q, kDefaultKeyBases, ws, L, perm, st));
        order = perm;
    }
    const bool rows_ordered = (flags & SA_MATCH_ROWS_ORDERED) != 0;
    if (rows_ordered && (!order || presort || stride_words == 0)) {
        sa_set_error("SA_MATCH_ROWS_ORDERED needs the order the rows were arranged in");
        return SA_EINVAL;
    }
    uint32_t big = 0, *dq = nullptr, *dcount = nullptr;
    uint2 *dbr = nullptr;
    if (defer) {
        const uint32_t lg = (flags >> 18) & 15u;
        big = 1u << (lg ? lg : 3u);
        dq = reinterpret_cast<uint32_t *>(ws + L.defer_q);
        dbr = reinterpret_cast<uint2 *>(ws + L.defer_br);
        dcount = reinterpret_cast<uint32_t *>(ws + L.defer_cnt);
    }
    return match_launch(idx, q_words, q_len, fixed_len, stride_words, Q, out_lohi, stats, order, rows_ordered, st,
                        (flags & SA_MATCH_COOPERATIVE) != 0, flags & (SA_MATCH_SMEM_TREE | 0x1FF00u | SA_MATCH_WIDE), big,
                        dq, dbr,
                        dcount);
}

// Synchronises the host pipeline's streams when sa_match_batch_host returns, on success and on every
// error path, so no copy into or out of the caller's host buffers outlives the call.
struct PipeSyncGuard {
    sa_index *idx;
    ~PipeSyncGuard() {
        for (int b = 0; b < 2; ++b)
            if (idx->pipe_stream[b]) cudaStreamSynchronize(idx->pipe_stream[b]);
    }
};

extern "C" sa_status sa_match_batch_host(sa_index *idx, const uint64_t *q_words, const uint32_t *q_len,
                                         uint32_t fixed_len, uint32_t stride, uint64_t Q, uint32_t *out_lohi,
                                         uint64_t chunk_Q) {
    sa_clear_error();
    SA_TRY(check_match_args(idx, q_words, q_len, fixed_len, stride, Q, out_lohi));
    if (Q == 0) return SA_OK;
    std::lock_guard<std::mutex> lock(idx->mu);
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    if (chunk_Q == 0) chunk_Q = 1ull << 21;  // 2 M reads: the best of 1 / 2 / 4 / 8 / 16 M (profiles/r02/r02j)
    chunk_Q = (chunk_Q + 31) & ~31ull;  // dense layout: every chunk starts on a word boundary
    if (chunk_Q > Q) chunk_Q = Q;
    // words of `cq` reads starting at read q0 (q0 a multiple of chunk_Q, hence of 32 for dense)
    auto words_of = [&](uint64_t cq) { return stride ? cq * stride : (cq * (uint64_t)fixed_len + 31) / 32; };
    const uint64_t need_words = words_of(chunk_Q);
    PresortLayout OL;
    SA_TRY(presort_layout(chunk_Q, false, true, true, OL));
    for (int b = 0; b < 2; ++b)
        if (!idx->pipe_stream[b]) SA_CUDA_TRY(cudaStreamCreateWithFlags(&idx->pipe_stream[b], cudaStreamNonBlocking));
    PipeSyncGuard guard{idx};
    if (idx->pipe_chunk < chunk_Q || idx->pipe_words_cap < need_words || idx->pipe_ws_bytes < OL.total) {
        for (int b = 0; b < 2; ++b) {
            cudaFree(idx->pipe_words[b]);
            cudaFree(idx->pipe_lens[b]);
            cudaFree(idx->pipe_out[b]);
            cudaFree(idx->pipe_order[b]);
            cudaFree(idx->pipe_ws[b]);
            idx->pipe_words[b] = nullptr;
            idx->pipe_lens[b] = nullptr;
            idx->pipe_out[b] = nullptr;
            idx->pipe_order[b] = nullptr;
            idx->pipe_ws[b] = nullptr;
        }
        idx->pipe_chunk = 0;
        idx->pipe_words_cap = 0;
        idx->pipe_ws_bytes = 0;
        for (int b = 0; b < 2; ++b) {
            SA_CUDA_TRY(cudaMalloc(&idx->pipe_words[b], need_words * sizeof(uint64_t)));
            SA_CUDA_TRY(cudaMalloc(&idx->pipe_lens[b], chunk_Q * sizeof(uint32_t)));
            SA_CUDA_TRY(cudaMalloc(&idx->pipe_out[b], chunk_Q * 2 * sizeof(uint32_t)));
            SA_CUDA_TRY(cudaMalloc(&idx->pipe_order[b], chunk_Q * sizeof(uint32_t)));
            SA_CUDA_TRY(cudaMalloc(&idx->pipe_ws[b], OL.total));
        }
        idx->pipe_chunk = chunk_Q;
        idx->pipe_words_cap = need_words;
        idx->pipe_ws_bytes = OL.total;
    }
    // chunk c uses buffer set c%2 on stream c%2: H2D -> order (a5) -> match (a6-a9) -> D2H; the two
    // streams overlap, so one chunk's copies run under the other's kernels.
    uint64_t c = 0;
    for (uint64_t q0 = 0; q0 < Q; q0 += chunk_Q, ++c) {
        const int b = (int)(c & 1);
        cudaStream_t st = idx->pipe_stream[b];
        const uint64_t cq = std::min<uint64_t>(chunk_Q, Q - q0);
        const uint64_t w0 = stride ? q0 * stride : q0 * (uint64_t)fixed_len / 32;
        SA_CUDA_TRY(cudaMemcpyAsync(idx->pipe_words[b], q_words + w0, words_of(cq) * sizeof(uint64_t),
                                    cudaMemcpyHostToDevice, st));
        const uint32_t *dl = nullptr;
        if (q_len) {
            SA_CUDA_TRY(cudaMemcpyAsync(idx->pipe_lens[b], q_len + q0, cq * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            dl = idx->pipe_lens[b];
        }
#ifndef SA_HOST_NO_ORDER  // (A/B build: chunks matched in input order)
        PresortLayout L;
        SA_TRY(presort_layout(cq, false, true, true, L));
        SA_TRY(order_reads(idx->pipe_words[b], dl, fixed_len, stride, cq, kDefaultKeyBases,
                           static_cast<uint8_t *>(idx->pipe_ws[b]), L, idx->pipe_order[b], st));
        const uint32_t *ord = idx->pipe_order[b];
#else
        const uint32_t *ord = nullptr;
#endif
        SA_TRY(match_launch(idx, idx->pipe_words[b], dl, fixed_len, stride, cq, idx->pipe_out[b], nullptr, ord, false,
                            st));
        SA_CUDA_TRY(cudaMemcpyAsync(out_lohi + 2 * q0, idx->pipe_out[b], cq * 2 * sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, st));
    }
    SA_CUDA_TRY(cudaStreamSynchronize(idx->pipe_stream[0]));
    SA_CUDA_TRY(cudaStreamSynchronize(idx->pipe_stream[1]));
    return SA_OK;
}

extern "C" sa_status sa_match_route(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len,
                                    uint32_t fixed_len, uint32_t stride_words, uint64_t Q, uint32_t *order,
                                    uint64_t *ordered_words, uint32_t *ordered_len, uint64_t *dest_offsets,
                                    void *workspace, size_t ws_bytes, void *stream) {
    sa_clear_error();
    SA_TRY(check_match_args(idx, q_words, q_len, fixed_len, stride_words, Q, order));
    if (!dest_offsets || !ordered_words || stride_words == 0) {
        sa_set_error("sa_match_route needs dest_offsets, ordered_words and strided reads");
        return SA_EINVAL;
    }
    if (idx->nparts < 2) { sa_set_error("not a partitioned index"); return SA_EINVAL; }
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    cudaStream_t st = (cudaStream_t)stream;
    const uint32_t nb = idx->nparts + 1;
    if (Q == 0) {
        SA_CUDA_TRY(cudaMemsetAsync(dest_offsets, 0, nb * sizeof(uint64_t), st));
        return SA_OK;
    }
    PresortLayout L;
    SA_TRY(presort_layout(Q, false, true, true, L));
    if (!workspace || ws_bytes < L.total) {
        sa_set_error("workspace too small: %zu < %zu bytes", ws_bytes, L.total);
        return SA_EINVAL;
    }
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    SA_TRY(order_reads(q_words, q_len, fixed_len, stride_words, Q, idx->route_bases, ws, L, order, st, true));
    uint64_t blocks = (Q + 255) / 256;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    const bool vec = stride_words == 4 && (reinterpret_cast<uintptr_t>(q_words) & 31) == 0 &&
                     (reinterpret_cast<uintptr_t>(ordered_words) & 31) == 0;
    k_gather_rows<<<(unsigned)blocks, 256, 0, st>>>(q_words, q_len, stride_words, vec, Q, order, ordered_words,
                                                   ordered_len);
    SA_CUDA_TRY(cudaGetLastError());
    DevBuf<uint32_t> bounds;
    SA_TRY(bounds.alloc(nb, st, "route bounds"));
    SA_CUDA_TRY(cudaMemcpyAsync(bounds.p, idx->part_keys.data(), nb * 4, cudaMemcpyHostToDevice, st));
    k_route_offsets<<<(nb + 63) / 64, 64, 0, st>>>(reinterpret_cast<const uint32_t *>(ws + L.keys_out), Q, bounds.p, nb,
                                                   dest_offsets);
    SA_CUDA_TRY(cudaGetLastError());
    SA_CUDA_TRY(cudaStreamSynchronize(st));  // bounds is freed on return; keep the copy stream-ordered
    return SA_OK;
}

extern "C" sa_status sa_scatter_results(const uint32_t *order, const uint32_t *in_lohi, uint64_t Q, uint32_t *out_lohi,
                                        void *stream) {
    sa_clear_error();
    if (Q == 0) return SA_OK;
    if (!order || !in_lohi || !out_lohi) { sa_set_error("NULL argument"); return SA_EINVAL; }
    uint64_t blocks = (Q + 255) / 256;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    k_scatter_results<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
        order, reinterpret_cast<const uint2 *>(in_lohi), Q, reinterpret_cast<uint2 *>(out_lohi));
    SA_CUDA_TRY(cudaGetLastError());
    return SA_OK;
}

extern "C" sa_status sa_locate_workspace_size(uint64_t Q, size_t *bytes) {
    sa_clear_error();
    if (!bytes) { sa_set_error("NULL argument"); return SA_EINVAL; }
    CountOp op{nullptr, Q};
    thrust::transform_iterator<CountOp, thrust::counting_iterator<uint64_t>, uint64_t> it(
        thrust::counting_iterator<uint64_t>(0), op);
    size_t b = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, b, it, (uint64_t *)nullptr, (int64_t)(Q + 1));
    if (e != cudaSuccess) { sa_set_error("scan size: %s", cudaGetErrorString(e)); return SA_ECUDA; }
    *bytes = b;
    return SA_OK;
}

extern "C" sa_status sa_locate_offsets(const sa_index *idx, const uint32_t *out_lohi, uint64_t Q, uint64_t *offsets,
                                       void *workspace, size_t ws_bytes, void *stream) {
    sa_clear_error();
    if (!idx || !offsets || (Q > 0 && !out_lohi)) { sa_set_error("NULL argument"); return SA_EINVAL; }
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    CountOp op{out_lohi, Q};
    thrust::transform_iterator<CountOp, thrust::counting_iterator<uint64_t>, uint64_t> it(
        thrust::counting_iterator<uint64_t>(0), op);
    size_t need = 0;
    SA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, need, it, offsets, (int64_t)(Q + 1), (cudaStream_t)stream));
    if (ws_bytes < need || (need > 0 && !workspace)) {
        sa_set_error("workspace too small: %zu < %zu bytes", ws_bytes, need);
        return SA_EINVAL;
    }
    SA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(workspace, need, it, offsets, (int64_t)(Q + 1), (cudaStream_t)stream));
    return SA_OK;
}

extern "C" sa_status sa_locate(const sa_index *idx, const uint32_t *out_lohi, const uint64_t *offsets, uint64_t Q,
                               uint32_t *positions, void *stream) {
    sa_clear_error();
    if (!idx) { sa_set_error("index is NULL"); return SA_EINVAL; }
    if (Q == 0) return SA_OK;
    // positions may be NULL only when offsets[Q] == 0 (nothing is written then)
    if (!out_lohi || !offsets) { sa_set_error("NULL argument"); return SA_EINVAL; }
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    cudaStream_t st = (cudaStream_t)stream;
    uint64_t blocks = (Q * 32 + 255) / 256;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    const SaView v = sa_view(idx);
    k_locate<<<(unsigned)blocks, 256, 0, st>>>(v.base, v.stride, out_lohi, offsets, Q, positions);
    SA_CUDA_TRY(cudaGetLastError());
    // heavy reads: exclusive scan of their chunk counts, then one block per chunk
    DevBuf<uint64_t> chunk_off;
    SA_TRY(chunk_off.alloc(Q + 1, st, "locate chunk offsets"));
    ChunksOfRead op{out_lohi};
    thrust::transform_iterator<ChunksOfRead, thrust::counting_iterator<uint64_t>, uint64_t> it(
        thrust::counting_iterator<uint64_t>(0), op);
    size_t bytes = 0;
    SA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, bytes, it, chunk_off.p, (int64_t)(Q + 1), st));
    DevBuf<uint8_t> tmp;
    SA_TRY(tmp.alloc(bytes, st, "locate scan"));
    // (entry Q of the transform reads lohi[2Q]: the scan input must stop at Q, so scan Q items and fix up)
    SA_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, it, chunk_off.p, (int64_t)Q, st));
    k_chunk_total<<<1, 1, 0, st>>>(out_lohi, Q, chunk_off.p);
    SA_CUDA_TRY(cudaGetLastError());
    k_locate_heavy<<<148 * 16, 256, 0, st>>>(v.base, v.stride, out_lohi, offsets, Q, chunk_off.p, positions);
    SA_CUDA_TRY(cudaGetLastError());
    return SA_OK;
}
