// sa_match.cu -- the hot path: per-query SA interval [lo, hi) by binary search (Sec. IV,
// Alg. 1 `cudaGeneBinSearch`, L173-230), plus locate and the host-buffer pipeline.
//
// B200 design, not a translation of Alg. 1:
//  * one thread per query (Alg. 1 line 2's mapping) with the query held in registers
//    (2 bits/base, MSB-first words) instead of the per-block shared tiles of lines 5, 14-15 (which
//    race as written, reading A9);
//  * the first k bases index the k-mer bracket table T: the search starts in
//    (T[x]-1, T[x+1]) instead of Alg. 1's (left, right) = (-1, n) (reading A4);
//  * Alg. 1's tiled do-while compare (lines 10-17) becomes a 32-bases-per-step compare of two
//    packed words (xor + clz; unsigned order of MSB-first words is lexicographic order);
//  * the LB and RB loops (lines 6-23 and 25-42, directions corrected per reading A6) run jointly:
//    one descent until the first pivot equal to P, then the RB search continues from that split;
//  * Manber-Myers skipping: compares start at min(lcp(P, t_L), lcp(P, t_R)).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>

#include "sa_internal.cuh"

namespace {

struct MatchArgs {
    const uint64_t *__restrict__ text;
    const uint32_t *__restrict__ sa;   // plain layout
    const uint4 *__restrict__ rec;     // record layout
    const uint32_t *__restrict__ table;
    uint64_t n;
    uint32_t k;
    const uint64_t *__restrict__ words;
    const uint32_t *__restrict__ lens;
    uint32_t fixed_len;
    uint32_t stride;
    uint64_t Q;
    uint32_t *__restrict__ out;
    uint32_t *__restrict__ stats;      // SA_MATCH_STATS
    const uint32_t *__restrict__ perm; // SA_MATCH_PRESORT: thread slot t handles read perm[t]
};

// Query words: QW > 0 -> registers (fully unrolled so indices are static); QW == 0 -> global.
template <int QW>
struct QueryWords {
    uint64_t w[QW];
    __device__ __forceinline__ void load(const uint64_t *__restrict__ p, uint32_t nw) {
#pragma unroll
        for (int j = 0; j < QW; ++j) w[j] = (j < (int)nw) ? __ldg(reinterpret_cast<const unsigned long long *>(p) + j) : 0ull;
    }
    __device__ __forceinline__ uint64_t first() const { return w[0]; }
    __device__ __forceinline__ uint64_t word(int j) const { return j < QW ? w[j] : 0ull; }
};
template <>
struct QueryWords<0> {
    const uint64_t *p;
    uint32_t nw;
    __device__ __forceinline__ void load(const uint64_t *__restrict__ q, uint32_t n) { p = q; nw = n; }
    __device__ __forceinline__ uint64_t first() const { return __ldg(reinterpret_cast<const unsigned long long *>(p)); }
    __device__ __forceinline__ uint64_t word(int j) const {
        return (uint32_t)j < nw ? __ldg(reinterpret_cast<const unsigned long long *>(p) + j) : 0ull;
    }
};

// One 32-base step of the compare: word j of P against the text at s + 32j.
// Returns 1 when decided (sign/lcp set), 0 to continue.
__device__ __forceinline__ int cmp_word(const uint64_t *__restrict__ text, uint64_t s, uint64_t slen, uint32_t m,
                                        uint32_t j, uint64_t pw, int &sign, uint32_t &lcp) {
    const uint32_t base = j << 5;
    const uint32_t plen = min(32u, m - base);
    const uint64_t rem = slen > base ? slen - base : 0;
    const uint32_t L = rem < plen ? (uint32_t)rem : plen;
    if (L) {
        const uint64_t tw = text_window(text, s + base);
        const uint64_t mask = prefix_mask(L);
        const uint64_t a = pw & mask, b = tw & mask;
        if (a != b) {
            lcp = base + ((uint32_t)__clzll((long long)(a ^ b)) >> 1);
            sign = a > b ? 1 : -1;
            return 1;
        }
    }
    if (L < plen) {  // the suffix ended first: it is a proper prefix of P (reading A7)
        lcp = base + L;
        sign = 1;
        return 1;
    }
    return 0;
}

// sign(P - t_s), t_s = S[s .. min(s+m, n)), comparing from word skip/32 on; lcp = lcp(P, t_s).
template <int QW>
__device__ __forceinline__ void compare(const uint64_t *__restrict__ text, uint64_t n, uint64_t s,
                                        const QueryWords<QW> &P, uint32_t m, uint32_t skip, int &sign,
                                        uint32_t &lcp) {
    const uint64_t slen = n - s;
    const uint32_t nw = (m + 31) >> 5;
    const uint32_t j0 = skip >> 5;
    if constexpr (QW > 0) {
#pragma unroll
        for (int j = 0; j < QW; ++j) {
            if ((uint32_t)j >= j0 && (uint32_t)j < nw) {
                if (cmp_word(text, s, slen, m, (uint32_t)j, P.w[j], sign, lcp)) return;
            }
        }
    } else {
        for (uint32_t j = j0; j < nw; ++j) {
            const uint64_t pw = __ldg(reinterpret_cast<const unsigned long long *>(P.p) + j);
            if (cmp_word(text, s, slen, m, j, pw, sign, lcp)) return;
        }
    }
    sign = 0;
    lcp = m;
}

// Compare P (m >= k, inside its k-mer bracket) with the suffix of SA record r.  The record caches
// the 48 bases after the first k, which every long suffix in the bracket shares with P; the text
// is read only when those 48 bases are equal and more remain, or for the < k suffixes shorter
// than k (which can sit at the end of a bracket without sharing its k-mer).
template <int QW>
__device__ __forceinline__ void rec_compare(const uint64_t *__restrict__ text, uint64_t n, uint32_t k, const uint4 r,
                                            const QueryWords<QW> &P, uint64_t pk01, uint32_t pk2, uint32_t m,
                                            uint32_t skip, int &sign, uint32_t &lcp, uint32_t &texts) {
    const uint64_t s = r.x;
    const uint64_t len = n - s;
    if (len < k || skip >= k + kCacheBases) {
        ++texts;
        compare<QW>(text, n, s, P, m, len < k ? 0u : skip, sign, lcp);
        return;
    }
    const uint32_t avail = (uint32_t)((m < len ? (uint64_t)m : len) - k);  // bases after k present in both
    const uint64_t c01 = ((uint64_t)r.w << 32) | r.z;
    const uint64_t mask1 = prefix_mask(min(32u, avail));
    const uint64_t a1 = pk01 & mask1, b1 = c01 & mask1;
    if (a1 != b1) {
        lcp = k + ((uint32_t)__clzll((long long)(a1 ^ b1)) >> 1);
        sign = a1 > b1 ? 1 : -1;
        return;
    }
    if (avail > 32) {
        const uint32_t L2 = min(16u, avail - 32);
        const uint32_t mask2 = L2 >= 16 ? ~0u : ~(~0u >> (2 * L2));
        const uint32_t a2 = pk2 & mask2, b2 = r.y & mask2;
        if (a2 != b2) {
            lcp = k + 32 + ((uint32_t)__clz((int)(a2 ^ b2)) >> 1);
            sign = a2 > b2 ? 1 : -1;
            return;
        }
        if (avail > kCacheBases) {
            ++texts;
            compare<QW>(text, n, s, P, m, k + kCacheBases, sign, lcp);
            return;
        }
    }
    // every base present in both is equal
    if (m <= len) { sign = 0; lcp = m; }            // P is a prefix of the suffix (case 1)
    else { sign = 1; lcp = (uint32_t)len; }          // the suffix is a proper prefix of P (reading A7)
}

enum : int { M_IDLE = 0, M_JOINT, M_HI, M_SHORT_LO, M_SHORT_HI };

// The search as a per-lane state machine.  Each loop iteration performs ONE binary-search step
// for whatever query the lane currently holds; a lane whose query is finished writes {lo, hi} and
// immediately takes its next query (grid-stride), so lanes of a warp stay busy even though reads
// need very different numbers of steps (repeats: up to ~32, unique reads: ~9).
//   M_JOINT     LB rule (R moves when P <= t) over the k-mer bracket, remembering the first pivot
//               where P is a prefix of the suffix (the split);
//   M_HI        RB rule (R moves when P < t) over (split, R at the split);
//   M_SHORT_*   m < k: LB then RB rule over the two small windows below T[xa] and T[xb].
// L is kept as L+1 (Lp1) so every bound fits uint32.
template <int QW, bool REC, bool STATS>
__global__ void __launch_bounds__(256) k_match(const MatchArgs a) {
    const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
    uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;  // slot; read q = perm[t] or t
    uint64_t q = 0;
    const uint32_t k = a.k;
    QueryWords<QW> P;
    uint64_t pk01 = 0;
    uint32_t pk2 = 0, m = 0;
    uint32_t Lp1 = 0, R = 0, lcpL = 0, lcpR = 0;
    uint32_t sLp1 = 0, sR = 0, slcpR = 0, lo = 0;
    uint32_t nsteps = 0, ntexts = 0;
    int mode = M_IDLE;
    bool split = false, first = true;
    for (;;) {
        if (mode == M_IDLE) {
            if (!first) t += nthreads;
            first = false;
            if (t >= a.Q) break;
            q = a.perm ? (uint64_t)__ldg(a.perm + t) : t;
            // lengths past the stride are clamped (include/sa.h requires m <= 32*stride_words)
            m = min(a.lens ? __ldg(a.lens + q) : a.fixed_len, 32u * a.stride);
            P.load(a.words + q * a.stride, (m + 31) >> 5);
            nsteps = ntexts = 0;
            lcpL = lcpR = 0;
            if (m == 0) {  // the empty query is a prefix of every suffix (reading A12)
                lo = 0;
                Lp1 = R = (uint32_t)a.n;
                mode = M_HI;
            } else if (m >= k) {
                // all suffixes before T[x] are < P, all from T[x+1] on are > P
                const uint64_t x = P.first() >> (64 - 2 * k);
                Lp1 = __ldg(a.table + x);
                R = __ldg(a.table + x + 1);
                split = false;
                mode = M_JOINT;
                if (REC) {
                    const uint64_t w0 = P.word(0), w1 = P.word(1), w2 = P.word(2);
                    pk01 = (w0 << (2 * k)) | (w1 >> (64 - 2 * k));
                    pk2 = (uint32_t)(((w1 << (2 * k)) | (w2 >> (64 - 2 * k))) >> 32);
                }
            } else {
                // m < k: lo in [T[xa]-(k-m), T[xa]], hi in [T[xb]-(k-1), T[xb]] with xa = x.a^(k-m),
                // xb = (x+1).a^(k-m); searched over T[.]-k .. T[.]
                const uint64_t x = P.first() >> (64 - 2 * m);
                const uint32_t Ta = __ldg(a.table + (x << (2 * (k - m))));
                const uint32_t Tb = __ldg(a.table + ((x + 1) << (2 * (k - m))));
                Lp1 = Ta > k ? Ta - k : 0;
                R = Ta;
                sLp1 = Tb > k ? Tb - k : 0;
                sR = Tb;
                mode = M_SHORT_LO;
            }
        }
        // finished intervals: move to the next phase or emit the result
        while (mode != M_IDLE && R <= Lp1) {
            if (mode == M_JOINT) {
                lo = R;
                if (split) {
                    Lp1 = sLp1; R = sR; lcpL = m; lcpR = slcpR;
                    mode = M_HI;
                    continue;
                }
            } else if (mode == M_SHORT_LO) {
                lo = R;
                Lp1 = sLp1; R = sR; lcpL = lcpR = 0;
                mode = M_SHORT_HI;
                continue;
            }
            // Alg. 1 lines 44-45: res[thd<<1] = LB, res[(thd<<1)+1] = RB (reading A8), half-open here
            const uint32_t hi = (mode == M_JOINT) ? lo : R;
            reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
            if (STATS) a.stats[q] = nsteps | (ntexts << 16);
            mode = M_IDLE;
        }
        if (mode == M_IDLE) continue;
        // ---- one binary-search step ----
        const uint32_t p = (uint32_t)(((uint64_t)Lp1 - 1 + R) >> 1);
        int sign;
        uint32_t lcp;
        const uint32_t skip = min(lcpL, lcpR);
        if constexpr (REC) {
            const uint4 r = __ldg(a.rec + p);
            if (mode <= M_HI) {
                rec_compare<QW>(a.text, a.n, k, r, P, pk01, pk2, m, skip, sign, lcp, ntexts);
            } else {
                ++ntexts;
                compare<QW>(a.text, a.n, r.x, P, m, skip, sign, lcp);
            }
        } else {
            const uint64_t s = __ldg(a.sa + p);
            ++ntexts;
            compare<QW>(a.text, a.n, s, P, m, skip, sign, lcp);
        }
        ++nsteps;
        if (mode == M_JOINT && sign == 0 && !split) {  // first pivot with P a prefix of its suffix
            split = true;
            sLp1 = p + 1;
            sR = R;
            slcpR = lcpR;
        }
        const bool go_left = sign < 0 || (sign == 0 && (mode == M_JOINT || mode == M_SHORT_LO));
        if (go_left) { R = p; lcpR = lcp; } else { Lp1 = p + 1; lcpL = lcp; }
    }
}

template <int QW, bool REC, bool STATS>
cudaError_t launch_match_t(const MatchArgs &a, bool simple, cudaStream_t st) {
    const int threads = 256;
    uint64_t blocks;
    if (simple) {
        blocks = (a.Q + threads - 1) / threads;  // one query per thread
    } else {
        static int per_sm[64] = {0};
        static int sms[64] = {0};
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 64 && per_sm[dev] == 0) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[dev], k_match<QW, REC, STATS>, threads, 0);
            cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
        }
        const uint64_t resident = (uint64_t)(dev < 64 ? per_sm[dev] * sms[dev] : 148 * 4);
        const uint64_t need = (a.Q + threads - 1) / threads;
        blocks = need < resident ? need : resident;  // persistent: one wave, lanes refill
    }
    if (blocks == 0) blocks = 1;
    k_match<QW, REC, STATS><<<(unsigned)blocks, threads, 0, st>>>(a);
    return cudaGetLastError();
}

template <int QW>
cudaError_t launch_match_qw(const MatchArgs &a, bool rec, bool stats, bool simple, cudaStream_t st) {
    if (rec) return stats ? launch_match_t<QW, true, true>(a, simple, st) : launch_match_t<QW, true, false>(a, simple, st);
    return stats ? launch_match_t<QW, false, true>(a, simple, st) : launch_match_t<QW, false, false>(a, simple, st);
}

// ---- presort (SA_MATCH_PRESORT) ---------------------------------------------------------------
// key = the read's first 16 bases (masked to its length), value = read index
__global__ void k_presort_keys(const uint64_t *__restrict__ words, const uint32_t *__restrict__ lens,
                               uint32_t fixed_len, uint32_t stride, uint64_t Q, uint32_t *__restrict__ keys,
                               uint32_t *__restrict__ perm) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Q; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t m = min(lens ? __ldg(lens + q) : fixed_len, 32u * stride);
        const uint64_t w0 = __ldg(reinterpret_cast<const unsigned long long *>(words + q * stride));
        keys[q] = (uint32_t)((w0 & prefix_mask(min(m, 16u))) >> 32);
        perm[q] = (uint32_t)q;
    }
}

struct PresortLayout {
    size_t stats = 0, keys_in = 0, keys_out = 0, perm_in = 0, perm_out = 0, cub = 0, cub_bytes = 0, total = 0;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// workspace of sa_match_order (order_only: the permutation goes to the caller's buffer) and of
// sa_match_batch (stats first, then, with SA_MATCH_PRESORT, the same sort scratch + the permutation)
sa_status presort_layout(uint64_t Q, bool stats, bool presort, bool order_only, PresortLayout &L) {
    size_t off = 0;
    if (stats) { L.stats = off; off = align256(off + Q * 4); }
    if (presort) {
        if (Q >= (1ull << 32)) { sa_set_error("read ordering needs Q < 2^32"); return SA_EINVAL; }
        L.keys_in = off; off = align256(off + Q * 4);
        L.keys_out = off; off = align256(off + Q * 4);
        L.perm_in = off; off = align256(off + Q * 4);
        if (!order_only) { L.perm_out = off; off = align256(off + Q * 4); }
        size_t b = 0;
        cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, b, (const uint32_t *)nullptr, (uint32_t *)nullptr,
                                                        (const uint32_t *)nullptr, (uint32_t *)nullptr, (int64_t)Q, 0, 32);
        if (e != cudaSuccess) { sa_set_error("order size query: %s", cudaGetErrorString(e)); return SA_ECUDA; }
        L.cub = off;
        L.cub_bytes = b;
        off = align256(off + b);
    }
    L.total = off;
    return SA_OK;
}

sa_status order_reads(const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len, uint32_t stride, uint64_t Q,
                      uint8_t *ws, const PresortLayout &L, uint32_t *order, cudaStream_t st) {
    uint32_t *keys_in = reinterpret_cast<uint32_t *>(ws + L.keys_in);
    uint32_t *keys_out = reinterpret_cast<uint32_t *>(ws + L.keys_out);
    uint32_t *perm_in = reinterpret_cast<uint32_t *>(ws + L.perm_in);
    uint64_t blocks = (Q + 255) / 256;
    if (blocks > 148ull * 16) blocks = 148ull * 16;
    k_presort_keys<<<(unsigned)blocks, 256, 0, st>>>(q_words, q_len, fixed_len, stride, Q, keys_in, perm_in);
    SA_CUDA_TRY(cudaGetLastError());
    size_t b = L.cub_bytes;
    SA_CUDA_TRY(cub::DeviceRadixSort::SortPairs(ws + L.cub, b, keys_in, keys_out, perm_in, order, (int64_t)Q, 0, 32, st));
    return SA_OK;
}

// ---- locate -----------------------------------------------------------------------------------
struct CountOp {
    const uint32_t *lohi;
    uint64_t Q;
    __host__ __device__ __forceinline__ uint64_t operator()(uint64_t q) const {
        return q < Q ? (uint64_t)(lohi[2 * q + 1] - lohi[2 * q]) : 0ull;
    }
};

// One warp per query: lanes copy SA[lo .. hi) to positions[off ..] (contiguous, coalesced).
// SA values are read through the layout's view (stride 1 = plain SA, 4 = 16-byte records).
__global__ void k_locate(const uint32_t *__restrict__ sa, uint32_t sa_stride, const uint32_t *__restrict__ lohi,
                         const uint64_t *__restrict__ offsets, uint64_t Q, uint32_t *__restrict__ pos) {
    const unsigned lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    for (uint64_t q = warp; q < Q; q += nwarps) {
        const uint32_t lo = lohi[2 * q], hi = lohi[2 * q + 1];
        const uint64_t off = offsets[q];
        for (uint64_t j = lane; j < (uint64_t)(hi - lo); j += 32) pos[off + j] = __ldg(sa + (lo + j) * sa_stride);
    }
}

sa_status check_match_args(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                           uint32_t stride, uint64_t Q, const uint32_t *out) {
    if (!idx) { sa_set_error("index is NULL"); return SA_EINVAL; }
    if (Q == 0) return SA_OK;
    if (!q_words || !out) { sa_set_error("q_words/out_lohi NULL with Q=%llu", (unsigned long long)Q); return SA_EINVAL; }
    if (stride == 0) { sa_set_error("stride_words must be >= 1"); return SA_EINVAL; }
    if (!q_len && fixed_len > 32u * stride) {
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

extern "C" sa_status sa_match_order(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len,
                                    uint32_t fixed_len, uint32_t stride_words, uint64_t Q, uint32_t *order,
                                    void *workspace, size_t ws_bytes, void *stream) {
    sa_clear_error();
    SA_TRY(check_match_args(idx, q_words, q_len, fixed_len, stride_words, Q, order));
    if (Q == 0) return SA_OK;
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    PresortLayout L;
    SA_TRY(presort_layout(Q, false, true, true, L));
    if (!workspace || ws_bytes < L.total) {
        sa_set_error("workspace too small: %zu < %zu bytes", ws_bytes, L.total);
        return SA_EINVAL;
    }
    return order_reads(q_words, q_len, fixed_len, stride_words, Q, static_cast<uint8_t *>(workspace), L, order,
                       (cudaStream_t)stream);
}

static sa_status match_launch(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len,
                              uint32_t stride, uint64_t Q, uint32_t *out, uint32_t *stats, const uint32_t *perm,
                              bool simple, cudaStream_t st) {
    MatchArgs a;
    a.perm = perm;
    a.text = idx->text;
    a.sa = idx->sa;
    a.rec = idx->rec;
    a.table = idx->table;
    a.n = idx->n;
    a.k = idx->k;
    a.words = q_words;
    a.lens = q_len;
    a.fixed_len = fixed_len;
    a.stride = stride;
    a.Q = Q;
    a.out = out;
    a.stats = stats;
    const bool rec = !idx->plain, st_on = stats != nullptr;
    cudaError_t e;
    if (stride <= 1) e = launch_match_qw<1>(a, rec, st_on, simple, st);
    else if (stride <= 2) e = launch_match_qw<2>(a, rec, st_on, simple, st);
    else if (stride <= 4) e = launch_match_qw<4>(a, rec, st_on, simple, st);
    else e = launch_match_qw<0>(a, rec, st_on, simple, st);
    if (e != cudaSuccess) { sa_set_error("match launch: %s", cudaGetErrorString(e)); return SA_ECUDA; }
    return SA_OK;
}

extern "C" sa_status sa_match_batch(const sa_index *idx, const uint64_t *q_words, const uint32_t *q_len,
                                    uint32_t fixed_len, uint32_t stride_words, uint64_t Q, const uint32_t *order,
                                    uint32_t *out_lohi, void *workspace, size_t ws_bytes, uint32_t flags,
                                    void *stream) {
    sa_clear_error();
    SA_TRY(check_match_args(idx, q_words, q_len, fixed_len, stride_words, Q, out_lohi));
    if (flags & ~(SA_MATCH_STATS | SA_MATCH_SIMPLE | SA_MATCH_PRESORT)) {
        sa_set_error("unknown flags 0x%x", flags);
        return SA_EINVAL;
    }
    if (Q == 0) return SA_OK;
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    const bool presort = (flags & SA_MATCH_PRESORT) && !order;
    PresortLayout L;
    SA_TRY(presort_layout(Q, flags & SA_MATCH_STATS, presort, false, L));
    if (L.total > 0 && (!workspace || ws_bytes < L.total)) {
        sa_set_error("workspace too small: %zu < %zu bytes", ws_bytes, L.total);
        return SA_EINVAL;
    }
    cudaStream_t st = (cudaStream_t)stream;
    uint8_t *ws = static_cast<uint8_t *>(workspace);
    uint32_t *stats = (flags & SA_MATCH_STATS) ? reinterpret_cast<uint32_t *>(ws + L.stats) : nullptr;
    if (presort) {
        uint32_t *perm = reinterpret_cast<uint32_t *>(ws + L.perm_out);
        SA_TRY(order_reads(q_words, q_len, fixed_len, stride_words, Q, ws, L, perm, st));
        order = perm;
    }
    return match_launch(idx, q_words, q_len, fixed_len, stride_words, Q, out_lohi, stats, order,
                        (flags & SA_MATCH_SIMPLE) != 0, st);
}

extern "C" sa_status sa_match_batch_host(sa_index *idx, const uint64_t *q_words, const uint32_t *q_len,
                                         uint32_t fixed_len, uint32_t stride, uint64_t Q, uint32_t *out_lohi,
                                         uint64_t chunk_Q) {
    sa_clear_error();
    SA_TRY(check_match_args(idx, q_words, q_len, fixed_len, stride, Q, out_lohi));
    if (Q == 0) return SA_OK;
    std::lock_guard<std::mutex> lock(idx->mu);
    SA_CUDA_TRY(cudaSetDevice(idx->device));
    if (chunk_Q == 0) chunk_Q = 1ull << 22;
    if (chunk_Q > Q) chunk_Q = Q;
    if (idx->pipe_chunk < chunk_Q || idx->pipe_stride < stride) {
        for (int b = 0; b < 2; ++b) {
            cudaFree(idx->pipe_words[b]);
            cudaFree(idx->pipe_lens[b]);
            cudaFree(idx->pipe_out[b]);
            idx->pipe_words[b] = nullptr;
            idx->pipe_lens[b] = nullptr;
            idx->pipe_out[b] = nullptr;
        }
        idx->pipe_chunk = 0;
        for (int b = 0; b < 2; ++b) {
            if (!idx->pipe_stream[b]) SA_CUDA_TRY(cudaStreamCreateWithFlags(&idx->pipe_stream[b], cudaStreamNonBlocking));
            SA_CUDA_TRY(cudaMalloc(&idx->pipe_words[b], chunk_Q * stride * sizeof(uint64_t)));
            SA_CUDA_TRY(cudaMalloc(&idx->pipe_lens[b], chunk_Q * sizeof(uint32_t)));
            SA_CUDA_TRY(cudaMalloc(&idx->pipe_out[b], chunk_Q * 2 * sizeof(uint32_t)));
        }
        idx->pipe_chunk = chunk_Q;
        idx->pipe_stride = stride;
    }
    // chunk c uses buffer set c%2 on stream c%2: H2D -> match -> D2H; the two streams overlap.
    uint64_t c = 0;
    for (uint64_t q0 = 0; q0 < Q; q0 += chunk_Q, ++c) {
        const int b = (int)(c & 1);
        cudaStream_t st = idx->pipe_stream[b];
        const uint64_t cq = std::min<uint64_t>(chunk_Q, Q - q0);
        SA_CUDA_TRY(cudaMemcpyAsync(idx->pipe_words[b], q_words + q0 * stride, cq * stride * sizeof(uint64_t),
                                    cudaMemcpyHostToDevice, st));
        const uint32_t *dl = nullptr;
        if (q_len) {
            SA_CUDA_TRY(cudaMemcpyAsync(idx->pipe_lens[b], q_len + q0, cq * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            dl = idx->pipe_lens[b];
        }
        SA_TRY(match_launch(idx, idx->pipe_words[b], dl, fixed_len, stride, cq, idx->pipe_out[b], nullptr, nullptr, false, st));
        SA_CUDA_TRY(cudaMemcpyAsync(out_lohi + 2 * q0, idx->pipe_out[b], cq * 2 * sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, st));
    }
    SA_CUDA_TRY(cudaStreamSynchronize(idx->pipe_stream[0]));
    SA_CUDA_TRY(cudaStreamSynchronize(idx->pipe_stream[1]));
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
    uint64_t blocks = (Q * 32 + 255) / 256;
    if (blocks > 148ull * 32) blocks = 148ull * 32;
    const SaView v = sa_view(idx);
    k_locate<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(v.base, v.stride, out_lohi, offsets, Q, positions);
    SA_CUDA_TRY(cudaGetLastError());
    return SA_OK;
}
