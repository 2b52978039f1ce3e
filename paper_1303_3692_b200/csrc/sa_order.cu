// sa_order.cu -- an A/B build (SA_ORDER_ONESWEEP) of the read ordering (SURVEY.md Sec. 8(a) a5,
// sa_match_order): a stable LSD radix sort of the reads by their first key_bases bases, hand-written for
// this key (<= 32 bits) and this value (the read index), in place of CUB's DeviceRadixSort::SortPairs.
// Measured (profiles/r02/r02m..r02r, 100 M C4 reads): 3.7-4.0 ms vs CUB's 2.77 ms -- the fused key +
// histogram kernel saves 0.19 ms, but each pass takes ~1.0-1.2 ms vs CUB's 0.68 ms (ncu: short-scoreboard
// and look-back stalls; the same DRAM bytes).  Default: CUB.
//
// What it does differently (DESIGN.md §6 "Read ordering"):
//   * the key extraction also builds the digit histograms of every pass (one kernel instead of CUB's
//     key kernel + its histogram kernel re-reading the keys);
//   * pass 0's values are implicit (value = the read's own index: nothing is written or read for
//     them), and the last pass writes only the values (the permutation), not the keys;
//   * a tile is 8192 items (512 threads x 16), twice CUB's, so the scattered runs per digit are longer
//     (fewer partial 32-byte sectors, each of which costs a DRAM read-modify-write for ECC).
// Each pass is one "onesweep" kernel: a CTA claims the next tile (atomic counter, so tiles are claimed in
// order), ranks its items stably within the tile (per warp: __match_any_sync on the digit, popc of the
// lower lanes, a per-warp digit counter; then an exclusive scan over the warps), finds the tile's global
// offset per digit by decoupled look-back over the preceding tiles (status = flag << 62 | count: A = the
// tile's own count, P = the inclusive prefix), stages the tile in shared memory in digit order, and
// writes it out: equal-digit items go to consecutive addresses.
#include <cuda_runtime.h>

#include <cstdint>

#include "sa_internal.cuh"

namespace {

#ifndef SA_OS_THREADS
#define SA_OS_THREADS 512
#endif
#ifndef SA_OS_ITEMS
#define SA_OS_ITEMS 16
#endif
#ifndef SA_OS_MINB
#define SA_OS_MINB (1024 / SA_OS_THREADS)
#endif
constexpr int kOsThreads = SA_OS_THREADS;
constexpr int kOsItems = SA_OS_ITEMS;
constexpr int kOsTile = kOsThreads * kOsItems;  // 8192
constexpr int kOsWarps = kOsThreads / 32;
constexpr int kOsSmem = 2 * kOsTile * 4;  // dynamic shared memory of k_onesweep
constexpr uint64_t kFlagA = 1ull << 62, kFlagP = 2ull << 62, kValMask = (1ull << 62) - 1;

// key of read q (as k_presort_keys of csrc/sa_match.cu) + the digit histograms of all passes
__global__ void __launch_bounds__(256) k_order_keys(const uint64_t *__restrict__ words, const uint32_t *__restrict__ lens,
                                                    uint32_t fixed_len, uint32_t stride, uint64_t dense_words, uint64_t Q,
                                                    uint32_t key_bases, int npasses, uint32_t *__restrict__ keys,
                                                    uint32_t *__restrict__ hist) {
    __shared__ uint32_t sh[4][256];
    for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < Q; q += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t m;
        uint64_t w0;
        if (stride == 0) {
            m = fixed_len;
            const uint64_t bit = 2ull * m * q, i = bit >> 6;
            const unsigned s = (unsigned)(bit & 63);
            const uint64_t lo = __ldg(reinterpret_cast<const unsigned long long *>(words) + i);
            const uint64_t hi = (s && i + 1 < dense_words) ? __ldg(reinterpret_cast<const unsigned long long *>(words) + i + 1) : 0ull;
            w0 = s ? (lo << s) | (hi >> (64 - s)) : lo;
        } else {
            m = min(lens ? __ldg(lens + q) : fixed_len, 32u * stride);
            w0 = __ldg(reinterpret_cast<const unsigned long long *>(words + q * stride));
        }
        const uint32_t key = (uint32_t)((w0 & prefix_mask(min(m, key_bases))) >> (64 - 2 * key_bases));
        keys[q] = key;
        for (int p = 0; p < npasses; ++p) atomicAdd(&sh[p][(key >> (8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npasses * 256; i += blockDim.x) {
        const uint32_t c = (&sh[0][0])[i];
        if (c) atomicAdd(hist + i, c);
    }
}

// bin_base[p][d] = exclusive prefix of hist[p][.] (one block of 256 threads per pass)
__global__ void k_order_bins(const uint32_t *__restrict__ hist, uint32_t *__restrict__ bin_base) {
    __shared__ uint32_t s[256];
    const int p = blockIdx.x, d = threadIdx.x;
    s[d] = hist[p * 256 + d];
    __syncthreads();
    for (int off = 1; off < 256; off <<= 1) {
        const uint32_t v = d >= off ? s[d - off] : 0u;
        __syncthreads();
        s[d] += v;
        __syncthreads();
    }
    bin_base[p * 256 + d] = s[d] - hist[p * 256 + d];
}

__device__ __forceinline__ uint64_t ld_status(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_status(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// one pass over bits [shift, shift+8): keys_in (and vals_in, or the implicit index) -> out
__global__ void __launch_bounds__(kOsThreads, SA_OS_MINB)
k_onesweep(const uint32_t *__restrict__ keys_in, const uint32_t *__restrict__ vals_in, uint64_t N, int shift,
           const uint32_t *__restrict__ bin_base, uint64_t *__restrict__ status, uint32_t *__restrict__ tile_counter,
           uint32_t *__restrict__ keys_out, uint32_t *__restrict__ vals_out) {
    extern __shared__ __align__(16) uint32_t s_dyn[];  // the staged tile: keys, then values (64 KB)
    uint32_t *s_keys = s_dyn, *s_vals = s_dyn + kOsTile;
    __shared__ uint32_t s_whist[kOsWarps][256];  // per-warp digit counts, then their exclusive prefix over warps
    __shared__ uint32_t s_toff[256];              // the tile's digit offsets (exclusive scan of its counts)
    __shared__ uint64_t s_goff[256];              // global position of the tile's first item of each digit, - s_toff
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_cnt[256];               // the tile's digit counts (published early)
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int i = tid; i < kOsWarps * 256; i += kOsThreads) (&s_whist[0][0])[i] = 0;
    if (tid < 256) s_cnt[tid] = 0;
    if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * kOsTile + (uint64_t)w * (kOsItems * 32);
    // load (coalesced per round) and rank within the warp, stably (round-major, lane order)
    uint32_t key[kOsItems], val[kOsItems], rank[kOsItems];
    const unsigned lt = (1u << lane) - 1u;
    // all of the thread's loads first (the ranking's __syncwarp would otherwise keep each round's loads
    // behind the previous round: 16 serial DRAM round trips per tile)
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        const bool ok = i < N;
        key[r] = ok ? keys_in[i] : 0u;
        val[r] = ok ? (vals_in ? vals_in[i] : (uint32_t)i) : 0u;
    }
    // early counts: the tile's histogram first, published as its aggregate at once, so that the tiles
    // after it find it when they look back (the ranking below takes longer)
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        if (i < N) atomicAdd(&s_cnt[(key[r] >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 256) {
        const uint64_t a = s_cnt[tid];
        st_status(status + tile * 256 + tid, (tile == 0 ? kFlagP : kFlagA) | a);
    }
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        const bool ok = i < N;
        const uint32_t d = ok ? ((key[r] >> shift) & 255u) : 256u;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t b = 0;
        if (lane == leader && ok) {
            b = s_whist[w][d];
            s_whist[w][d] = b + (uint32_t)__popc(peers);
        }
        b = __shfl_sync(0xFFFFFFFFu, b, leader);
        rank[r] = b + (uint32_t)__popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over the warps, the tile's count
    uint32_t cnt = 0;
    if (tid < 256) {
        for (int ww = 0; ww < kOsWarps; ++ww) {
            const uint32_t c = s_whist[ww][tid];
            s_whist[ww][tid] = cnt;
            cnt += c;
        }
        s_toff[tid] = cnt;
    }
    __syncthreads();
    // the tile's digit offsets: exclusive scan of the counts over the 256 digits
    for (int off = 1; off < 256; off <<= 1) {
        uint32_t v = 0;
        if (tid < 256 && tid >= off) v = s_toff[tid - off];
        __syncthreads();
        if (tid < 256) s_toff[tid] += v;
        __syncthreads();
    }
    if (tid < 256) {
        s_toff[tid] -= cnt;  // exclusive
        // decoupled look-back: this tile's count, then the sum of the preceding tiles' counts
        uint64_t *my = status + tile * 256 + tid;
        if (tile == 0) {
            s_goff[tid] = (uint64_t)bin_base[tid] - s_toff[tid];
        } else {
            uint64_t excl = 0;
            for (int64_t pt = (int64_t)tile - 1; pt >= 0; --pt) {
                uint64_t v;
                do {
                    v = ld_status(status + (uint64_t)pt * 256 + tid);
                } while ((v >> 62) == 0);
                excl += v & kValMask;
                if ((v >> 62) == 2) break;
            }
            st_status(my, kFlagP | (excl + cnt));
            s_goff[tid] = (uint64_t)bin_base[tid] + excl - s_toff[tid];
        }
    }
    __syncthreads();
    // stage the tile in digit order
#pragma unroll
    for (int r = 0; r < kOsItems; ++r) {
        const uint64_t i = base + (uint64_t)r * 32 + lane;
        if (i < N) {
            const uint32_t d = (key[r] >> shift) & 255u;
            const uint32_t at = s_toff[d] + s_whist[w][d] + rank[r];
            s_keys[at] = key[r];
            s_vals[at] = val[r];
        }
    }
    __syncthreads();
    const uint64_t t0 = tile * kOsTile;
    const uint32_t nvalid = (uint32_t)(N - t0 < (uint64_t)kOsTile ? N - t0 : (uint64_t)kOsTile);
    for (uint32_t i = tid; i < nvalid; i += kOsThreads) {
        const uint32_t k = s_keys[i];
        const uint64_t pos = s_goff[(k >> shift) & 255u] + i;
        if (keys_out) keys_out[pos] = k;
        vals_out[pos] = s_vals[i];
    }
}

inline unsigned grid_keys(uint64_t Q) {
    uint64_t b = (Q + 255) / 256;
    if (b > 148ull * 16) b = 148ull * 16;
    return (unsigned)(b ? b : 1);
}

}  // namespace

// workspace bytes of sa_order_onesweep for Q reads
size_t sa_order_onesweep_bytes(uint64_t Q) {
    const uint64_t tiles = (Q + kOsTile - 1) / kOsTile;
    auto a = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
    return a(Q * 4) * 4 + a(tiles * 256 * 8) * 4 + a(4 * 256 * 4) * 2 + a(4 * 4);
}

// order (Q uint32) = the stable permutation sorting the reads by their first key_bases bases
sa_status sa_order_onesweep(const uint64_t *q_words, const uint32_t *q_len, uint32_t fixed_len, uint32_t stride,
                            uint64_t Q, uint32_t key_bases, uint8_t *ws, uint32_t *order, cudaStream_t st) {
    if (Q == 0) return SA_OK;
    if (Q >= (1ull << 32)) { sa_set_error("read ordering needs Q < 2^32"); return SA_EINVAL; }
    const uint64_t tiles = (Q + kOsTile - 1) / kOsTile;
    auto a = [](uint64_t x) { return (x + 255) & ~uint64_t(255); };
    uint8_t *p = ws;
    uint32_t *k0 = reinterpret_cast<uint32_t *>(p); p += a(Q * 4);
    uint32_t *k1 = reinterpret_cast<uint32_t *>(p); p += a(Q * 4);
    uint32_t *v1 = reinterpret_cast<uint32_t *>(p); p += a(Q * 4);
    uint32_t *v2 = reinterpret_cast<uint32_t *>(p); p += a(Q * 4);
    uint64_t *status[4];
    for (int i = 0; i < 4; ++i) { status[i] = reinterpret_cast<uint64_t *>(p); p += a(tiles * 256 * 8); }
    uint32_t *hist = reinterpret_cast<uint32_t *>(p); p += a(4 * 256 * 4);
    uint32_t *bins = reinterpret_cast<uint32_t *>(p); p += a(4 * 256 * 4);
    uint32_t *counters = reinterpret_cast<uint32_t *>(p);
    const int bits = 2 * (int)key_bases;
    const int npasses = (bits + 7) / 8;
    // the zeroed state of every pass (histograms, counters, look-back status) in one memset each
    SA_CUDA_TRY(cudaMemsetAsync(status[0], 0, (size_t)(reinterpret_cast<uint8_t *>(counters) + a(16) -
                                                       reinterpret_cast<uint8_t *>(status[0])), st));
    const uint64_t dense_words = (Q * (uint64_t)fixed_len + 31) / 32;
    k_order_keys<<<grid_keys(Q), 256, 0, st>>>(q_words, q_len, fixed_len, stride, dense_words, Q, key_bases, npasses,
                                                k0, hist);
    SA_CUDA_TRY(cudaGetLastError());
    k_order_bins<<<npasses, 256, 0, st>>>(hist, bins);
    SA_CUDA_TRY(cudaGetLastError());
    // pass chain: keys k0 -> k1 -> k0 ..., values (implicit) -> v1 -> v2 -> v1 ..., the last pass's
    // values into `order` (its keys are not written)
    static bool attr_set = false;  // (set once, outside any graph capture: the first call is a warm-up)
    if (!attr_set) {
        SA_CUDA_TRY(cudaFuncSetAttribute(k_onesweep, cudaFuncAttributeMaxDynamicSharedMemorySize, kOsSmem));
        attr_set = true;
    }
    const uint32_t *kin = k0, *vin = nullptr;
    for (int ps = 0; ps < npasses; ++ps) {
        const bool last = ps == npasses - 1;
        uint32_t *kout = last ? nullptr : (kin == k0 ? k1 : k0);
        uint32_t *vout = last ? order : ((ps & 1) ? v2 : v1);
        k_onesweep<<<(unsigned)tiles, kOsThreads, kOsSmem, st>>>(kin, vin, Q, 8 * ps, bins + 256 * ps, status[ps],
                                                           counters + ps, kout, vout);
        SA_CUDA_TRY(cudaGetLastError());
        kin = kout;
        vin = vout;
    }
    return SA_OK;
}
