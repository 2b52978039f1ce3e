// sa_search.cuh -- device side of the hot path: per-read SA interval [lo, hi) by binary search
// (Sec. IV, Alg. 1 `cudaGeneBinSearch`, L173-230), re-designed for B200:
//
//  * one thread per read (Alg. 1 line 2's mapping), the read held in registers at 2 bits per
//    base (MSB-first words) instead of the per-block shared tiles of lines 5, 14-15 (which race as
//    written, reading A9);
//  * the first k bases index the k-mer bracket table T: the search starts in (T[x]-1, T[x+1])
//    instead of Alg. 1's undefined (left, right) (reading A4: (-1, n));
//  * Alg. 1's tiled do-while compare (lines 10-17) becomes a 32-bases-per-step compare of two packed
//    words (xor + clz; the unsigned order of MSB-first words is lexicographic order);
//  * the SA is stored as records {SA[r], bases k .. k+C-1 of that suffix} (C = 48 or 112), so one
//    32-byte sector per step decides the compare; the packed text is read only past the cache;
//  * the LB and RB loops (lines 6-23 and 25-42, directions corrected per reading A6) run jointly:
//    one descent until the first pivot equal to P (the split), then the RB search continues from it;
//  * Manber-Myers skipping: text compares start at min(lcp(P, t_L), lcp(P, t_R)).
#pragma once

#include "sa_internal.cuh"

namespace sa_search {

// SA layouts (sa_index::layout)
enum : int { L_PLAIN = 0, L_REC16 = 1, L_REC32 = 2 };

struct MatchArgs {
    const uint64_t *__restrict__ text;
    const uint32_t *__restrict__ sa;    // L_PLAIN
    const uint4 *__restrict__ rec;      // L_REC16 (1 uint4 per suffix) / L_REC32 (2 uint4 per suffix)
    const uint32_t *__restrict__ table;
    uint64_t n;
    uint64_t text_words;                // words of `text` (incl. the zero guard words)
    uint32_t k;
    const uint64_t *__restrict__ words;
    const uint32_t *__restrict__ lens;
    uint32_t fixed_len;
    uint32_t stride;
    uint64_t Q;
    uint32_t *__restrict__ out;
    uint32_t *__restrict__ stats;       // SA_MATCH_STATS: [Q] steps | text windows << 16, [Q] useful bytes
    const uint32_t *__restrict__ order; // thread slot t takes read order[t] (or t)
    bool vec_rows;                      // read rows can be loaded with one vector load (aligned, stride == QW)
    uint64_t dense_words;               // stride == 0: dense layout, words = one 2-bit stream of this many words
    bool rows_ordered;                  // SA_MATCH_ROWS_ORDERED: row t is read order[t]
    // the index's SA ranks [clo, chi): [0, n) for a whole index; a partition's slice (csrc/sa_part.cu),
    // every bracket is clamped to it, so a read is answered as clamp(lo), clamp(hi)
    uint32_t clo, chi;
    const uint32_t *__restrict__ route;  // partition: route-level table T_r (4^rb + 1 entries), else NULL
    uint32_t route_bases;                // partition: rb (reads with m < rb use T_r), else 0
    const unsigned long long *__restrict__ big_hash; // SA_INDEX_SUBTABLE: x << 32 | sub-table id, empty = ~0
    const uint32_t *__restrict__ big_sub;
    uint32_t big_bits;
    const unsigned long long *__restrict__ tree_hash;  // SA_INDEX_BUCKET_TREE: x << 32 | first line, empty = ~0
    const uint4 *__restrict__ tree;                     // its lines (4 records of 32 bytes, 3 used)
    uint32_t tree_bits;
    bool wide;  // a large batch (>= kWideQ reads): 64-byte L2 fetches for the read row and the table pair
};

// ---- the read ---------------------------------------------------------------------------------
// QW > 0: QW words in registers (loops over them are fully unrolled so indices are static; 1, 2 or 4
// words = reads up to 128 bases; an 8-word variant measured 16% slower for 150-250-base reads,
// profiles/r01x, as the extra registers cost occupancy);
// QW == 0: long reads, words read from global memory (L1-cached) as needed.
template <int QW>
struct QueryWords {
    uint64_t w[QW];
    // the whole read row in one vector load (one request, one sector) when the stride equals QW:
    // 256-bit (LDG.E.ENL2.256) for 4 words, 128-bit for 2; rows are then 32- / 16-byte aligned
    __device__ __forceinline__ void load(const uint64_t *__restrict__ p, uint32_t nw, bool vec, bool wide = false) {
        if constexpr (QW == 4) {
            if (vec) {
                ld_row_v4u64(p, wide, w[0], w[1], w[2], w[3]);
                return;
            }
        } else if constexpr (QW == 2) {
            if (vec) {
                ld_row_v2u64(p, wide, w[0], w[1]);
                return;
            }
        }
#pragma unroll
        for (int j = 0; j < QW; ++j)
            w[j] = (j < (int)nw) ? ld_row_u64(p + j, wide) : 0ull;
    }
    // dense layout: the read starts at bit `bit` of a continuous stream of `total` words
    __device__ __forceinline__ void load_dense(const uint64_t *__restrict__ s, uint64_t bit, uint32_t nw,
                                               uint64_t total) {
        const uint64_t w0 = bit >> 6;
        const unsigned sh = (unsigned)(bit & 63);
        uint64_t r[QW + 1];
#pragma unroll
        for (int j = 0; j <= QW; ++j)
            r[j] = (j <= (int)nw && w0 + j < total) ? ld_u64(s + w0 + j) : 0ull;
#pragma unroll
        for (int j = 0; j < QW; ++j)
            w[j] = j < (int)nw ? (sh ? (r[j] << sh) | (r[j + 1] >> (64 - sh)) : r[j]) : 0ull;
    }
    __device__ __forceinline__ uint64_t first() const { return w[0]; }
    __device__ __forceinline__ uint64_t word(int j) const { return j < QW ? w[j] : 0ull; }
};
// Long reads: words 0..4 (the k-mer, the record-cached bases and the first text word) are kept in
// registers; the rest is read from the row in 4-word chunks (one 256-bit load when the row is
// 32-byte aligned and the stride a multiple of 4 words) as the text compare reaches it.
#ifndef SA_QW0_HEAD
#define SA_QW0_HEAD 5  // words of a long read kept in registers (A/B builds: variants/)
#endif
template <>
struct QueryWords<0> {
    static constexpr int kHead = SA_QW0_HEAD;
    const uint64_t *p;
    uint32_t nw;
    unsigned sh = 0;     // dense layout: bit shift of the read inside its first word
    uint64_t left = ~0ull;  // dense layout: words readable from p
    bool vec = false;    // chunk c = one 256-bit load at p + 4c
    uint64_t h[kHead];   // words 0..4
    __device__ __forceinline__ void fill_head() {
#pragma unroll
        for (int j = 0; j < kHead; ++j) h[j] = gword((uint32_t)j);
    }
    // (the large-batch row hint of QueryWords<QW> is not used here: L1::no_allocate.L2::64B on the row
    // words of 150-250-base reads measured 9.90 / 10.37 vs 8.24 / 8.55 ms per 50 M reads -- their words
    // are read more than once -- profiles/r02/r02ai)
    __device__ __forceinline__ void load(const uint64_t *__restrict__ q, uint32_t n, bool v, bool = false) {
        p = q;
        nw = n;
        vec = v;
        fill_head();
    }
    __device__ __forceinline__ void load_dense(const uint64_t *__restrict__ s, uint64_t bit, uint32_t n, uint64_t total) {
        p = s + (bit >> 6);
        sh = (unsigned)(bit & 63);
        nw = n;
        left = total - (bit >> 6);
        fill_head();
    }
    __device__ __forceinline__ uint64_t raw(uint64_t j) const {
        return j < left ? ld_u64(p + j) : 0ull;
    }
    __device__ __forceinline__ uint64_t gword(uint32_t j) const {
        if (j >= nw) return 0ull;
        return sh ? (raw(j) << sh) | (raw(j + 1) >> (64 - sh)) : raw(j);
    }
    __device__ __forceinline__ uint64_t word(int j) const { return j < kHead ? h[j] : gword((uint32_t)j); }
    // words 4c .. 4c+3 (0 past the read)
    __device__ __forceinline__ void chunk(uint32_t c, uint64_t (&w)[4]) const {
        if (vec && 4 * c + 3 < nw) {
            ld_v4u64(p + 4 * c, w[0], w[1], w[2], w[3]);
            return;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) w[u] = gword(4 * c + u);
    }
    __device__ __forceinline__ uint64_t first() const { return h[0]; }
    // words j .. nw-1 of the row into L2 (TMA bulk prefetch)
    __device__ __forceinline__ void prefetch_rows(uint32_t j) const {
        if (j < nw) {
            const uint64_t last = sh ? nw : nw - 1;  // (dense: one more word for the shift)
            if (j < left) bulk_prefetch_l2(p + j, ((last < left ? last : left - 1) + 1 - j) * 8);
        }
    }
};

// ---- compare against the packed text --------------------------------------------------------
// One 32-base step: word j of P against the text at s + 32j.  Returns true when decided.
__device__ __forceinline__ bool cmp_text_word(const uint64_t *__restrict__ text, uint64_t s, uint64_t slen, uint32_t m,
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
            return true;
        }
    }
    if (L < plen) {  // the suffix ended first: it is a proper prefix of P (reading A7)
        lcp = base + L;
        sign = 1;
        return true;
    }
    return false;
}

// cmp_text_word with the 32-base text window at s + 32j already loaded (tw)
__device__ __forceinline__ bool cmp_word_window(uint64_t slen, uint32_t m, uint32_t j, uint64_t pw, uint64_t tw,
                                                int &sign, uint32_t &lcp) {
    const uint32_t base = j << 5;
    const uint32_t plen = min(32u, m - base);
    const uint64_t rem = slen > base ? slen - base : 0;
    const uint32_t L = rem < plen ? (uint32_t)rem : plen;
    if (L) {
        const uint64_t mask = prefix_mask(L);
        const uint64_t a = pw & mask, b = tw & mask;
        if (a != b) {
            lcp = base + ((uint32_t)__clzll((long long)(a ^ b)) >> 1);
            sign = a > b ? 1 : -1;
            return true;
        }
    }
    if (L < plen) {
        lcp = base + L;
        sign = 1;
        return true;
    }
    return false;
}

// four consecutive 32-base windows of the text from base b (b < n): text words w0 .. w0+4 from three
// 16-byte loads (w0 <= ceil(n/32)-1, so the last word read is inside the zero guard words)
__device__ __forceinline__ void text_windows4(const uint64_t *__restrict__ text, uint64_t b, uint64_t (&tw)[4]) {
    const uint64_t w0 = b >> 5;
    const uint64_t a = w0 & ~1ull;
    uint64_t x[6];
    ld_v2u64(text + a, x[0], x[1]);
    ld_v2u64(text + a + 2, x[2], x[3]);
    ld_v2u64(text + a + 4, x[4], x[5]);
    const bool odd = (w0 & 1) != 0;
    uint64_t r[5];
#pragma unroll
    for (int u = 0; u < 5; ++u) r[u] = odd ? x[u + 1] : x[u];
    const unsigned sh = (unsigned)(b & 31u) << 1;
#pragma unroll
    for (int u = 0; u < 4; ++u) tw[u] = sh ? (r[u] << sh) | (r[u + 1] >> (64u - sh)) : r[u];
}

// sign(P - t_s), t_s = S[s .. min(s+m, n)), comparing from word skip/32 on; lcp = lcp(P, t_s).
template <int QW>
__device__ __forceinline__ void compare_text(const uint64_t *__restrict__ text, uint64_t n, uint64_t s,
                                             const QueryWords<QW> &P, uint32_t m, uint32_t skip, int &sign,
                                             uint32_t &lcp) {
    const uint64_t slen = n - s;
    const uint32_t nw = (m + 31) >> 5;
    const uint32_t j0 = skip >> 5;
    if constexpr (QW > 0) {
#pragma unroll
        for (int j = 0; j < QW; ++j) {
            if ((uint32_t)j >= j0 && (uint32_t)j < nw) {
                if (cmp_text_word(text, s, slen, m, (uint32_t)j, P.w[j], sign, lcp)) return;
            }
        }
    } else {
        if (nw <= j0 + 2) {  // one or two words left (e.g. bases 128..149 of a 150-base read past rec32's
                             // cache): word by word, no 4-window load (profiles/r01-3/l_*: 10% at m = 150)
            for (uint32_t j = j0; j < nw; ++j)  // (gword: the row word from L1, not a dynamic index into h)
                if (cmp_text_word(text, s, slen, m, j, P.gword(j), sign, lcp)) return;
            sign = 0;
            lcp = m;
            return;
        }
        // 4 words per step: the read chunk and four text windows are loaded together (vector loads),
        // so a long verification is ~m/128 dependent round trips instead of ~m/32.  (SA_BULK_PREFETCH:
        // once 128 bases are known equal, the rest of the text window and of the read row are brought
        // into L2 by one TMA bulk prefetch each -- measured slower, kept as an A/B build.)
        bool fetched = false;
        auto prefetch_rest = [&](uint32_t jfrom) {
            if (fetched) return;
            fetched = true;
            const uint64_t b0 = s + 32ull * jfrom;                  // first base still to compare
            const uint64_t b1 = s + (m < slen ? (uint64_t)m : slen);  // past the last one
            if (b1 > b0) bulk_prefetch_l2(text + (b0 >> 5), (((b1 + 31) >> 5) + 1 - (b0 >> 5)) * 8);
            P.prefetch_rows(jfrom);
        };
#ifdef SA_BULK_PREFETCH  // A/B build only: measured slower (r02b: m = 500 +18%, m = 1000 +7%)
        if (j0 >= 4) prefetch_rest(j0);
#endif
#ifdef SA_CHUNK2  // A/B build: two chunks (8 words, 256 bases) loaded per round trip
        for (uint32_t c = j0 >> 2; 4 * c < nw; c += 2) {
            uint64_t pa[4], pb[4] = {0, 0, 0, 0}, ta[4] = {0, 0, 0, 0}, tb[4] = {0, 0, 0, 0};
            P.chunk(c, pa);
            const bool two = 4 * (c + 1) < nw;
            if (two) P.chunk(c + 1, pb);
            if (128ull * c < slen) text_windows4(text, s + 128ull * c, ta);
            if (two && 128ull * (c + 1) < slen) text_windows4(text, s + 128ull * (c + 1), tb);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t j = 4 * c + u;
                if (j >= j0 && j < nw && cmp_word_window(slen, m, j, pa[u], ta[u], sign, lcp)) return;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t j = 4 * c + 4 + u;
                if (j >= j0 && j < nw && cmp_word_window(slen, m, j, pb[u], tb[u], sign, lcp)) return;
            }
        }
#else
        for (uint32_t c = j0 >> 2; 4 * c < nw; ++c) {
#ifdef SA_BULK_PREFETCH
            if (4 * c > j0) prefetch_rest(4 * c);
#endif
            uint64_t pw[4], tw[4] = {0, 0, 0, 0};
            P.chunk(c, pw);
            if (128ull * c < slen) text_windows4(text, s + 128ull * c, tw);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint32_t j = 4 * c + u;
                if (j >= j0 && j < nw && cmp_word_window(slen, m, j, pw[u], tw[u], sign, lcp)) return;
            }
        }
#endif
    }
    sign = 0;
    lcp = m;
}

// ---- SA records ---------------------------------------------------------------------------------
// L_REC16: uint4 {SA, bases k+32..k+47 (high half), bases k..k+31 (lo, hi)}               -> 48 bases
// L_REC32: uint4 {SA, bases k+96..k+111 (high half), bases k..k+31 (lo, hi)},
//          uint4 {bases k+32..k+63 (lo, hi), bases k+64..k+95 (lo, hi)}                   -> 112 bases
template <int L>
struct Rec {
    static constexpr int kWords = (L == L_REC32) ? 4 : 2;             // 64-bit cache words
    static constexpr uint32_t kBases = (L == L_REC32) ? 112u : 48u;   // cached bases
    static constexpr int kU4 = (L == L_REC32) ? 2 : 1;                 // uint4 per record
    uint32_t sa;
    uint64_t c[kWords];  // c[j] = bases k+32j .. k+32j+31 (the last word holds 16)
    // a record staged in shared memory (k_match_tree)
    __device__ __forceinline__ void load_shared(const uint4 *s) {
        if constexpr (L == L_REC32) {
            const ulonglong2 x = reinterpret_cast<const ulonglong2 *>(s)[0];
            const ulonglong2 y = reinterpret_cast<const ulonglong2 *>(s)[1];
            sa = (uint32_t)x.x;
            c[0] = x.y;
            c[1] = y.x;
            c[2] = y.y;
            c[3] = x.x & 0xFFFFFFFF00000000ull;
        } else {
            const uint4 v = s[0];
            sa = v.x;
            c[0] = ((uint64_t)v.w << 32) | v.z;
            c[1] = (uint64_t)v.y << 32;
        }
    }
    __device__ __forceinline__ void load(const uint4 *__restrict__ rec, uint64_t p) {
        if constexpr (L == L_REC32) {
            uint64_t w0, w1, w2, w3;
            // one 256-bit load (LDG.E.ENL2.256 on sm_100a): the whole 32-byte record, one sector
            ld_v4u64(rec + 2 * p, w0, w1, w2, w3);
            sa = (uint32_t)w0;
            c[0] = w1;
            c[1] = w2;
            c[2] = w3;
            c[3] = w0 & 0xFFFFFFFF00000000ull;
        } else {
            const uint4 a = ld_v4u32(rec + p);
            sa = a.x;
            c[0] = ((uint64_t)a.w << 32) | a.z;
            c[1] = (uint64_t)a.y << 32;
        }
    }
};

// T[x] and T[x+1]: one aligned 16-byte load unless x sits in the last slot of its 16-byte group.
__device__ __forceinline__ void table_pair(const uint32_t *__restrict__ T, uint64_t x, uint32_t &a, uint32_t &b,
                                           bool wide = false) {
    const uint4 v = ld_tab_v4u32(T + (x & ~3ull), wide);
    switch (x & 3) {
    case 0: a = v.x; b = v.y; break;
    case 1: a = v.y; b = v.z; break;
    case 2: a = v.z; b = v.w; break;
    default: a = v.w; b = ld_u32(T + x + 1); break;
    }
}

// Bases k+32j .. k+32j+31 of P (k < 32).
template <int QW>
__device__ __forceinline__ uint64_t read_after_k(const QueryWords<QW> &P, uint32_t k, int j) {
    return (P.word(j) << (2 * k)) | (P.word(j + 1) >> (64 - 2 * k));
}

template <int QW>
__device__ __forceinline__ uint64_t after_k0(const QueryWords<QW> &P, uint32_t k) { return read_after_k<QW>(P, k, 0); }

// Compare P (m >= k, inside its k-mer bracket) with the suffix of a record.  Every suffix with >= k
// bases in the bracket starts with P's k-mer, so the compare starts at base k on the cached bases;
// the text is read only when all cached bases are equal and more remain, or for the < k suffixes
// shorter than k (which can sit at the end of a bracket without sharing its k-mer).
template <int QW, int L>
__device__ __forceinline__ void compare_rec(const MatchArgs &a, const Rec<L> &r, const QueryWords<QW> &P, uint32_t m,
                                            uint32_t skip, int &sign, uint32_t &lcp, uint32_t &texts) {
    const uint32_t k = a.k;
    const uint64_t s = r.sa, len = a.n - s;
    constexpr uint32_t CB = Rec<L>::kBases;
    if (len < k || skip >= k + CB) {
        ++texts;
        compare_text<QW>(a.text, a.n, s, P, m, len < k ? 0u : skip, sign, lcp);
        return;
    }
    const uint32_t avail = (uint32_t)((m < len ? (uint64_t)m : len) - k);  // bases after k present in both
#pragma unroll
    for (int j = 0; j < Rec<L>::kWords; ++j) {
        const uint32_t base = 32u * j;
        if (base < avail) {
            const uint32_t Lj = min(min(32u, avail - base), CB - base);
            const uint64_t mask = prefix_mask(Lj);
            const uint64_t x = read_after_k<QW>(P, k, j) & mask, y = r.c[j] & mask;
            if (x != y) {
                lcp = k + base + ((uint32_t)__clzll((long long)(x ^ y)) >> 1);
                sign = x > y ? 1 : -1;
                return;
            }
        }
    }
    if (avail > CB) {
        ++texts;
        compare_text<QW>(a.text, a.n, s, P, m, k + CB, sign, lcp);
        return;
    }
    // every base present in both is equal
    if (m <= len) { sign = 0; lcp = m; }            // P is a prefix of the suffix (case 1)
    else { sign = 1; lcp = (uint32_t)len; }          // the suffix is a proper prefix of P (reading A7)
}

// A probe of pivot p, split into its load (issued early) and its compare (sign(P - t_SA[p]), lcp).
// in_bracket: P has >= k bases and the pivot lies inside its k-mer bracket, so a record's cache applies.
template <int L>
struct Probe {
    Rec<L> r;
    __device__ __forceinline__ void load(const MatchArgs &a, uint64_t p) { r.load(a.rec, p); }
    __device__ __forceinline__ uint64_t sa() const { return r.sa; }
};
template <>
struct Probe<L_PLAIN> {
    uint64_t s;
    __device__ __forceinline__ void load(const MatchArgs &a, uint64_t p) { s = ld_u32(a.sa + p); }
    __device__ __forceinline__ uint64_t sa() const { return s; }
};

template <int QW, int L>
__device__ __forceinline__ void compare_probe(const MatchArgs &a, const Probe<L> &pr, const QueryWords<QW> &P,
                                              uint32_t m, uint32_t skip, bool in_bracket, int &sign, uint32_t &lcp,
                                              uint32_t &texts) {
    if constexpr (L == L_PLAIN) {
        ++texts;
        compare_text<QW>(a.text, a.n, pr.s, P, m, skip, sign, lcp);
    } else {
        if (in_bracket) {
            compare_rec<QW, L>(a, pr.r, P, m, skip, sign, lcp, texts);
        } else {
            ++texts;
            compare_text<QW>(a.text, a.n, pr.r.sa, P, m, skip, sign, lcp);
        }
    }
}

// ---- group-cooperative reads (long reads, m > 128) ---------------------------------------------
// G lanes (8, 16 or 32) hold one read: word j of P sits in lane j % G (WPL words per lane in
// registers; WPL == 0: read from global memory when needed).  One compare step covers G words (32·G
// bases): every lane compares its own word with the text (adjacent lanes, adjacent text words: one
// coalesced request), __ballot_sync over the group finds the first differing word and __shfl_sync
// broadcasts its lcp and sign (north_star's warp-cooperative compare).  A 1000-base compare is one
// round trip instead of ~30 dependent ones; the search's control state stays uniform in the group.
template <int G, int WPL>
struct GroupRead {
    static constexpr int kRegs = WPL > 0 ? WPL : 1;
    uint64_t w[kRegs];       // w[i] = word lane + G*i of P (0 past the read)
    uint64_t w0, w1;         // words 0 and 1, in every lane
    const uint64_t *p;       // the row
    unsigned sh;             // dense layout: bit shift of the read inside its first word
    uint64_t left;           // dense layout: words readable from p
    uint32_t nw;             // words of the read
    unsigned lane, base, mask;  // lane in the group, the group's first lane in the warp, its lane mask

    __device__ __forceinline__ uint64_t raw(uint64_t j) const { return j < left ? ld_u64(p + j) : 0ull; }
    __device__ __forceinline__ uint64_t gword(uint32_t j) const {
        if (j >= nw) return 0ull;
        return sh ? (raw(j) << sh) | (raw(j + 1) >> (64 - sh)) : raw(j);
    }
    __device__ __forceinline__ uint64_t own(int i) const {  // word lane + G*i
        if constexpr (WPL > 0) return w[i];
        else return gword(lane + G * (uint32_t)i);
    }
    __device__ __forceinline__ void init(const uint64_t *row, unsigned shift, uint64_t readable, uint32_t n) {
        p = row;
        sh = shift;
        left = readable;
        nw = n;
        lane = threadIdx.x & (G - 1);
        base = (threadIdx.x & 31) & ~(G - 1);
        mask = G == 32 ? 0xFFFFFFFFu : (((1u << (G & 31)) - 1) << base);
#pragma unroll
        for (int i = 0; i < kRegs; ++i) w[i] = gword(lane + G * i);
        w0 = __shfl_sync(mask, w[0], 0, G);
        w1 = __shfl_sync(mask, w[0], 1, G);
    }
    __device__ __forceinline__ uint64_t first() const { return w0; }
    // the first lane of the group with pred set, -1 if none
    __device__ __forceinline__ int first_lane(bool pred) const {
        unsigned b = __ballot_sync(mask, pred) >> base;
        if constexpr (G < 32) b &= (1u << G) - 1;
        return b ? __ffs(b) - 1 : -1;
    }
    __device__ __forceinline__ void take(int f, int sg, uint32_t lc, int &sign, uint32_t &lcp) const {
        sign = __shfl_sync(mask, sg, f, G);
        lcp = __shfl_sync(mask, lc, f, G);
    }
};

template <int G, int WPL>
__device__ __forceinline__ uint64_t after_k0(const GroupRead<G, WPL> &P, uint32_t k) {
    return (P.w0 << (2 * k)) | (P.w1 >> (64 - 2 * k));
}

// sign(P - t_s) and lcp, from word skip/32 on, G words per step
template <int G, int WPL>
__device__ __forceinline__ void gcompare_text(const uint64_t *__restrict__ text, uint64_t n, uint64_t s,
                                              const GroupRead<G, WPL> &P, uint32_t m, uint32_t skip, int &sign,
                                              uint32_t &lcp) {
    const uint64_t slen = n - s;
    const uint32_t nw = (m + 31) >> 5;
    const uint32_t j0 = skip >> 5;
    auto step = [&](int i, bool &done) {
        const uint32_t j = P.lane + G * (uint32_t)i;
        int sg = 0;
        uint32_t lc = 0;
        bool dec = false;
        if (j >= j0 && j < nw) dec = cmp_text_word(text, s, slen, m, j, P.own(i), sg, lc);
        const int f = P.first_lane(dec);
        if (f >= 0) {
            P.take(f, sg, lc, sign, lcp);
            done = true;
        }
    };
    bool done = false;
    if constexpr (WPL > 0) {
#pragma unroll
        for (int i = 0; i < WPL; ++i) {
            if (G * (uint32_t)(i + 1) <= j0) continue;
            if (G * (uint32_t)i >= nw) break;
            step(i, done);
            if (done) return;
        }
    } else {
        for (uint32_t i = j0 / G; G * i < nw; ++i) {
            step((int)i, done);
            if (done) return;
        }
    }
    sign = 0;
    lcp = m;
}

// the record compare of compare_rec: lane j < kWords takes cached word j (bases k+32j ..) against
// P's bases k+32j .. (its own word and the next lane's)
template <int G, int WPL, int L>
__device__ __forceinline__ void gcompare_rec(const MatchArgs &a, const Rec<L> &r, const GroupRead<G, WPL> &P,
                                             uint32_t m, uint32_t skip, int &sign, uint32_t &lcp, uint32_t &texts) {
    const uint32_t k = a.k;
    const uint64_t s = r.sa, len = a.n - s;
    constexpr uint32_t CB = Rec<L>::kBases;
    if (len < k || skip >= k + CB) {
        ++texts;
        gcompare_text(a.text, a.n, s, P, m, len < k ? 0u : skip, sign, lcp);
        return;
    }
    const uint32_t avail = (uint32_t)((m < len ? (uint64_t)m : len) - k);
    const uint64_t mine = P.own(0);
    const uint64_t next = __shfl_down_sync(P.mask, mine, 1, G);
    const uint32_t j = P.lane;
    int sg = 0;
    uint32_t lc = 0;
    bool dec = false;
    if (j < (uint32_t)Rec<L>::kWords && 32u * j < avail) {
        const uint32_t b = 32u * j;
        uint64_t c = r.c[0];
#pragma unroll
        for (int u = 1; u < Rec<L>::kWords; ++u)
            if (j == (uint32_t)u) c = r.c[u];
        const uint64_t msk = prefix_mask(min(min(32u, avail - b), CB - b));
        const uint64_t x = ((mine << (2 * k)) | (next >> (64 - 2 * k))) & msk, y = c & msk;
        if (x != y) {
            dec = true;
            lc = k + b + ((uint32_t)__clzll((long long)(x ^ y)) >> 1);
            sg = x > y ? 1 : -1;
        }
    }
    const int f = P.first_lane(dec);
    if (f >= 0) {
        P.take(f, sg, lc, sign, lcp);
        return;
    }
    if (avail > CB) {
        ++texts;
        gcompare_text(a.text, a.n, s, P, m, k + CB, sign, lcp);
        return;
    }
    if (m <= len) { sign = 0; lcp = m; }            // P is a prefix of the suffix (case 1)
    else { sign = 1; lcp = (uint32_t)len; }          // the suffix is a proper prefix of P (reading A7)
}

template <int G, int WPL, int L>
__device__ __forceinline__ void compare_probe(const MatchArgs &a, const Probe<L> &pr, const GroupRead<G, WPL> &P,
                                              uint32_t m, uint32_t skip, bool in_bracket, int &sign, uint32_t &lcp,
                                              uint32_t &texts) {
    if constexpr (L == L_PLAIN) {
        ++texts;
        gcompare_text(a.text, a.n, pr.s, P, m, skip, sign, lcp);
    } else {
        if (in_bracket) {
            gcompare_rec(a, pr.r, P, m, skip, sign, lcp, texts);
        } else {
            ++texts;
            gcompare_text(a.text, a.n, pr.r.sa, P, m, skip, sign, lcp);
        }
    }
}

// SA_INDEX_BUCKET_TREE: a large bucket's binary search is an implicit tree (BFS node i: root 1, children
// 2i, 2i+1 -- the probes of search_read and bound ARE its nodes); nodes above depth `depth` have their
// records copied into lines of three (a node at even depth and its two children)
struct TreeLoc {
    uint64_t line0;  // the bucket's first line
    uint32_t depth;  // levels stored (2E); 0 = no tree
};

__device__ __forceinline__ uint64_t tree_rec(const TreeLoc &tl, uint32_t i) {  // record index (32-byte units)
    const uint32_t r = (ilog2_u32(i) & 1) ? (i >> 1) : i;
    const uint32_t slot = i == r ? 0u : 1u + (i & 1u);
    return (tl.line0 + tree_line(r)) * 4 + slot;
}

// the node's child after a probe (0: past the stored levels, or no tree)
__device__ __forceinline__ uint32_t tree_child(const TreeLoc &tl, uint32_t node, bool left) {
    if (!node) return 0;
    const uint32_t c = 2 * node + (left ? 0u : 1u);
    return c < (1u << tl.depth) ? c : 0u;
}

// (returns the pivot's suffix position SA[p])
template <int L, class RD>
__device__ __forceinline__ uint64_t probe(const MatchArgs &a, const RD &P, uint32_t m, uint64_t p,
                                          uint32_t skip, bool in_bracket, int &sign, uint32_t &lcp, uint32_t &texts,
                                          const TreeLoc &tl = TreeLoc{0, 0}, uint32_t node = 0) {
    Probe<L> pr;
    if constexpr (L == L_REC32) {
        if (node) pr.r.load(a.tree, tree_rec(tl, node));  // the same record, from the bucket's tree
        else pr.load(a, p);
    } else {
        pr.load(a, p);
    }
    compare_probe(a, pr, P, m, skip, in_bracket, sign, lcp, texts);
    return pr.sa();
}

// Binary search over (Lp1-1, R): LB rule (lower: R moves when P <= t) or RB rule (R moves when P < t).
// SA_MATCH_STATS: the algorithmic bytes of one probe (SURVEY.md Sec. 8(d) "useful bytes"): the 4-byte SA
// entry plus the bases that decide the compare, from the known common prefix `skip` up to and including
// the first difference (all m - skip bases when P is a prefix of the suffix), 2 bits each.
__device__ __forceinline__ uint32_t probe_bytes(uint32_t m, uint32_t skip, uint32_t lcp) {
    const uint32_t end = lcp + 1 < m ? lcp + 1 : m;
    return 4u + (end > skip ? (end - skip + 3) >> 2 : 0u);
}

template <int L, class RD>
__device__ __forceinline__ uint32_t bound(const MatchArgs &a, const RD &P, uint32_t m, uint32_t Lp1,
                                          uint32_t R, uint32_t lcpL, uint32_t lcpR, bool lower, bool in_bracket,
                                          uint32_t &steps, uint32_t &texts, uint32_t &ubytes,
                                          const TreeLoc &tl = TreeLoc{0, 0}, uint32_t node = 0) {
    while (R > Lp1) {
        const uint32_t p = (uint32_t)(((uint64_t)Lp1 - 1 + R) >> 1);
        int sign;
        uint32_t lcp;
        const uint32_t skip = min(lcpL, lcpR);
        probe<L>(a, P, m, p, skip, in_bracket, sign, lcp, texts, tl, node);
        ++steps;
        ubytes += probe_bytes(m, skip, lcp);
        const bool left = sign < 0 || (lower && sign == 0);
        if (left) { R = p; lcpR = lcp; } else { Lp1 = p + 1; lcpL = lcp; }
        node = tree_child(tl, node, left);
    }
    return R;
}

// ---- the shared-memory top tree (SA_MATCH_SMEM_TREE, k_match_tree) ----------------------------
// The first `levels` levels of the binary search over a CTA's rank range (Lp1 - 1, R): BFS node i
// (1-based) holds the record of its pivot, staged in shared memory by TMA bulk copies.
struct TreeCtx {
    const uint4 *nodes;   // shared: node i at nodes[(i - 1) * kU4]
    uint32_t Lp1, R;      // the root's range
    uint32_t levels;
};

// Walk the tree with the read's own search state (Lp1 - 1, R): a node's pivot inside that interval is
// a probe that costs no DRAM access; the walk follows the side that still holds the interval.  Returns
// true at the split (P a prefix of the pivot's suffix), with the RB search's start state set.
template <int L, class RD>
__device__ __forceinline__ bool tree_descent(const MatchArgs &a, const TreeCtx &tc, const RD &P, uint32_t m,
                                             uint32_t &Lp1, uint32_t &R, uint32_t &lcpL, uint32_t &lcpR,
                                             uint32_t &hLp1, uint32_t &hR, uint32_t &hlcpL, uint32_t &hlcpR,
                                             uint32_t &steps, uint32_t &texts) {
    uint32_t tL = tc.Lp1, tR = tc.R, node = 1;
    for (uint32_t d = 0; d < tc.levels && tR > tL; ++d) {
        const uint32_t p = (uint32_t)(((uint64_t)tL - 1 + tR) >> 1);
        if (p >= Lp1 && p < R) {
            Probe<L> pr;
            pr.r.load_shared(tc.nodes + (uint64_t)(node - 1) * Rec<L>::kU4);
            int sign;
            uint32_t lcp;
            compare_probe(a, pr, P, m, min(lcpL, lcpR), true, sign, lcp, texts);
            ++steps;
            if (sign == 0) {
                hLp1 = p + 1; hR = R; hlcpL = lcp; hlcpR = lcpR;
                R = p; lcpR = lcp;
                return true;
            }
            if (sign < 0) { R = p; lcpR = lcp; } else { Lp1 = p + 1; lcpL = lcp; }
        }
        if (R <= p) { tR = p; node = 2 * node; } else { tL = p + 1; node = 2 * node + 1; }
    }
    return false;
}

template <int L, bool TREE, class RD>
__device__ __forceinline__ void joint_search(const MatchArgs &a, const RD &P, uint32_t m, uint32_t Lp1, uint32_t R,
                                             uint32_t lcp0, const TreeLoc &tl, uint32_t node, uint32_t &lo,
                                             uint32_t &hi, uint32_t &steps, uint32_t &texts, uint32_t &ubytes,
                                             const TreeCtx *tc, uint32_t *split_sa = nullptr);

// One read: [lo, hi).  L is carried as L+1 (Lp1) so every bound fits uint32.  BT: the index may have
// bucket trees (SA_INDEX_BUCKET_TREE; a separate instantiation keeps the default kernel's registers).
template <int L, bool TREE = false, bool BT = false, class RD>
__device__ __forceinline__ void search_read(const MatchArgs &a, const RD &P, uint32_t m, uint32_t &lo,
                                            uint32_t &hi, uint32_t &steps, uint32_t &texts, uint32_t &ubytes,
                                            const TreeCtx *tc = nullptr, uint32_t *split_sa = nullptr) {
    const uint32_t k = a.k;
    auto clamp = [&](uint32_t v) { return min(max(v, a.clo), a.chi); };
    if (m == 0) {  // the empty read is a prefix of every suffix (reading A12): [0, n), clamped
        lo = a.clo;
        hi = a.chi;
        return;
    }
    if (m < k) {
        // lo in [T[xa]-(k-m), T[xa]], hi in [T[xb]-(k-1), T[xb]], xa = x.a^(k-m), xb = (x+1).a^(k-m)
        // (DESIGN.md "Bracket, short reads"); each searched over (T[.]-k-1, T[.]).  A partition answers a
        // read shorter than its route key with the route-level table T_r (the same rule at rb bases).
        const bool rt = m < a.route_bases;
        const uint32_t kk = rt ? a.route_bases : k;
        const uint32_t *T = rt ? a.route : a.table;
        const uint64_t x = P.first() >> (64 - 2 * m);
        const uint32_t Ta = ld_u32(T + (x << (2 * (kk - m))));
        const uint32_t Tb = ld_u32(T + ((x + 1) << (2 * (kk - m))));
        ubytes += 8;  // the two table entries
        lo = bound<L>(a, P, m, clamp(Ta > kk ? Ta - kk : 0), clamp(Ta), 0, 0, true, false, steps, texts, ubytes);
        hi = bound<L>(a, P, m, clamp(Tb > kk ? Tb - kk : 0), clamp(Tb), 0, 0, false, false, steps, texts, ubytes);
        return;
    }
    // all suffixes before T[x] are < P, all from T[x+1] on are > P
    const uint64_t x = P.first() >> (64 - 2 * k);
    uint32_t Lp1, R;
    table_pair(a.table, x, Lp1, R, a.wide);
    Lp1 = clamp(Lp1);
    R = clamp(R);
    ubytes += 8;  // T[x], T[x+1]
    if (a.big_sub && R - Lp1 > kBigBucket && m >= k + 4) {
        // a large bucket (repeats): its (k+4)-base sub-table narrows the bracket by the next 4 bases
        const uint64_t mask = (1ull << a.big_bits) - 1;
        uint64_t h = (uint64_t)(((uint32_t)x * 0x9E3779B1u) >> (32 - a.big_bits));
        for (uint64_t tries = 0; tries <= mask; ++tries, h = (h + 1) & mask) {
            const uint64_t e = ld_u64(reinterpret_cast<const uint64_t *>(a.big_hash) + h);
            if (e == ~0ull) break;  // empty slot: x has no sub-table (tested before the key)
            if ((uint32_t)(e >> 32) == (uint32_t)x) {
                const uint32_t *T2 = a.big_sub + (uint64_t)(uint32_t)e * 257;
                const uint32_t y = (uint32_t)(after_k0(P, k) >> 56);  // bases k .. k+3
                Lp1 = ld_u32(T2 + y);
                R = ld_u32(T2 + y + 1);
                break;
            }
        }
    }
    TreeLoc tl{0, 0};  // SA_INDEX_BUCKET_TREE: a large bucket's line-packed top levels
    uint32_t node = 0;
    if (BT && !TREE && a.tree_hash && R - Lp1 >= kTreeMin) {
        const uint64_t mask = (1ull << a.tree_bits) - 1;
        uint64_t h = (uint64_t)(((uint32_t)x * 0x9E3779B1u) >> (32 - a.tree_bits));
        for (uint64_t tries = 0; tries <= mask; ++tries, h = (h + 1) & mask) {
            const uint64_t e = ld_u64(reinterpret_cast<const uint64_t *>(a.tree_hash) + h);
            if (e == ~0ull) break;
            if ((uint32_t)(e >> 32) == (uint32_t)x) {
                tl.line0 = (uint32_t)e;
                tl.depth = 2 * tree_pairs(R - Lp1);
                node = 1;
                break;
            }
        }
    }
    joint_search<L, TREE>(a, P, m, Lp1, R, 0, tl, node, lo, hi, steps, texts, ubytes, tc, split_sa);
}

// The joint lo/hi search over the bracket (Lp1 - 1, R) -- every suffix in it shares P's first lcp0
// bases (lcp0 = 0: only the bracket property is known) -- with the split of search_read.
template <int L, bool TREE, class RD>
__device__ __forceinline__ void joint_search(const MatchArgs &a, const RD &P, uint32_t m, uint32_t Lp1, uint32_t R,
                                             uint32_t lcp0, const TreeLoc &tl, uint32_t node, uint32_t &lo,
                                             uint32_t &hi, uint32_t &steps, uint32_t &texts, uint32_t &ubytes,
                                             const TreeCtx *tc, uint32_t *split_sa) {
    uint32_t lcpL = lcp0, lcpR = lcp0;
    uint32_t hLp1 = 0, hR = 0, hlcpL = 0, hlcpR = 0, hnode = 0;
    bool split = false;
    if constexpr (TREE) split = tree_descent<L>(a, *tc, P, m, Lp1, R, lcpL, lcpR, hLp1, hR, hlcpL, hlcpR, steps, texts);
    while (!split && R > Lp1) {  // LB rule until the first pivot where P is a prefix of the suffix (the split)
        const uint32_t p = (uint32_t)(((uint64_t)Lp1 - 1 + R) >> 1);
        int sign;
        uint32_t lcp;
        const uint32_t skip = min(lcpL, lcpR);
        const uint64_t sp = probe<L>(a, P, m, p, skip, true, sign, lcp, texts, tl, node);
        ++steps;
        ubytes += probe_bytes(m, skip, lcp);
        if (sign == 0) {  // lo lies in (L, p], hi in (p, R]: the RB search starts from here
            split = true;
            if (split_sa) *split_sa = (uint32_t)sp;  // (the staged long-read kernel: SA[p] of the split)
            hLp1 = p + 1; hR = R; hlcpL = lcp; hlcpR = lcpR;
            R = p; lcpR = lcp;
            hnode = tree_child(tl, node, false);
            node = tree_child(tl, node, true);
            break;
        }
        if (sign < 0) { R = p; lcpR = lcp; } else { Lp1 = p + 1; lcpL = lcp; }
        node = tree_child(tl, node, sign < 0);
    }
    if (!split) {  // no suffix has P as a prefix: an empty interval at the insertion point
        lo = hi = R;
        return;
    }
    // finish the LB search in (L, p], then the RB search in (p, R at the split].  (Interleaving the
    // two chains, both probes issued before either compare, measured 3% slower at C4: profiles/r01n.)
    lo = bound<L>(a, P, m, Lp1, R, lcpL, lcpR, true, true, steps, texts, ubytes, tl, node);
    hi = bound<L>(a, P, m, hLp1, hR, hlcpL, hlcpR, false, true, steps, texts, ubytes, tl, hnode);
}

__device__ __forceinline__ uint32_t read_len(const MatchArgs &a, uint64_t q) {
    if (a.stride == 0) return a.fixed_len;  // dense layout: fixed length
    // lengths past the stride are clamped (include/sa.h requires m <= 32*stride_words)
    return min(a.lens ? __ldg(a.lens + q) : a.fixed_len, 32u * a.stride);
}

template <int QW>
__device__ __forceinline__ void load_read(const MatchArgs &a, uint64_t row, uint32_t m, QueryWords<QW> &P) {
    if (a.stride == 0) P.load_dense(a.words, 2ull * m * row, (m + 31) >> 5, a.dense_words);
    else P.load(a.words + row * a.stride, (m + 31) >> 5, a.vec_rows, a.wide);
}

// One read per thread slot, all lanes of a warp in lock step (with sa_match_order the lanes hold
// lexicographically adjacent reads and walk neighbouring parts of the SA and table).  Measured and
// dropped on B200 at C4: a persistent lane-refilling variant (a finished lane takes the next read;
// profiles/r01b, r01c: it de-correlates the lanes' addresses), and a software-pipelined variant that
// prefetches the next read's row during the current search (profiles/r01t: 2% slower -- the kernel is
// bound by DRAM line throughput, not by the latency of the chain's head).
#ifndef SA_MATCH_THREADS
// block size of k_match (A/B builds: variants/).  64: a block retires as soon as its two warps finish, so a
// slow (repeat or long) read holds 64 thread slots instead of 256 -- k_match 9.97 vs 10.05 ms per 100 M
// reads, 1.40 vs 1.47 per 12.5 M, 2.68 vs 2.80 per 25 M, C5 m = 150 / 500 7.45 / 10.22 vs 8.16 / 10.79 per
// 50 M (profiles/r02/r02am, r02an; round 1's kernel had measured flat, profiles/r01-3/e_*)
#define SA_MATCH_THREADS 64
#endif
// minimum resident blocks per SM requested from ptxas (a register cap): 1280 threads per SM (20 x 64) =
// 62.5% occupancy = at most 48 registers, the plateau measured in r01-3 (profiles/r01-3/e_*: 40 registers
// spill and run slower, 64 registers (50%) run 9% slower; again with 64-thread blocks, profiles/r02/r02ap)
#ifndef SA_MATCH_MINB
#define SA_MATCH_MINB (1280 / SA_MATCH_THREADS)
#endif
// (the long-read instantiation, QW = 0: 1024 threads per SM = 64 registers, the r01 build's allocation)
#ifndef SA_MATCH_MINB_LONG
#define SA_MATCH_MINB_LONG (1024 / SA_MATCH_THREADS)
#endif
#define SA_MATCH_BOUNDS __launch_bounds__(SA_MATCH_THREADS, QW > 0 ? SA_MATCH_MINB : SA_MATCH_MINB_LONG)
template <int QW, int L, bool STATS, bool BT = false>
__global__ void SA_MATCH_BOUNDS k_match(const MatchArgs a) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.Q) return;
    uint64_t q = a.order ? (uint64_t)__ldg(a.order + t) : t;  // the read; its result goes to out[q]
    const uint64_t row = a.rows_ordered ? t : q;               // where its bases are
    const uint32_t m = read_len(a, row);
    QueryWords<QW> P;
    load_read<QW>(a, row, m, P);
    // ubytes (SA_MATCH_STATS): the read (2 bits/base) + the 8-byte result + what the search adds
    uint32_t lo, hi, steps = 0, texts = 0, ubytes = ((m + 3) >> 2) + 8;
    if constexpr (QW == 0 && L != L_PLAIN) {
        // Long reads in two phases.  (A) the search for P' = P's first mt = k + (cached bases) bases: the
        // records decide every probe, no text is read.  Its interval holds P's: [lo, hi) within
        // [lo', hi') (P' is a prefix of P).  (B) the joint search for P over [lo', hi'), where every
        // suffix shares P' (compares start at base mt): for a unique hit one probe, the verification of
        // P's remaining bases.  All lanes of a warp finish (A) before any starts (B), so the long
        // text compares of (B) run with the warp's lanes together instead of one by one (ncu r02c: the
        // one-phase kernel ran its text loop with 6 of 32 lanes active).
        const uint32_t mt = min(m, a.k + Rec<L>::kBases);
        // (A direct compare for a unique P' against (A)'s split pivot -- skipping the joint search's reload
        // of that record -- measured slower: 8.34 / 11.52 vs 8.16 / 10.87 ms per 50 M reads at m = 150 /
        // 500, profiles/r02/r02w: the unique and the repeat lanes of a warp then run apart.)
        search_read<L, false, BT>(a, P, mt, lo, hi, steps, texts, ubytes);
        __syncwarp();
        if (m > mt) {
            if (hi > lo) joint_search<L, false>(a, P, m, lo, hi, mt, TreeLoc{0, 0}, 0, lo, hi, steps, texts, ubytes,
                                                nullptr);
            else hi = lo;
        }
    } else {
        search_read<L, false, BT>(a, P, m, lo, hi, steps, texts, ubytes);
    }
    // Alg. 1 lines 44-45: res[thd<<1] = LB, res[(thd<<1)+1] = RB (reading A8), half-open here.
    // The read index is loaded again here (an L1 hit) rather than kept live across the search: at the
    // 48 registers of the 62.5%-occupancy build ptxas otherwise spills it to local memory.
    if (a.order) q = reload_u32(a.order + t);
#ifdef SA_OUT_PAD  // experiment: one full 32-byte sector per read (no ECC read-modify-write of a partial sector)
    reinterpret_cast<uint4 *>(a.out)[2 * q] = make_uint4(lo, hi, 0u, 0u);
    reinterpret_cast<uint4 *>(a.out)[2 * q + 1] = make_uint4(0u, 0u, 0u, 0u);
#else
    reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
#endif
    if (STATS) {
        a.stats[q] = min(steps, 0xFFFFu) | (min(texts, 0xFFFFu) << 16);
        a.stats[a.Q + q] = ubytes;
    }
}

// ---- deferred heavy reads (SA_MATCH_DEFER) -----------------------------------------------------
// The lanes of a warp search in lock step, so a warp takes as long as its slowest read: one read in a
// repeat bucket (10-60 probes) holds 31 finished lanes.  Two passes instead: k_match_light does every read
// whose k-mer bracket holds at most `big` suffixes (<= ~log2(big) + 2 probes) and appends the others --
// read index and bracket -- to a list (one atomic per warp, lane order kept, so the list stays roughly in
// key order); k_match_heavy then searches the listed reads with full warps, from the saved bracket.  The
// same search (search_read / joint_search), the same results.
template <int QW, int L>
__global__ void SA_MATCH_BOUNDS k_match_light(const MatchArgs a, uint32_t big, uint32_t *__restrict__ dq,
                                              uint2 *__restrict__ dbr, uint32_t *__restrict__ dcount) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= a.Q) return;
    const unsigned act = __activemask();
    uint64_t q = a.order ? (uint64_t)__ldg(a.order + t) : t;
    const uint64_t row = a.rows_ordered ? t : q;
    const uint32_t m = read_len(a, row);
    QueryWords<QW> P;
    load_read<QW>(a, row, m, P);
    uint32_t lo, hi, steps = 0, texts = 0, ubytes = 0;
    bool heavy = false;
    uint32_t Lp1 = 0, R = 0;
    if (m >= a.k && !a.big_sub && !a.tree_hash) {
        const uint64_t x = P.first() >> (64 - 2 * a.k);
        table_pair(a.table, x, Lp1, R);
        Lp1 = min(max(Lp1, a.clo), a.chi);
        R = min(max(R, a.clo), a.chi);
        heavy = R - Lp1 > big;
    }
    const unsigned hv = __ballot_sync(act, heavy);
    if (hv) {
        const unsigned lane = threadIdx.x & 31, leader = (unsigned)(__ffs(act) - 1);
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(dcount, (uint32_t)__popc(hv));
        base = __shfl_sync(act, base, (int)leader);
        if (heavy) {
            const uint32_t i = base + __popc(hv & ((1u << lane) - 1u));
            dq[i] = (uint32_t)q;
            dbr[i] = make_uint2(Lp1, R);
            return;
        }
    }
    if (m >= a.k && !a.big_sub && !a.tree_hash)
        joint_search<L, false>(a, P, m, Lp1, R, 0, TreeLoc{0, 0}, 0, lo, hi, steps, texts, ubytes, nullptr);
    else
        search_read<L>(a, P, m, lo, hi, steps, texts, ubytes);
    if (a.order) q = reload_u32(a.order + t);
    reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
}

// the listed reads (*dcount of them), grid-stride: slot i searches read dq[i] from bracket dbr[i]
template <int QW, int L>
__global__ void SA_MATCH_BOUNDS k_match_heavy(const MatchArgs a, const uint32_t *__restrict__ dq,
                                              const uint2 *__restrict__ dbr, const uint32_t *__restrict__ dcount) {
    const uint64_t cnt = *dcount;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t q = __ldg(dq + i);
        const uint2 br = __ldg(dbr + i);
        const uint32_t m = read_len(a, q);  // (rows_ordered is rejected with SA_MATCH_DEFER)
        QueryWords<QW> P;
        load_read<QW>(a, q, m, P);
        uint32_t lo, hi, steps = 0, texts = 0, ubytes = 0;
        joint_search<L, false>(a, P, m, br.x, br.y, 0, TreeLoc{0, 0}, 0, lo, hi, steps, texts, ubytes, nullptr);
        reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
    }
}

// k_match with the shared-memory top tree (north_star's "top levels of the SA
// binary-search tree staged in shared memory via TMA"; the B200 form of the paper's shared-memory
// tiles).  The reads are ordered (sa_match_order by key_bases bases), so a CTA's 256
// reads share one range of the suffix array: [T[first read's key], T[last read's key + 1]).  The
// CTA stages the records of the first `levels` levels of the binary search over that range into
// shared memory with one cp.async.bulk per record (mbarrier completion), and every read walks them
// (tree_descent) before its own DRAM probes.
template <int QW, int L>
__global__ void __launch_bounds__(256, 4) k_match_tree(const MatchArgs a, uint32_t levels, uint32_t key_bases) {
    extern __shared__ __align__(128) uint4 s_nodes[];
    __shared__ __align__(8) uint64_t s_bar;
    __shared__ uint32_t s_lo, s_hi;
    constexpr uint32_t U4 = Rec<L>::kU4;
    const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x;
    const uint64_t t = t0 + threadIdx.x;
    const uint32_t nodes = (1u << levels) - 1;
    const uint32_t bar = (uint32_t)__cvta_generic_to_shared(&s_bar);
    const uint32_t k = a.k, kb = key_bases;
    if (threadIdx.x == 0) {
        // the ordering keys of the block's first and last read
        auto key_of = [&](uint64_t slot) -> uint64_t {
            const uint64_t q = a.order ? (uint64_t)__ldg(a.order + slot) : slot;
            const uint64_t row = a.rows_ordered ? slot : q;
            const uint32_t m = read_len(a, row);
            uint64_t w0;
            if (a.stride == 0) {
                const uint64_t bit = 2ull * m * row, i = bit >> 6;
                const unsigned sh = (unsigned)(bit & 63);
                const uint64_t lo = ld_u64(a.words + i);
                const uint64_t hi = (sh && i + 1 < a.dense_words) ? ld_u64(a.words + i + 1) : 0ull;
                w0 = sh ? (lo << sh) | (hi >> (64 - sh)) : lo;
            } else {
                w0 = ld_u64(a.words + row * a.stride);
            }
            return (w0 & prefix_mask(min(m, kb))) >> (64 - 2 * kb);
        };
        const uint64_t kf = key_of(t0), kl = key_of(min(t0 + blockDim.x, a.Q) - 1);
        const uint64_t xlo = k >= kb ? kf << (2 * (k - kb)) : kf >> (2 * (kb - k));
        const uint64_t xhi = k >= kb ? (kl + 1) << (2 * (k - kb)) : (kl >> (2 * (kb - k))) + 1;
        s_lo = min(max(ld_u32(a.table + xlo), a.clo), a.chi);
        s_hi = min(max(ld_u32(a.table + xhi), a.clo), a.chi);
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nodes * U4 * 16u)
                     : "memory");
    }
    __syncthreads();
    const uint32_t tlo = s_lo, thi = s_hi;
    for (uint32_t i = threadIdx.x; i < nodes; i += blockDim.x) {
        // the pivot of BFS node i+1: its path from the root, the same midpoints tree_descent takes
        uint32_t Lp1 = tlo, R = thi;
        const uint32_t node = i + 1;
        for (int b = 30 - __clz(node); b >= 0; --b) {
            const uint32_t p = (uint32_t)(((uint64_t)Lp1 - 1 + R) >> 1);
            if ((node >> b) & 1) Lp1 = p + 1; else R = p;
        }
        uint64_t p = ((uint64_t)Lp1 - 1 + R) >> 1;
        if (p < a.clo) p = a.clo;  // (an empty node's copy is never compared; keep its address valid)
        if (p >= a.chi) p = a.chi - 1;
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(s_nodes + (uint64_t)i * U4);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(a.rec + p * U4), "r"(U4 * 16u), "r"(bar) : "memory");
    }
    if (t < a.Q) {
        uint64_t q = a.order ? (uint64_t)__ldg(a.order + t) : t;
        const uint64_t row = a.rows_ordered ? t : q;
        const uint32_t m = read_len(a, row);
        QueryWords<QW> P;
        load_read<QW>(a, row, m, P);
        uint32_t done = 0;  // the staged tree is complete (phase 0 of the barrier)
        while (!done) {
            asm volatile("{ .reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0; selp.u32 %0, 1, 0, P1; }"
                         : "=r"(done) : "r"(bar) : "memory");
        }
        const TreeCtx tc{s_nodes, tlo, thi, levels};
        // (ubytes: the staged records are the CTA's, not counted per read)
        uint32_t lo, hi, steps = 0, texts = 0, ubytes = ((m + 3) >> 2) + 8;
        if (m >= k) search_read<L, true>(a, P, m, lo, hi, steps, texts, ubytes, &tc);
        else search_read<L>(a, P, m, lo, hi, steps, texts, ubytes);
        if (a.order) q = reload_u32(a.order + t);
        reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
        if (a.stats) {
            a.stats[q] = min(steps, 0xFFFFu) | (min(texts, 0xFFFFu) << 16);
            a.stats[a.Q + q] = ubytes;
        }
    } else {  // (every thread of the block waits before the block's shared memory can go away)
        uint32_t done = 0;
        while (!done) {
            asm volatile("{ .reg .pred P1; mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0; selp.u32 %0, 1, 0, P1; }"
                         : "=r"(done) : "r"(bar) : "memory");
        }
    }
}

// Long reads (m > 128): G lanes per read slot (GroupRead), the same search as k_match.
template <int G, int WPL, int L, bool STATS>
__global__ void __launch_bounds__(256) k_match_group(const MatchArgs a) {
    const uint64_t t = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    if (t >= a.Q) return;  // whole groups leave together
    const uint64_t q = a.order ? (uint64_t)__ldg(a.order + t) : t;
    const uint64_t row = a.rows_ordered ? t : q;
    const uint32_t m = read_len(a, row);
    GroupRead<G, WPL> P;
    if (a.stride == 0) {
        const uint64_t bit = 2ull * m * row;
        P.init(a.words + (bit >> 6), (unsigned)(bit & 63), a.dense_words - (bit >> 6), (m + 31) >> 5);
    } else {
        P.init(a.words + row * a.stride, 0u, ~0ull, (m + 31) >> 5);
    }
    uint32_t lo, hi, steps = 0, texts = 0, ubytes = ((m + 3) >> 2) + 8;
    search_read<L>(a, P, m, lo, hi, steps, texts, ubytes);
    if (P.lane == 0) {
        reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
        if (STATS) {
            a.stats[q] = min(steps, 0xFFFFu) | (min(texts, 0xFFFFu) << 16);
            a.stats[a.Q + q] = ubytes;
        }
    }
}

}  // namespace sa_search
