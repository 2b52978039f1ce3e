// sa_search_long.cuh -- the search for long reads (more than 4 words, m > 128): the same result as
// sa_search.cuh's search_read (Alg. 1, corrected per DESIGN.md A4-A8; the joint lo/hi
// search, the k-mer bracket, the records), re-organised so that the long text compares -- the cost
// of a read of several hundred bases -- are done by the whole warp (north_star's warp-cooperative
// compare with __shfl / __ballot).
//
// Why: with one thread per read the verification of a 1000-base match is a per-lane loop of ~8 chunk
// steps, and the lanes of a warp reach it at different probes, so the loop ran with 6 of 32 lanes
// active on average and took 68% of the kernel's instructions (ncu, profiles/r02c: C5 m = 1000 was
// issue-bound, 57% issue-active, 1.8 TB/s of DRAM).  Here every lane still runs its own binary search,
// but one probe per lane per round, in warp lock step (an explicit state machine instead of nested
// loops).  A probe is decided by the record's cached bases when it can be; a lane that needs the text
// raises a request, and after each round the warp serves the requests one by one: lane l compares
// word j0 + l (32 bases) of the requesting read with the text, the first differing word is found with
// one ballot, and its lcp and sign go back with one shuffle -- 1024 bases per step, loads coalesced.
#pragma once

#include "sa_search.cuh"

namespace sa_search {

// the phases of one lane's search (sa_search.cuh's search_read, flattened)
enum : uint32_t {
    PH_DONE = 0,
    PH_DESC = 1,  // LB rule until the split (the first pivot with P a prefix of its suffix)
    PH_LO = 2,    // lower bound in (L, split]
    PH_HI = 3,    // upper bound in (split, R at the split]
    PH_SLO = 4,   // m < k: lower bound over the widened table window (no record cache)
    PH_SHI = 5,   // m < k: upper bound
};

// one warp-cooperative compare of (the read of lane `src`) against the suffix at s, from word j0 on:
// sign(P - t_s) and lcp (all lanes of the warp take part; the result is valid in every lane)
__device__ __forceinline__ void warp_compare_text(const uint64_t *__restrict__ text, uint64_t n, uint64_t s,
                                                  const uint64_t *__restrict__ rp, unsigned rsh, uint64_t rleft,
                                                  uint32_t m, uint32_t j0, unsigned lane, int &sign, uint32_t &lcp) {
    const uint64_t slen = n - s;
    const uint32_t nw = (m + 31) >> 5;
    for (uint32_t jb = j0; jb < nw; jb += 32) {
        const uint32_t j = jb + lane;
        const bool live = j < nw;       // lane compares word j
        const bool feeds = j <= nw;     // lane loads words for itself and for lane - 1 (the next raw word)
        // the read's word j: raw words j and j+1 of its row (the dense layout's shift needs both)
        const uint64_t r0 = (feeds && j < rleft) ? ld_u64(rp + j) : 0ull;
        uint64_t r1 = __shfl_down_sync(0xFFFFFFFFu, r0, 1);
        if (lane == 31 && rsh && live && j + 1 < rleft) r1 = ld_u64(rp + j + 1);
        const uint64_t pw = rsh ? (r0 << rsh) | (r1 >> (64 - rsh)) : r0;
        // the text's 32 bases at s + 32j: words w and w+1 of the packed text (bases past n read as 0:
        // base < slen + 32 keeps w within the zero guard words)
        const uint64_t base = 32ull * j;
        const uint64_t w = (s + base) >> 5;
        const bool inside = feeds && base < slen + 32;
        const uint64_t x0 = inside ? ld_u64(text + w) : 0ull;
        uint64_t x1 = __shfl_down_sync(0xFFFFFFFFu, x0, 1);
        const unsigned tsh = (unsigned)((s & 31u) << 1);
        if (lane == 31 && live && base < slen + 32 && tsh) x1 = ld_u64(text + w + 1);
        const uint64_t tw = tsh ? (x0 << tsh) | (x1 >> (64u - tsh)) : x0;
        int sg = 0;
        uint32_t lc = 0;
        const bool dec = live && cmp_word_window(slen, m, j, pw, tw, sg, lc);
        const unsigned b = __ballot_sync(0xFFFFFFFFu, dec);
        if (b) {
            const int f = __ffs(b) - 1;
            sign = __shfl_sync(0xFFFFFFFFu, sg, f);
            lcp = __shfl_sync(0xFFFFFFFFu, lc, f);
            return;
        }
    }
    sign = 0;
    lcp = m;
}

// The record part of a probe (compare_rec without its text fallback): returns true when the cached
// bases decide (sign, lcp); else `from` = the base from which the text must be compared.
template <int L>
__device__ __forceinline__ bool rec_decides(const MatchArgs &a, const Rec<L> &r, const QueryWords<0> &P, uint32_t m,
                                            uint32_t skip, int &sign, uint32_t &lcp, uint32_t &from) {
    const uint32_t k = a.k;
    const uint64_t s = r.sa, len = a.n - s;
    constexpr uint32_t CB = Rec<L>::kBases;
    if (len < k || skip >= k + CB) {
        from = len < k ? 0u : skip;
        return false;
    }
    const uint32_t avail = (uint32_t)((m < len ? (uint64_t)m : len) - k);
#pragma unroll
    for (int j = 0; j < Rec<L>::kWords; ++j) {
        const uint32_t base = 32u * j;
        if (base < avail) {
            const uint32_t Lj = min(min(32u, avail - base), CB - base);
            const uint64_t mask = prefix_mask(Lj);
            const uint64_t x = read_after_k<0>(P, k, j) & mask, y = r.c[j] & mask;
            if (x != y) {
                lcp = k + base + ((uint32_t)__clzll((long long)(x ^ y)) >> 1);
                sign = x > y ? 1 : -1;
                return true;
            }
        }
    }
    if (avail > CB) {
        from = k + CB;
        return false;
    }
    if (m <= len) { sign = 0; lcp = m; } else { sign = 1; lcp = (uint32_t)len; }
    return true;
}

// Long reads: one read per thread slot, every lane's search advanced one probe per round in warp lock
// step; text compares served by the whole warp (warp_compare_text).  Results equal k_match's.
template <int L, bool STATS>
#ifndef SA_LONG_MINB
#define SA_LONG_MINB 4  // 4 x 256 threads: 64 registers
#endif
__global__ void __launch_bounds__(256, SA_LONG_MINB) k_match_long(const MatchArgs a) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned lane = threadIdx.x & 31;
    const bool valid = t < a.Q;  // (lanes past Q stay to the end: the warp's collectives need all 32)
    uint64_t q = 0;
    uint32_t m = 0;
    QueryWords<0> P;  // (sh = 0, left = ~0 by default: the strided layout)
    P.p = a.words;
    P.nw = 0;
    if (valid) {
        q = a.order ? (uint64_t)__ldg(a.order + t) : t;
        const uint64_t row = a.rows_ordered ? t : q;
        m = read_len(a, row);
        load_read<0>(a, row, m, P);
    }
    const uint32_t k = a.k;
    auto clamp = [&](uint32_t v) { return min(max(v, a.clo), a.chi); };
    uint32_t phase = PH_DONE, lo = 0, hi = 0, steps = 0, texts = 0, ubytes = ((m + 3) >> 2) + 8;
    uint32_t Lp1 = 0, R = 0, lcpL = 0, lcpR = 0, hLp1 = 0, hR = 0, hlcpL = 0, hlcpR = 0;
    TreeLoc tl{0, 0};  // SA_INDEX_BUCKET_TREE (as search_read)
    uint32_t node = 0, hnode = 0;
    if (valid) {
        if (m == 0) {  // reading A12: [0, n), clamped
            lo = a.clo;
            hi = a.chi;
        } else if (m < k) {  // the widened windows of search_read (a partition: the route table below rb)
            const bool rt = m < a.route_bases;
            const uint32_t kk = rt ? a.route_bases : k;
            const uint32_t *T = rt ? a.route : a.table;
            const uint64_t x = P.first() >> (64 - 2 * m);
            const uint32_t Ta = ld_u32(T + (x << (2 * (kk - m))));
            const uint32_t Tb = ld_u32(T + ((x + 1) << (2 * (kk - m))));
            ubytes += 8;
            Lp1 = clamp(Ta > kk ? Ta - kk : 0);
            R = clamp(Ta);
            hLp1 = clamp(Tb > kk ? Tb - kk : 0);
            hR = clamp(Tb);
            phase = PH_SLO;
        } else {
            const uint64_t x = P.first() >> (64 - 2 * k);
            table_pair(a.table, x, Lp1, R);
            Lp1 = clamp(Lp1);
            R = clamp(R);
            ubytes += 8;
            if (a.big_sub && R - Lp1 > kBigBucket && m >= k + 4) {  // (SA_INDEX_SUBTABLE, as search_read)
                const uint64_t mask = (1ull << a.big_bits) - 1;
                uint64_t h = (uint64_t)(((uint32_t)x * 0x9E3779B1u) >> (32 - a.big_bits));
                for (uint64_t tries = 0; tries <= mask; ++tries, h = (h + 1) & mask) {
                    const uint64_t e = ld_u64(reinterpret_cast<const uint64_t *>(a.big_hash) + h);
                    if (e == ~0ull) break;
                    if ((uint32_t)(e >> 32) == (uint32_t)x) {
                        const uint32_t *T2 = a.big_sub + (uint64_t)(uint32_t)e * 257;
                        const uint32_t y = (uint32_t)(after_k0(P, k) >> 56);
                        Lp1 = ld_u32(T2 + y);
                        R = ld_u32(T2 + y + 1);
                        break;
                    }
                }
            }
            if (a.tree_hash && R - Lp1 >= kTreeMin) {
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
            phase = PH_DESC;
        }
    }
    while (true) {
        // phase transitions at an empty interval (no probe needed)
        while (phase != PH_DONE && R <= Lp1) {
            if (phase == PH_DESC) { lo = hi = R; phase = PH_DONE; }          // no split: the insertion point
            else if (phase == PH_LO) { lo = R; Lp1 = hLp1; R = hR; lcpL = hlcpL; lcpR = hlcpR; node = hnode; phase = PH_HI; }
            else if (phase == PH_SLO) { lo = R; Lp1 = hLp1; R = hR; lcpL = lcpR = 0; phase = PH_SHI; }
            else { hi = R; phase = PH_DONE; }                                 // PH_HI, PH_SHI
        }
        if (__ballot_sync(0xFFFFFFFFu, phase != PH_DONE) == 0) break;
        // this round's probe: the record (or SA entry) at the pivot, decided by the cache if it can be
        const bool probing = phase != PH_DONE;
        const bool in_bracket = phase == PH_DESC || phase == PH_LO || phase == PH_HI;
        uint32_t p = 0, skip = 0, from = 0, lcp = 0;
        int sign = 0;
        uint64_t s = 0;
        bool need_text = false;
        if (probing) {
            p = (uint32_t)(((uint64_t)Lp1 - 1 + R) >> 1);
            skip = min(lcpL, lcpR);
            Probe<L> pr;
            if constexpr (L == L_REC32) {
                if (node) pr.r.load(a.tree, tree_rec(tl, node)); else pr.load(a, p);
            } else {
                pr.load(a, p);
            }
            s = pr.sa();
            if constexpr (L == L_PLAIN) {
                need_text = true;
                from = skip;
            } else {
                if (in_bracket) need_text = !rec_decides<L>(a, pr.r, P, m, skip, sign, lcp, from);
                else { need_text = true; from = skip; }
            }
        }
        // the warp serves the text compares, one request at a time, all 32 lanes on each
        unsigned req = __ballot_sync(0xFFFFFFFFu, need_text);
        while (req) {
            const int i = __ffs(req) - 1;
            req &= req - 1;
            const uint64_t si = __shfl_sync(0xFFFFFFFFu, s, i);
            const uint32_t ji = __shfl_sync(0xFFFFFFFFu, from >> 5, i);
            const uint32_t mi = __shfl_sync(0xFFFFFFFFu, m, i);
            const uint64_t rpi = __shfl_sync(0xFFFFFFFFu, reinterpret_cast<uint64_t>(P.p), i);
            const unsigned shi = __shfl_sync(0xFFFFFFFFu, P.sh, i);
            const uint64_t lefti = __shfl_sync(0xFFFFFFFFu, P.left, i);
            int sg;
            uint32_t lc;
            warp_compare_text(a.text, a.n, si, reinterpret_cast<const uint64_t *>(rpi), shi, lefti, mi, ji, lane, sg, lc);
            if ((int)lane == i) {
                sign = sg;
                lcp = lc;
            }
        }
        if (probing) {
            ++steps;
            texts += need_text;
            ubytes += probe_bytes(m, skip, lcp);
            if (phase == PH_DESC) {
                if (sign == 0) {  // the split: lo in (L, p], hi in (p, R]
                    hLp1 = p + 1; hR = R; hlcpL = lcp; hlcpR = lcpR;
                    R = p; lcpR = lcp;
                    hnode = tree_child(tl, node, false);
                    node = tree_child(tl, node, true);
                    phase = PH_LO;
                } else {
                    if (sign < 0) { R = p; lcpR = lcp; } else { Lp1 = p + 1; lcpL = lcp; }
                    node = tree_child(tl, node, sign < 0);
                }
            } else {
                const bool lower = phase == PH_LO || phase == PH_SLO;
                const bool left = sign < 0 || (lower && sign == 0);
                if (left) { R = p; lcpR = lcp; } else { Lp1 = p + 1; lcpL = lcp; }
                node = tree_child(tl, node, left);
            }
        }
    }
    if (valid) {
        reinterpret_cast<uint2 *>(a.out)[q] = make_uint2(lo, hi);
        if (STATS) {
            a.stats[q] = min(steps, 0xFFFFu) | (min(texts, 0xFFFFu) << 16);
            a.stats[a.Q + q] = ubytes;
        }
    }
}

}  // namespace sa_search
